"""Config 3 sweep (diagnostic): complex fp64 forward + inverse, N = 2^4 .. 2^20,
batch = 2^26 / N rows (1 GiB in), exact order (bitwise the reference) and
fast order where it exists; round-trip error on a row sample."""
import json
import sys
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1404_1810_b200 as amqft

res = {}
lo = int(sys.argv[1]) if len(sys.argv) > 1 else 4
hi = int(sys.argv[2]) if len(sys.argv) > 2 else 20
for lg in range(lo, hi + 1):
    n = 1 << lg
    batch = (1 << 26) // n
    x = torch.rand(batch, 2 * n, dtype=torch.float64, device="cuda") * 2 - 1
    y = torch.empty_like(x)
    z = torch.empty_like(x)
    for order in (amqft.Order.Exact, amqft.Order.Fast):
        try:
            p = amqft.Plan(4, amqft.FunctionId.Cdft, n, batch, dtype="f64", order=order)
        except Exception as e:  # noqa: BLE001
            res[f"{lg}/{int(order)}"] = str(e)
            continue
        path = p.path()[0]
        if order == amqft.Order.Fast and path < 2:
            continue
        p.forward(x, y)
        p.inverse(y, z)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(3):
            p.forward(x, y)
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / 3
        err = float((z - x).norm() / x.norm())
        res[f"{lg}/{'exact' if order == amqft.Order.Exact else 'fast'}"] = {
            "path": path, "ms": round(ms, 3), "GBs": round(batch * 32 * n / ms / 1e6, 1),
            "roundtrip_rel_l2": err}
        print(lg, res[f"{lg}/{'exact' if order == amqft.Order.Exact else 'fast'}"], flush=True)
        del p
    del x, y, z
    torch.cuda.empty_cache()
print(json.dumps(res))
