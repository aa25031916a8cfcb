"""Config 3 sweep (BASELINE.json configs[2]): complex fp64 forward and
inverse DFT, N = 2^lo .. 2^hi, batch = 2^26 / N rows (1 GiB in), values
iid U[-1, 1) from a seed, ALL 8 variants, fast order (the path the plan picks
per N); per N and variant: forward and inverse throughput, round-trip error
over the batch, row 0 against the CPU oracle of the same variant (bitwise
flag; N <= 2^16) and against numpy's fp64 FFT.  The exact order (the generic
recursion, bitwise the reference at every N) is timed for variant 4.

  python tools/sweep_c3.py [lo] [hi] > profiles/r02_sweep_c3_all_variants.log
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1404_1810_b200 as amqft  # noqa: E402
from oracle import oracle as O  # noqa: E402  (the checker, after the timed calls)


def timed(fn, it=3):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(it):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / it


def main():
    lo = int(sys.argv[1]) if len(sys.argv) > 1 else 4
    hi = int(sys.argv[2]) if len(sys.argv) > 2 else 20
    r = O.restatement()
    res = {}
    g = torch.Generator(device="cuda").manual_seed(3)
    for lg in range(lo, hi + 1):
        n = 1 << lg
        batch = (1 << 26) // n
        x = torch.rand(batch, 2 * n, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
        y = torch.empty_like(x)
        z = torch.empty_like(x)
        x0 = x[0].cpu().numpy()
        f = np.fft.fft(x0[0::2] + 1j * x0[1::2])
        fft0 = np.empty(2 * n)
        fft0[0::2], fft0[1::2] = f.real, f.imag
        for v in range(1, 9):
            p = amqft.Plan(v, amqft.FunctionId.Cdft, n, batch, dtype="f64", order=amqft.Order.Fast)
            path, launches = p.path()
            ms_f = timed(lambda: p.forward(x, y))
            ms_i = timed(lambda: p.inverse(y, z))
            rt = float((z - x).norm() / x.norm())
            y0 = y[0].cpu().numpy()
            row = {"path": path, "launches": launches, "fwd_ms": round(ms_f, 4), "inv_ms": round(ms_i, 4),
                   "fwd_GBs": round(batch * 32 * n / ms_f / 1e6, 1), "inv_GBs": round(batch * 32 * n / ms_i / 1e6, 1),
                   "roundtrip_rel_l2": rt, "row0_vs_numpy_fft": float(np.linalg.norm(y0 - fft0) / np.linalg.norm(fft0))}
            if lg <= 16:
                want = r.execute(v, O.F_CDFT, n, x0)
                row["row0_vs_cpu_same_variant"] = float(np.linalg.norm(y0 - want) / np.linalg.norm(want))
                row["row0_bitwise_cpu"] = bool(y0.tobytes() == want.tobytes())
            if v == 4:
                pe = amqft.Plan(4, amqft.FunctionId.Cdft, n, batch, dtype="f64", order=amqft.Order.Exact)
                ms_e = timed(lambda: pe.forward(x, y), it=1)
                row["exact_order_fwd_GBs"] = round(batch * 32 * n / ms_e / 1e6, 1)
                del pe
            res[f"{lg}/v{v}"] = row
            print(lg, v, json.dumps(row), flush=True)
            del p
        del x, y, z
        torch.cuda.empty_cache()
    print(json.dumps(res))


if __name__ == "__main__":
    main()
