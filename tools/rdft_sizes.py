"""Throughput of the real-row transforms per size on one GPU (diagnostic):
RDFT (N reals -> packed spectrum), DCT-0 (N/2 + 1 cells), DST-0 (N/2 - 1 cells),
fp32, variant 4, fast order -> the path the plan picks; GB/s on the rows' own
bytes (one read + one write).  python tools/rdft_sizes.py [rdft|dct|dst]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1404_1810_b200 as amqft  # noqa: E402

kind = sys.argv[1] if len(sys.argv) > 1 else "rdft"
fn = {"rdft": amqft.FunctionId.Rdft, "dct": amqft.FunctionId.Dct, "dst": amqft.FunctionId.Dst}[kind]
for n in (128, 256, 512, 1024, 2048, 4096):
    cells = amqft.cell_count(fn, n)
    batch = (1 << 28) // n
    x = torch.randn(batch, cells, device="cuda")
    y = torch.empty_like(x)
    p = amqft.Plan(4, fn, n, batch, dtype="f32", order=amqft.Order.Fast)
    for _ in range(2):
        p.forward(x, y)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(3):
        p.forward(x, y)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 3
    print(f"{kind.upper()} N={n} path {p.path()}: {ms:.3f} ms, {batch / ms * 1e3:.3e} rows/s, "
          f"{batch * 8 * cells / ms / 1e6:.0f} GB/s", flush=True)
