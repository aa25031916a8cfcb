"""A/B of two builds of the library on one plan (diagnostic):
   python tools/ab_lib.py OTHER_SO variant n dtype"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1404_1810_b200 as amqft  # noqa: E402
from paper_1404_1810_b200 import _native  # noqa: E402

other, v, n, dt = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
batch = (1 << 26) // n if dt == "f64" else (1 << 28) // n
x = torch.rand(batch, 2 * n, device="cuda", dtype=torch.float64 if dt == "f64" else torch.float32) * 2 - 1
y = torch.empty_like(x)
for label in ("current", "other"):
    if label == "other":
        _native.LIB_PATH = os.path.abspath(other)
        _native._lib = None
        amqft._native._lib = None
    p = amqft.Plan(v, amqft.FunctionId.Cdft, n, batch, dtype=dt, order=amqft.Order.Fast)
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
    print(f"{label}: v{v} N={n} {dt}: {ms:.3f} ms", flush=True)
    del p
