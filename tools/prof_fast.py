"""Runs one plan a few times for profiling (ncu) -- not a benchmark."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1404_1810_b200 as amqft  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--variant", type=int, default=4)
p.add_argument("--n", type=int, default=4096)
p.add_argument("--batch", type=int, default=4096)
p.add_argument("--dtype", default="f32")
p.add_argument("--order", default="fast")
p.add_argument("--iters", type=int, default=3)
a = p.parse_args()
plan = amqft.Plan(a.variant, amqft.FunctionId.Cdft, a.n, a.batch, dtype=a.dtype,
                  order=amqft.Order.Fast if a.order == "fast" else amqft.Order.Exact)
dt = torch.float32 if a.dtype == "f32" else torch.float64
x = torch.randn(a.batch, 2 * a.n, device="cuda", dtype=dt)
y = torch.empty_like(x)
for _ in range(a.iters):
    plan.forward(x, y)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
plan.forward(x, y)
e.record()
torch.cuda.synchronize()
ms = s.elapsed_time(e)
print(f"v{a.variant} N={a.n} batch={a.batch} {a.dtype}: {ms:.3f} ms, {a.batch / ms * 1e3:.3e} transforms/s, "
      f"{a.batch * 16 * a.n / ms / 1e6:.1f} GB/s (fp32 bytes)")
