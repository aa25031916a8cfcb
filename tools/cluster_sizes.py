"""fp32 CDFT throughput at N = 2^13 .. 2^16 (diagnostic, not a benchmark):
the cluster four-step against the previous multi-pass four-step (forced by
table_max_n... no: by the A/B hook for 8192) -- prints GB/s on fp32 bytes."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1404_1810_b200 as amqft  # noqa: E402


def t(plan, x, y, it=5):
    for _ in range(2):
        plan.forward(x, y)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(it):
        plan.forward(x, y)
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / it


for v in [int(a) for a in (sys.argv[1:] or ["4"])]:
    for lg in (13, 14, 15, 16):
        n = 1 << lg
        batch = (1 << 28) // n
        x = torch.randn(batch, 2 * n, device="cuda")
        y = torch.empty_like(x)
        p = amqft.Plan(v, amqft.FunctionId.Cdft, n, batch, dtype="f32", order=amqft.Order.Fast)
        ms = t(p, x, y)
        print(f"v{v} N=2^{lg} path={p.path()} batch={batch}: {ms:.3f} ms  {batch * 16 * n / ms / 1e6:.0f} GB/s",
              flush=True)
