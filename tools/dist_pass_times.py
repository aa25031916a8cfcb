"""Per-kernel device times of the distributed four-step at world size 1
(config 5 shape, diagnostic)."""
import sys
import torch
sys.path.insert(0, ".")
import paper_1404_1810_b200 as a  # noqa: E402
from paper_1404_1810_b200.dist import DistFourStep  # noqa: E402
from torch.profiler import profile, ProfilerActivity  # noqa: E402

n = 1 << int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 30
d = DistFourStep(4, n, device=0, trig_mode=a.TrigMode.OnTheFly)
x = torch.randn(d.rows1, 2 * d.n1, device="cuda")
bufs = d.buffers(x)
for _ in range(2):
    d.forward(x, bufs=bufs)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    d.forward(x, bufs=bufs)
    torch.cuda.synchronize()
tot = 0.0
for e in prof.key_averages():
    if e.self_device_time_total > 0:
        tot += e.self_device_time_total / 1000
        print(f"  {e.key[:70]:70s} {e.self_device_time_total / 1000:.3f} ms  x{e.count}")
print(f"total {tot:.3f} ms (n1 = {d.n1}, n2 = {d.n2})")
