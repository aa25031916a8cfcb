"""Per-kernel device time of one large four-step plan (diagnostic):
  python tools/pass_times.py [lgN] [batch] [table|onthefly]"""
import sys
import torch
sys.path.insert(0, ".")
import paper_1404_1810_b200 as a  # noqa: E402
from torch.profiler import profile, ProfilerActivity  # noqa: E402

lg = int(sys.argv[1]) if len(sys.argv) > 1 else 24
batch = int(sys.argv[2]) if len(sys.argv) > 2 else 1
trig = a.TrigMode.OnTheFly if (len(sys.argv) > 3 and sys.argv[3] == "onthefly") else a.TrigMode.Precomputed
n = 1 << lg
p = a.Plan(4, a.FunctionId.Cdft, n, batch, dtype="f32", order=a.Order.Fast, trig_mode=trig)
x = torch.randn(batch, 2 * n, device="cuda")
y = torch.empty_like(x)
for _ in range(3):
    p.forward(x, y)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(5):
        p.forward(x, y)
    torch.cuda.synchronize()
tot = 0.0
for e in prof.key_averages():
    if e.self_device_time_total > 0:
        ms = e.self_device_time_total / 5 / 1000
        tot += ms
        print(f"  {e.key[:70]:70s} {ms:.3f} ms/step  x{e.count // 5}")
print(f"N=2^{lg} batch {batch} {sys.argv[3] if len(sys.argv) > 3 else 'table'}: {tot:.3f} ms/step")
