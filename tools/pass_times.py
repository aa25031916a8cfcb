import sys, torch
sys.path.insert(0, ".")
import paper_1404_1810_b200 as a
from torch.profiler import profile, ProfilerActivity
for batch in (1, 16):
    n = 1 << 24
    p = a.Plan(4, a.FunctionId.Cdft, n, batch, dtype="f32", order=a.Order.Fast)
    x = torch.randn(batch, 2 * n, device="cuda"); y = torch.empty_like(x)
    for _ in range(3): p.forward(x, y)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(5): p.forward(x, y)
        torch.cuda.synchronize()
    print("batch", batch)
    for e in prof.key_averages():
        if e.device_type is not None and e.self_device_time_total > 0:
            print(f"  {e.key[:70]:70s} {e.self_device_time_total/5/1000:.3f} ms/step  x{e.count//5}")
