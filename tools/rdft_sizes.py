import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1404_1810_b200 as amqft
for n in (128, 256, 512, 1024, 2048, 4096):
    batch = (1 << 28) // n
    x = torch.randn(batch, n, device="cuda")
    y = torch.empty_like(x)
    p = amqft.Plan(4, amqft.FunctionId.Rdft, n, batch, dtype="f32", order=amqft.Order.Fast)
    for _ in range(3): p.forward(x, y)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5): p.forward(x, y)
    b.record(); torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 5
    print(f"RDFT N={n} path {p.path()}: {ms:.3f} ms, {batch * 8 * n / ms / 1e6:.0f} GB/s", flush=True)
