import torch, sys
sys.path.insert(0, '.')
import paper_1404_1810_b200 as amqft
for n, batch in ((1 << 24, 1), (1 << 24, 4), (1 << 20, 64)):
    for trig in (amqft.TrigMode.Precomputed, amqft.TrigMode.OnTheFly):
        p = amqft.Plan(4, amqft.FunctionId.Cdft, n, batch, dtype="f32", order=amqft.Order.Fast, trig_mode=trig)
        x = torch.randn(batch, 2 * n, device="cuda"); y = torch.empty_like(x)
        for _ in range(3): p.forward(x, y)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(10): p.forward(x, y)
        b.record(); torch.cuda.synchronize()
        ms = a.elapsed_time(b) / 10
        gbs = batch * 16 * n / ms / 1e6
        print(f"N=2^{n.bit_length()-1} batch {batch} trig {int(trig)}: {ms:.3f} ms, {gbs:.0f} GB/s algorithmic, {gbs/6548.5:.3f} of HBM")
