"""In-shared-memory four-step (path 6) against the CPU oracle and numpy's fp64
FFT, and its timing against the path the plan picks without it
(AMQFT_AB_TILE=none: fused / cooperative kernels).  Diagnostic, run on the GPU
box: python tools/tile_check.py [variants] [log2 sizes]"""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1404_1810_b200 as amqft  # noqa: E402
from oracle import oracle as O  # noqa: E402


def timed(plan, x, y, iters=5):
    for _ in range(3):
        plan.forward(x, y)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        plan.forward(x, y)
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters


def main():
    variants = [int(v) for v in sys.argv[1].split(",")] if len(sys.argv) > 1 else [4]
    lgs = [int(v) for v in sys.argv[2].split(",")] if len(sys.argv) > 2 else [8, 9, 10, 11, 12]
    dtype = sys.argv[3] if len(sys.argv) > 3 else "f32"
    tdt = torch.float32 if dtype == "f32" else torch.float64
    esize = 4 if dtype == "f32" else 8
    child = os.environ.get("AMQFT_AB_TILE", "") == "none"
    r = O.restatement()
    for lg in lgs:
        n = 1 << lg
        batch = (1 << (28 if dtype == "f32" else 27)) // n
        x = torch.randn(batch, 2 * n, device="cuda", dtype=tdt)
        y = torch.empty_like(x)
        for v in variants:
            plan = amqft.Plan(v, amqft.FunctionId.Cdft, n, batch, dtype=dtype, order=amqft.Order.Fast)
            ms = timed(plan, x, y)
            gbs = batch * 4 * esize * n / ms / 1e6
            line = f"v{v} N={n} path {plan.path()}: {ms:.3f} ms, {gbs:.0f} GB/s"
            if not child:
                rows = [0, 1, batch - 1]
                xs = x[rows].double().cpu().numpy()
                ys = y[rows].double().cpu().numpy()
                e_or = max(r.rel_l2(ys[i], r.execute(v, O.F_CDFT, n, xs[i])) for i in range(len(rows)))
                ref = np.fft.fft(xs[:, 0::2] + 1j * xs[:, 1::2], axis=1)
                got = ys[:, 0::2] + 1j * ys[:, 1::2]
                e_np = float(np.linalg.norm(got - ref) / np.linalg.norm(ref))
                z = torch.empty_like(x[:64])
                p2 = amqft.Plan(v, amqft.FunctionId.Cdft, n, 64, dtype=dtype, order=amqft.Order.Fast)
                p2.forward(x[:64], z)
                w = torch.empty_like(z)
                p2.inverse(z, w)
                torch.cuda.synchronize()
                rt = float((w - x[:64]).double().norm() / x[:64].double().norm())
                line += f", vs oracle {e_or:.2e}, vs numpy {e_np:.2e}, round trip {rt:.2e}"
            print(line, flush=True)
        del x, y
    if not child:
        env = dict(os.environ, AMQFT_AB_TILE="none")
        print("--- AMQFT_AB_TILE=none", flush=True)
        subprocess.run([sys.executable, os.path.abspath(__file__)] + sys.argv[1:], env=env, check=False)


if __name__ == "__main__":
    main()
