"""Quick fp32 parity check of one variant's fused kernel against the CPU
oracle (diagnostic, for A/B builds)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1404_1810_b200 as amqft  # noqa: E402
from oracle import oracle as O  # noqa: E402

v, n = int(sys.argv[1]), int(sys.argv[2])
r = O.restatement()
x = np.random.default_rng(1).standard_normal((8, 2 * n)).astype(np.float32)
p = amqft.Plan(v, amqft.FunctionId.Cdft, n, 8, dtype="f32", order=amqft.Order.Fast)
dx = torch.tensor(x, device="cuda")
dy = torch.empty_like(dx)
p.forward(dx, dy)
p.inverse(dy, dx)
torch.cuda.synchronize()
y = dy.double().cpu().numpy()
errs = [r.rel_l2(y[i], r.execute(v, O.F_CDFT, n, x[i].astype(np.float64))) for i in range(8)]
rt = float(np.linalg.norm(dx.double().cpu().numpy() - x) / np.linalg.norm(x))
print(f"v{v} N={n}: max rel-L2 vs oracle {max(errs):.3e}, round trip {rt:.3e}, path {p.path()}")
