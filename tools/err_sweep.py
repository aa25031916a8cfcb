"""fp32 fast-order error per variant and N against the CPU oracle of the same
variant (diagnostic; tests assert the tolerance).  Prints one line per
(variant, N): the plan path, rel-L2 vs the oracle, and the tolerance
1e-5 log2 N.  The oracle is the checker only."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1404_1810_b200 as amqft  # noqa: E402
from oracle import oracle as O  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--lgmin", type=int, default=1)
p.add_argument("--lgmax", type=int, default=16)
p.add_argument("--rows", type=int, default=2)
p.add_argument("--variants", default="1,2,3,4,5,6,7,8")
p.add_argument("--dtype", default="f32")
a = p.parse_args()
r = O.restatement()
rng = np.random.default_rng(11)
for v in [int(s) for s in a.variants.split(",")]:
    for lg in range(a.lgmin, a.lgmax + 1):
        n = 1 << lg
        batch = max(a.rows, 64)
        try:
            plan = amqft.Plan(v, amqft.FunctionId.Cdft, n, batch, dtype=a.dtype, order=amqft.Order.Fast)
        except amqft.AmqftError as e:
            print(f"v{v} N=2^{lg}: no plan ({e})")
            continue
        dt = torch.float32 if a.dtype == "f32" else torch.float64
        x = torch.tensor(rng.standard_normal((batch, 2 * n)), dtype=dt, device="cuda")
        y = torch.empty_like(x)
        plan.forward(x, y)
        torch.cuda.synchronize()
        errs = []
        for b in range(a.rows):
            want = r.execute(v, O.F_CDFT, n, x[b].double().cpu().numpy())
            errs.append(r.rel_l2(y[b].double().cpu().numpy(), want))
        tol = 1e-5 * lg
        print(f"v{v} N=2^{lg:2d} path={plan.path()[0]} rel_l2_vs_cpu_same_variant={max(errs):.3e} "
              f"tol={tol:.1e} {'OK' if max(errs) <= tol else 'FAIL'}", flush=True)
