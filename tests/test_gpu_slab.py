"""Column-slab four-step plans (csrc/slab_kernel.cuh, fourstep.cu SlabPlan):
N = L1 L2 in two passes over HBM, N = L1 L2 L3 in three, L in {128 .. 1024},
natural order in and out, no transpose kernel.  Checked against numpy's fp64
FFT (all variants), the CPU reference of the same variant (variants 1-4, where
the reference is itself accurate at these sizes), inverses, in-place calls,
batches and the op meter.  AMQFT_AB_SLAB=all selects the slab plan at every
size it covers (2^14 .. 2^30), so the small cases stay cheap on the CPU side."""
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_1404_1810_b200 as amqft  # noqa: E402
from test_gpu_parity import DEV, numpy_dft, run_plan  # noqa: E402


@pytest.fixture
def slab_all(monkeypatch):
    monkeypatch.setenv("AMQFT_AB_SLAB", "all")
    monkeypatch.setenv("AMQFT_AB_TILE", "none")


def _plan(v, n, batch, dtype, passes):
    p = amqft.Plan(v, amqft.FunctionId.Cdft, n, batch, dtype=dtype, order=amqft.Order.Fast)
    assert p.path() == (3, passes), "slab plan expected (four-step path, one launch per pass)"
    return p


def _factors(n, dtype="f32"):
    lg = n.bit_length() - 1
    if lg <= 20 or (dtype == "f32" and lg <= 23):   # fp32: 2048- / 4096-point passes up to 2^23
        return [1 << ((lg + 1) // 2), 1 << (lg // 2)]
    a = (lg + 2) // 3
    b = (lg - a + 1) // 2
    return [1 << a, 1 << b, 1 << (lg - a - b)]


@pytest.mark.parametrize("lg,dtype", [(14, "f32"), (15, "f32"), (17, "f32"), (19, "f32"), (20, "f32"), (21, "f32"),
                                      (23, "f32"), (24, "f32"),
                                      (14, "f64"), (16, "f64"), (19, "f64"), (21, "f64")])
def test_slab_all_variants(oracle, restatement, slab_all, lg, dtype):
    r, O = restatement, oracle
    n = 1 << lg
    f = _factors(n, dtype)
    rows = 2
    xs = np.random.default_rng(lg).standard_normal((rows, 2 * n))
    if dtype == "f32":
        xs = xs.astype(np.float32).astype(np.float64)
    tol = 2e-6 if dtype == "f32" else 1e-13
    refs = [numpy_dft(xs[row]) for row in range(rows)]
    for v in (range(1, 9) if lg < 23 else (4, 7)):   # the largest sizes: two variants (host-side FFTs and copies)
        plan = _plan(v, n, rows, dtype, len(f))
        assert plan.fourstep_factors() == (f[0], f[1] if len(f) == 3 else 1, f[-1])
        got = run_plan(plan, xs)
        for row in range(rows):
            assert r.rel_l2(got[row], refs[row]) <= tol, (v, lg, dtype)
        if v <= 4 and lg <= 17:
            want = r.execute(v, O.F_CDFT, n, xs[0])
            assert r.rel_l2(got[0], want) <= (1e-5 * lg if dtype == "f32" else 1e-12), (v, lg)
        back = run_plan(plan, got.astype(np.float32) if dtype == "f32" else got, inverse=True)
        assert r.rel_l2(back.ravel(), xs.ravel()) <= tol, (v, lg, dtype)


@pytest.mark.parametrize("lg", [16, 21, 24])
def test_slab_in_place_and_batch_rows_independent(slab_all, lg):
    """d_in == d_out goes through the plan's scratch buffer (the first pass
    transposes); a row's result does not depend on its batch position."""
    n = 1 << lg
    rows = 5
    x = torch.tensor(np.random.default_rng(lg + 1).standard_normal((rows, 2 * n)), dtype=torch.float32, device=DEV)
    plan = _plan(3, n, rows, "f32", len(_factors(n)))
    y = torch.empty_like(x)
    plan.forward(x, y)
    z = x.clone()
    plan.forward(z, z)
    torch.cuda.synchronize()
    assert torch.equal(y, z)
    single = _plan(3, n, 1, "f32", len(_factors(n)))
    w = torch.empty_like(x[:1])
    single.forward(x[3:4].contiguous(), w)
    torch.cuda.synchronize()
    assert torch.equal(w[0], y[3])
    plan.inverse(z, z)
    torch.cuda.synchronize()
    assert float((z - x).norm() / x.norm()) <= 2e-6


def test_slab_op_counts(oracle, restatement, slab_all):
    """Meter of the executed schedule: per pass N / L columns of the
    two-factor length-L schedule (its factor meters + one twiddle multiply
    per element), and one twiddle multiply per element between passes."""
    r, O = restatement, oracle
    split = {128: (8, 16), 256: (16, 16), 512: (16, 32), 1024: (32, 32), 2048: (64, 32), 4096: (64, 64)}
    for n in (1 << 16, 1 << 19, 1 << 22, 1 << 24):
        f = _factors(n)
        want = [0, 0, 0]
        for L in f:
            col = [0, 0, 0]
            for nf in split[L]:
                m = r.execute(4, O.F_CDFT, nf, np.zeros(2 * nf), meter=True)[1]
                for i in range(3):
                    col[i] += (L // nf) * m[i]
            col[0] += 2 * L
            col[1] += 4 * L
            for i in range(3):
                want[i] += (n // L) * col[i]
        want[0] += 2 * n * (len(f) - 1)
        want[1] += 4 * n * (len(f) - 1)
        assert _plan(4, n, 1, "f32", len(f)).op_counts() == tuple(want), n


def test_slab_is_the_default_where_measured_faster():
    for lg, dtype, passes in ((17, "f32", 2), (20, "f32", 2), (22, "f32", 2), (24, "f32", 3), (16, "f64", 2), (20, "f64", 2),
                              (22, "f64", 3)):
        p = amqft.Plan(4, amqft.FunctionId.Cdft, 1 << lg, 1, dtype=dtype, order=amqft.Order.Fast)
        assert p.path() == (3, passes), (lg, dtype)
    # where the column / tile-row / transpose four-step wins, it stays
    p = amqft.Plan(4, amqft.FunctionId.Cdft, 1 << 17, 1, dtype="f64", order=amqft.Order.Fast)
    assert p.path()[0] == 3 and p.fourstep_factors() != (512, 1, 256)
