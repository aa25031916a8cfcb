"""Cluster four-step (fast_kernel.cuh k_fast<..., P>): CDFT N = 2^13 .. 2^16
as P = N / 4096 fused rows on one thread-block cluster, one pass over HBM
(north_star "one fused pass up to N ~ 2^16").

Checked per variant against the fp64 oracle of the same variant (v1-4, fp32
tolerance 1e-5 log2 N) and against numpy's fp64 FFT (all variants: the
reference's own fp64 v5-8 drift from the true DFT from N = 2^13),
inverse round trips, batch rows independent of their neighbours, and the op
meter of the executed schedule."""
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_1404_1810_b200 as amqft  # noqa: E402
from test_gpu_parity import numpy_dft, run_plan  # noqa: E402

# Since the in-shared-memory four-step (tile_kernel.cuh) covers N <= 2^14 in one pass at 0.78-0.88 of
# HBM, the plan no longer picks the cluster kernel anywhere; AMQFT_AB_CLUSTER=all keeps it testable.
ALL = [1 << 13, 1 << 14, 1 << 15, 1 << 16]


def _plan(v, n, batch):
    p = amqft.Plan(v, amqft.FunctionId.Cdft, n, batch, dtype="f32", order=amqft.Order.Fast)
    assert p.path() == (2, 1), "cluster four-step expected (fused path, one launch)"
    return p


@pytest.fixture
def all_cluster_sizes(monkeypatch):
    """Every cluster size (P = 2 .. 16) through the A/B override (and the
    tile path, the default at N <= 2^14, off)."""
    monkeypatch.setenv("AMQFT_AB_CLUSTER", "all")
    monkeypatch.setenv("AMQFT_AB_TILE", "none")


@pytest.mark.parametrize("n", ALL)
def test_cluster_all_variants(oracle, restatement, n, all_cluster_sizes):
    r, O = restatement, oracle
    lg = n.bit_length() - 1
    tol = 1e-5 * lg
    rng = np.random.default_rng(n)
    xs = rng.standard_normal((3, 2 * n)).astype(np.float32).astype(np.float64)
    refs = [numpy_dft(x) for x in xs]
    for v in range(1, 9):
        plan = _plan(v, n, 3)
        got = run_plan(plan, xs)
        for i in range(3):
            assert r.rel_l2(got[i], refs[i]) <= tol, (v, n, i)
        if v <= 4 and n <= (1 << 15):
            want = r.execute(v, O.F_CDFT, n, xs[0])
            assert r.rel_l2(got[0], want) <= tol, (v, n)
        back = run_plan(plan, got.astype(np.float32), inverse=True)
        assert r.rel_l2(back.ravel(), xs.ravel()) <= tol, (v, n)


@pytest.mark.parametrize("n", [8192, 1 << 14])
def test_default_at_cluster_sizes_is_the_tile_path(n):
    p = amqft.Plan(4, amqft.FunctionId.Cdft, n, 1, dtype="f32", order=amqft.Order.Fast)
    assert p.path() == (6, 1)


def test_cluster_rows_independent_and_deterministic(all_cluster_sizes):
    """A row's result does not depend on its batch position or on the
    persistent cluster schedule (rows > resident clusters)."""
    n = 1 << 14
    rows = 700                      # more rows than resident clusters
    g = torch.Generator(device="cuda:0").manual_seed(3)
    x = torch.randn(rows, 2 * n, device="cuda:0", generator=g)
    y = torch.empty_like(x)
    plan = _plan(4, n, rows)
    plan.forward(x, y)
    y1 = torch.empty(1, 2 * n, device="cuda:0")
    p1 = _plan(4, n, 1)
    for i in (0, 1, 347, rows - 1):
        p1.forward(x[i:i + 1].contiguous(), y1)
        torch.cuda.synchronize()
        assert torch.equal(y1[0], y[i]), i
    ref = numpy_dft(x[rows - 1].double().cpu().numpy())
    got = y[rows - 1].double().cpu().numpy()
    assert np.linalg.norm(got - ref) / np.linalg.norm(ref) <= 1.4e-4


def test_cluster_op_counts(all_cluster_sizes):
    """Meter of the executed schedule: P rows of the 4096-point AM-QFT DAG
    (reference closed forms) + the radix-2 P-point DFTs + (2P-3) N/P twiddle
    multiplies (the twiddles and their powers)."""
    for n in ALL:
        P = n // 4096
        lgp = P.bit_length() - 1
        base = amqft.Plan(4, amqft.FunctionId.Cdft, 4096, 1, dtype="f32", order=amqft.Order.Fast).op_counts()
        bfly = (n // P) * (P // 2) * lgp
        tw = (2 * P - 3) * (n // P)
        want = (P * base[0] + 6 * bfly + 2 * tw, P * base[1] + 4 * bfly + 4 * tw, P * base[2])
        assert _plan(4, n, 1).op_counts() == want, n
