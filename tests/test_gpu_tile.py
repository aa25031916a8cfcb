"""In-shared-memory four-step (path 6, tile_kernel.cuh): fp32 CDFT N = 16 ..
65536 as N1 x N2 (x N3 from N = 8192) register-resident AM-QFT factors, one
pass over HBM -- the default fast-order path for these sizes (config 2 is
N = 4096).  N = 2^15 / 2^16 run one row per thread-block cluster of 2 / 4
CTAs with the phase-A outputs exchanged over distributed shared memory.

Checked for ALL 8 variants against the fp64 CPU reference of the same variant
(tolerance 1e-5 log2 N, BASELINE north_star; the factors are <= 64 points, where
the sine-family variants 5-8 are stable in fp32, so no variant needs fp64
compute here), against numpy's fp64 FFT, against the compiled reference
library (oracle/_ref) at config 2's size, inverse round trips, in-place rows,
ragged batches (rows not a multiple of the tile, fewer rows than CTAs, more
rows than one wave), and the op meter of the executed schedule."""
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_1404_1810_b200 as amqft  # noqa: E402
from test_gpu_parity import DEV, numpy_dft, run_plan  # noqa: E402

SIZES = [16, 32, 64, 128, 256, 512, 1024, 2048, 4096, 8192, 16384, 32768, 65536]
# the kernel's split (tile_kernel.cuh make_tile): N1 (phase A) x N2 (phase B) [x N3 (phase C)]
SPLIT = {16: (4, 4), 32: (4, 8), 64: (8, 8), 128: (8, 16), 256: (16, 16), 512: (16, 32), 1024: (32, 32),
         2048: (64, 32), 4096: (64, 64), 8192: (32, 16, 16), 16384: (32, 16, 32), 32768: (32, 32, 32),
         65536: (32, 32, 64)}


def rows_per_tile(n):
    return 1 if len(SPLIT[n]) == 3 else max(1, 64 // min(SPLIT[n]))
# measured on the B200: 1e-7 .. 4e-7 (v1-4), up to 6e-7 vs numpy for v5-8;
# the bar below is 10x tighter than the north-star tolerance
TIGHT = 2e-6


def _plan(v, n, batch):
    p = amqft.Plan(v, amqft.FunctionId.Cdft, n, batch, dtype="f32", order=amqft.Order.Fast)
    assert p.path() == (6, 1), "in-shared-memory four-step expected (one launch)"
    return p


@pytest.mark.parametrize("n", SIZES)
def test_tile_all_variants_match_cpu(oracle, restatement, n):
    r, O = restatement, oracle
    rows = 5
    xs = np.random.default_rng(n).standard_normal((rows, 2 * n)).astype(np.float32).astype(np.float64)
    tol = 1e-5 * math.log2(n)
    for v in range(1, 9):
        plan = _plan(v, n, rows)
        got = run_plan(plan, xs)
        for row in (0, rows - 1):
            assert r.rel_l2(got[row], numpy_dft(xs[row])) <= TIGHT, (v, n)
            if v >= 5 and n > 4096:
                continue   # the reference's own fp64 v5-8 drift from the DFT (1e-3 at 2^13, O(1) at 2^14)
            want = r.execute(v, O.F_CDFT, n, xs[row])
            err = r.rel_l2(got[row], want)
            # the reference's own fp64 v5-8 result is ~1e-6 from the DFT at 4096
            assert err <= (tol if v >= 5 else TIGHT), (v, n, err)
        back = run_plan(plan, got.astype(np.float32), inverse=True)
        assert r.rel_l2(back.ravel(), xs.ravel()) <= TIGHT, (v, n)


def test_tile_matches_reference_library_config2(oracle, reference, restatement):
    """Config 2's size against the compiled reference itself (oracle/_ref)."""
    n = 4096
    x = np.random.default_rng(2).standard_normal(2 * n).astype(np.float32).astype(np.float64)
    for v in range(1, 9):
        got = run_plan(_plan(v, n, 1), [x])[0]
        want = reference.execute(v, oracle.F_CDFT, n, x)
        assert restatement.rel_l2(got, want) <= 1e-5 * 12, v


@pytest.mark.parametrize("n", SIZES)
def test_tile_ragged_batches_and_rows_independent(n):
    """Row counts around the tile size (R = 64 / min(N1, N2) rows per CTA
    iteration) and beyond one wave of CTAs: every row equals the same row
    transformed alone (bitwise: a row's arithmetic does not depend on its
    position in the batch)."""
    R = rows_per_tile(n)
    big = min(148 * 16 * R + R + 1, (1 << 27) // n + 3)   # more tiles than resident CTAs / clusters, last tile partial
    rng = np.random.default_rng(n + 1)
    x = torch.tensor(rng.standard_normal((big, 2 * n)), dtype=torch.float32, device=DEV)
    plan = _plan(4, n, big)
    y = torch.empty_like(x)
    plan.forward(x, y)
    torch.cuda.synchronize()
    single = _plan(4, n, 1)
    for row in (0, 1, R - 1, R, big // 2, big - 2, big - 1):
        z = torch.empty_like(x[row:row + 1])
        single.forward(x[row:row + 1].contiguous(), z)
        torch.cuda.synchronize()
        assert torch.equal(z[0], y[row]), (n, row)
    for rows in (1, R - 1 if R > 1 else 1, R + 1, 3 * R + 2):
        z = torch.full_like(x[:rows + 1], float("nan"))
        plan.forward(x[:rows].contiguous(), z, rows=rows)
        torch.cuda.synchronize()
        assert torch.equal(z[:rows], y[:rows]), (n, rows)
        assert torch.isnan(z[rows]).all(), "rows past the batch must not be written"


@pytest.mark.parametrize("n", [256, 4096])
def test_tile_in_place(n):
    x = torch.tensor(np.random.default_rng(n + 2).standard_normal((37, 2 * n)), dtype=torch.float32, device=DEV)
    plan = _plan(2, n, 37)
    y = torch.empty_like(x)
    plan.forward(x, y)
    z = x.clone()
    plan.forward(z, z)
    torch.cuda.synchronize()
    assert torch.equal(y, z)
    plan.inverse(z, z)
    torch.cuda.synchronize()
    assert float((z - x).norm() / x.norm()) <= TIGHT


@pytest.mark.parametrize("n", SIZES)
def test_tile_op_counts(oracle, restatement, n):
    """Meter of the executed schedule: N2 reference DAGs of length N1, N1 of
    length N2 (the reference meter of each) and one complex twiddle multiply
    per element (4 muls + 2 adds), the four-step's accounting (three factors:
    two twiddle passes)."""
    r, O = restatement, oracle
    f = SPLIT[n]
    for v in (1, 4, 6):
        want = [0, 0, 0]
        for nf in f:   # n / nf reference DAGs of length nf per factor
            m = r.execute(v, O.F_CDFT, nf, np.zeros(2 * nf), meter=True)[1]
            for i in range(3):
                want[i] += (n // nf) * m[i]
        want[0] += 2 * n * (len(f) - 1)   # one twiddle pass per extra factor
        want[1] += 4 * n * (len(f) - 1)
        assert _plan(v, n, 1).op_counts() == tuple(want), (v, n)


def test_tile_rejects_misaligned_buffers():
    """Device buffers of fast-order plans must be 16-byte aligned (the C ABI's
    contract for every fast path); the host-buffer pipeline of this path is
    covered by test_gpu_parity.py::test_host_pipeline_matches_device_path."""
    n = 4096
    plan = _plan(4, n, 1)
    x = torch.zeros(2 * n + 2, dtype=torch.float32, device=DEV)
    with pytest.raises(amqft.InvalidArgument):
        plan.forward(x[1:2 * n + 1], x[1:2 * n + 1], rows=1)


# ---- fp64 instances: factors <= 32 points, N = 64 .. 2^15.  The plan takes this path only where
# the result stays within 1e-12 of the CPU reference of the same variant (fast.cu tile_covers):
# variants 1-4 at every size, variants 5-8 up to N = 256 (beyond, the reference's own v5-8 drift from
# the DFT, and the plan keeps the reference DAG: the fused kernel's fp64 instance, bitwise).
SIZES64 = [64, 128, 256, 512, 1024, 2048, 4096, 8192, 16384, 32768]
SPLIT64 = {64: (8, 8), 128: (8, 16), 256: (16, 16), 512: (16, 32), 1024: (32, 32), 2048: (8, 16, 16),
           4096: (16, 16, 16), 8192: (32, 16, 16), 16384: (32, 16, 32), 32768: (32, 32, 32)}


@pytest.mark.parametrize("n", SIZES64)
def test_tile_fp64_within_1e12_of_cpu(oracle, restatement, n):
    r, O = restatement, oracle
    rows = 3
    xs = np.stack([O.seeded_signal(41, O.CDFT, n, k, r) for k in range(rows)])
    for v in range(1, 9):
        plan = amqft.Plan(v, amqft.FunctionId.Cdft, n, rows, dtype="f64", order=amqft.Order.Fast)
        if v >= 5 and n > 256:
            assert plan.path()[0] != 6, (v, n)   # the reference DAG (bitwise) or its four-step
            continue
        assert plan.path() == (6, 1), (v, n)
        got = run_plan(plan, xs)
        for row in range(rows):
            assert r.rel_l2(got[row], r.execute(v, O.F_CDFT, n, xs[row])) <= 1e-12, (v, n)
            assert r.rel_l2(got[row], numpy_dft(xs[row])) <= 1e-14, (v, n)
        back = run_plan(plan, got, inverse=True)
        assert r.rel_l2(back.ravel(), xs.ravel()) <= 1e-14, (v, n)
        f = SPLIT64[n]
        want = [0, 0, 0]
        for nf in f:
            m = r.execute(v, O.F_CDFT, nf, np.zeros(2 * nf), meter=True)[1]
            for i in range(3):
                want[i] += (n // nf) * m[i]
        want[0] += 2 * n * (len(f) - 1)
        want[1] += 4 * n * (len(f) - 1)
        assert plan.op_counts() == tuple(want), (v, n)


@pytest.mark.parametrize("n", [256, 4096, 32768])
def test_tile_fp64_ragged_rows_independent(n):
    R = 1 if len(SPLIT64[n]) == 3 else max(1, 64 // min(SPLIT64[n]))
    big = min(148 * 12 * R + R + 1, (1 << 26) // n + 3)
    x = torch.tensor(np.random.default_rng(n).uniform(-1, 1, (big, 2 * n)), dtype=torch.float64, device=DEV)
    plan = amqft.Plan(2, amqft.FunctionId.Cdft, n, big, dtype="f64", order=amqft.Order.Fast)
    assert plan.path() == (6, 1)
    y = torch.empty_like(x)
    plan.forward(x, y)
    torch.cuda.synchronize()
    single = amqft.Plan(2, amqft.FunctionId.Cdft, n, 1, dtype="f64", order=amqft.Order.Fast)
    for row in (0, R, big // 2, big - 1):
        z = torch.empty_like(x[row:row + 1])
        single.forward(x[row:row + 1].contiguous(), z)
        torch.cuda.synchronize()
        assert torch.equal(z[0], y[row]), (n, row)


def test_fast_dag_order_keeps_the_reference_dag(oracle, restatement):
    """Order.FastDag: the whole-DAG kernels (no split inside shared memory);
    its fp64 instances are bitwise amqft::execute where Order.Fast is within
    1e-12."""
    r, O = restatement, oracle
    for n in (256, 4096):
        x = O.seeded_signal(43, O.CDFT, n, 0, r)
        want = r.execute(4, O.F_CDFT, n, x)
        dag = amqft.Plan(4, amqft.FunctionId.Cdft, n, 1, dtype="f64", order=amqft.Order.FastDag)
        assert dag.path()[0] in (2, 4)
        assert run_plan(dag, [x])[0].tobytes() == want.tobytes()
        fast = amqft.Plan(4, amqft.FunctionId.Cdft, n, 1, dtype="f64", order=amqft.Order.Fast)
        assert fast.path() == (6, 1)
        assert r.rel_l2(run_plan(fast, [x])[0], want) <= 1e-12
    p32 = amqft.Plan(4, amqft.FunctionId.Cdft, 4096, 1, dtype="f32", order=amqft.Order.FastDag)
    assert p32.path() == (2, 1)


# ---- RDFT rows (FunctionId::Rdft) on the two-factor kernel: the CDFT of x + 0 i,
# stored as the packed spectrum (signal.hpp:122-124).  fp32 N = 256 .. 4096 (only the generic
# interpreter covered 256 / 512 before), fp64 N = 128 .. 1024.
@pytest.mark.parametrize("n,dtype", [(256, "f32"), (512, "f32"), (1024, "f32"), (2048, "f32"), (4096, "f32"),
                                     (128, "f64"), (256, "f64"), (1024, "f64")])
def test_tile_rdft_rows_match_cpu(oracle, restatement, n, dtype):
    r, O = restatement, oracle
    rows = 70                                    # partial last tile
    xs = np.random.default_rng(n + 9).standard_normal((rows, n))
    if dtype == "f32":
        xs = xs.astype(np.float32).astype(np.float64)
    for v in range(1, 9):
        plan = amqft.Plan(v, amqft.FunctionId.Rdft, n, rows, dtype=dtype, order=amqft.Order.Fast)
        if dtype == "f64" and v >= 5 and n > 256:
            assert plan.path()[0] != 6          # the whole-DAG kernel (bitwise) keeps these
            continue
        assert plan.path() == (6, 1), (v, n, dtype)
        got = run_plan(plan, xs)
        for row in (0, rows - 1):
            want = r.execute(v, O.F_RDFT, n, xs[row])
            err = r.rel_l2(got[row], want)
            assert err <= (1e-5 * math.log2(n) if dtype == "f32" else 1e-12), (v, n, dtype, err)
        # the packed spectrum against numpy: P[k] = Re X[k] (k <= N/2), P[N - k] = -Im X[k]
        f = np.fft.fft(xs[0])
        ref = np.concatenate([f.real[:n // 2 + 1], (-f.imag[1:n // 2])[::-1]])
        assert r.rel_l2(got[0], ref) <= (2e-6 if dtype == "f32" else 1e-13), (v, n, dtype)
        # inverse (DCT-0 / DST-0 sub-plans, csrc/inverse.cu) round trip
        back = run_plan(plan, got.astype(np.float32) if dtype == "f32" else got, inverse=True)
        assert r.rel_l2(back.ravel(), xs.ravel()) <= (1e-5 * math.log2(n) if dtype == "f32" else 1e-9), (v, n, dtype)


# ---- DCT-0 / DST-0 rows (FunctionId::Dct / Dst: N/2 + 1 / N/2 - 1 cells, oracle.hpp:38-41) on the
# two-factor kernel: the CDFT of the even / odd extension.  fp32 N = 512 .. 4096, fp64 256 .. 1024
# (above the scalar small kernels, where only the generic interpreter was left).
@pytest.mark.parametrize("n,dtype", [(512, "f32"), (1024, "f32"), (4096, "f32"), (256, "f64"), (1024, "f64")])
def test_tile_dct_dst_rows_match_cpu(oracle, restatement, n, dtype):
    r, O = restatement, oracle
    rows = 70
    for f in (O.F_DCT, O.F_DST):
        cells = amqft.cell_count(f, n)
        xs = np.random.default_rng(n + f).standard_normal((rows, cells))
        if dtype == "f32":
            xs = xs.astype(np.float32).astype(np.float64)
        for v in range(1, 9):
            plan = amqft.Plan(v, f, n, rows, dtype=dtype, order=amqft.Order.Fast)
            if dtype == "f64" and v >= 5 and n > 256:
                assert plan.path()[0] != 6
                continue
            assert plan.path() == (6, 1), (v, f, n, dtype)
            got = run_plan(plan, xs)
            for row in (0, rows - 1):
                want = r.execute(v, f, n, xs[row])
                err = r.rel_l2(got[row], want)
                assert err <= (1e-5 * math.log2(n) if dtype == "f32" else 1e-12), (v, f, n, dtype, err)
            # in place, and the inverse (weights + the same forward, csrc/inverse.cu) round trip
            t = torch.tensor(xs, dtype=torch.float32 if dtype == "f32" else torch.float64, device=DEV)
            plan.forward(t, t)
            torch.cuda.synchronize()
            assert np.array_equal(t.double().cpu().numpy(), got), (v, f, n, dtype)
            back = run_plan(plan, got.astype(np.float32) if dtype == "f32" else got, inverse=True)
            assert r.rel_l2(back.ravel(), xs.ravel()) <= (1e-5 * math.log2(n) if dtype == "f32" else 1e-9), (v, f, n)


@pytest.mark.parametrize("n", [4096, 1 << 15, 1 << 18])
def test_exec_is_cuda_graph_capturable(n):
    """include/amqft_b200.h: the device entry points allocate nothing and are
    stream-ordered -- a forward of the tile kernel (4096), the cluster tile
    kernel (2^15, cudaLaunchKernelEx) and the column-slab plan (2^18, two
    launches through the plan's scratch) captures into a CUDA graph and replays
    with the same bits."""
    rows = 6
    x = torch.tensor(np.random.default_rng(n + 5).standard_normal((rows, 2 * n)), dtype=torch.float32, device=DEV)
    plan = amqft.Plan(4, amqft.FunctionId.Cdft, n, rows, dtype="f32", order=amqft.Order.Fast)
    want = torch.empty_like(x)
    plan.forward(x, want)
    torch.cuda.synchronize()
    y = torch.zeros_like(x)
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(side):
        plan.forward(x, y, stream=side)          # warm-up on the capture stream
        side.synchronize()
        y.zero_()
        with torch.cuda.graph(g, stream=side):
            plan.forward(x, y, stream=side)
    torch.cuda.synchronize()
    assert float(y.abs().max()) == 0.0, "capture must not execute"
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(y, want)
