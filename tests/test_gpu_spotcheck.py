"""Independent checks of the transforms the CPU oracle cannot reach (SURVEY
§8(c)-(d)): direct per-bin DFT sums on the device with exact integer phase
reduction (amqft_direct_bins, csrc/verify.cu; the reference naive DFT's
discipline, src/oracle.cpp:30-35) against config 4 (N = 2^24) and config 5
(N = 2^30, the distributed four-step on one GPU), all 8 variants at 2^24."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_1404_1810_b200 as amqft  # noqa: E402
from paper_1404_1810_b200.dist import DistFourStep  # noqa: E402

DEV = "cuda:0"


def spot_bins(n, count=64, seed=1):
    rng = np.random.default_rng(seed)
    edge = [0, 1, 2, n // 4, n // 2 - 1, n // 2, n // 2 + 1, n - 1]
    return np.unique(np.concatenate([edge, rng.integers(0, n, count - len(edge))])).astype(np.uint64)


def rel(got, want):
    return float(np.linalg.norm(got - want) / np.linalg.norm(want))


def test_direct_bins_against_numpy():
    """The checker itself: fp64 direct bins of a 2^12 signal equal numpy's
    FFT to ~1e-15 (strided slab layout too)."""
    n = 4096
    x = torch.randn(2 * n, dtype=torch.float64, device=DEV)
    xc = x.cpu().numpy()
    ref = np.fft.fft(xc[0::2] + 1j * xc[1::2])
    bins = spot_bins(n)
    got = amqft.direct_bins(x, n, bins)
    assert rel(got, ref[bins.astype(np.int64)]) < 1e-14
    # column slab: rows = 64 columns i2 of length 64, sample (r, c) = x[r + 64 c]
    slab = x.view(64, 64, 2).permute(1, 0, 2).contiguous()
    got = amqft.direct_bins(slab, n, bins, rows=64, row_len=64, stride=64)
    assert rel(got, ref[bins.astype(np.int64)]) < 1e-14
    f32 = x.float()
    got = amqft.direct_bins(f32, n, bins)
    ref32 = np.fft.fft(f32.double().cpu().numpy()[0::2] + 1j * f32.double().cpu().numpy()[1::2])
    assert rel(got, ref32[bins.astype(np.int64)]) < 1e-14


@pytest.mark.parametrize("v", range(1, 9))
def test_config4_spot_bins_all_variants(v):
    n = 1 << 24
    g = torch.Generator(device=DEV).manual_seed(24)
    x = torch.randn(1, 2 * n, generator=g, device=DEV)
    y = torch.empty_like(x)
    plan = amqft.Plan(v, amqft.FunctionId.Cdft, n, 1, dtype="f32", order=amqft.Order.Fast)
    plan.forward(x, y)
    torch.cuda.synchronize()
    bins = spot_bins(n, seed=v)
    want = amqft.direct_bins(x, n, bins)
    yc = y.view(-1, 2)[torch.as_tensor(bins.astype(np.int64), device=DEV)].double().cpu().numpy()
    got = yc[:, 0] + 1j * yc[:, 1]
    assert rel(got, want) <= 1e-5 * 24, v


def test_config5_spot_bins_one_gpu():
    """N = 2^30 through the distributed four-step (world 1): 64 output bins
    against their direct sums over the 2^30 input samples."""
    n = 1 << 30
    d = DistFourStep(4, n, device=0, trig_mode=amqft.TrigMode.OnTheFly, world=1, rank=0)
    g = torch.Generator(device=DEV).manual_seed(30)
    a0 = torch.randn(d.rows1, 2 * d.n1, generator=g, device=DEV)
    a = a0.clone()
    z = d.forward(a)
    torch.cuda.synchronize()
    bins = spot_bins(n, seed=30)
    # input slab: row i2 holds x[n2 i1 + i2] along i1
    want = amqft.direct_bins(a0, n, bins, rows=d.rows1, row_len=d.n1, stride=d.n2)
    k1 = torch.as_tensor((bins % d.n1).astype(np.int64), device=DEV)
    k2 = torch.as_tensor((bins // d.n1).astype(np.int64), device=DEV)
    zc = z.view(d.w, d.n2, 2)[k1, k2].double().cpu().numpy()
    got = zc[:, 0] + 1j * zc[:, 1]
    assert rel(got, want) <= 1e-5 * 30
