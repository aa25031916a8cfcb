"""CPU model of the in-shared-memory four-step (csrc/tile_kernel.cuh): the
kernel's index algebra -- two and three factors, decimation in frequency,
twiddles w_N^(n2 k1) / w_M^(n3 k2) -- restated in numpy over the ORACLE's
AM-QFT sub-transforms, and checked against the oracle's full-length transform
of the same variant.  Runs without a GPU; the device kernels themselves are
checked in tests/test_gpu_tile.py."""
import numpy as np
import pytest


def _cplx(x):
    return x[0::2] + 1j * x[1::2]


def _interleave(z):
    out = np.empty(2 * z.size)
    out[0::2], out[1::2] = z.real, z.imag
    return out


def _sub(r, O, v, n, z):
    """AM-QFT of length n (the oracle) of one complex vector."""
    return _cplx(r.execute(v, O.F_CDFT, n, _interleave(z)))


def two_factor(r, O, v, x, n1, n2):
    """n = N2 n1 + n2, k = k1 + N1 k2 (tile_kernel.cuh k_tile)."""
    n = n1 * n2
    a = x.reshape(n1, n2)                       # a[n1][n2]
    p = np.empty((n1, n2), dtype=complex)       # phase A: P[k1][n2]
    for c in range(n2):
        p[:, c] = _sub(r, O, v, n1, a[:, c]) * np.exp(-2j * np.pi * c * np.arange(n1) / n)
    out = np.empty(n, dtype=complex)            # phase B: X[k1 + N1 k2]
    for k1 in range(n1):
        out[k1::n1] = _sub(r, O, v, n2, p[k1])
    return out


def three_factor(r, O, v, x, n1, n2, n3):
    """n = N2 N3 n1 + N3 n2 + n3, k = k1 + N1 k2 + N1 N2 k3 (k_tile3)."""
    m, n = n2 * n3, n1 * n2 * n3
    a = x.reshape(n1, m)
    y = np.empty((n1, n2, n3), dtype=complex)
    for c in range(m):                          # phase A: Y[k1][n2][n3], times w_N^(m k1)
        y[:, c // n3, c % n3] = _sub(r, O, v, n1, a[:, c]) * np.exp(-2j * np.pi * c * np.arange(n1) / n)
    for k1 in range(n1):                        # phase B: in place over n2, times w_M^(n3 k2)
        for c in range(n3):
            y[k1, :, c] = _sub(r, O, v, n2, y[k1, :, c]) * np.exp(-2j * np.pi * c * np.arange(n2) / m)
    out = np.empty(n, dtype=complex)
    for k1 in range(n1):                        # phase C: X[k1 + N1 (k2 + N2 k3)]
        for k2 in range(n2):
            out[k1 + n1 * k2::n1 * n2] = _sub(r, O, v, n3, y[k1, k2])
    return out


@pytest.mark.parametrize("v", [1, 2, 4])
@pytest.mark.parametrize("split", [(4, 4), (4, 8), (8, 16), (16, 32), (64, 32)])
def test_two_factor_split_matches_the_full_transform(oracle, restatement, v, split):
    r, O = restatement, oracle
    n = split[0] * split[1]
    x = O.seeded_signal(51, O.CDFT, n, v, r)
    want = _cplx(r.execute(v, O.F_CDFT, n, x))
    got = two_factor(r, O, v, _cplx(x), *split)
    assert np.linalg.norm(got - want) / np.linalg.norm(want) <= 1e-13
    assert np.linalg.norm(got - np.fft.fft(_cplx(x))) / np.linalg.norm(want) <= 1e-13


@pytest.mark.parametrize("split", [(8, 16, 16), (32, 16, 16)])
def test_three_factor_split_matches_the_full_transform(oracle, restatement, split):
    r, O = restatement, oracle
    n = split[0] * split[1] * split[2]
    x = O.seeded_signal(52, O.CDFT, n, 0, r)
    want = _cplx(r.execute(4, O.F_CDFT, n, x))
    got = three_factor(r, O, 4, _cplx(x), *split)
    assert np.linalg.norm(got - want) / np.linalg.norm(want) <= 1e-13


def test_sine_variants_are_stable_inside_the_factors(oracle, restatement):
    """Why variants 5-8 need no fp64 compute on this path: the reference's own
    v5-8 error explodes with N but stays ~1e-15 up to the factor
    sizes the kernel uses (<= 64), so the split result is closer to the DFT
    than the reference's full-length result."""
    r, O = restatement, oracle
    n = 4096
    x = O.seeded_signal(53, O.CDFT, n, 0, r)
    f = np.fft.fft(_cplx(x))
    for v in (5, 6, 7, 8):
        full = _cplx(r.execute(v, O.F_CDFT, n, x))
        split = two_factor(r, O, v, _cplx(x), 64, 64)
        e_full = np.linalg.norm(full - f) / np.linalg.norm(f)
        e_split = np.linalg.norm(split - f) / np.linalg.norm(f)
        assert e_split <= 1e-13 < e_full, (v, e_split, e_full)
