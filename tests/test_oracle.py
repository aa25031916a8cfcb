"""Pins the CPU oracle (oracle/amqft_oracle.c) before it is trusted.

1. Bitwise equality with the reference library compiled from its own sources
   (oracle/_ref/libamqft_ref.so) -- when it is built.
2. Bitwise equality with the committed golden fixtures generated from that
   library (tests/golden/make_golden.py) -- always (also on the GPU box).
3. The reference tests' own known-answer values (file:line cited).
"""
import math
import os

import numpy as np
import pytest

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def test_restatement_matches_reference_bitwise(oracle, restatement, reference):
    r, ref, O = restatement, reference, oracle
    for v in range(1, 9):
        for f in O.wired_functions(v):
            n = O.FUNCTION_BASE[f]
            while n <= 1024:
                t = O.FUNCTION_OPERAND[f]
                x = r.uniform(r.mix_seed(4242, v, f, n), r.cell_count(t, n))
                a, ma = r.execute(v, f, n, x, meter=True)
                b, mb = ref.execute(v, f, n, x, meter=True)
                assert a.tobytes() == b.tobytes(), (v, f, n)
                assert ma == mb, (v, f, n)
                n *= 2


def test_restatement_matches_reference_on_the_fly_and_large_table(oracle, restatement, reference):
    O = oracle
    for v in (1, 4, 6, 7):
        x = restatement.uniform(99 + v, 2 * 256)
        for kw in (dict(on_the_fly=True), dict(table_max_n=4096), dict(corrupt=True)):
            a = restatement.execute(v, O.F_CDFT, 256, x, **kw)
            b = reference.execute(v, O.F_CDFT, 256, x, **kw)
            assert a.tobytes() == b.tobytes(), (v, kw)


def test_restatement_pinned_at_config_sizes(oracle, restatement, reference):
    """Beyond N = 1024: the restatement is bitwise the compiled reference at
    config 2's N = 4096 (every wired function), at 2^13 and at 2^16 (CDFT,
    all 8 variants, meters too) and at 2^18 (CDFT v4) -- the sizes the GPU
    parity tests compare the device against."""
    r, ref, O = restatement, reference, oracle
    for v in range(1, 9):
        for f in O.wired_functions(v):
            t = O.FUNCTION_OPERAND[f]
            x = r.uniform(r.mix_seed(4096, v, f, 0), r.cell_count(t, 4096))
            a, ma = r.execute(v, f, 4096, x, meter=True)
            b, mb = ref.execute(v, f, 4096, x, meter=True)
            assert a.tobytes() == b.tobytes() and ma == mb, (v, f)
        for lg in (13, 16):
            n = 1 << lg
            x = r.uniform(r.mix_seed(lg, v, 0, n), 2 * n)
            a, ma = r.execute(v, O.F_CDFT, n, x, meter=True)
            b, mb = ref.execute(v, O.F_CDFT, n, x, meter=True)
            assert a.tobytes() == b.tobytes() and ma == mb, (v, lg)
    n = 1 << 18
    x = r.uniform(18, 2 * n)
    assert r.execute(4, O.F_CDFT, n, x).tobytes() == ref.execute(4, O.F_CDFT, n, x).tobytes()


def test_golden_config1(oracle, restatement):
    g = np.load(os.path.join(GOLD, "config1_cdft1024.npz"))
    x = g["input"]
    assert x.tobytes() == oracle.seeded_signal(1, oracle.CDFT, 1024, 0, restatement).tobytes()
    for v in range(1, 9):
        y, m = restatement.execute(v, oracle.F_CDFT, 1024, x, meter=True)
        assert y.tobytes() == g[f"v{v}"].tobytes(), v
        assert m == tuple(int(t) for t in g[f"meter_v{v}"])
    naive = restatement.naive(oracle.CDFT_FULL, 1024, x)
    assert np.array_equal(naive, g["naive_working"])
    ext = restatement.reference_spectrum(oracle.CDFT_FULL, 1024, x)
    assert np.array_equal(ext, g["extended"])


def test_golden_functions_small(oracle, restatement):
    g = np.load(os.path.join(GOLD, "functions_small.npz"))
    count = 0
    for key in g.files:
        if not key.startswith("x_"):
            continue
        _, v, f, n = key.split("_")
        v, f, n = int(v), int(f), int(n)
        y, m = restatement.execute(v, f, n, g[key], meter=True)
        assert y.tobytes() == g[f"y_{v}_{f}_{n}"].tobytes(), key
        assert m == tuple(int(t) for t in g[f"m_{v}_{f}_{n}"]), key
        count += 1
    assert count > 200


def test_golden_tables(restatement):
    g = np.load(os.path.join(GOLD, "tables.npz"))
    for v in range(1, 9):
        for m in (8, 16, 1024):
            assert np.array_equal(restatement.trig_constants(v, m), g[f"v{v}_{m}"])
    assert np.array_equal(restatement.uniform(12345, 64), g["uniform_seed12345"])
    assert restatement.mix_seed(1, 0, 1024, 0) == int(g["mix_seed_1_0_1024_0"][0])


def test_known_answers(oracle, restatement):
    r, O = restatement, oracle
    # variants_test.cpp:291-295 / oracle_test.cpp:48-56: CDFT N=2.
    for v in range(1, 9):
        assert list(r.execute(v, O.F_CDFT, 2, [1, 2, 3, 4])) == [4, 6, -2, -2]
        # variants_test.cpp:283-289: Dct N=2 [5,3] -> [8,2]
        assert list(r.execute(v, O.F_DCT, 2, [5, 3])) == [8, 2]
        # variants_test.cpp:298-304: OddOdd N=8, s(1)=2 -> 2*cos(pi/4), meter {0,1,0}
        y, m = r.execute(v, O.F_DCT_OO, 8, [2.0], meter=True)
        assert y[0] == 2.0 * r.base_constant() and m == (0, 1, 0)
    # oracle_test.cpp:58-88: RDFT N=4, DCT, DST pinned sums.
    assert np.allclose(r.naive(O.RDFT_FULL, 4, [1, 2, 3, 4]), [10, -2, -2, -2], atol=1e-15)
    assert np.allclose(r.naive(O.DCT_FULL, 4, [1, 2, 3]), [6, -2, 2], atol=1e-15)
    s = math.sqrt(2)
    assert np.allclose(r.naive(O.DST_FULL, 8, [1, 2, 3]), [2 * s + 2, -2, 2 * s - 2], atol=1e-14)
    # The fast transforms agree: RDFT N=4 via the recursion.
    for v in range(1, 9):
        assert np.allclose(r.execute(v, O.F_RDFT, 4, [1, 2, 3, 4]), [10, -2, -2, -2])
    # elaborations_test.cpp:323-355 constants; variants_test.cpp:221-246 tables.
    assert r.modulation_value(0, 1, 8) == pytest.approx(s, rel=1e-15)
    assert r.modulation_value(3, 2, 8) == pytest.approx(0.5, rel=1e-15)
    c16 = r.trig_constants(4, 16)
    for p in (1, 2, 3):
        assert c16[p - 1] == pytest.approx(1 / (2 * math.cos(2 * math.pi * p / 16)), rel=1e-15)
    assert c16[1] == pytest.approx(c16[3], rel=1e-15)


def test_measured_counts(oracle, restatement):
    """metering_test.cpp:108-135: pinned meters and closed forms."""
    r, O = restatement, oracle

    def measure(v, kind, n):
        x = r.uniform(r.mix_seed(1, v, kind, n), r.cell_count(O.KIND_TYPE[kind], n))
        return r.execute(v, [O.F_CDFT, O.F_RDFT, O.F_DCT, O.F_DST][kind], n, x, meter=True)[1]

    assert measure(1, O.CDFT, 16) == (148, 20, 4)
    assert measure(4, O.CDFT, 16) == (148, 20, 0)
    assert measure(1, O.DST, 16) == (19, 5, 1)
    assert measure(6, O.DCT, 64) == (185, 49, 0)
    for v in range(1, 9):
        for kind in range(4):
            n = 4
            while n <= 256:
                a, m, bt = r.predicted_cost(kind, n)
                got = measure(v, kind, n)
                assert got == (a, m, bt if v % 2 == 1 else 0), (v, kind, n)
                n *= 2


def test_accuracy_against_extended(oracle, restatement):
    """acceptance_test.cpp:131-185 tolerances at small N."""
    r, O = restatement, oracle
    for n in (8, 64, 256):
        x = O.seeded_signal(8101, O.CDFT, n, 0, r)
        for v in range(1, 9):
            y = r.execute(v, O.F_CDFT, n, x)
            err = r.rel_error_extended(O.CDFT_FULL, n, x, y)
            tol = 1e-10 if v <= 4 else (1e-8 if n <= 64 else 1e-6)
            assert err <= tol, (v, n, err)


def test_inverse_round_trip(oracle, restatement):
    r, O = restatement, oracle
    n = 256
    x = O.seeded_signal(5, O.CDFT, n, 0, r)
    for v in range(1, 9):
        y = r.execute(v, O.F_CDFT, n, x)
        back = r.inverse_cdft(v, n, y)
        assert r.rel_l2(back, x) < (1e-14 if v <= 4 else 1e-9)


def test_rejections(oracle, restatement):
    r, O = restatement, oracle
    with pytest.raises(O.OracleError):
        r.execute(0, O.F_CDFT, 8, np.zeros(16))
    with pytest.raises(O.OracleError):
        r.execute(2, O.F_DCT_ODD_TIME, 16, np.zeros(4))   # harmonic-major has no odd-time fn
    with pytest.raises(O.OracleError):
        r.execute(1, O.F_CDFT, 12, np.zeros(24))           # not a power of two
    with pytest.raises(O.OracleError):
        r.execute(1, O.F_DCT_OO, 4, np.zeros(1))           # below base size
