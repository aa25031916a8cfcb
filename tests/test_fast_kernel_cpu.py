"""CPU checks of the fused fast kernel's formulation and generated code.

* tests/fast_model.py -- recursive and phase-structured numpy models of the
  index-space formulation, bitwise against the oracle.
* tests/kernel_emu.py -- the kernel's phases with the generated straight-
  line functions (csrc/gen/fast_gen.cuh, generated at build time, compiled as host C++), bitwise.
"""
import pytest

from fast_model import (fast_cdft_harmonic_major, fast_cdft_time_major, phased_harmonic_major,
                        phased_time_major)
from kernel_emu import emulate


@pytest.mark.parametrize("v", range(1, 9))
def test_models_bitwise(oracle, restatement, v):
    r, O = restatement, oracle
    for n in (8, 16, 64, 256):
        x = O.seeded_signal(7, O.CDFT, n, v, r)
        want = r.execute(v, O.F_CDFT, n, x).tobytes()
        tab = r.trig_constants(v, n)
        f = fast_cdft_time_major if v in (1, 4, 5, 8) else fast_cdft_harmonic_major
        assert f(v, n, x, tab, n, r.base_constant()).tobytes() == want, n
    for n, lb in ((256, 16), (1024, 32)):
        x = O.seeded_signal(8, O.CDFT, n, v, r)
        want = r.execute(v, O.F_CDFT, n, x).tobytes()
        f = phased_time_major if v in (1, 4, 5, 8) else phased_harmonic_major
        assert f(v, n, x, r.trig_constants(v, n), n, r.base_constant(), lb).tobytes() == want


@pytest.mark.parametrize("v", range(1, 9))
@pytest.mark.parametrize("n,lb", [(1024, 64), (2048, 64), (4096, 64), (8192, 64)])
def test_kernel_emulator_bitwise(oracle, restatement, v, n, lb):
    r, O = restatement, oracle
    x = O.seeded_signal(9, O.CDFT, n, 100 + v, r)
    want = r.execute(v, O.F_CDFT, n, x)
    got = emulate(v, n, lb, x, r.trig_constants(v, n), r.base_constant())
    assert got.tobytes() == want.tobytes()
