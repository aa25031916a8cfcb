"""Drop-in boundary: the reference's own callers on the B200 library.

oracle/_ref/libamqft_dropin.so is the reference's unmodified caller sources
(src/metering.cpp `measure`, src/accuracy.cpp `measure_accuracy` /
`ordering_check`, src/oracle.cpp) plus the same extern "C" wrapper as the
reference build (oracle/ref_capi.cpp), compiled against OUR headers
(include/amqft/*.hpp -> include/amqft_b200.hpp) and linked to
libamqft_b200.so (oracle/Makefile).  Every `amqft::execute` those callers
make runs on the device.  The tests compare it call for call with
oracle/_ref/libamqft_ref.so, the same wrapper over the reference library:

* host metadata (layout, traits, wiring, TrigTable, the naive DFT computed
  on our layout) -- CPU, no device;
* every transform, meter and accuracy figure -- bitwise, on the GPU.
"""
import ctypes as C
import os

import numpy as np
import pytest

from oracle import oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DROPIN = os.path.join(ROOT, "oracle", "_ref", "libamqft_dropin.so")
_szp = np.ctypeslib.ndpointer(dtype=np.uintp, flags="C_CONTIGUOUS")


class Wrapper(O.Reference):
    """The ref_capi.cpp entry points of one build (reference or drop-in)."""

    def __init__(self, path=None):
        if path is not None:
            self.path = path
        super().__init__()
        L = self.lib
        L.ref_ordering_check.argtypes = [C.c_int, C.c_size_t, C.c_int, C.c_uint64,
                                         np.ctypeslib.ndpointer(np.float64), np.ctypeslib.ndpointer(np.int32)]
        L.ref_stored_range.argtypes = [C.c_int, C.c_size_t, C.c_int, _szp]
        L.ref_type_info.argtypes = [C.c_int, np.ctypeslib.ndpointer(np.int32), C.c_char_p, C.c_size_t]
        L.ref_plan_encode.argtypes = [C.c_int, np.ctypeslib.ndpointer(np.int64), C.c_int]
        L.ref_trig_value.argtypes = [C.c_int, C.c_size_t, C.c_int, C.c_int, C.c_int, C.c_size_t, C.c_size_t,
                                     np.ctypeslib.ndpointer(np.float64)]
        L.ref_modulation_value.argtypes = [C.c_int, C.c_size_t, C.c_size_t]
        L.ref_modulation_value.restype = C.c_double
        for name in ("ref_ordering_check", "ref_stored_range", "ref_type_info", "ref_plan_encode", "ref_trig_value"):
            getattr(L, name).restype = C.c_int

    def err(self):
        return self._err().decode()

    def stored_range(self, t, n, freq):
        out = np.zeros(3, dtype=np.uintp)
        rc = self.lib.ref_stored_range(t, n, int(freq), out)
        return None if rc else tuple(int(v) for v in out)

    def type_info(self, t):
        out = np.zeros(4, dtype=np.int32)
        name = C.create_string_buffer(64)
        rc = self.lib.ref_type_info(t, out, name, 64)
        return None if rc else (tuple(int(v) for v in out), name.value.decode())

    def plan(self, v):
        out = np.zeros(512, dtype=np.int64)
        k = self.lib.ref_plan_encode(v, out, out.size)
        return None if k < 0 else out[:k].tolist()

    def trig_value(self, v, max_n, otf, corrupt, kind, idx, m):
        out = np.zeros(1)
        rc = self.lib.ref_trig_value(v, max_n, int(otf), int(corrupt), kind, idx, m, out)
        return None if rc else out[0]

    def constants(self, v, max_n):
        out = np.zeros(max_n // 4)
        self._check(self._tc(v, max_n, out))
        return out

    def ordering(self, kind, n, trials, seed):
        out = np.zeros(17)
        flags = np.zeros(4, dtype=np.int32)
        self._check(self.lib.ref_ordering_check(kind, n, trials, seed, out, flags))
        return out, tuple(int(f) for f in flags)

    def cost(self, kind, n):
        out = np.zeros(3, dtype=np.int64)
        rc = self._pc(kind, n, out)
        return None if rc else tuple(int(v) for v in out)


@pytest.fixture(scope="module")
def pair():
    if not os.path.exists(DROPIN) or not os.path.exists(Wrapper.path):
        pytest.skip("drop-in / reference builds absent (built by oracle/Makefile where /root/reference exists)")
    return Wrapper(), Wrapper(DROPIN)


SIZES = [2, 4, 8, 16, 32, 64, 128, 1024]


# ------------------------------------------------------------------ CPU

def test_dropin_library_is_linked_to_the_product(pair):
    """The drop-in build resolves amqft::execute from libamqft_b200.so (the
    reference library is not in it)."""
    import subprocess
    out = subprocess.run(["ldd", DROPIN], capture_output=True, text=True).stdout
    assert "libamqft_b200.so" in out
    syms = subprocess.run(["nm", "-D", "--defined-only", DROPIN], capture_output=True, text=True).stdout
    assert "_ZN5amqft7executeE" not in syms          # execute is not defined in the caller build
    und = subprocess.run(["nm", "-D", "--undefined-only", DROPIN], capture_output=True, text=True).stdout
    assert "_ZN5amqft7executeE" in und


def test_layout_metadata_matches_reference(pair):
    ref, ours = pair
    for t in range(18):
        assert ref.type_info(t) == ours.type_info(t), t
        for n in [0, 1, 2, 3, 4, 6, 8, 16, 64, 1 << 20]:
            for freq in (0, 1):
                assert ref.stored_range(t, n, freq) == ours.stored_range(t, n, freq), (t, n, freq)
            assert ref.cell_count(t, n) == ours.cell_count(t, n), (t, n)


def test_wiring_and_trig_table_match_reference(pair):
    ref, ours = pair
    for v in range(1, 9):
        assert ref.plan(v) == ours.plan(v), v
        for max_n in (8, 16, 1024, 1 << 16):
            assert ref.constants(v, max_n).tobytes() == ours.constants(v, max_n).tobytes(), (v, max_n)
        for k in range(4):
            for (mx, idx, m) in [(1024, 1, 16), (1024, 3, 256), (1024, 255, 1024), (16, 1, 32), (64, 0, 64),
                                 (64, 16, 64), (64, 5, 48)]:
                for otf in (0, 1):
                    for corrupt in (0, 1):
                        a = ref.trig_value(v, mx, otf, corrupt, k, idx, m)
                        b = ours.trig_value(v, mx, otf, corrupt, k, idx, m)
                        assert (a is None) == (b is None), (v, k, mx, idx, m, otf)
                        if a is not None:
                            assert np.float64(a).tobytes() == np.float64(b).tobytes(), (v, k, mx, idx, m)
    for k in range(4):
        for (idx, n) in [(1, 16), (7, 1024), (1000, 4096)]:
            assert ref.lib.ref_modulation_value(k, idx, n) == ours.lib.ref_modulation_value(k, idx, n)


def test_reference_naive_dft_on_our_layout(pair):
    """src/oracle.cpp (the callers' naive DFT) compiled on our layout
    functions gives the reference's bits; predicted_cost likewise."""
    ref, ours = pair
    rng = np.random.default_rng(5)
    for t in range(18):
        for n in (8, 16, 64):
            cells = ref.cell_count(t, n)
            if cells == 0:
                continue
            x = rng.uniform(-1, 1, cells)
            for ext in (False, True):
                assert ref.pruned_transform(t, n, x, ext).tobytes() == ours.pruned_transform(t, n, x, ext).tobytes()
    for kind in range(4):
        for n in (2, 4, 16, 1024, 1 << 20):
            assert ref.cost(kind, n) == ours.cost(kind, n)


def test_execute_without_device_raises_not_computes(pair):
    """No CUDA device here: the drop-in execute fails (runtime_error from
    AMQFT_ECUDA), it never computes on the host."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("device present")
    _, ours = pair
    x = np.zeros(2 * 16)
    with pytest.raises(O.OracleError, match="CUDA"):
        ours.execute(4, O.F_CDFT, 16, x)


# ------------------------------------------------------------------ GPU

@pytest.mark.gpu
def test_dropin_execute_bitwise_all_functions(pair):
    ref, ours = pair
    for v in range(1, 9):
        for f in O.wired_functions(v):
            n = O.FUNCTION_BASE[f]
            while n <= 1024:
                t = O.FUNCTION_OPERAND[f]
                x = ref.uniform(ref.mix_seed(77, v, f, n), ref.cell_count(t, n))
                a, ma = ref.execute(v, f, n, x, meter=True)
                b, mb = ours.execute(v, f, n, x, meter=True)
                assert a.tobytes() == b.tobytes(), (v, f, n)
                assert ma == mb, (v, f, n)
                n *= 4 if n >= 64 else 2
        # unwired functions raise in both
        for f in range(10):
            if f not in O.wired_functions(v):
                with pytest.raises(O.OracleError):
                    ref.execute(v, f, 16, np.zeros(4))
                with pytest.raises(O.OracleError):
                    ours.execute(v, f, 16, np.zeros(4))


@pytest.mark.gpu
def test_dropin_execute_trig_modes_and_errors(pair):
    ref, ours = pair
    x = ref.uniform(11, 2 * 256)
    for v in (1, 4, 5, 6):
        for kw in (dict(on_the_fly=True), dict(table_max_n=4096), dict(corrupt=True),
                   dict(table_max_n=4096, on_the_fly=True, corrupt=True)):
            assert ref.execute(v, O.F_CDFT, 256, x, **kw).tobytes() == \
                ours.execute(v, O.F_CDFT, 256, x, **kw).tobytes(), (v, kw)
    # a table smaller than the transform: both reject (TrigTable::value)
    for lib in (ref, ours):
        with pytest.raises(O.OracleError):
            lib.execute(4, O.F_CDFT, 256, x, table_max_n=64)


@pytest.mark.gpu
def test_dropin_execute_large_n_against_reference(pair):
    """Config 2 / 3 sizes straight against the compiled reference (not the
    restatement): CDFT N = 4096, 2^13, 2^16, all 8 variants, bitwise."""
    ref, ours = pair
    for n in (4096, 1 << 13, 1 << 16):
        for v in range(1, 9):
            x = ref.uniform(ref.mix_seed(3, v, 0, n), 2 * n)
            assert ref.execute(v, O.F_CDFT, n, x).tobytes() == ours.execute(v, O.F_CDFT, n, x).tobytes(), (n, v)


@pytest.mark.gpu
def test_dropin_measure_and_accuracy_bitwise(pair):
    """metering.cpp measure() and accuracy.cpp measure_accuracy() /
    ordering_check() -- the reference's own code -- give identical numbers
    when their execute() runs on the device."""
    ref, ours = pair
    for v in range(1, 9):
        for kind in range(4):
            for n in (16, 256, 4096):
                assert ref.measure(v, kind, n, 1) == ours.measure(v, kind, n, 1), (v, kind, n)
            for n in (64, 1024):
                a = ref.measure_accuracy(v, kind, n, 2, 7)
                b = ours.measure_accuracy(v, kind, n, 2, 7)
                assert np.array(a).tobytes() == np.array(b).tobytes(), (v, kind, n)
    for kind in (0, 3):
        a, fa = ref.ordering(kind, 256, 2, 1)
        b, fb = ours.ordering(kind, 256, 2, 1)
        assert a.tobytes() == b.tobytes() and fa == fb


@pytest.mark.gpu
def test_dropin_execute_rows_threads(pair):
    """The reference's per-signal loop (ref_execute_rows: one TrigTable per
    thread, execute per row) on 8 host threads through the device library."""
    ref, ours = pair
    rows = ref.uniform(5, 64 * 2 * 512).reshape(64, -1)
    a = ref.execute_rows(4, 0, 512, rows, 8)
    b = ours.execute_rows(4, 0, 512, rows, 8)
    assert a.tobytes() == b.tobytes()
