"""ctypes front end of the CPU parity oracle.

TEST INFRASTRUCTURE ONLY.  Imported by tests/, ``__graft_entry__.smoke()``
and bench.py's ``cpu_baseline`` / ``--impl reference`` legs -- never by the
product package ``paper_1404_1810_b200`` (which fails loudly without its
CUDA library instead of falling back to anything here).

Two back ends share one interface:

* ``Restatement`` -- ``oracle/liboracle.so``, our C restatement of the
  reference recursion (``oracle/amqft_oracle.c``, every function citing the
  reference file:line it follows);
* ``Reference``   -- ``oracle/_ref/libamqft_ref.so``, the unmodified
  reference library compiled from ``/root/reference/proj/src`` by
  ``oracle/Makefile`` (present wherever it was built; it travels to the GPU
  box with the repo snapshot).

Enumerations follow the reference's declaration order
(``include/amqft/signal.hpp:28-48``, ``include/amqft/variants.hpp:55-66``).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))

# SignalType (signal.hpp:28-48)
CDFT_FULL, RDFT_FULL, DCT_FULL = 0, 1, 2
DCT_ODD_TIME, DCT_ODD_HARM, DCT_OO = 4, 6, 9
DST_FULL, DST_ODD_TIME, DST_ODD_HARM, DST_OO = 10, 12, 14, 17
# TransformKind (signal.hpp:18)
CDFT, RDFT, DCT, DST = 0, 1, 2, 3
# FunctionId (variants.hpp:55-66)
F_CDFT, F_RDFT, F_DCT, F_DST = 0, 1, 2, 3
F_DCT_ODD_TIME, F_DST_ODD_TIME, F_DCT_ODD_HARM, F_DST_ODD_HARM = 4, 5, 6, 7
F_DCT_OO, F_DST_OO = 8, 9
FUNCTION_OPERAND = [CDFT_FULL, RDFT_FULL, DCT_FULL, DST_FULL, DCT_ODD_TIME,
                    DST_ODD_TIME, DCT_ODD_HARM, DST_ODD_HARM, DCT_OO, DST_OO]
FUNCTION_BASE = [2, 2, 2, 4, 4, 4, 4, 4, 8, 8]
KIND_TYPE = [CDFT_FULL, RDFT_FULL, DCT_FULL, DST_FULL]


def time_major(v: int) -> bool:
    """variants.cpp:32-35."""
    return v in (1, 4, 5, 8)


def wired_functions(v: int):
    """Functions build_plan(v) wires (variants.cpp:184-231)."""
    odd = (F_DCT_ODD_TIME, F_DST_ODD_TIME) if time_major(v) else (F_DCT_ODD_HARM, F_DST_ODD_HARM)
    return [F_CDFT, F_RDFT, F_DCT, F_DST, *odd, F_DCT_OO, F_DST_OO]


_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(dtype=np.uint64, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
_sz = C.c_size_t


class OracleError(ValueError):
    """Mirrors the reference's std::invalid_argument."""


class _Backend:
    prefix = ""
    path = ""

    def __init__(self):
        if not os.path.exists(self.path):
            raise FileNotFoundError(
                f"{self.path} is missing: run `make -C oracle` (python -c 'import __graft_entry__ as g; g.build()')")
        self.lib = C.CDLL(self.path)
        p = self.prefix
        f = getattr(self.lib, p + "execute")
        f.argtypes = [C.c_int, C.c_int, _sz, _dp, _dp, _sz, C.c_int, C.c_int, C.c_void_p]
        f.restype = C.c_int
        self._exec = f
        err = getattr(self.lib, p + "last_error")
        err.restype = C.c_char_p
        self._err = err
        cc = getattr(self.lib, p + "cell_count")
        cc.argtypes = [C.c_int, _sz]
        cc.restype = _sz
        self._cc = cc
        mix = getattr(self.lib, p + "mix_seed")
        mix.argtypes = [C.c_uint64] * 4
        mix.restype = C.c_uint64
        self._mix = mix
        uf = getattr(self.lib, p + "uniform_fill")
        uf.argtypes = [C.c_uint64, _sz, _dp]
        uf.restype = None
        self._uf = uf
        tc = getattr(self.lib, p + "trig_constants")
        tc.argtypes = [C.c_int, _sz, _dp]
        tc.restype = C.c_int
        self._tc = tc
        pc = getattr(self.lib, p + "predicted_cost")
        pc.argtypes = [C.c_int, _sz, _i64p]
        pc.restype = C.c_int
        self._pc = pc

    def _check(self, rc):
        if rc != 0:
            raise OracleError(self._err().decode())

    def cell_count(self, signal_type: int, n: int) -> int:
        return int(self._cc(signal_type, n))

    def execute(self, v: int, f: int, n: int, x, *, table_max_n: int = 0,
                on_the_fly: bool = False, corrupt: bool = False, meter: bool = False):
        """amqft::execute(v, f, input, trig[, meter]) on one signal."""
        x = np.ascontiguousarray(x, dtype=np.float64)
        cells = self.cell_count(FUNCTION_OPERAND[f], n) if f in range(10) else 0
        if cells == 0 or x.size != cells:
            if f not in range(10):
                raise OracleError("unknown function")
            if cells != 0:
                raise OracleError(f"expected {cells} cells, got {x.size}")
        out = np.zeros(max(cells, 1), dtype=np.float64)
        m = np.zeros(3, dtype=np.uint64)
        rc = self._exec(v, f, n, x if x.size else np.zeros(1), out, table_max_n,
                        int(on_the_fly), int(corrupt), m.ctypes.data if meter else None)
        self._check(rc)
        out = out[:cells]
        return (out, tuple(int(t) for t in m)) if meter else out

    def mix_seed(self, base, a=0, b=0, c=0) -> int:
        return int(self._mix(base, a, b, c))

    def uniform(self, seed: int, count: int) -> np.ndarray:
        out = np.empty(count, dtype=np.float64)
        self._uf(seed, count, out)
        return out

    def trig_constants(self, v: int, max_n: int) -> np.ndarray:
        out = np.empty(max_n // 4, dtype=np.float64)
        self._check(self._tc(v, max_n, out))
        return out

    def predicted_cost(self, kind: int, n: int):
        out = np.zeros(3, dtype=np.int64)
        self._check(self._pc(kind, n, out))
        return tuple(int(t) for t in out)


class Restatement(_Backend):
    """oracle/amqft_oracle.c -- our CPU restatement."""
    prefix = "oracle_"
    path = os.path.join(HERE, "liboracle.so")

    def __init__(self):
        super().__init__()
        lib = self.lib
        lib.oracle_inverse_cdft.argtypes = [C.c_int, _sz, _dp, _dp]
        lib.oracle_inverse_cdft.restype = C.c_int
        lib.oracle_reference_spectrum.argtypes = [C.c_int, _sz, _dp, _dp]
        lib.oracle_reference_spectrum.restype = C.c_int
        lib.oracle_naive_working.argtypes = [C.c_int, _sz, _dp, _dp]
        lib.oracle_naive_working.restype = C.c_int
        lib.oracle_rel_error_extended.argtypes = [C.c_int, _sz, _dp, _dp]
        lib.oracle_rel_error_extended.restype = C.c_double
        lib.oracle_rel_l2.argtypes = [_sz, _dp, _dp]
        lib.oracle_rel_l2.restype = C.c_double
        lib.oracle_modulation_value.argtypes = [C.c_int, _sz, _sz]
        lib.oracle_modulation_value.restype = C.c_double
        lib.oracle_base_constant.restype = C.c_double

    def inverse_cdft(self, v: int, n: int, spectrum) -> np.ndarray:
        """Swap-trick inverse on top of the reference forward."""
        x = np.ascontiguousarray(spectrum, dtype=np.float64)
        out = np.empty(2 * n, dtype=np.float64)
        self._check(self.lib.oracle_inverse_cdft(v, n, x, out))
        return out

    def inverse_real(self, v: int, f: int, n: int, spectrum) -> np.ndarray:
        """Builder-defined inverses of the real transforms on top of the
        reference forward (csrc/inverse.cu): DCT-0 (4/N) W DCT(W C), DST-0
        (4/N) DST(S), RDFT through both on the split packed spectrum; the
        same operations in the same order as the device."""
        y = np.ascontiguousarray(spectrum, dtype=np.float64)
        h = n // 2
        if f == F_DST:
            return self.execute(v, F_DST, n, y) * (4.0 / n)
        w = np.ones(h + 1)
        w[0] = w[-1] = 0.5
        if f == F_DCT:
            sc = np.full(h + 1, 4.0 / n)
            sc[0] = sc[-1] = 2.0 / n
            return self.execute(v, F_DCT, n, y * w) * sc
        assert f == F_RDFT
        c = self.execute(v, F_DCT, n, y[:h + 1] * w) * (4.0 / n)
        s = self.execute(v, F_DST, n, y[h + 1:][::-1].copy()) * (4.0 / n)
        x = np.empty(n)
        x[0], x[h] = c[0] * 0.5, c[h] * 0.5
        m = np.arange(1, h)
        x[m] = (c[m] + s[m - 1]) * 0.5
        x[n - m] = (c[m] - s[m - 1]) * 0.5
        return x

    def reference_spectrum(self, signal_type: int, n: int, x) -> np.ndarray:
        x = np.ascontiguousarray(x, dtype=np.float64)
        out = np.empty(self.cell_count(signal_type, n), dtype=np.float64)
        self._check(self.lib.oracle_reference_spectrum(signal_type, n, x, out))
        return out

    def naive(self, signal_type: int, n: int, x) -> np.ndarray:
        """pruned_transform(..., Working): the naive O(N^2) fp64 DFT."""
        x = np.ascontiguousarray(x, dtype=np.float64)
        out = np.empty(self.cell_count(signal_type, n), dtype=np.float64)
        self._check(self.lib.oracle_naive_working(signal_type, n, x, out))
        return out

    def rel_error_extended(self, signal_type: int, n: int, x, got) -> float:
        return float(self.lib.oracle_rel_error_extended(
            signal_type, n, np.ascontiguousarray(x, dtype=np.float64),
            np.ascontiguousarray(got, dtype=np.float64)))

    def rel_l2(self, got, want) -> float:
        got = np.ascontiguousarray(got, dtype=np.float64).ravel()
        want = np.ascontiguousarray(want, dtype=np.float64).ravel()
        return float(self.lib.oracle_rel_l2(got.size, got, want))

    def modulation_value(self, kind: int, index: int, n: int) -> float:
        return float(self.lib.oracle_modulation_value(kind, index, n))

    def base_constant(self) -> float:
        return float(self.lib.oracle_base_constant())


class Reference(_Backend):
    """oracle/_ref/libamqft_ref.so -- the unmodified reference library."""
    prefix = "ref_"
    path = os.path.join(HERE, "_ref", "libamqft_ref.so")

    def __init__(self):
        super().__init__()
        lib = self.lib
        lib.ref_execute_rows.argtypes = [C.c_int, C.c_int, _sz, _sz, _dp, _dp, C.c_int]
        lib.ref_execute_rows.restype = C.c_int
        lib.ref_pruned_transform.argtypes = [C.c_int, _sz, _dp, _dp, C.c_int]
        lib.ref_pruned_transform.restype = C.c_int
        lib.ref_measure.argtypes = [C.c_int, C.c_int, _sz, C.c_uint64, _u64p]
        lib.ref_measure.restype = C.c_int
        lib.ref_measure_accuracy.argtypes = [C.c_int, C.c_int, _sz, C.c_int, C.c_uint64, _dp]
        lib.ref_measure_accuracy.restype = C.c_int

    def execute_rows(self, v: int, kind: int, n: int, rows, threads: int) -> np.ndarray:
        rows = np.ascontiguousarray(rows, dtype=np.float64)
        out = np.empty_like(rows)
        cells = self.cell_count(KIND_TYPE[kind], n)
        nrows = rows.size // cells
        self._check(self.lib.ref_execute_rows(v, kind, n, nrows, rows, out, threads))
        return out

    def pruned_transform(self, signal_type: int, n: int, x, extended: bool) -> np.ndarray:
        x = np.ascontiguousarray(x, dtype=np.float64)
        out = np.empty(self.cell_count(signal_type, n), dtype=np.float64)
        self._check(self.lib.ref_pruned_transform(signal_type, n, x, out, int(extended)))
        return out

    def measure(self, v: int, kind: int, n: int, seed: int = 1):
        out = np.zeros(3, dtype=np.uint64)
        self._check(self.lib.ref_measure(v, kind, n, seed, out))
        return tuple(int(t) for t in out)

    def measure_accuracy(self, v, kind, n, trials, seed):
        out = np.zeros(2, dtype=np.float64)
        self._check(self.lib.ref_measure_accuracy(v, kind, n, trials, seed, out))
        return float(out[0]), float(out[1])


_cache = {}


def restatement() -> Restatement:
    if "r" not in _cache:
        _cache["r"] = Restatement()
    return _cache["r"]


def reference():
    """The compiled reference, or None where it was never built."""
    if "ref" not in _cache:
        try:
            _cache["ref"] = Reference()
        except (FileNotFoundError, OSError):
            _cache["ref"] = None
    return _cache["ref"]


def seeded_signal(seed: int, kind: int, n: int, trial: int, backend=None) -> np.ndarray:
    """The accuracy harness' input: UniformSource(mix_seed(seed, kind, n,
    trial)).fill(...) (accuracy.cpp:20-28)."""
    b = backend or restatement()
    cells = b.cell_count(KIND_TYPE[kind], n)
    return b.uniform(b.mix_seed(seed, kind, n, trial), cells)
