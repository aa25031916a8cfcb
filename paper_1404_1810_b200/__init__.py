"""B200-native AM-QFT (arXiv:1404.1810): host mirror of the reference API.

The names follow the reference C++ library (``/root/reference/proj/include/
amqft``): ``VariantId`` 1..8, ``FunctionId``, ``TransformKind``, ``TrigMode``
and ``execute`` (variants.hpp:148-153).  Everything runs through the C ABI of
``libamqft_b200.so`` (``include/amqft_b200.h``) on a CUDA device; there is no
CPU implementation here.

* ``execute(v, f, n, cells)`` -- one signal, host in / host out, exact fp64
  order: bitwise equal to ``amqft::execute``.
* ``Plan`` -- batched device execution (fp32 / fp64, exact or fast order,
  forward and swap-trick inverse) on caller-owned device buffers (torch
  tensors or raw pointers) and a CUDA stream.
"""
from __future__ import annotations

import ctypes as C
import enum

import numpy as np

from . import _native
from ._native import AmqftError, InvalidArgument, check, lib

__all__ = [
    "VariantId", "FunctionId", "TransformKind", "TrigMode", "Order", "Plan",
    "execute", "execute_inverse", "cell_count", "AmqftError", "InvalidArgument",
    "schedule_dump", "function_base", "wired",
]


class VariantId(enum.IntEnum):
    """variants.hpp:25-30."""
    V1 = 1
    V2 = 2
    V3 = 3
    V4 = 4
    V5 = 5
    V6 = 6
    V7 = 7
    V8 = 8


class FunctionId(enum.IntEnum):
    """variants.hpp:55-66 (declaration order = numeric value)."""
    Cdft = 0
    Rdft = 1
    Dct = 2
    Dst = 3
    DctOddTime = 4
    DstOddTime = 5
    DctOddHarm = 6
    DstOddHarm = 7
    DctOddOdd = 8
    DstOddOdd = 9


class TransformKind(enum.IntEnum):
    """signal.hpp:18."""
    Cdft = 0
    Rdft = 1
    Dct = 2
    Dst = 3


class TrigMode(enum.IntEnum):
    """variants.hpp:108: Precomputed table or on-the-fly constants."""
    Precomputed = _native.TRIG_TABLE
    OnTheFly = _native.TRIG_ONTHEFLY


class Order(enum.IntEnum):
    Exact = _native.ORDER_EXACT
    Fast = _native.ORDER_FAST
    FastDag = _native.ORDER_FAST_DAG   # Fast without the split inside shared memory: whole-DAG kernels


_BASE = [2, 2, 2, 4, 4, 4, 4, 4, 8, 8]


def function_base(f: int) -> int:
    """FunctionPlan::base_size (variants.cpp:190-231)."""
    return _BASE[int(f)]


def wired(v: int, f: int) -> bool:
    """VariantPlan::has_function (variants.cpp:158-163)."""
    tm = int(v) in (1, 4, 5, 8)
    if f in (FunctionId.DctOddTime, FunctionId.DstOddTime):
        return tm
    if f in (FunctionId.DctOddHarm, FunctionId.DstOddHarm):
        return not tm
    return 0 <= int(f) < 10


def cell_count(f: int, n: int) -> int:
    """Cells of the operand of function f at periodization n
    (signal.cpp:254-258 through operand_type, variants.cpp:132-156)."""
    f = int(f)
    if f == 0:
        return 2 * n
    if f == 1:
        return n
    if f == 2:
        return n // 2 + 1
    if f == 3:
        return n // 2 - 1
    if f in (4, 5, 6, 7):
        return n // 4
    return n // 8


def _dtype_code(dtype) -> int:
    s = str(dtype)
    if s in ("f32", "float32", "torch.float32", "<class 'numpy.float32'>"):
        return _native.F32
    if s in ("f64", "float64", "torch.float64", "<class 'numpy.float64'>"):
        return _native.F64
    raise InvalidArgument(_native.EINVAL, f"unsupported dtype {dtype!r}")


class Plan:
    """A compiled batched transform on one device (amqft_plan_create)."""

    def __init__(self, variant: int, function: int, n: int, batch: int = 1, *,
                 dtype="f32", order=Order.Fast, trig_mode=TrigMode.Precomputed,
                 device: int = 0, table_max_n: int = 0, corrupt_constants: bool = False,
                 transposable: bool = False):
        d = _native.PlanDesc()
        d.variant = int(variant)
        d.function = int(function)
        d.n = int(n)
        d.batch = int(batch)
        d.dtype = _dtype_code(dtype)
        d.trig_mode = int(trig_mode)
        d.order = int(order)
        d.device = int(device)
        d.table_max_n = int(table_max_n)
        d.corrupt_constants = int(bool(corrupt_constants))
        self._h = C.c_void_p()
        # transposable: prefer a four-step plan with a transposed output (amqft_exec_rows_transposed)
        create = lib().amqft_plan_create_transposable if transposable else lib().amqft_plan_create
        check(create(C.byref(self._h), C.byref(d)))
        self.variant, self.function, self.n, self.batch = d.variant, d.function, d.n, d.batch
        self.dtype = "f64" if d.dtype == _native.F64 else "f32"
        self.device = d.device
        self.cells = int(lib().amqft_plan_cells(self._h))

    def close(self):
        if getattr(self, "_h", None) and self._h.value:
            lib().amqft_plan_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @staticmethod
    def _ptr(x) -> int:
        return int(x.data_ptr()) if hasattr(x, "data_ptr") else int(x)

    @staticmethod
    def _stream(stream) -> int:
        if stream is None:
            return 0
        if hasattr(stream, "cuda_stream"):
            return int(stream.cuda_stream)
        return int(stream)

    def _check_dtype(self, t):
        import torch
        want = torch.float64 if self.dtype == "f64" else torch.float32
        if t.dtype != want:
            raise InvalidArgument(_native.EINVAL, f"tensor dtype {t.dtype} does not match plan dtype {self.dtype}")

    def _check_tensor(self, t, rows):
        if hasattr(t, "is_cuda"):
            if not t.is_cuda:
                raise InvalidArgument(_native.EINVAL, "device tensors required")
            if t.device.index is not None and t.device.index != self.device:
                raise InvalidArgument(_native.EINVAL,
                                      f"tensor on cuda:{t.device.index}, plan on cuda:{self.device}")
            if not t.is_contiguous():
                raise InvalidArgument(_native.EINVAL, "contiguous tensors required")
            self._check_dtype(t)
            if t.numel() < rows * self.cells:
                raise InvalidArgument(_native.EINVAL, "tensor smaller than rows * cells")

    def forward(self, d_in, d_out, rows: int | None = None, stream=None):
        rows = self.batch if rows is None else int(rows)
        self._check_tensor(d_in, rows)
        self._check_tensor(d_out, rows)
        check(lib().amqft_exec_rows(self._h, self._ptr(d_in), self._ptr(d_out), rows, 0,
                                    self._stream(stream)))

    def inverse(self, d_in, d_out, rows: int | None = None, stream=None):
        rows = self.batch if rows is None else int(rows)
        self._check_tensor(d_in, rows)
        self._check_tensor(d_out, rows)
        check(lib().amqft_exec_rows(self._h, self._ptr(d_in), self._ptr(d_out), rows, 1,
                                    self._stream(stream)))

    def _check_host(self, t, rows):
        if hasattr(t, "is_cuda"):
            if t.is_cuda:
                raise InvalidArgument(_native.EINVAL, "host tensors required")
            if not t.is_contiguous():
                raise InvalidArgument(_native.EINVAL, "contiguous tensors required")
            self._check_dtype(t)
            if t.numel() < rows * self.cells:
                raise InvalidArgument(_native.EINVAL, "tensor smaller than rows * cells")

    def forward_host(self, h_in, h_out, rows: int | None = None, stream=None, inverse: bool = False):
        """Host (ideally pinned) tensors in and out; the batch streams through
        the device as an H2D | transform | D2H pipeline (amqft_exec_host_rows).
        Stream-ordered on `stream`; synchronise before reading h_out."""
        rows = self.batch if rows is None else int(rows)
        self._check_host(h_in, rows)
        self._check_host(h_out, rows)
        check(lib().amqft_exec_host_rows(self._h, self._ptr(h_in), self._ptr(h_out), rows,
                                         1 if inverse else 0, self._stream(stream)))

    def op_counts(self):
        out = (C.c_uint64 * 3)()
        check(lib().amqft_plan_op_counts(self._h, out))
        return tuple(int(v) for v in out)

    def fourstep_factors(self):
        """(A, B, C) with n = A B C for a four-step plan (B = 1: two factors)."""
        f = (C.c_size_t * 3)()
        check(lib().amqft_plan_fourstep_factors(self._h, f))
        return tuple(int(v) for v in f)

    def path(self):
        p, n = C.c_int(), C.c_int()
        check(lib().amqft_plan_path(self._h, C.byref(p), C.byref(n)))
        return int(p.value), int(n.value)


def execute(variant: int, function: int, n: int, cells, *, trig_mode=TrigMode.Precomputed,
            table_max_n: int = 0, corrupt_constants: bool = False, meter: bool = False):
    """amqft::execute(v, f, input, trig[, meter]) on one signal (host arrays),
    computed on the device in exact fp64 order."""
    x = np.ascontiguousarray(cells, dtype=np.float64)
    want = cell_count(function, n) if 0 <= int(function) < 10 else -1
    if want >= 0 and x.size != want and want > 0:
        raise InvalidArgument(_native.EINVAL, f"expected {want} cells, got {x.size}")
    out = np.zeros(max(x.size, 1), dtype=np.float64)
    m = (C.c_uint64 * 3)()
    check(lib().amqft_execute_host(int(variant), int(function), int(n),
                                   x.ctypes.data if x.size else out.ctypes.data, out.ctypes.data,
                                   int(trig_mode), int(table_max_n), int(bool(corrupt_constants)),
                                   m))
    out = out[:x.size]
    return (out, tuple(int(v) for v in m)) if meter else out


def execute_inverse(variant: int, n: int, spectrum, *, device: int = 0):
    """Swap-trick inverse CDFT of one host spectrum (exact fp64 order)."""
    import torch
    x = torch.as_tensor(np.ascontiguousarray(spectrum, dtype=np.float64)).to(f"cuda:{device}")
    y = torch.empty_like(x)
    p = Plan(variant, FunctionId.Cdft, n, 1, dtype="f64", order=Order.Exact, device=device)
    p.inverse(x, y)
    torch.cuda.synchronize(device)
    return y.cpu().numpy()


EI_DTYPE = np.dtype([("op", "u1"), ("lens", "u1"), ("flags", "u1"), ("am", "u1"),
                     ("n", "<u4"), ("off", "<u4"), ("aux", "<u4")])


def schedule_dump(variant: int, function: int, n: int, capacity_cells: int = 1 << 20):
    """Host-only: the compiled single-CTA stage program (EI records, stage
    boundaries) and its op counts.  No device needed."""
    L = lib()
    cnt, nst = C.c_size_t(), C.c_size_t()
    check(L.amqft_schedule_dump(int(variant), int(function), int(n), int(capacity_cells),
                                None, 0, C.byref(cnt), None, 0, C.byref(nst), None))
    recs = np.zeros(cnt.value, dtype=EI_DTYPE)
    st = np.zeros(2 * nst.value, dtype=np.uint32)
    ops = (C.c_uint64 * 3)()
    check(L.amqft_schedule_dump(int(variant), int(function), int(n), int(capacity_cells),
                                recs.ctypes.data, recs.size, C.byref(cnt), st.ctypes.data,
                                nst.value, C.byref(nst), ops))
    return recs, st.reshape(-1, 2), tuple(int(v) for v in ops)


def direct_bins(x, n: int, bins, *, rows: int = 1, row_len: int | None = None, row0: int = 0,
                stride: int = 1, stream=None):
    """Direct fp64 evaluation of selected DFT bins of a device signal
    (amqft_direct_bins: O(N) per bin, exact integer phase reduction) -- the
    verification utility for transforms too large for the CPU oracle
    (config 5).  x: device tensor of interleaved complex samples, fp32 or
    fp64, `rows` x `row_len` of them; sample (r, c) is the signal's element
    (row0 + r + stride c) mod n.  Returns complex128 bins (numpy)."""
    import torch
    row_len = (x.numel() // 2) // rows if row_len is None else int(row_len)
    dt = _native.F64 if x.dtype == torch.float64 else _native.F32
    b = np.ascontiguousarray(bins, dtype=np.uint64)
    out = np.zeros(2 * b.size, dtype=np.float64)
    check(lib().amqft_direct_bins(int(x.data_ptr()), dt, int(rows), int(row_len), int(row0), int(stride), int(n),
                                  b.ctypes.data, b.size, out.ctypes.data, Plan._stream(stream)))
    return out[0::2] + 1j * out[1::2]
