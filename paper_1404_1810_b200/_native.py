"""ctypes binding of libamqft_b200.so (declarations: include/amqft_b200.h).

The library is the product: there is no Python or CPU implementation of the
transform in this package.  Importing fails loudly when the shared library
has not been built, and every device entry point returns AMQFT_ECUDA on a
machine without a CUDA device.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libamqft_b200.so")

OK, EINVAL, ECUDA, ENCCL, ENOMEM = 0, 1, 2, 3, 4
F32, F64 = 0, 1
TRIG_TABLE, TRIG_ONTHEFLY = 0, 1
ORDER_EXACT, ORDER_FAST, ORDER_FAST_DAG = 0, 1, 2


class PlanDesc(C.Structure):
    """amqft_plan_desc (include/amqft_b200.h)."""
    _fields_ = [
        ("variant", C.c_int),
        ("function", C.c_int),
        ("n", C.c_size_t),
        ("batch", C.c_size_t),
        ("dtype", C.c_int),
        ("trig_mode", C.c_int),
        ("order", C.c_int),
        ("device", C.c_int),
        ("table_max_n", C.c_size_t),
        ("corrupt_constants", C.c_int),
    ]


class AmqftError(RuntimeError):
    def __init__(self, status: int, message: str):
        super().__init__(f"amqft status {status}: {message}")
        self.status = status


class InvalidArgument(AmqftError, ValueError):
    """AMQFT_EINVAL -- the reference's std::invalid_argument."""


_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; g.build()'` "
            "(the AM-QFT package has no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    vp, sz, u64p = C.c_void_p, C.c_size_t, C.POINTER(C.c_uint64)
    L.amqft_plan_create.argtypes = [C.POINTER(vp), C.POINTER(PlanDesc)]
    L.amqft_plan_create_transposable.argtypes = [C.POINTER(vp), C.POINTER(PlanDesc)]
    L.amqft_plan_destroy.argtypes = [vp]
    L.amqft_plan_cells.argtypes = [vp]
    L.amqft_plan_cells.restype = sz
    L.amqft_exec_forward.argtypes = [vp, vp, vp, vp]
    L.amqft_exec_inverse.argtypes = [vp, vp, vp, vp]
    L.amqft_exec_rows.argtypes = [vp, vp, vp, sz, C.c_int, vp]
    L.amqft_exec_host_rows.argtypes = [vp, vp, vp, sz, C.c_int, vp]
    L.amqft_dist_twiddle_scatter.argtypes = [vp, C.POINTER(vp), sz, sz, sz, sz, C.c_int, C.c_int, C.c_int, vp]
    L.amqft_transpose_c64.argtypes = [vp, vp, sz, sz, sz, vp]
    L.amqft_plan_transposed_factor.argtypes = [vp, C.POINTER(sz)]
    L.amqft_exec_rows_transposed.argtypes = [vp, vp, vp, sz, vp]
    L.amqft_dist_twiddle_scatter_direct.argtypes = [vp, C.POINTER(vp), sz, sz, sz, sz, C.c_int, C.c_int, sz, vp]
    L.amqft_dist_twiddle_scatter_t.argtypes = [vp, C.POINTER(vp), sz, sz, sz, sz, C.c_int, C.c_int, C.c_int, sz,
                                               vp]
    L.amqft_execute_host.argtypes = [C.c_int, C.c_int, sz, vp, vp, C.c_int, sz, C.c_int, vp]
    L.amqft_execute_host_constants.argtypes = [C.c_int, C.c_int, sz, vp, vp, vp, sz, vp]
    L.amqft_execute_host_inverse.argtypes = [C.c_int, sz, vp, vp]
    L.amqft_plan_create_with_constants.argtypes = [C.POINTER(vp), C.POINTER(PlanDesc), vp, sz]
    L.amqft_direct_bins.argtypes = [vp, C.c_int, sz, sz, sz, sz, sz, vp, sz, vp, vp]
    L.amqft_direct_bins_extended.argtypes = [vp, sz, vp, sz, C.c_int, vp]
    L.amqft_dist_unique_id.argtypes = [vp]
    L.amqft_dist_plan_create.argtypes = [C.POINTER(vp), C.c_int, sz, C.c_int, C.c_int, C.c_int, C.c_int, vp]
    L.amqft_dist_plan_shape.argtypes = [vp, C.POINTER(sz), C.POINTER(sz), C.POINTER(sz), C.POINTER(sz)]
    L.amqft_dist_exec_forward.argtypes = [vp, vp, vp, vp]
    L.amqft_dist_plan_destroy.argtypes = [vp]
    L.amqft_plan_op_counts.argtypes = [vp, vp]
    L.amqft_plan_path.argtypes = [vp, C.POINTER(C.c_int), C.POINTER(C.c_int)]
    L.amqft_plan_fourstep_factors.argtypes = [vp, C.POINTER(sz)]
    L.amqft_plan_dump.argtypes = [vp, C.c_int, vp, sz, C.POINTER(sz), vp, sz, C.POINTER(sz)]
    L.amqft_schedule_dump.argtypes = [C.c_int, C.c_int, sz, sz, vp, sz, C.POINTER(sz), vp, sz,
                                      C.POINTER(sz), vp]
    L.amqft_device_synchronize.argtypes = [C.c_int]
    L.amqft_last_error.restype = C.c_char_p
    L.amqft_version.restype = C.c_char_p
    for name in ("amqft_plan_create", "amqft_plan_create_transposable", "amqft_dist_twiddle_scatter_direct", "amqft_plan_destroy", "amqft_exec_forward",
                 "amqft_exec_inverse", "amqft_exec_rows", "amqft_exec_host_rows", "amqft_execute_host",
                 "amqft_execute_host_constants", "amqft_execute_host_inverse", "amqft_plan_create_with_constants",
                 "amqft_direct_bins", "amqft_direct_bins_extended", "amqft_dist_unique_id",
                 "amqft_dist_plan_create", "amqft_dist_plan_shape", "amqft_dist_exec_forward",
                 "amqft_dist_plan_destroy",
                 "amqft_dist_twiddle_scatter", "amqft_transpose_c64", "amqft_plan_transposed_factor",
                 "amqft_exec_rows_transposed", "amqft_dist_twiddle_scatter_t",
                 "amqft_plan_op_counts", "amqft_plan_path", "amqft_plan_fourstep_factors", "amqft_plan_dump",
                 "amqft_schedule_dump", "amqft_device_synchronize"):
        getattr(L, name).restype = C.c_int
    _lib = L
    return L


def check(status: int) -> None:
    if status == OK:
        return
    msg = lib().amqft_last_error().decode(errors="replace")
    if status == EINVAL:
        raise InvalidArgument(status, msg)
    raise AmqftError(status, msg)
