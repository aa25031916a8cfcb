"""Per-phase cycle breakdown of the fused kernel (diagnostic)."""
import ctypes as C
import os
import sys

import numpy as np
import torch

HERE = os.path.dirname(os.path.abspath(__file__))
lib = C.CDLL(os.path.join(HERE, os.environ.get("PT_LIB", "libphase_timing.so")))
lib.pt_run.argtypes = [C.c_int, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p, C.c_int,
                       C.c_void_p, C.c_int]
N = int(os.environ.get("PT_N", "4096"))
names = ["load", "top||small / chainfold+AM_F", "bottom", "AM_B levels", "chain recomb / top bwd",
         "store"]
for v in [int(a) for a in sys.argv[1:]] or [4]:
    kind = {1: 0, 4: 2, 2: 2}[v]
    p = np.arange(1, N // 4, dtype=np.longdouble)
    ang = 2 * np.pi * p / N
    f = {0: 2 * np.cos(ang), 2: 1 / (2 * np.cos(ang))}[kind]
    tab = np.concatenate([f.astype(np.float64), [np.cos(np.longdouble(np.pi) / 4)]]).astype(np.float32)
    dtab = torch.tensor(tab, device="cuda")
    rows = 65536 * 4096 // N
    x = torch.randn(rows, 2 * N, device="cuda")
    y = torch.empty_like(x)
    cyc = (C.c_ulonglong * 16)()
    grid = 148 * int(os.environ.get("PT_CTAS", "0"))   # 0: occupancy-derived
    for _ in range(2):
        rc = lib.pt_run(v, x.data_ptr(), y.data_ptr(), rows, dtab.data_ptr(), N, cyc, grid)
    per = rows / cyc[15]   # CTA iterations = rows / (grid * rows per CTA)
    tot = sum(cyc[i] for i in range(6))
    print(f"variant {v}: {tot / per:.0f} cycles/transform on CTA 0 (rc={rc})")
    for i, nm in enumerate(names):
        print(f"  {nm:32s} {cyc[i] / per:8.0f} cyc  {100 * cyc[i] / max(tot, 1):5.1f}%")
