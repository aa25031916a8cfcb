"""A/B timing of fused-kernel build variants tools/ab_*.so (diagnostic).

  python tools/ab_kernel.py [variants...]
"""
import ctypes as C
import glob
import os
import sys

import numpy as np
import torch

HERE = os.path.dirname(os.path.abspath(__file__))
N, rows = 4096, 65536
vs = [int(a) for a in sys.argv[1:]] or [4, 2]
x = torch.randn(rows, 2 * N, device="cuda")
y = torch.empty_like(x)
p = np.arange(1, N // 4, dtype=np.longdouble)
tab = np.concatenate([(1 / (2 * np.cos(2 * np.pi * p / N))).astype(np.float64),
                      [np.cos(np.longdouble(np.pi) / 4)]]).astype(np.float32)
dtab = torch.tensor(tab, device="cuda")
libs = sorted(glob.glob(os.path.join(HERE, "ab_*.so")))
res = {}
for rnd in range(2):                      # two interleaved rounds against drift
    for path in libs:
        lib = C.CDLL(path)
        lib.ab_run.argtypes = [C.c_int, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p, C.c_int, C.c_int]
        lib.ab_run.restype = C.c_float
        for v in vs:
            ms = lib.ab_run(v, x.data_ptr(), y.data_ptr(), rows, dtab.data_ptr(), N, 6)
            key = (os.path.basename(path), v)
            res[key] = min(res.get(key, 1e9), ms)
for (name, v), ms in sorted(res.items()):
    print(f"{name:24s} v{v}: {ms:.3f} ms  {rows / ms / 1e3:.2f} M transforms/s")
