"""A/B timing of kernel build variants (diagnostic; tools/libphase_timing_*.so)."""
import ctypes as C
import glob
import os

import numpy as np
import torch

HERE = os.path.dirname(os.path.abspath(__file__))
N = 4096
rows = 65536
x = torch.randn(rows, 2 * N, device="cuda")
y = torch.empty_like(x)
p = np.arange(1, N // 4, dtype=np.longdouble)
tab = np.concatenate([(1 / (2 * np.cos(2 * np.pi * p / N))).astype(np.float64),
                      [np.cos(np.longdouble(np.pi) / 4)]]).astype(np.float32)
dtab = torch.tensor(tab, device="cuda")
for path in sorted(glob.glob(os.path.join(HERE, "ab_*.so"))):
    lib = C.CDLL(path)
    lib.pt_run.argtypes = [C.c_int, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p, C.c_int,
                           C.c_void_p, C.c_int]
    cyc = (C.c_ulonglong * 16)()
    for v in (4, 2):
        ts = []
        for rep in range(4):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            lib.pt_run(v, x.data_ptr(), y.data_ptr(), rows, dtab.data_ptr(), N, cyc, 148 * int(os.path.basename(path).split('_m')[-1].split('.')[0]) if '_m' in path else 296)
            e.record()
            torch.cuda.synchronize()
            ts.append(s.elapsed_time(e))
        print(f"{os.path.basename(path):28s} v{v}: {min(ts[1:]):.3f} ms")
