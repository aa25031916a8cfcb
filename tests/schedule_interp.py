"""Host (numpy fp64) interpreter of the compiled stage program.

Test-only: an independent restatement of the EI semantics of
paper_1404_1810_b200/csrc/generic.cuh, used to check the PLAN COMPILER on the
CPU (no GPU needed) against the oracle, bitwise.  numpy fp64 element-wise
add/sub/mul are single IEEE operations (no contraction), as on the device.
"""
from __future__ import annotations

import numpy as np

OP = dict(SC_F=1, SC_B=2, SR_F=3, SR_B=4, GATHER=5, SCATTER=6, SH_F_DCT=7, SH_F_DST=8,
          SH_F_ODD=9, ST_B_DCT=10, ST_B_DST=11, ST_B_ODD=12, AM_F=13, AM_B=14,
          BASE_CDFT2=15, BASE_PAIR2=16, BASE_OO8=17, CHAIN_F=18, CHAIN_B=19)
FL_DESC, FL_ADD = 4, 8


def _items(op, n):
    if op in (OP["SC_F"], OP["SC_B"]):
        return 2 * n
    if op in (OP["SR_F"], OP["SR_B"], OP["GATHER"], OP["SCATTER"]):
        return n
    if op in (OP["SH_F_DCT"], OP["ST_B_DCT"]):
        return n // 2 + 1
    if op in (OP["SH_F_DST"], OP["ST_B_DST"]):
        return n // 2 - 1
    if op in (OP["SH_F_ODD"], OP["ST_B_ODD"]):
        return n // 4
    if op in (OP["AM_F"], OP["AM_B"]):
        return n // 8
    return {OP["BASE_CDFT2"]: 4, OP["BASE_PAIR2"]: 2, OP["BASE_OO8"]: 1}.get(op, 1)


def _eval(e, x, trig, nmax):
    """Return (dst positions, values) of all items of EI e (relative)."""
    op, lens, am, n, aux = int(e["op"]), int(e["lens"]), int(e["am"]), int(e["n"]), int(e["aux"])
    i = np.arange(_items(op, n))
    L = lambda p: x[p]  # noqa: E731
    if op == OP["SC_F"]:
        src = np.where(i < n, 2 * i, 2 * (i - n) + 1)
        return i, L(src)
    if op == OP["SC_B"]:
        k, im = i >> 1, i & 1
        v = np.empty(i.size)
        for t in range(i.size):
            kk, ii = int(k[t]), int(im[t])
            if kk == 0 or kk == n // 2:
                v[t] = x[n + kk] if ii else x[kk]
            elif kk < n // 2:
                v[t] = (x[n + kk] - x[n - kk]) if ii else (x[kk] + x[2 * n - kk])
            else:
                j = n - kk
                v[t] = (x[n + j] + x[kk]) if ii else (x[j] - x[n + kk])
        return i, v
    if op == OP["SR_F"]:
        v = np.empty(i.size)
        for t in range(i.size):
            if t == 0 or t == n // 2:
                v[t] = x[t]
            elif t < n // 2:
                v[t] = x[t] + x[n - t]
            else:
                m = t - n // 2
                v[t] = x[m] - x[n - m]
        return i, v
    if op == OP["SR_B"]:
        return i, L(np.where(i <= n // 2, i, 3 * n // 2 - i))
    if op == OP["GATHER"]:
        return i, L(np.where(i < aux, 2 * i + lens, 2 * (i - aux) + 1 - lens))
    if op == OP["SCATTER"]:
        return i, L(np.where((i & 1) == lens, i >> 1, aux + (i >> 1)))
    if op == OP["SH_F_DCT"]:
        v = np.empty(i.size)
        for t in range(i.size):
            if t <= n // 4:
                v[t] = x[t] if t == n // 4 else x[t] + x[n // 2 - t]
            else:
                j = t - (n // 4 + 1)
                v[t] = x[j] - x[n // 2 - j]
        return i, v
    if op == OP["SH_F_DST"]:
        v = np.empty(i.size)
        for t in range(i.size):
            if t < n // 4 - 1:
                v[t] = x[t] - x[n // 2 - t - 2]
            else:
                idx = t - (n // 4 - 1) + 1
                v[t] = x[idx - 1] if idx == n // 4 else x[idx - 1] + x[n // 2 - idx - 1]
        return i, v
    if op == OP["SH_F_ODD"]:
        mc = n // 4
        v = np.empty(i.size)
        for t in range(i.size):
            if t < mc // 2:
                v[t] = (x[t] - x[mc - 1 - t]) if lens else (x[t] + x[mc - 1 - t])
            else:
                j = t - mc // 2
                v[t] = (x[j] + x[mc - 1 - j]) if lens else (x[j] - x[mc - 1 - j])
        return i, v
    if op == OP["ST_B_DCT"]:
        o = n // 4 + 1
        v = np.empty(i.size)
        for t in range(i.size):
            if t < n // 4:
                v[t] = x[t] + x[o + t]
            elif t == n // 4:
                v[t] = x[t]
            else:
                j = n // 2 - t
                v[t] = x[j] - x[o + j]
        return i, v
    if op == OP["ST_B_DST"]:
        o = n // 4 - 1
        v = np.empty(i.size)
        for t in range(i.size):
            k = t + 1
            if k < n // 4:
                v[t] = x[o + k - 1] + x[k - 1]
            elif k == n // 4:
                v[t] = x[o + n // 4 - 1]
            else:
                j = n // 2 - k
                v[t] = x[o + j - 1] - x[j - 1]
        return i, v
    if op == OP["ST_B_ODD"]:
        mc = n // 4
        o = mc // 2
        v = np.empty(i.size)
        for t in range(i.size):
            if t < o:
                v[t] = x[o + t] + x[t] if lens else x[t] + x[o + t]
            else:
                j = mc - 1 - t
                v[t] = (x[o + j] - x[j]) if lens else (x[j] - x[o + j])
        return i, v
    if op in (OP["AM_F"], OP["AM_B"]):
        q = aux
        pointwise = (am in (1, 4, 5, 8)) if op == OP["AM_F"] else (am in (2, 3, 6, 7))
        if pointwise:
            slots = (2 * i + 1) * (nmax // n) - 1
            return i, x[i] * trig[slots]
        v = np.empty(q)
        for t in range(q):
            if op == OP["AM_F"] and am == 2:
                v[t] = (x[0] if t == 0 else x[t] + x[t - 1]) if lens == 0 else \
                       (x[q - 1] if t == q - 1 else x[t + 1] + x[t])
            elif op == OP["AM_F"]:  # 6
                v[t] = (x[q - 1] if t == q - 1 else x[t] - x[t + 1]) if lens == 0 else \
                       (x[0] if t == 0 else x[t] - x[t - 1])
            elif am == 4:
                v[t] = (x[t] + x[t + 1] if t < q - 1 else x[q - 1]) if lens == 0 else \
                       (x[0] if t == 0 else x[t - 1] + x[t])
            else:  # 8
                v[t] = (x[0] if t == 0 else x[t] - x[t - 1]) if lens == 0 else \
                       (x[t] - x[t + 1] if t < q - 1 else x[q - 1])
        return i, v
    if op == OP["BASE_CDFT2"]:
        return i, np.array([x[0] + x[2], x[1] + x[3], x[0] - x[2], x[1] - x[3]])
    if op == OP["BASE_PAIR2"]:
        return i, np.array([x[0] + x[1], x[0] - x[1]])
    if op == OP["BASE_OO8"]:
        return i, np.array([x[0] * trig[nmax // 4 - 1]])
    raise ValueError(f"unknown op {op}")


def _chain(e, x):
    q, fl = int(e["aux"]), int(e["flags"])
    desc, add = bool(fl & FL_DESC), bool(fl & FL_ADD)
    s, d = (q - 1, -1) if desc else (0, 1)
    y = x.copy()
    f = (lambda a, b: a + b) if add else (lambda a, b: a - b)
    if int(e["op"]) == OP["CHAIN_F"]:
        if q == 1:
            y[0] = 0.5 * x[0]
            return y
        prev = x[s]
        y[s] = prev
        p = s
        for _ in range(1, q - 1):
            p += d
            prev = f(x[p], prev)
            y[p] = prev
        p += d
        y[p] = 0.5 * f(x[p], prev)
        return y
    prev = 0.5 * x[s]
    y[s] = prev
    p = s
    for _ in range(1, q):
        p += d
        prev = f(x[p], prev)
        y[p] = prev
    return y


def interpret(recs, stages, cells, trig, nmax):
    """Run the stage program on cells (fp64) in place semantics."""
    x = np.array(cells, dtype=np.float64)
    for b, e in stages:
        writes = []
        for k in range(int(b), int(e)):
            ei = recs[k]
            off = int(ei["off"])
            if int(ei["op"]) in (OP["CHAIN_F"], OP["CHAIN_B"]):
                q = int(ei["aux"])
                writes.append((off + np.arange(q), _chain(ei, x[off:off + q])))
            else:
                dst, val = _eval(ei, x[off:], trig, nmax)
                writes.append((off + dst, val))
        for dst, val in writes:
            x[dst] = val
    return x
