"""CPU emulator of the fused kernel (csrc/fast_kernel.cuh), test-only.

Runs the kernel's phases in the kernel's order with the kernel's index
arithmetic: the generated straight-line functions (fast_gen.cuh) are called
through tests/native/libgen_host.so (the same header compiled as host C++),
the cooperative phases are restated here line by line from the CUDA source.
Threads of one phase touch disjoint cells, so running them one after the
other is equivalent to the device's barrier-separated execution.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "native", "libgen_host.so")
SRC = os.path.join(HERE, "native", "gen_host.cpp")
GEN = os.path.join(os.path.dirname(HERE), "paper_1404_1810_b200", "csrc", "gen", "fast_gen.cuh")
GEN_PY = os.path.join(os.path.dirname(HERE), "paper_1404_1810_b200", "codegen", "gen_fast.py")


def ensure_generated():
    """The generated header normally comes from the library build; make it
    here when the CPU tests run on a tree that was never built."""
    if not os.path.exists(GEN) or os.path.getmtime(GEN) < os.path.getmtime(GEN_PY):
        import subprocess
        import sys
        os.makedirs(os.path.dirname(GEN), exist_ok=True)
        out = subprocess.run([sys.executable, GEN_PY], check=True, capture_output=True, text=True).stdout
        with open(GEN + ".tmp", "w") as f:
            f.write(out)
        os.replace(GEN + ".tmp", GEN)

_lib = None


def lib():
    global _lib
    if _lib is None:
        ensure_generated()
        if (not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(GEN)
                or os.path.getmtime(LIB) < os.path.getmtime(SRC)):
            import subprocess
            subprocess.run(["g++", "-std=c++17", "-O1", "-ffp-contract=off", "-fPIC", "-shared",
                            "-o", LIB, SRC], check=True)
        L = C.CDLL(LIB)
        dp, i, d = C.c_void_p, C.c_int, C.c_double
        L.host_top.argtypes = [i, i, i, i, i, i, dp, i, dp, d]
        L.host_bottom.argtypes = [i, i, i, i, dp, dp, i, dp, i, d, i, i, i, i]
        L.host_small.argtypes = [i, i, i, i, i, dp, dp, dp, d]
        L.host_recomb.argtypes = [i, i, i, dp, i]
        L.host_fold.argtypes = [i, i, i, dp, i]
        L.host_smallpar.argtypes = [i, i, i, i, i, i, dp, dp, dp, d, i, dp]
        _lib = L
    return _lib


def _swz(i, lam):
    return i + ((i + (0 if lam else 31)) >> 5)


def _par(x):
    return bin(x).count("1") & 1


def seg_params(sine, lam_c, s, d):
    rho = 0 if d == 0 else (s & 1)
    lens = lam_c ^ (sine & _par(s ^ (s >> 1)))
    res, ln, prev = 0, lam_c, 0
    for i in range(1, d + 1):
        b = (s >> (d - i)) & 1
        is_o = 1 if b != prev else 0
        res |= (is_o ^ ln) << (i - 1)
        ln ^= sine & is_o
        prev = b
    return rho, lens, res


def _am_level(B, CS, N, LOGLB, depth, v, sine, tm):
    """AmLevel<C, DEPTH>::run / am_chains (fast_kernel.cuh)."""
    stride = 2 << depth
    chain = v in (1, 3, 5, 7)
    new = B.copy()
    for c in range(4):
        lam_c = c & 1
        for t in range(LOGLB):
            q = N >> (t + depth + 3)
            if q < 2:
                continue
            hi = (N >> (t + 1)) - lam_c
            for r in range(1 << depth):
                lens = ((r >> (depth - 1)) & 1) if (sine and depth > 0) else lam_c
                rO = r + ((1 - lens) << depth)
                cells = [c * CS + _swz(hi - rO - j * stride, lam_c) for j in range(q)]
                Cv = [B[p] for p in cells]
                if chain:
                    out = _chain(v, tm, lens, Cv)
                else:
                    if tm:
                        right = (lens == 0) if v == 4 else (lens == 1)
                    else:
                        right = (lens == 1) if v == 2 else (lens == 0)
                    out = []
                    for j in range(q):
                        cj = Cv[j]
                        if right:
                            if j == q - 1:
                                o = cj
                            else:
                                cn = Cv[j + 1]
                                o = (cj + cn if v == 4 else cj - cn) if tm else \
                                    (cn + cj if v == 2 else cj - cn)
                        else:
                            if j == 0:
                                o = cj
                            else:
                                cp = Cv[j - 1]
                                o = (cp + cj if v == 4 else cj - cp) if tm else \
                                    (cj + cp if v == 2 else cj - cp)
                        out.append(o)
                for p, o in zip(cells, out):
                    new[p] = o
    B[:] = new


def _chain(v, tm, lens, X):
    q = len(X)
    Y = list(X)
    if tm:
        addop = v == 5
        desc = (lens == 1) if v == 1 else (lens == 0)
        s0, d = (q - 1, -1) if desc else (0, 1)
        prev = 0.5 * Y[s0]
        Y[s0] = prev
        p = s0
        for _ in range(1, q):
            p += d
            prev = (Y[p] + prev) if addop else (Y[p] - prev)
            Y[p] = prev
    else:
        addop = v == 7
        desc = (lens == 0) if v == 3 else (lens == 1)
        s0, d = (q - 1, -1) if desc else (0, 1)
        prev = Y[s0]
        p = s0
        for _ in range(1, q - 1):
            p += d
            prev = (Y[p] + prev) if addop else (Y[p] - prev)
            Y[p] = prev
        p += d
        t = (Y[p] + prev) if addop else (Y[p] - prev)
        Y[p] = 0.5 * t
    return Y


def _chain_level(B, CS, n, fwd):
    q = n >> 2
    for c in range(4):
        lam = c & 1
        for k in range(q):
            if lam and k == 0:
                continue
            i0, i1 = c * CS + _swz(k, lam), c * CS + _swz((n >> 1) - k, lam)
            e, o = B[i0], B[i1]
            if not fwd:
                B[i0], B[i1] = (o + e, o - e) if lam else (e + o, e - o)
            else:
                B[i0], B[i1] = (e - o, e + o) if lam else (e + o, e - o)


def emulate(v, N, LB, x, tab, base):
    L = lib()
    H = N // 2
    LOGN = N.bit_length() - 1
    LOGLB = LB.bit_length() - 1
    LT = LOGN - 1 - LOGLB
    HP = H // LB
    NSEG = 4 * HP
    NT = max(4 * LB, NSEG, 128)
    CS = (max(H + HP + 1, H + H // 32 + 1) + 31) // 32 * 32 + 16
    TM = v in (1, 4, 5, 8)
    SINE = 1 if v >= 5 else 0
    skew = lambda i: i + (i >> LOGLB)  # noqa: E731
    def tpos(i):  # Cfg::ipos: odd LB-segments stored reversed
        s_, u_ = i >> LOGLB, i & (LB - 1)
        j = i + LB - 2 * u_ if (s_ & 1) and u_ else i
        return j + s_
    pt = (lambda i, lam: tpos(i)) if TM else _swz
    pf = _swz if TM else (lambda i, lam: tpos(i))
    T = np.zeros(4 * CS + 8)
    F = np.zeros(4 * CS + 8)
    tab = np.ascontiguousarray(tab, dtype=np.float64)
    tp = tab.ctypes.data
    # per-level compacted table for the top levels (fast_kernel.cuh k_level_table)
    lt = []
    for lvl in range(1, LT + 1):
        Lv = H >> (lvl - 1)
        lt += [0.0 if u == 0 else tab[u * (N // (2 * Lv)) - 1] for u in range(Lv // 2)]
    ltab = np.ascontiguousarray(lt + [0.0], dtype=np.float64)
    ltp = ltab.ctypes.data
    Tp, Fp = T.ctypes.data, F.ctypes.data
    x = np.asarray(x, dtype=np.float64)
    re, im = x[0::2], x[1::2]
    for m in range(H + 1):
        if m in (0, H):
            T[0 * CS + pt(m, 0)] = re[m]
            T[2 * CS + pt(m, 0)] = im[m]
        else:
            T[0 * CS + pt(m, 0)] = re[m] + re[N - m]
            T[1 * CS + pt(m, 1)] = re[m] - re[N - m]
            T[2 * CS + pt(m, 0)] = im[m] + im[N - m]
            T[3 * CS + pt(m, 1)] = im[m] - im[N - m]
    if TM:
        for c in range(4):
            for vv in range(1, LB):
                assert L.host_top(LB, LT, LOGN, SINE, 0, c & 1, Tp + 8 * c * CS, vv, ltp, base) == 0
    else:
        # generated folds on the sets {j W +- k} for n = N .. 2W, then the
        # levels below 2W (down to 2N/LB) level by level (fast_kernel.cuh)
        W = max(64, N // LB)
        for c in range(4):
            for k in range(W // 2):
                assert L.host_fold(W, H // W, c & 1, Tp + 8 * c * CS, k) == 0
        n = W
        while n >= 2 * (N // LB):
            _chain_level(T, CS, n, True)
            n >>= 1
        if v in (3, 7):
            for depth in range(LT):
                _am_level(T, CS, N, LOGLB, depth, v, SINE, False)
        else:
            am_phase_regs(T, CS, N, LOGLB, LT, v, SINE, False)
        for c in range(4):
            assert L.host_smallpar(v, HP, LOGN, LB, c & 1, 0, None, None, tp, base, 1, Tp + 8 * c * CS) == 0
    half = HP // 2
    for tid in range(NSEG):
        h = tid % half
        rest = tid // half
        part, rho_bit, lam_bit = rest & 1, (rest >> 1) & 1, (rest >> 2) & 1
        c = part * 2 + lam_bit
        s = 2 * h + rho_bit
        rho, lens, r = seg_params(SINE, lam_bit, s, LT)
        rho = 0  # reversed odd segments (Cfg::ipos)
        assert L.host_bottom(v, LB, rho, lens, Tp + 8 * c * CS, Fp + 8 * c * CS, s * LB, tp, N,
                             base, N, LT, r, lam_bit) == 0
    if TM:  # the small chain runs beside the bottom (disjoint cells)
        for c in range(4):
            for cls in range(LT + 1):
                assert L.host_smallpar(v, HP, LOGN, LB, c & 1, cls, Tp + 8 * c * CS, Fp + 8 * c * CS,
                                       tp, base, 0, None) == 0
    for c in range(4):
        if TM:
            assert L.host_smallpar(v, HP, LOGN, LB, c & 1, 0, None, None, tp, base, 1, Fp + 8 * c * CS) == 0
        else:
            for cls in range(LT + 1):
                assert L.host_smallpar(v, HP, LOGN, LB, c & 1, cls, Tp + 8 * c * CS, Fp + 8 * c * CS,
                                       tp, base, 0, None) == 0
    if TM:
        if v in (1, 5):
            for depth in range(LT - 1, -1, -1):
                _am_level(F, CS, N, LOGLB, depth, v, SINE, True)
        else:
            am_phase_regs(F, CS, N, LOGLB, LT, v, SINE, True)
        W = max(64, N // LB)
        n = 2 * (N // LB)
        while n < 2 * W:
            _chain_level(F, CS, n, False)
            n <<= 1
        for c in range(4):
            for k in range(W // 2):
                assert L.host_recomb(W, H // W, c & 1, Fp + 8 * c * CS, k) == 0
    else:
        for c in range(4):
            for vv in range(1, LB):
                assert L.host_top(LB, LT, LOGN, SINE, 1, c & 1, Fp + 8 * c * CS, vv, ltp, base) == 0
    out = np.zeros(2 * N)
    for k in range(H + 1):
        rd, idd = F[0 * CS + pf(k, 0)], F[2 * CS + pf(k, 0)]
        if k in (0, H):
            out[2 * k], out[2 * k + 1] = rd, idd
        else:
            rs, is_ = F[1 * CS + pf(k, 1)], F[3 * CS + pf(k, 1)]
            out[2 * k], out[2 * k + 1] = rd + is_, idd - rs
            out[2 * (N - k)], out[2 * (N - k) + 1] = rd - is_, idd + rs
    return out


def am_phase_regs(B, CS, N, LOGLB, LT, v, sine, bwd):
    """Mirror of fast_kernel.cuh am_phase_regs: per-lane runs of RR cells,
    halo exchange between adjacent lanes of the same warp (shuffles)."""
    RR = N // 128
    LOGR = RR.bit_length() - 1
    lanes = []  # (warp, lane, c, t, i, active)
    for warp in range(8):
        for lane in range(32):
            c = warp >> 1
            if warp % 2 == 0:
                t, i = 0, lane
            else:
                t = 1 + (lane >= 16) + (lane >= 24) + (lane >= 28) + (lane >= 30) + (lane >= 31)
                i = lane - (32 - (64 >> t))
            active = t < LOGLB
            lanes.append((warp, lane, c, t if active else 0, i, active))
    X = {}
    for (warp, lane, c, t, i, active) in lanes:
        lam_c = c & 1
        basep = (N >> (t + 1)) - lam_c - (i << LOGR)
        X[(warp, lane)] = [B[c * CS + _swz(basep - l, lam_c)] if active else 0.0 for l in range(RR)]
    depths = list(range(LT - 1, -1, -1)) if bwd else list(range(LT))
    for D in depths:
        S = 2 << D
        new = {}
        for (warp, lane, c, t, i, active) in lanes:
            lam_c = c & 1
            Mt = N >> (t + 2)
            blk_ok = (Mt >> (D + 1)) >= 2
            x = X[(warp, lane)]
            xr = X[(warp, lane + 1)] if lane < 31 else x     # shfl_down (lane 31 keeps own)
            xl = X[(warp, lane - 1)] if lane > 0 else x      # shfl_up (lane 0 keeps own)
            y = []
            for l in range(RR):
                p = (i << LOGR) + l
                obit = (p >> D) & 1
                lens = ((p >> (D - 1)) & 1) if (sine and D > 0) else lam_c
                is_o = blk_ok and (obit == 1 - lens)
                if bwd:
                    right = (lens == 0) if v == 4 else (lens == 1)
                else:
                    right = (lens == 1) if v == 2 else (lens == 0)
                cj = x[l]
                if right:
                    cn = x[l + S] if l + S < RR else (xr[l + S - RR] if S <= RR else cj)
                    edge = p + S >= Mt
                else:
                    cn = x[l - S] if l - S >= 0 else (xl[l - S + RR] if S <= RR else cj)
                    edge = p - S < 0
                o = cj
                if not edge:
                    if bwd:
                        o = ((cj + cn) if v == 4 else (cj - cn)) if right else \
                            ((cn + cj) if v == 4 else (cj - cn))
                    else:
                        o = ((cn + cj) if v == 2 else (cj - cn)) if right else \
                            ((cj + cn) if v == 2 else (cj - cn))
                y.append(o if is_o else cj)
            new[(warp, lane)] = y
        X = new
    for (warp, lane, c, t, i, active) in lanes:
        if not active:
            continue
        lam_c = c & 1
        basep = (N >> (t + 1)) - lam_c - (i << LOGR)
        for l in range(RR):
            B[c * CS + _swz(basep - l, lam_c)] = X[(warp, lane)][l]
