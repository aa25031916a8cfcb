"""Reference model (numpy fp64) of the fused fast-kernel formulation.

Test infrastructure: the spec the CUDA fast kernel (csrc/fast*.cu) follows,
proven bitwise against the oracle on the CPU.

Time-major variants (1, 4, 5, 8), "Dct-index space": after SplitComplex and
SplitReal the four chains (Re/Im x Dct/Dst) are kept in natural temporal
index order m = 0..N/2.  The Dct-chain gathers (SplitTimeParity) are then
pure relabellings: oddC(N/2^t) owns the indices with exactly t trailing
zeros.  Every oddC fold pairs mirror indices, so the whole forward is an
in-place mirror-butterfly network over nested segments [a, a+L]: pairs
(a+v, a+L-v), orientation (normal for a lower half, reversed for an upper
half) deciding which cell carries the block position j, and the AM
constant f(pi v / L) (table slot v*Nmax/(2L)), or the base constant
cos(pi/4) for v = L/4 (the OO(8) base case).  The backward rebuilds each
block's spectrum from its E child (same segment class) and its AM child,
and the Dct chains recombine with SplitTimeParity butterflies in natural
frequency order.
"""
from __future__ import annotations

import numpy as np


def _interleave(first, second):
    out = []
    for a, b in zip(first, second):
        out += [a, b]
    return out


def am_backward_tm(v, lens, C):
    """AM_B of the time-major variants on a child spectrum C (positions).
    lens: 0 = Dct mother, 1 = Dst mother (elaborations.cpp:472-526)."""
    q = len(C)
    O = [0.0] * q
    if v == 4:
        if lens == 0:
            for j in range(q - 1):
                O[j] = C[j] + C[j + 1]
            O[q - 1] = C[q - 1]
        else:
            O[0] = C[0]
            for j in range(1, q):
                O[j] = C[j - 1] + C[j]
    elif v == 8:
        if lens == 0:
            O[0] = C[0]
            for j in range(1, q):
                O[j] = C[j] - C[j - 1]
        else:
            for j in range(q - 1):
                O[j] = C[j] - C[j + 1]
            O[q - 1] = C[q - 1]
    elif v == 1:
        if lens == 0:
            O[0] = 0.5 * C[0]
            for j in range(1, q):
                O[j] = C[j] - O[j - 1]
        else:
            O[q - 1] = 0.5 * C[q - 1]
            for j in range(q - 2, -1, -1):
                O[j] = C[j] - O[j + 1]
    elif v == 5:
        if lens == 0:
            O[q - 1] = 0.5 * C[q - 1]
            for j in range(q - 2, -1, -1):
                O[j] = C[j] + O[j + 1]
        else:
            O[0] = 0.5 * C[0]
            for j in range(1, q):
                O[j] = C[j] + O[j - 1]
    else:
        raise ValueError(v)
    return O


def mnet_forward(S, a, L, rho, lens, sine, tab, nmax, base):
    """In-place mirror network on segment [a, a+L] (recursive)."""
    if L < 4:
        return
    for v in range(1, L // 2):
        lo, hi = a + v, a + L - v
        x, y = (S[lo], S[hi]) if rho == 0 else (S[hi], S[lo])
        if lens == 0:
            e, o = x + y, x - y
        else:
            e, o = x - y, x + y
        k = base if v == L // 4 else tab[v * (nmax // (2 * L)) - 1]
        o = o * k
        if rho == 0:
            S[lo], S[hi] = e, o
        else:
            S[hi], S[lo] = e, o
    lo_lens = lens if rho == 0 else lens ^ sine
    hi_lens = lens ^ sine if rho == 0 else lens
    mnet_forward(S, a, L // 2, 0, lo_lens, sine, tab, nmax, base)
    mnet_forward(S, a + L // 2, L // 2, 1, hi_lens, sine, tab, nmax, base)


def spectrum(S, v, a, L, rho, lens, sine, tcls):
    """Spectrum (natural order) of the class-tcls block of segment [a, a+L]."""
    m = L >> (tcls + 1)
    if m == 1:
        return [S[a + L // 2]]
    lower = (a, L // 2, 0)
    upper = (a + L // 2, L // 2, 1)
    e_seg, o_seg = (lower, upper) if rho == 0 else (upper, lower)
    E = spectrum(S, v, *e_seg, lens, sine, tcls)
    C = spectrum(S, v, *o_seg, lens ^ sine, sine, tcls)
    # a 2-cell block's odd child is the OO(8) base case (no AM conversion;
    # its base-constant multiply happened in the forward network).
    O = am_backward_tm(v, lens, C) if m > 2 else C
    return _interleave(E, O) if lens == 0 else _interleave(O, E)


def fast_cdft_time_major(v, N, x, tab, nmax, base):
    assert v in (1, 4, 5, 8)
    H = N // 2
    sine = 1 if v >= 5 else 0
    x = np.asarray(x, dtype=np.float64)
    parts = (x[0::2], x[1::2])
    out = np.zeros(2 * N)
    specs = []
    for part in parts:
        dct = np.zeros(H + 1)
        dst = np.zeros(H + 1)
        dct[0], dct[H] = part[0], part[H]
        for m in range(1, H):
            dct[m] = part[m] + part[N - m]
            dst[m] = part[m] - part[N - m]
        pair = []
        for S, lam in ((dct, 0), (dst, 1)):
            mnet_forward(S, 0, H, 0, lam, sine, tab, nmax, base)
            F = np.zeros(H + 1)
            lg = H.bit_length() - 1
            top_classes = lg if lam == 0 else lg - 1
            for t in range(top_classes):
                sp = spectrum(S, v, 0, H, 0, lam, sine, t)
                hi = N >> (t + 1)
                for p, val in enumerate(sp):
                    F[hi - p - lam] = val
            # chain recombination (SplitTimeParity backward, elab.cpp:304-332)
            if lam == 0:
                F[0], F[1] = S[0] + S[H], S[0] - S[H]
                n = 4
                F[2] = F[2]  # oddC(4) spectrum already at cell 2
            else:
                F[1] = S[H // 2]
                n = 8
            while n <= N:
                if lam == 0:
                    for k in range(n // 4):
                        e, o = F[k], F[n // 2 - k]
                        F[k], F[n // 2 - k] = e + o, e - o
                else:
                    for k in range(1, n // 4):
                        e, o = F[k], F[n // 2 - k]
                        F[k], F[n // 2 - k] = o + e, o - e
                n *= 2
            pair.append(F)
        specs.append(pair)
    (rdct, rdst), (idct, idst) = specs
    # SplitReal bwd + SplitComplex bwd (elab.cpp:162-208)
    out[0], out[1] = rdct[0], idct[0]
    out[2 * H], out[2 * H + 1] = rdct[H], idct[H]
    for k in range(1, H):
        out[2 * k] = rdct[k] + idst[k]
        out[2 * (N - k)] = rdct[k] - idst[k]
        out[2 * k + 1] = idct[k] - rdst[k]
        out[2 * (N - k) + 1] = idct[k] + rdst[k]
    return out


# ---------------------------------------------------------------------------
# Harmonic-major variants (2, 3, 6, 7): the transpose.  Forward in natural
# temporal order: the Dct/Dst chain folds (SplitHarmonicParity, prefix
# segments [0, n/2], elab.cpp:229-257) leave oddC(n) reversed in (n/4, n/2];
# each block's forward is gathers (even/odd positions) plus AM_F on the odd
# part.  Backward in natural FREQUENCY order: the same in-place mirror
# network as the time-major forward, run bottom-up, with AM_B pointwise on
# the mirror cell before each SplitTimeParity butterfly.

def am_forward_hm(v, lens, A):
    """AM_F of the harmonic-major variants (elaborations.cpp:370-448)."""
    q = len(A)
    C = [0.0] * q
    if v == 2:
        if lens == 0:
            C[0] = A[0]
            for j in range(1, q):
                C[j] = A[j] + A[j - 1]
        else:
            C[q - 1] = A[q - 1]
            for j in range(q - 1):
                C[j] = A[j + 1] + A[j]
    elif v == 6:
        if lens == 0:
            C[q - 1] = A[q - 1]
            for j in range(q - 1):
                C[j] = A[j] - A[j + 1]
        else:
            C[0] = A[0]
            for j in range(1, q):
                C[j] = A[j] - A[j - 1]
    elif v == 3:
        if lens == 0:
            C[q - 1] = A[q - 1]
            for j in range(q - 2, 0, -1):
                C[j] = A[j] - C[j + 1]
            C[0] = 0.5 * (A[0] - C[1])
        else:
            C[0] = A[0]
            for j in range(1, q - 1):
                C[j] = A[j] - C[j - 1]
            C[q - 1] = 0.5 * (A[q - 1] - C[q - 2])
    elif v == 7:
        if lens == 0:
            C[0] = A[0]
            for j in range(1, q - 1):
                C[j] = A[j] + C[j - 1]
            C[q - 1] = 0.5 * (A[q - 1] + C[q - 2])
        else:
            C[q - 1] = A[q - 1]
            for j in range(q - 2, 0, -1):
                C[j] = A[j] + C[j + 1]
            C[0] = 0.5 * (A[0] + C[1])
    else:
        raise ValueError(v)
    return C


def place_forward(v, vals, lens, sine, F, a, L, rho):
    """Forward of one block given its temporal values (natural positions):
    gathers + AM_F, leaves written to the centres of the frequency-space
    mirror network segments."""
    m = len(vals)
    if m == 1:
        F[a + L // 2] = vals[0]
        return
    if lens == 0:
        E, A = vals[0::2], vals[1::2]
    else:
        E, A = vals[1::2], vals[0::2]
    C = am_forward_hm(v, lens, A) if m > 2 else A
    lower = (a, L // 2, 0)
    upper = (a + L // 2, L // 2, 1)
    e_seg, o_seg = (lower, upper) if rho == 0 else (upper, lower)
    place_forward(v, E, lens, sine, F, *e_seg)
    place_forward(v, C, lens ^ sine, sine, F, *o_seg)


def mnet_backward(F, a, L, rho, lens, sine, tab, nmax, base):
    if L < 4:
        return
    lo_lens = lens if rho == 0 else lens ^ sine
    hi_lens = lens ^ sine if rho == 0 else lens
    mnet_backward(F, a, L // 2, 0, lo_lens, sine, tab, nmax, base)
    mnet_backward(F, a + L // 2, L // 2, 1, hi_lens, sine, tab, nmax, base)
    for v in range(1, L // 2):
        lo, hi = a + v, a + L - v
        jc, mc = (lo, hi) if rho == 0 else (hi, lo)
        E, C = F[jc], F[mc]
        k = base if v == L // 4 else tab[v * (nmax // (2 * L)) - 1]
        O = C * k
        if lens == 0:
            F[jc], F[mc] = E + O, E - O
        else:
            F[jc], F[mc] = O + E, O - E


def fast_cdft_harmonic_major(v, N, x, tab, nmax, base):
    assert v in (2, 3, 6, 7)
    H = N // 2
    sine = 1 if v >= 5 else 0
    x = np.asarray(x, dtype=np.float64)
    specs = []
    for part in (x[0::2], x[1::2]):
        dct = np.zeros(H + 1)
        dst = np.zeros(H + 1)
        dct[0], dct[H] = part[0], part[H]
        for m in range(1, H):
            dct[m] = part[m] + part[N - m]
            dst[m] = part[m] - part[N - m]
        pair = []
        for S, lam in ((dct, 0), (dst, 1)):
            F = np.zeros(H + 1)
            n = N
            while n >= (4 if lam == 0 else 8):
                if lam == 0:
                    for m in range(n // 4):
                        a, b = S[m], S[n // 2 - m]
                        S[m], S[n // 2 - m] = a + b, a - b
                else:
                    for m in range(1, n // 4):
                        a, b = S[m], S[n // 2 - m]
                        S[m], S[n // 2 - m] = a - b, a + b
                t = (N // n).bit_length() - 1
                vals = [S[n // 2 - p - lam] for p in range(n // 4)]
                place_forward(v, vals, lam, sine, F, 0, H, 0)
                n //= 2
            if lam == 0:
                F[0], F[H] = S[0] + S[1], S[0] - S[1]
            else:
                F[H // 2] = S[1]
            mnet_backward(F, 0, H, 0, lam, sine, tab, nmax, base)
            pair.append(F)
        specs.append(pair)
    (rdct, rdst), (idct, idst) = specs
    out = np.zeros(2 * N)
    out[0], out[1] = rdct[0], idct[0]
    out[2 * H], out[2 * H + 1] = rdct[H], idct[H]
    for k in range(1, H):
        out[2 * k] = rdct[k] + idst[k]
        out[2 * (N - k)] = rdct[k] - idst[k]
        out[2 * k + 1] = idct[k] - rdst[k]
        out[2 * (N - k) + 1] = idct[k] + rdst[k]
    return out


# ---------------------------------------------------------------------------
# Phase-structured model: the exact decomposition the CUDA kernel uses
# (top levels, bottom segments of length LB, small chain, depth-ordered upper
# levels, chain recombination).  Must equal the recursive models bitwise.

def _parity(x):
    return bin(x).count("1") & 1


def segment_params(lam_c, s, LT, sine):
    """(orientation, lens, residue) of segment s at depth LT."""
    rho = 0 if LT == 0 else (s & 1)
    lens = lam_c ^ (sine & _parity(s ^ (s >> 1)))
    r = 0
    ln = lam_c
    prev = 0
    for i in range(1, LT + 1):
        b = (s >> (LT - i)) & 1
        is_o = 1 if b != prev else 0
        bit = is_o ^ ln
        r |= bit << (i - 1)
        ln ^= sine & is_o
        prev = b
    return rho, lens, r


def sub_lens(lam_c, depth, r, sine):
    """Lens of the depth-`depth` sub-block with residue r (upper levels)."""
    if not sine or depth == 0:
        return lam_c
    return (r >> (depth - 1)) & 1


def phased_time_major(v, N, x, tab, nmax, base, LB):
    H = N // 2
    sine = 1 if v >= 5 else 0
    LT = (H // LB).bit_length() - 1
    lgLB = LB.bit_length() - 1
    x = np.asarray(x, dtype=np.float64)
    chains = []
    for part in (x[0::2], x[1::2]):
        dct = np.zeros(H + 1)
        dst = np.zeros(H + 1)
        dct[0], dct[H] = part[0], part[H]
        for m in range(1, H):
            dct[m] = part[m] + part[N - m]
            dst[m] = part[m] - part[N - m]
        chains += [(dct, 0), (dst, 1)]
    results = []
    for T, lam_c in chains:
        F = np.zeros(H + 1)
        # phase T: levels 1..LT
        for lvl in range(1, LT + 1):
            L = H >> (lvl - 1)
            for s in range(1 << (lvl - 1)):
                rho, lens, _ = segment_params(lam_c, s, lvl - 1, sine)
                a = s * L
                for vv in range(1, L // 2):
                    lo, hi = a + vv, a + L - vv
                    j, m = (lo, hi) if rho == 0 else (hi, lo)
                    p, q = T[j], T[m]
                    e, o = (p + q, p - q) if lens == 0 else (p - q, p + q)
                    k = base if vv == L // 4 else tab[vv * (nmax // (2 * L)) - 1]
                    T[j], T[m] = e, o * k
        # phase B: segments of length LB
        for s in range(H // LB):
            rho, lens, r = segment_params(lam_c, s, LT, sine)
            seg = T.copy()
            mnet_forward(seg, s * LB, LB, rho, lens, sine, tab, nmax, base)
            for t in range(lgLB):
                sp = spectrum(seg, v, s * LB, LB, rho, lens, sine, t)
                hi = (N >> (t + 1)) - lam_c - r
                for p, val in enumerate(sp):
                    F[hi - (p << LT)] = val
        # small chain
        HP = H // LB
        y = {k: T[k * LB] for k in range(HP + 1)}
        G = [0.0] * (HP + 1)
        lg = HP.bit_length() - 1
        ntop = lg if lam_c == 0 else lg - 1
        for t in range(ntop):
            sp = spectrum(y, v, 0, HP, 0, lam_c, sine, t)
            hi = (2 * HP) >> (t + 1)
            for p, val in enumerate(sp):
                G[hi - p - lam_c] = val
        if lam_c == 0:
            G[0], G[1] = y[0] + y[HP], y[0] - y[HP]
            n = 4
        else:
            G[1] = y[HP // 2]
            n = 8
        while n <= 2 * HP:
            for k in (range(n // 4) if lam_c == 0 else range(1, n // 4)):
                e, o = G[k], G[n // 2 - k]
                G[k], G[n // 2 - k] = (e + o, e - o) if lam_c == 0 else (o + e, o - e)
            n *= 2
        for k in range(HP + 1):
            if lam_c == 0 or 1 <= k < HP:
                F[k] = G[k]
        # phase U: depth LT-1 .. 0, blocks of top classes t < lgLB
        for depth in range(LT - 1, -1, -1):
            new = F.copy()
            for t in range(lgLB):
                Mt = N >> (t + 2)
                m = Mt >> depth
                hi = (N >> (t + 1)) - lam_c
                for r in range(1 << depth):
                    lens = sub_lens(lam_c, depth, r, sine)
                    rO = r + ((1 - lens) << depth)
                    q = m // 2
                    C = [F[hi - (j * (2 << depth) + rO)] for j in range(q)]
                    O = am_backward_tm(v, lens, C) if m > 2 else C
                    for j in range(q):
                        new[hi - (j * (2 << depth) + rO)] = O[j]
            F = new
        # phase F: chain recombination n = 2N'..N
        n = 2 * (N // LB)
        while n <= N:
            for k in (range(n // 4) if lam_c == 0 else range(1, n // 4)):
                e, o = F[k], F[n // 2 - k]
                F[k], F[n // 2 - k] = (e + o, e - o) if lam_c == 0 else (o + e, o - e)
            n *= 2
        results.append(F)
    rdct, rdst, idct, idst = results
    out = np.zeros(2 * N)
    out[0], out[1] = rdct[0], idct[0]
    out[2 * H], out[2 * H + 1] = rdct[H], idct[H]
    for k in range(1, H):
        out[2 * k] = rdct[k] + idst[k]
        out[2 * (N - k)] = rdct[k] - idst[k]
        out[2 * k + 1] = idct[k] - rdst[k]
        out[2 * (N - k) + 1] = idct[k] + rdst[k]
    return out


def phased_harmonic_major(v, N, x, tab, nmax, base, LB):
    H = N // 2
    sine = 1 if v >= 5 else 0
    LT = (H // LB).bit_length() - 1
    lgLB = LB.bit_length() - 1
    HP = H // LB
    x = np.asarray(x, dtype=np.float64)
    chains = []
    for part in (x[0::2], x[1::2]):
        dct = np.zeros(H + 1)
        dst = np.zeros(H + 1)
        dct[0], dct[H] = part[0], part[H]
        for m in range(1, H):
            dct[m] = part[m] + part[N - m]
            dst[m] = part[m] - part[N - m]
        chains += [(dct, 0), (dst, 1)]
    results = []
    for T, lam_c in chains:
        F = np.zeros(H + 1)
        # phase F': chain folds n = N .. 2N'
        n = N
        while n >= 2 * (N // LB):
            for m in (range(n // 4) if lam_c == 0 else range(1, n // 4)):
                a_, b_ = T[m], T[n // 2 - m]
                T[m], T[n // 2 - m] = (a_ + b_, a_ - b_) if lam_c == 0 else (a_ - b_, a_ + b_)
            n //= 2
        # phase U': depth 0 .. LT-1 (top-down), AM_F on odd classes
        for depth in range(LT):
            new = T.copy()
            for t in range(lgLB):
                Mt = N >> (t + 2)
                m = Mt >> depth
                hi = (N >> (t + 1)) - lam_c
                for r in range(1 << depth):
                    lens = sub_lens(lam_c, depth, r, sine)
                    rO = r + ((1 - lens) << depth)
                    q = m // 2
                    A = [T[hi - (j * (2 << depth) + rO)] for j in range(q)]
                    C = am_forward_hm(v, lens, A) if m > 2 else A
                    for j in range(q):
                        new[hi - (j * (2 << depth) + rO)] = C[j]
            T = new
        # phase B': segments in frequency space
        for s in range(H // LB):
            rho, lens, r = segment_params(lam_c, s, LT, sine)
            seg = {}
            for t in range(lgLB):
                hi = (N >> (t + 1)) - lam_c - r
                vals = [T[hi - (p << LT)] for p in range(LB >> (t + 1))]
                place_forward(v, vals, lens, sine, seg, s * LB, LB, rho)
            arr = np.zeros(H + 1)
            for k, val in seg.items():
                arr[k] = val
            mnet_backward(arr, s * LB, LB, rho, lens, sine, tab, nmax, base)
            for u in range(1, LB):
                F[s * LB + u] = arr[s * LB + u]
        # small chain: temporal [0, HP] -> frequency k*LB
        S = {k: T[k] for k in range(HP + 1)}
        seg = {}
        n = 2 * HP
        while n >= (4 if lam_c == 0 else 8):
            for m in (range(n // 4) if lam_c == 0 else range(1, n // 4)):
                a_, b_ = S[m], S[n // 2 - m]
                S[m], S[n // 2 - m] = (a_ + b_, a_ - b_) if lam_c == 0 else (a_ - b_, a_ + b_)
            vals = [S[n // 2 - p - lam_c] for p in range(n // 4)]
            place_forward(v, vals, lam_c, sine, seg, 0, HP, 0)
            n //= 2
        if lam_c == 0:
            seg[0], seg[HP] = S[0] + S[1], S[0] - S[1]
        else:
            seg[HP // 2] = S[1]
        for k, val in seg.items():
            F[k * LB] = val
        # phase T': mirror levels LT .. 1 (L = 2LB .. H), bottom-up
        for lvl in range(LT, 0, -1):
            L = H >> (lvl - 1)
            for s in range(1 << (lvl - 1)):
                rho, lens, _ = segment_params(lam_c, s, lvl - 1, sine)
                a = s * L
                for vv in range(1, L // 2):
                    lo, hi = a + vv, a + L - vv
                    j, m = (lo, hi) if rho == 0 else (hi, lo)
                    E, C = F[j], F[m]
                    k = base if vv == L // 4 else tab[vv * (nmax // (2 * L)) - 1]
                    O = C * k
                    F[j], F[m] = (E + O, E - O) if lens == 0 else (O + E, O - E)
        results.append(F)
    rdct, rdst, idct, idst = results
    out = np.zeros(2 * N)
    out[0], out[1] = rdct[0], idct[0]
    out[2 * H], out[2 * H + 1] = rdct[H], idct[H]
    for k in range(1, H):
        out[2 * k] = rdct[k] + idst[k]
        out[2 * (N - k)] = rdct[k] - idst[k]
        out[2 * k + 1] = idct[k] - rdst[k]
        out[2 * (N - k) + 1] = idct[k] + rdst[k]
    return out
