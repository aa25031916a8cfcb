#!/usr/bin/env python3
"""Generates csrc/gen/fast_gen.cuh (at build time, csrc/Makefile): straight-line per-thread code for the
bottom of the AM-QFT recursion (see tests/fast_model.py for the proven
formulation and csrc/fast.cu for the kernel that calls these functions).

Per variant family:
  time-major (1,4,5,8)
    tmB  one index-space segment [a, a+LB]: remaining mirror folds (forward),
         then the spectra of every block inside (AM_B neighbour ops / serial
         recurrences), scattered to the frequency layout.
    tmS  the cells at multiples of LB (small top blocks + Dct(2)/Dst(4)):
         their backward and the chain recombination up to Dct/Dst(N/LB).
  harmonic-major (2,3,6,7)
    hmB  one frequency-space segment: gathers + AM_F of the blocks inside
         (read from the temporal layout), then the bottom mirror levels.
    hmS  the small top blocks: chain folds up to N/LB, their forward, leaves
         placed at multiples of LB, and the Dct(2)/Dst(4) bases.

Every emitted operation is one of the reference's add/sub/mul on the
reference's operands (AR::add/sub/mul = __fadd_rn/__dadd_rn..., never
contracted), so the fp64 instantiation is bitwise the reference recursion.

  python3 paper_1404_1810_b200/codegen/gen_fast.py > paper_1404_1810_b200/csrc/gen/fast_gen.cuh
"""
from __future__ import annotations

import sys

TM = (1, 4, 5, 8)
HM = (2, 3, 6, 7)


class Emitter:
    def __init__(self):
        self.lines = []
        self.tmp = 0

    def emit(self, s):
        self.lines.append("  " + s)

    def new(self, expr):
        self.tmp += 1
        name = f"t{self.tmp}"
        self.emit(f"const R {name} = {expr};")
        return name


def add(a, b):
    return f"AR::add({a}, {b})"


def sub(a, b):
    return f"AR::sub({a}, {b})"


def mul(a, b):
    return f"AR::mul({a}, {b})"


def half(a):
    return f"AR::mul(R(0.5), {a})"


def const_expr(v, L):
    """AM constant f(pi v / L): table slot v*nmax/(2L) (variants.cpp:281)."""
    if v == L // 4:
        return "base"
    lg = (2 * L).bit_length() - 1
    return f"AMQFT_TABLD(tab, ({v} * (nmax >> {lg}) - 1))"


# --------------------------------------------------------------- time-major
def am_b_tm(em, v, lens, C):
    q = len(C)
    O = [None] * q
    if v == 4:
        if lens == 0:
            for j in range(q - 1):
                O[j] = em.new(add(C[j], C[j + 1]))
            O[q - 1] = C[q - 1]
        else:
            O[0] = C[0]
            for j in range(1, q):
                O[j] = em.new(add(C[j - 1], C[j]))
    elif v == 8:
        if lens == 0:
            O[0] = C[0]
            for j in range(1, q):
                O[j] = em.new(sub(C[j], C[j - 1]))
        else:
            for j in range(q - 1):
                O[j] = em.new(sub(C[j], C[j + 1]))
            O[q - 1] = C[q - 1]
    elif v == 1:
        if lens == 0:
            O[0] = em.new(half(C[0]))
            for j in range(1, q):
                O[j] = em.new(sub(C[j], O[j - 1]))
        else:
            O[q - 1] = em.new(half(C[q - 1]))
            for j in range(q - 2, -1, -1):
                O[j] = em.new(sub(C[j], O[j + 1]))
    elif v == 5:
        if lens == 0:
            O[q - 1] = em.new(half(C[q - 1]))
            for j in range(q - 2, -1, -1):
                O[j] = em.new(add(C[j], O[j + 1]))
        else:
            O[0] = em.new(half(C[0]))
            for j in range(1, q):
                O[j] = em.new(add(C[j], O[j - 1]))
    return O


def interleave(lens, E, O):
    out = []
    for e, o in zip(E, O):
        out += [e, o] if lens == 0 else [o, e]
    return out


def tz(u):
    return (u & -u).bit_length() - 1


def mnet_fwd(em, x, a, L, rho, lens, sine, cls=None):
    if L < 4:
        return
    for v in range(1, L // 2):
        if cls is not None and tz(v) != cls:
            continue
        lo, hi = a + v, a + L - v
        j, m = (lo, hi) if rho == 0 else (hi, lo)
        p, q = x[j], x[m]
        s, d = add(p, q), sub(p, q)
        e_expr, o_expr = (s, d) if lens == 0 else (d, s)
        e_name = em.new(e_expr)
        o_name = em.new(mul(o_expr, const_expr(v, L)))
        x[j], x[m] = e_name, o_name
    lo_l = lens if rho == 0 else lens ^ sine
    hi_l = lens ^ sine if rho == 0 else lens
    mnet_fwd(em, x, a, L // 2, 0, lo_l, sine, cls)
    mnet_fwd(em, x, a + L // 2, L // 2, 1, hi_l, sine, cls)


def spectrum_tm(em, v, x, a, L, rho, lens, sine, tcls):
    m = L >> (tcls + 1)
    if m == 1:
        return [x[a + L // 2]]
    lower, upper = (a, L // 2, 0), (a + L // 2, L // 2, 1)
    es, os_ = (lower, upper) if rho == 0 else (upper, lower)
    E = spectrum_tm(em, v, x, *es, lens, sine, tcls)
    C = spectrum_tm(em, v, x, *os_, lens ^ sine, sine, tcls)
    O = am_b_tm(em, v, lens, C) if m > 2 else C
    return interleave(lens, E, O)


def store_off(p):
    """Offset of F[SW(hi - p*2^D)] from F[SW(hi)] for compile-time D >= 5:
    SW(hi - 32m) = SW(hi) - 33m  (SW(i) = i + i/32)."""
    return f"-({p} * ((1 << D) + (1 << (D >= 5 ? D - 5 : 0))))"


def gen_tmB(v, LB, rho, lam, part=None):
    """Class by class: mirror folds never mix trailing-zero classes
    (tz(v) == tz(L - v)), so each class is transformed and stored on its own
    -- small live register set.  Addresses are immediate offsets from two
    per-thread bases (segment start in T, class top in F).  part 0 = class
    0, part 1 = classes 1.., part 2 = all classes with every T load hoisted
    to the top (the stores of one class would otherwise keep the next
    class's loads waiting: both are shared memory)."""
    sine = 1 if v >= 5 else 0
    lg = LB.bit_length() - 1
    em = Emitter()
    ld = Emitter()
    hoist = part == 2
    ld.emit("const R* __restrict__ Tp = T + a + (a >> LOGLB);")
    ld.emit("const int swsh = dsto ? 0 : 31;")
    for t in range(lg):
        if part in (0, 1) and (t == 0) != (part == 0):
            continue
        x = {}
        for u in range(1, LB):
            if tz(u) == t:
                (ld if hoist else em).emit(f"const R x{u} = Tp[{u}];")
                x[u] = f"x{u}"
        mnet_fwd(em, x, 0, LB, rho, lam, sine, cls=t)
        sp = spectrum_tm(em, v, x, 0, LB, rho, lam, sine, t)
        em.emit(f"{{ const int hi = (N >> {t + 1}) - dsto - r;")
        em.emit("  R* __restrict__ Fq = F + SW(hi);")
        for p, name in enumerate(sp):
            em.emit(f"  if constexpr (D >= 5) Fq[{store_off(p)}] = {name}; "
                    f"else F[SW(hi - ({p} << D))] = {name};")
        em.emit("}")
        if not hoist:
            em.emit("AMQFT_CLASS_FENCE();  // keep classes apart (register pressure)")
    sfx = "" if part is None else f"_p{part}"
    sig = (f"template <typename R, typename AR, int LOGLB, int D>\n__device__ __forceinline__ void "
           f"tmB_v{v}_lb{LB}_r{rho}_l{lam}{sfx}(const R* __restrict__ T, R* __restrict__ F, int a, "
           f"const R* __restrict__ tab, int nmax, R base, int N, int r, int dsto)")
    return sig + " {\n" + "\n".join(ld.lines + em.lines) + "\n}\n"


def gen_tmS(v, HP, LB, lam):
    """Small chain: cells k*LB, k = 0..HP (Dct) / 1..HP-1 (Dst)."""
    sine = 1 if v >= 5 else 0
    em = Emitter()
    y = {}
    ks = range(0, HP + 1) if lam == 0 else range(1, HP)
    for k in ks:
        em.emit(f"const R y{k} = T[PH({k} * {LB})];")
        y[k] = f"y{k}"
    G = [None] * (HP + 1)
    lg = HP.bit_length() - 1
    ntop = lg if lam == 0 else lg - 1
    Np = 2 * HP
    for t in range(ntop):
        sp = spectrum_tm(em, v, y, 0, HP, 0, lam, sine, t)
        hi = Np >> (t + 1)
        for p, name in enumerate(sp):
            G[hi - p - lam] = name
    if lam == 0:
        G[0] = em.new(add(y[0], y[HP]))
        G[1] = em.new(sub(y[0], y[HP]))
        n = 4
    else:
        G[1] = y[HP // 2]
        n = 8
    while n <= Np:
        if lam == 0:
            for k in range(n // 4):
                e, o = G[k], G[n // 2 - k]
                G[k], G[n // 2 - k] = em.new(add(e, o)), em.new(sub(e, o))
        else:
            for k in range(1, n // 4):
                e, o = G[k], G[n // 2 - k]
                G[k], G[n // 2 - k] = em.new(add(o, e)), em.new(sub(o, e))
        n *= 2
    for k in ks:
        em.emit(f"F[PH({k})] = {G[k]};")
    sig = (f"template <typename R, typename AR, int LOGLB>\n__device__ __forceinline__ void "
           f"tmS_v{v}_hp{HP}_l{lam}(const R* __restrict__ T, R* __restrict__ F, R base)")
    return sig + " {\n" + "\n".join(em.lines) + "\n}\n"


# ----------------------------------------------------------- harmonic-major
def am_f_hm(em, v, lens, A):
    q = len(A)
    C = [None] * q
    if v == 2:
        if lens == 0:
            C[0] = A[0]
            for j in range(1, q):
                C[j] = em.new(add(A[j], A[j - 1]))
        else:
            C[q - 1] = A[q - 1]
            for j in range(q - 1):
                C[j] = em.new(add(A[j + 1], A[j]))
    elif v == 6:
        if lens == 0:
            C[q - 1] = A[q - 1]
            for j in range(q - 1):
                C[j] = em.new(sub(A[j], A[j + 1]))
        else:
            C[0] = A[0]
            for j in range(1, q):
                C[j] = em.new(sub(A[j], A[j - 1]))
    elif v == 3:
        if lens == 0:
            C[q - 1] = A[q - 1]
            for j in range(q - 2, 0, -1):
                C[j] = em.new(sub(A[j], C[j + 1]))
            C[0] = em.new(half(sub(A[0], C[1])))
        else:
            C[0] = A[0]
            for j in range(1, q - 1):
                C[j] = em.new(sub(A[j], C[j - 1]))
            C[q - 1] = em.new(half(sub(A[q - 1], C[q - 2])))
    elif v == 7:
        if lens == 0:
            C[0] = A[0]
            for j in range(1, q - 1):
                C[j] = em.new(add(A[j], C[j - 1]))
            C[q - 1] = em.new(half(add(A[q - 1], C[q - 2])))
        else:
            C[q - 1] = A[q - 1]
            for j in range(q - 2, 0, -1):
                C[j] = em.new(add(A[j], C[j + 1]))
            C[0] = em.new(half(add(A[0], C[1])))
    return C


def place_hm(em, v, vals, lens, sine, x, a, L, rho):
    m = len(vals)
    if m == 1:
        x[a + L // 2] = vals[0]
        return
    if lens == 0:
        E, A = vals[0::2], vals[1::2]
    else:
        E, A = vals[1::2], vals[0::2]
    C = am_f_hm(em, v, lens, A) if m > 2 else A
    lower, upper = (a, L // 2, 0), (a + L // 2, L // 2, 1)
    es, os_ = (lower, upper) if rho == 0 else (upper, lower)
    place_hm(em, v, E, lens, sine, x, *es)
    place_hm(em, v, C, lens ^ sine, sine, x, *os_)


def mnet_bwd(em, x, a, L, rho, lens, sine, cls=None):
    if L < 4:
        return
    lo_l = lens if rho == 0 else lens ^ sine
    hi_l = lens ^ sine if rho == 0 else lens
    mnet_bwd(em, x, a, L // 2, 0, lo_l, sine, cls)
    mnet_bwd(em, x, a + L // 2, L // 2, 1, hi_l, sine, cls)
    for v in range(1, L // 2):
        if cls is not None and tz(v) != cls:
            continue
        lo, hi = a + v, a + L - v
        j, m = (lo, hi) if rho == 0 else (hi, lo)
        E, C = x[j], x[m]
        O = em.new(mul(C, const_expr(v, L)))
        if lens == 0:
            x[j], x[m] = em.new(add(E, O)), em.new(sub(E, O))
        else:
            x[j], x[m] = em.new(add(O, E)), em.new(sub(O, E))


def gen_hmB(v, LB, rho, lam, part=None):
    """Class by class (see gen_tmB; part 2 hoists every T load)."""
    sine = 1 if v >= 5 else 0
    lg = LB.bit_length() - 1
    em = Emitter()
    ld = Emitter()
    hoist = part == 2
    ld.emit("R* __restrict__ Fp = F + a + (a >> LOGLB);")
    ld.emit("const int swsh = dsto ? 0 : 31;")
    for t in range(lg):
        if part in (0, 1) and (t == 0) != (part == 0):
            continue
        x = {}
        cnt = LB >> (t + 1)
        tgt = ld if hoist else em
        if not hoist:
            em.emit("{")
        tgt.emit(f"const int hi{t} = (N >> {t + 1}) - dsto - r;")
        tgt.emit(f"const R* __restrict__ Tq{t} = T + SW(hi{t});")
        vals = []
        for p in range(cnt):
            nm = f"v{t}_{p}"
            tgt.emit(f"const R {nm} = (D >= 5) ? Tq{t}[{store_off(p)}] : T[SW(hi{t} - ({p} << D))];")
            vals.append(nm)
        if hoist:
            em.emit("{")
        place_hm(em, v, vals, lam, sine, x, 0, LB, rho)
        mnet_bwd(em, x, 0, LB, rho, lam, sine, cls=t)
        for u in sorted(x):
            em.emit(f"Fp[{u}] = {x[u]};")
        em.emit("}")
        if not hoist:
            em.emit("AMQFT_CLASS_FENCE();  // keep classes apart (register pressure)")
    sfx = "" if part is None else f"_p{part}"
    sig = (f"template <typename R, typename AR, int LOGLB, int D>\n__device__ __forceinline__ void "
           f"hmB_v{v}_lb{LB}_r{rho}_l{lam}{sfx}(const R* __restrict__ T, R* __restrict__ F, int a, "
           f"const R* __restrict__ tab, int nmax, R base, int N, int r, int dsto)")
    return sig + " {\n" + "\n".join(ld.lines + em.lines) + "\n}\n"


def gen_hmS(v, HP, LB, lam):
    """Temporal cells [0, HP] (Dct(N/LB) after the big folds) -> leaves at
    frequency cells k*LB."""
    sine = 1 if v >= 5 else 0
    em = Emitter()
    S = {}
    ks = range(0, HP + 1) if lam == 0 else range(1, HP)
    for k in ks:
        em.emit(f"const R s{k} = T[PH({k})];")
        S[k] = f"s{k}"
    x = {}
    Np = 2 * HP
    n = Np
    while n >= (4 if lam == 0 else 8):
        if lam == 0:
            for m in range(n // 4):
                a_, b_ = S[m], S[n // 2 - m]
                S[m], S[n // 2 - m] = em.new(add(a_, b_)), em.new(sub(a_, b_))
        else:
            for m in range(1, n // 4):
                a_, b_ = S[m], S[n // 2 - m]
                S[m], S[n // 2 - m] = em.new(sub(a_, b_)), em.new(add(a_, b_))
        vals = [S[n // 2 - p - lam] for p in range(n // 4)]
        place_hm(em, v, vals, lam, sine, x, 0, HP, 0)
        n //= 2
    if lam == 0:
        x[0] = em.new(add(S[0], S[1]))
        x[HP] = em.new(sub(S[0], S[1]))
    else:
        x[HP // 2] = S[1]
    for k in ks:
        em.emit(f"F[PH({k} * {LB})] = {x[k]};")
    sig = (f"template <typename R, typename AR, int LOGLB>\n__device__ __forceinline__ void "
           f"hmS_v{v}_hp{HP}_l{lam}(const R* __restrict__ T, R* __restrict__ F, R base)")
    return sig + " {\n" + "\n".join(em.lines) + "\n}\n"


# ------------------------------------------------------------- top levels
def gen_top(LB, LT, direction, lam, sine, nlog, kmode=None, collect=None):
    """Mirror levels 1..LT of one chain for the thread owning offset v in
    [1, LB): cells z_2k = kW + v, z_2k+1 = (k+1)W - v (W = 2 LB), closed
    under every top level.  direction 'fwd' = time-major forward fold,
    'bwd' = harmonic-major backward butterfly (levels LT..1).  Table size
    nmax = N = 2^nlog (compile time).  kmode "tm": the constants come from
    the register array kk (filled from tensor memory, top_cols order)
    instead of the per-level table; collect: a set receiving the (level,
    offset, expression) keys.  Skewed addresses:
    PH(kW+v) = v + k(W+2), PH((k+1)W-v) = (k+1)(W+2) - v - 1."""
    W = 2 * LB
    K = 1 << (LT - 1)          # cells per parity
    H = W * K
    em = Emitter()
    # The index-space buffer (T time-major, F harmonic-major) stores odd
    # LB-segments reversed (cell a + u at a + LB - u, see Cfg::ipos), so
    # (k+1)W - v sits at (2k+1) LB + v: every cell of the thread is
    # B + v + s (LB + 1).
    rev = True
    def addr(z):
        k = z // 2
        if rev:
            return "pe", z * (LB + 1)
        return ("pe", k * (W + 2)) if z % 2 == 0 else ("po", (k + 1) * (W + 2))
    em.emit("R* __restrict__ pe = B + v;")
    if not rev:
        em.emit("R* __restrict__ po = B - v - 1;")
    x = {}
    for k in range(K):
        x[2 * k] = f"x{2 * k}"
        x[2 * k + 1] = f"x{2 * k + 1}"
        for z in (2 * k, 2 * k + 1):
            b_, o_ = addr(z)
            em.emit(f"R x{z} = {b_}[{o_}];")
    # offsets of cells from 0: z_2k = kW + v (+v), z_2k+1 = (k+1)W - v (-v)
    def off(z):
        k = z // 2
        return (k * W, +1) if z % 2 == 0 else ((k + 1) * W, -1)
    nmax = 1 << nlog
    levels = list(range(1, LT + 1))
    if direction == "bwd":
        levels = levels[::-1]
    for i in levels:
        L = H >> (i - 1)
        lg2L = (2 * L).bit_length() - 1
        sc = nmax >> lg2L
        # per-level compacted table: ltab[off_i + u] = f(pi u / L), u < L/2
        off_i = sum((H >> (j - 1)) // 2 for j in range(1, i))
        if kmode == "tm":
            em.emit("{")
        else:
            em.emit(f"{{ const R* __restrict__ tp = ltab + {off_i} + v;")
            em.emit(f"  const R* __restrict__ tm = ltab + {off_i} - v;")
        done = set()
        for z in range(2 * K):
            if z in done:
                continue
            c0, sg = off(z)
            seg = c0 // L if sg > 0 else (c0 - 1) // L
            a = seg * L
            # mirror cell
            mc0, msg = a + L - (c0 - a), -sg
            mz = None
            for z2 in range(2 * K):
                if off(z2) == (mc0, msg):
                    mz = z2
            assert mz is not None
            done.add(z)
            done.add(mz)
            # lower cell: offset < L/2
            u_z = (c0 - a, sg)
            z_is_lower = (c0 - a) < L // 2 if sg > 0 else (c0 - a) <= L // 2
            lower, upper = (z, mz) if z_is_lower else (mz, z)
            lc0, lsg = off(lower)
            u0 = lc0 - a                  # u = u0 + lsg * v
            rho = 0 if i == 1 else (seg & 1)
            par = bin(seg ^ (seg >> 1)).count("1") & 1
            lens = lam ^ (sine & par)
            jc, mcz = (lower, upper) if rho == 0 else (upper, lower)
            kexpr = f"__ldg({'tp' if lsg > 0 else 'tm'} + {u0})"
            if u0 == 0 and lsg > 0 and i == LT:
                kexpr = f"(v == {LB // 2} ? base : {kexpr})"
            if collect is not None:
                collect.add((i, off_i, kexpr))
            if kmode == "tm":
                kexpr = f"kk[{top_cols(LB, LT, nlog).index((i, off_i, kexpr))}]"
            p_, q_ = x[jc], x[mcz]
            em.tmp += 1
            t = em.tmp
            em.emit(f"  const R k{t} = {kexpr};")
            if direction == "fwd":
                em.emit(f"  const R s{t} = {add(p_, q_)}, d{t} = {sub(p_, q_)};")
                if lens == 0:
                    em.emit(f"  {p_} = s{t}; {q_} = {mul('d' + str(t), 'k' + str(t))};")
                else:
                    em.emit(f"  {p_} = d{t}; {q_} = {mul('s' + str(t), 'k' + str(t))};")
            else:
                em.emit(f"  const R o{t} = {mul(q_, 'k' + str(t))};")
                if lens == 0:
                    em.emit(f"  const R e{t} = {p_}; {p_} = {add('e' + str(t), 'o' + str(t))}; "
                            f"{q_} = {sub('e' + str(t), 'o' + str(t))};")
                else:
                    em.emit(f"  const R e{t} = {p_}; {p_} = {add('o' + str(t), 'e' + str(t))}; "
                            f"{q_} = {sub('o' + str(t), 'e' + str(t))};")
        em.emit("}")
    for z in range(2 * K):
        b_, o_ = addr(z)
        em.emit(f"{b_}[{o_}] = x{z};")
    if kmode == "tm":
        sig = (f"template <typename R, typename AR>\n__device__ __forceinline__ void "
               f"top_{direction}_lb{LB}_lt{LT}_n{nlog}_l{lam}_s{sine}_tm(R* __restrict__ B, int v, "
               f"const R* kk)")
        return sig + " {\n" + "\n".join(em.lines) + "\n}\n"
    sig = (f"template <typename R, typename AR>\n__device__ __forceinline__ void "
           f"top_{direction}_lb{LB}_lt{LT}_n{nlog}_l{lam}_s{sine}(R* __restrict__ B, int v, "
           f"const R* __restrict__ ltab, R base)")
    return sig + " {\n" + "\n".join(em.lines) + "\n}\n"


_TOP_COLS = {}


def top_cols(LB, LT, nlog):
    """The distinct top-level constants of one thread, in column order:
    (level, per-level table offset, expression).  They depend on v only
    (not on the chain, lens or direction), so one fill serves every top."""
    key = (LB, LT, nlog)
    if key not in _TOP_COLS:
        keys = set()
        for direction in ("fwd", "bwd"):
            for lam in (0, 1):
                for sine in (0, 1):
                    gen_top(LB, LT, direction, lam, sine, nlog, collect=keys)
        _TOP_COLS[key] = sorted(keys)
    return _TOP_COLS[key]


def gen_top_fill(LB, LT, nlog):
    """Evaluates the top_cols constants for offset v (the tensor-memory
    fill, once per kernel); out[j] = column j."""
    lines = []
    for j, (i, off_i, kexpr) in enumerate(top_cols(LB, LT, nlog)):
        lines.append(f"  {{ const R* __restrict__ tp = ltab + {off_i} + v; const R* __restrict__ tm = ltab + {off_i} - v; "
                     f"(void)tp; (void)tm; out[{j}] = {kexpr}; }}")
    sig = (f"template <typename R>\n__device__ __forceinline__ void "
           f"top_fill_lb{LB}_lt{LT}_n{nlog}(R* out, int v, const R* __restrict__ ltab, R base)")
    return sig + " {\n" + "\n".join(lines) + "\n}\n"


def scaled_mnet(em, y, HP, lam, sine, direction, nlog, LB):
    """Mirror network on the cells at multiples of LB (scaled segment
    [0, HP]); constants f(pi u/L) with the scaled u and L."""
    nmax = 1 << nlog
    def rec(a, L, rho, lens):
        if L < 4:
            return
        if direction == "bwd":
            lo_l = lens if rho == 0 else lens ^ sine
            hi_l = lens ^ sine if rho == 0 else lens
            rec(a, L // 2, 0, lo_l)
            rec(a + L // 2, L // 2, 1, hi_l)
        lg2L = (2 * L).bit_length() - 1
        for vv in range(1, L // 2):
            lo, hi = a + vv, a + L - vv
            j, m = (lo, hi) if rho == 0 else (hi, lo)
            k = "base" if vv == L // 4 else f"AMQFT_TABLD(tab, {vv * (nmax >> lg2L) - 1})"
            if direction == "fwd":
                p_, q_ = y[j], y[m]
                s_, d_ = add(p_, q_), sub(p_, q_)
                e_, o_ = (s_, d_) if lens == 0 else (d_, s_)
                y[j] = em.new(e_)
                y[m] = em.new(mul(o_, k))
            else:
                E, C = y[j], y[m]
                O = em.new(mul(C, k))
                if lens == 0:
                    y[j], y[m] = em.new(add(E, O)), em.new(sub(E, O))
                else:
                    y[j], y[m] = em.new(add(O, E)), em.new(sub(O, E))
        if direction == "fwd":
            lo_l = lens if rho == 0 else lens ^ sine
            hi_l = lens ^ sine if rho == 0 else lens
            rec(a, L // 2, 0, lo_l)
            rec(a + L // 2, L // 2, 1, hi_l)
    rec(0, HP, 0, lam)


def gen_small_full(v, HP, lam, nlog):
    """Cells at multiples of LB: time-major = full forward (scaled mirror
    network) + backward (tmS); harmonic-major = hmS + scaled backward."""
    sine = 1 if v >= 5 else 0
    em = Emitter()
    em.emit(f"constexpr int swsh = {0 if lam else 31};")
    ks = range(0, HP + 1) if lam == 0 else range(1, HP)
    if v in TM:
        y = {}
        for k in ks:
            em.emit(f"const R y{k} = T[PH({k} * LBV)];")
            y[k] = f"y{k}"
        scaled_mnet(em, y, HP, lam, sine, "fwd", nlog, None)
        G = [None] * (HP + 1)
        lg = HP.bit_length() - 1
        ntop = lg if lam == 0 else lg - 1
        Np = 2 * HP
        for t in range(ntop):
            sp = spectrum_tm(em, v, y, 0, HP, 0, lam, sine, t)
            hi = Np >> (t + 1)
            for p, name in enumerate(sp):
                G[hi - p - lam] = name
        if lam == 0:
            G[0] = em.new(add(y[0], y[HP]))
            G[1] = em.new(sub(y[0], y[HP]))
            n = 4
        else:
            G[1] = y[HP // 2]
            n = 8
        while n <= Np:
            for k in (range(n // 4) if lam == 0 else range(1, n // 4)):
                e, o = G[k], G[n // 2 - k]
                if lam == 0:
                    G[k], G[n // 2 - k] = em.new(add(e, o)), em.new(sub(e, o))
                else:
                    G[k], G[n // 2 - k] = em.new(add(o, e)), em.new(sub(o, e))
            n *= 2
        for k in ks:
            em.emit(f"F[SW({k})] = {G[k]};")
    else:
        S = {}
        for k in ks:
            em.emit(f"const R s{k} = T[SW({k})];")
            S[k] = f"s{k}"
        x = {}
        Np = 2 * HP
        n = Np
        while n >= (4 if lam == 0 else 8):
            for m in (range(n // 4) if lam == 0 else range(1, n // 4)):
                a_, b_ = S[m], S[n // 2 - m]
                if lam == 0:
                    S[m], S[n // 2 - m] = em.new(add(a_, b_)), em.new(sub(a_, b_))
                else:
                    S[m], S[n // 2 - m] = em.new(sub(a_, b_)), em.new(add(a_, b_))
            vals = [S[n // 2 - p - lam] for p in range(n // 4)]
            place_hm(em, v, vals, lam, sine, x, 0, HP, 0)
            n //= 2
        if lam == 0:
            x[0] = em.new(add(S[0], S[1]))
            x[HP] = em.new(sub(S[0], S[1]))
        else:
            x[HP // 2] = S[1]
        scaled_mnet(em, x, HP, lam, sine, "bwd", nlog, None)
        for k in ks:
            em.emit(f"F[PH({k} * LBV)] = {x[k]};")
    sig = (f"template <typename R, typename AR, int LOGLB, int LBV>\n__device__ __forceinline__ void "
           f"smallfull_v{v}_hp{HP}_n{nlog}_l{lam}(const R* __restrict__ T, R* __restrict__ F, "
           f"const R* __restrict__ tab, R base)")
    return sig + " {\n" + "\n".join(em.lines) + "\n}\n"


# --------------------------------------------- chain recombination (phase F)
def emit_pair(em, e, o, t, lam, fold):
    """Recombination (SplitTimeParity bwd, elab.cpp:310-329):
    Dct (E+O, E-O), Dst (O+E, O-E).  Fold (SplitHarmonicParity fwd,
    elab.cpp:238-255): Dct (a+b, a-b), Dst (a-b, a+b)."""
    if not fold:
        if lam == 0:
            em.emit(f"{{ const R e{t} = {e}; {e} = {add('e' + str(t), o)}; {o} = {sub('e' + str(t), o)}; }}")
        else:
            em.emit(f"{{ const R e{t} = {e}; {e} = {add(o, 'e' + str(t))}; {o} = {sub(o, 'e' + str(t))}; }}")
    else:
        if lam == 0:
            em.emit(f"{{ const R e{t} = {e}; {e} = {add('e' + str(t), o)}; {o} = {sub('e' + str(t), o)}; }}")
        else:
            em.emit(f"{{ const R e{t} = {e}; {e} = {sub('e' + str(t), o)}; {o} = {add('e' + str(t), o)}; }}")


def gen_recomb(W, HW, lam, special, fold=False):
    """SplitTimeParity recombination Dct/Dst(n), n = 2W .. 2 W HW (= N), for
    the thread owning k in [1, W/2): cells j*W + k (j < HW) and j*W - k
    (1 <= j <= HW), closed under every level (pairs (y, n/2 - y), y < n/4).
    special: the multiples of W/2 (k = 0 class).  Buffer padded by 1 per 32:
    phys(y) = y + y/32; for W = 64, j*W + k -> j*66 + k, j*W - k -> j*66 - 1 - k."""
    em = Emitter()
    N = 2 * W * HW
    if not special:
        cells = [("a", j) for j in range(HW)] + [("b", j) for j in range(1, HW + 1)]
        def val(c):  # symbolic (jW, sign)
            return (c[1] * W, 1 if c[0] == "a" else -1)
        name = {c: f"{c[0]}{c[1]}" for c in cells}
        assert W >= 64 and W % 32 == 0
        # phys(y) = y + (y + sh)/32, sh = 31 (Dct chain) / 0 (Dst chain):
        # phys(jW +- k) = j (W + W/32) +- k + ((sh +- k) >> 5), the last term a
        # per-thread constant (arithmetic shift = floor)
        JS = W + W // 32
        em.emit(f"constexpr int swsh = {31 if lam == 0 else 0};")
        em.emit("R* __restrict__ pa = F + k + ((k + swsh) >> 5);")
        em.emit("R* __restrict__ pb = F - k + ((swsh - k) >> 5);")
        for c in cells:
            off = c[1] * JS
            em.emit(f"R {name[c]} = {'pa' if c[0] == 'a' else 'pb'}[{off}];")
        levels = []
        n = 2 * W
        while n <= N:
            levels.append(n)
            n *= 2
        if fold:
            levels = levels[::-1]
        for n in levels:
            m = n // (2 * W)          # n/4 = m W/2
            for c in cells:
                jW, sg = val(c)
                j = c[1]
                lower = (2 * j < m) if sg > 0 else (2 * j <= m)
                if not lower:
                    continue
                # partner n/2 - y
                pj = n // (2 * W) - j
                pc = ("b", pj) if sg > 0 else ("a", pj)
                e, o = name[c], name[pc]
                em.tmp += 1
                t = em.tmp
                emit_pair(em, e, o, t, lam, fold)
        for c in cells:
            off = c[1] * JS
            em.emit(f"{'pa' if c[0] == 'a' else 'pb'}[{off}] = {name[c]};")
        nm = "fold" if fold else "recomb"
        sig = (f"template <typename R, typename AR>\n__device__ __forceinline__ void "
               f"{nm}_w{W}_hw{HW}_l{lam}(R* __restrict__ F, int k)")
    else:
        hw2 = W // 2
        ys = [i * hw2 for i in range(0, 2 * HW + 1)]
        if lam == 1:
            ys = [y for y in ys if 1 <= y <= N // 2 - 1]
        name = {y: f"s{y}" for y in ys}
        sh = 31 if lam == 0 else 0
        for y in ys:
            em.emit(f"R s{y} = F[{y + ((y + sh) >> 5)}];")
        levels = []
        n = 2 * W
        while n <= N:
            levels.append(n)
            n *= 2
        if fold:
            levels = levels[::-1]
        for n in levels:
            for y in ys:
                if y < n // 4 and (lam == 0 or y >= 1):
                    e, o = name[y], name[n // 2 - y]
                    em.tmp += 1
                    t = em.tmp
                    emit_pair(em, e, o, t, lam, fold)
        for y in ys:
            em.emit(f"F[{y + ((y + sh) >> 5)}] = s{y};")
        nm = "foldsp" if fold else "recombsp"
        sig = (f"template <typename R, typename AR>\n__device__ __forceinline__ void "
               f"{nm}_w{W}_hw{HW}_l{lam}(R* __restrict__ F)")
    return sig + " {\n" + "\n".join(em.lines) + "\n}\n"


# ------------------------------------ small chain, split for parallel lanes
def scaled_mnet_cls(em, y, HP, lam, sine, direction, nlog, cls):
    """scaled_mnet restricted to one trailing-zero class (classes never mix)."""
    nmax = 1 << nlog
    def rec(a, L, rho, lens):
        if L < 4:
            return
        lo_l = lens if rho == 0 else lens ^ sine
        hi_l = lens ^ sine if rho == 0 else lens
        if direction == "bwd":
            rec(a, L // 2, 0, lo_l)
            rec(a + L // 2, L // 2, 1, hi_l)
        lg2L = (2 * L).bit_length() - 1
        for vv in range(1, L // 2):
            if tz(vv) != cls:
                continue
            lo, hi = a + vv, a + L - vv
            j, m = (lo, hi) if rho == 0 else (hi, lo)
            k = "base" if vv == L // 4 else f"AMQFT_TABLD(tab, {vv * (nmax >> lg2L) - 1})"
            if direction == "fwd":
                p_, q_ = y[j], y[m]
                s_, d_ = add(p_, q_), sub(p_, q_)
                e_, o_ = (s_, d_) if lens == 0 else (d_, s_)
                y[j] = em.new(e_)
                y[m] = em.new(mul(o_, k))
            else:
                E, C = y[j], y[m]
                O = em.new(mul(C, k))
                if lens == 0:
                    y[j], y[m] = em.new(add(E, O)), em.new(sub(E, O))
                else:
                    y[j], y[m] = em.new(add(O, E)), em.new(sub(O, E))
        if direction == "fwd":
            rec(a, L // 2, 0, lo_l)
            rec(a + L // 2, L // 2, 1, hi_l)
    rec(0, HP, 0, lam)


def gen_small_tm_class(v, HP, lam, nlog, cls):
    """Time-major: one class of the cells at multiples of LB -- forward
    mirror levels and the spectrum of its small top block, written to F;
    cls == log2(HP) is the Dct(2)/Dst(4) base."""
    sine = 1 if v >= 5 else 0
    em = Emitter()
    em.emit(f"constexpr int swsh = {0 if lam else 31};")
    lg = HP.bit_length() - 1
    Np = 2 * HP
    if cls == lg:
        if lam == 0:
            em.emit("const R y0 = T[PH(0)], yh = T[PH(" + str(HP) + " * LBV)];")
            em.emit(f"F[SW(0)] = {add('y0', 'yh')};")
            em.emit(f"F[SW(1)] = {sub('y0', 'yh')};")
        else:
            em.emit(f"F[SW(1)] = T[PH({HP // 2} * LBV)];")
    elif lam == 1 and cls == lg - 1:
        pass  # Dst chain: the centre is Dst(4), handled by the base lane
    else:
        y = {}
        for k in range(1, HP):
            if tz(k) == cls:
                em.emit(f"const R y{k} = T[PH({k} * LBV)];")
                y[k] = f"y{k}"
        scaled_mnet_cls(em, y, HP, lam, sine, "fwd", nlog, cls)
        sp = spectrum_tm(em, v, y, 0, HP, 0, lam, sine, cls)
        hi = (Np >> (cls + 1)) - lam
        for p, name in enumerate(sp):
            em.emit(f"F[SW({hi - p})] = {name};")
    sig = (f"template <typename R, typename AR, int LOGLB, int LBV>\n__device__ __forceinline__ void "
           f"smtm_v{v}_hp{HP}_n{nlog}_l{lam}_c{cls}(const R* __restrict__ T, R* __restrict__ F, "
           f"const R* __restrict__ tab, R base)")
    return sig + " {\n" + "\n".join(em.lines) + "\n}\n"


def gen_small_tm_recomb(HP, lam):
    """Time-major: SplitTimeParity recombination Dct/Dst(n), n = 4|8 .. 2HP,
    on F cells [0, HP] in registers."""
    em = Emitter()
    em.emit(f"constexpr int swsh = {0 if lam else 31};")
    ks = range(0, HP + 1) if lam == 0 else range(1, HP)
    G = {}
    for k in ks:
        em.emit(f"const R g{k} = F[SW({k})];")
        G[k] = f"g{k}"
    n = 4 if lam == 0 else 8
    while n <= 2 * HP:
        for k in (range(n // 4) if lam == 0 else range(1, n // 4)):
            e, o = G[k], G[n // 2 - k]
            if lam == 0:
                G[k], G[n // 2 - k] = em.new(add(e, o)), em.new(sub(e, o))
            else:
                G[k], G[n // 2 - k] = em.new(add(o, e)), em.new(sub(o, e))
        n *= 2
    for k in ks:
        em.emit(f"F[SW({k})] = {G[k]};")
    sig = (f"template <typename R, typename AR>\n__device__ __forceinline__ void "
           f"smtm_recomb_hp{HP}_l{lam}(R* __restrict__ F)")
    return sig + " {\n" + "\n".join(em.lines) + "\n}\n"


def gen_small_hm_fold(HP, lam):
    """Harmonic-major: SplitHarmonicParity folds n = 2HP .. 4|8 on T cells
    [0, HP] in registers (in place)."""
    em = Emitter()
    em.emit(f"constexpr int swsh = {0 if lam else 31};")
    ks = range(0, HP + 1) if lam == 0 else range(1, HP)
    S_ = {}
    for k in ks:
        em.emit(f"const R s{k} = T[SW({k})];")
        S_[k] = f"s{k}"
    n = 2 * HP
    while n >= (4 if lam == 0 else 8):
        for m in (range(n // 4) if lam == 0 else range(1, n // 4)):
            a_, b_ = S_[m], S_[n // 2 - m]
            if lam == 0:
                S_[m], S_[n // 2 - m] = em.new(add(a_, b_)), em.new(sub(a_, b_))
            else:
                S_[m], S_[n // 2 - m] = em.new(sub(a_, b_)), em.new(add(a_, b_))
        n //= 2
    for k in ks:
        em.emit(f"T[SW({k})] = {S_[k]};")
    sig = (f"template <typename R, typename AR>\n__device__ __forceinline__ void "
           f"smhm_fold_hp{HP}_l{lam}(R* __restrict__ T)")
    return sig + " {\n" + "\n".join(em.lines) + "\n}\n"


def gen_small_hm_class(v, HP, lam, nlog, cls):
    """Harmonic-major: one small top block (after the folds, its temporal
    cells are reversed in T (n/4, n/2]): gathers + AM_F placing its leaves
    on the scaled segment, then its mirror levels, written to F at
    multiples of LB; cls == log2(HP) is the Dct(2)/Dst(4) base."""
    sine = 1 if v >= 5 else 0
    em = Emitter()
    em.emit(f"constexpr int swsh = {0 if lam else 31};")
    lg = HP.bit_length() - 1
    Np = 2 * HP
    if cls == lg:
        if lam == 0:
            em.emit("const R t0 = T[SW(0)], t1 = T[SW(1)];")
            em.emit(f"F[PH(0)] = {add('t0', 't1')};")
            em.emit(f"F[PH({HP} * LBV)] = {sub('t0', 't1')};")
        else:
            em.emit(f"F[PH({HP // 2} * LBV)] = T[SW(1)];")
    elif lam == 1 and cls == lg - 1:
        pass
    else:
        n = Np >> cls
        vals = []
        for p in range(n // 4):
            em.emit(f"const R u{p} = T[SW({n // 2 - p - lam})];")
            vals.append(f"u{p}")
        x = {}
        place_hm(em, v, vals, lam, sine, x, 0, HP, 0)
        scaled_mnet_cls(em, x, HP, lam, sine, "bwd", nlog, cls)
        for k in sorted(x):
            em.emit(f"F[PH({k} * LBV)] = {x[k]};")
    sig = (f"template <typename R, typename AR, int LOGLB, int LBV>\n__device__ __forceinline__ void "
           f"smhm_v{v}_hp{HP}_n{nlog}_l{lam}_c{cls}(const R* __restrict__ T, R* __restrict__ F, "
           f"const R* __restrict__ tab, R base)")
    return sig + " {\n" + "\n".join(em.lines) + "\n}\n"


# (LB, nlog) pairs of the fused kernels: LT = nlog - 1 - log2(LB), HP = 2^LT
FULL_SIZES = [(64, 10), (64, 11), (64, 12), (64, 13)]


# Sizes instantiated by csrc/fast.cu (LB, HP = N/(2 LB)).
CONFIGS = [
    # (LB, [HP...])
    (64, [8, 16, 32, 64]),
]


def main():
    out = [
        "// fast_gen.cuh -- GENERATED by codegen/gen_fast.py; do not edit.",
        "// Straight-line bottom-of-recursion code for the fused AM-QFT kernels.",
        "#pragma once",
        "#define PH(i) ((i) + ((i) >> LOGLB))",
        "#define SW(i) ((i) + (((i) + swsh) >> 5))",
        "// constant-table read: __ldg from global memory by default; the fused",
        "// kernel reads it from its parameter space (constant bank operands)",
        "#ifndef AMQFT_TABLD",
        "#define AMQFT_TABLD(t, i) __ldg((t) + (i))",
        "#endif",
        "#ifndef AMQFT_CLASS_FENCE",
        "#define AMQFT_CLASS_FENCE() asm volatile(\"\" ::: \"memory\")",
        "#endif",
        "namespace amqft_b200 {",
        "namespace gen {",
    ]
    hp_all = sorted({hp for _, hps in CONFIGS for hp in hps})
    for LB, hps in CONFIGS:
        for v in range(1, 9):
            for rho in (0,):   # odd segments are stored reversed (Cfg::ipos)
                for lam in (0, 1):
                    for part in (0, 1, 2):
                        out.append(gen_tmB(v, LB, rho, lam, part) if v in TM else gen_hmB(v, LB, rho, lam, part))
    for v in range(1, 9):
        for hp in hp_all:
            for lam in (0, 1):
                body = gen_tmS(v, hp, "LBV", lam) if v in TM else gen_hmS(v, hp, "LBV", lam)
                body = body.replace("template <typename R, typename AR, int LOGLB>",
                                    "template <typename R, typename AR, int LOGLB, int LBV>")
                out.append(body)
    for LB, nlog in FULL_SIZES:
        LT = nlog - 1 - (LB.bit_length() - 1)
        for direction in ("fwd", "bwd"):
            for lam in (0, 1):
                for sine in (0, 1):
                    out.append(gen_top(LB, LT, direction, lam, sine, nlog))
                    out.append(gen_top(LB, LT, direction, lam, sine, nlog, kmode="tm"))
        out.append(gen_top_fill(LB, LT, nlog))
        HP = 1 << LT
        for v in range(1, 9):
            for lam in (0, 1):
                out.append(gen_small_full(v, HP, lam, nlog))
    small_hps = set()
    for LB, nlog in FULL_SIZES:
        LT = nlog - 1 - (LB.bit_length() - 1)
        HP = 1 << LT
        small_hps.add(HP)
        for v in range(1, 9):
            for lam in (0, 1):
                for cls in range(LT + 1):
                    out.append(gen_small_tm_class(v, HP, lam, nlog, cls) if v in TM
                               else gen_small_hm_class(v, HP, lam, nlog, cls))
    for HP in sorted(small_hps):
        for lam in (0, 1):
            out.append(gen_small_tm_recomb(HP, lam))
            out.append(gen_small_hm_fold(HP, lam))
    for LB, nlog in FULL_SIZES:
        N = 1 << nlog
        W = max(64, N // LB)      # recombination thread sets {j W +- k}
        HW = (N // 2) // W
        for lam in (0, 1):
            for fold in (False, True):
                out.append(gen_recomb(W, HW, lam, False, fold))
                out.append(gen_recomb(W, HW, lam, True, fold))
    out.append("}  // namespace gen")
    out.append("template <int W, int HW> struct Recomb;")
    for LB, nlog in FULL_SIZES:
        N = 1 << nlog
        W = max(64, N // LB)
        HW = (N // 2) // W
        if True:
            out.append(f"template <> struct Recomb<{W}, {HW}> {{")
            out.append("  template <typename R, typename AR>")
            out.append("  static __device__ __forceinline__ void run(int lam, R* F, int k) {")
            out.append(f"    if (k == 0) {{ if (lam == 0) gen::recombsp_w{W}_hw{HW}_l0<R, AR>(F); else gen::recombsp_w{W}_hw{HW}_l1<R, AR>(F); }}")
            out.append(f"    else {{ if (lam == 0) gen::recomb_w{W}_hw{HW}_l0<R, AR>(F, k); else gen::recomb_w{W}_hw{HW}_l1<R, AR>(F, k); }}")
            out.append("  }")
            out.append("  template <typename R, typename AR>")
            out.append("  static __device__ __forceinline__ void fold(int lam, R* F, int k) {")
            out.append(f"    if (k == 0) {{ if (lam == 0) gen::foldsp_w{W}_hw{HW}_l0<R, AR>(F); else gen::foldsp_w{W}_hw{HW}_l1<R, AR>(F); }}")
            out.append(f"    else {{ if (lam == 0) gen::fold_w{W}_hw{HW}_l0<R, AR>(F, k); else gen::fold_w{W}_hw{HW}_l1<R, AR>(F, k); }}")
            out.append("  }")
            out.append("};")
    out.append("template <int LB, int LT, int NLOG, int SINE> struct Top;")
    for LB, nlog in FULL_SIZES:
        LT = nlog - 1 - (LB.bit_length() - 1)
        for sine in (0, 1):
            out.append(f"template <> struct Top<{LB}, {LT}, {nlog}, {sine}> {{")
            out.append(f"  static constexpr int NK = {len(top_cols(LB, LT, nlog))};   // distinct constants per thread")
            for direction in ("fwd", "bwd"):
                out.append("  template <typename R, typename AR>")
                out.append(f"  static __device__ __forceinline__ void {direction}(int lam, R* B, int v, const R* ltab, R base) {{")
                out.append(f"    if (lam == 0) gen::top_{direction}_lb{LB}_lt{LT}_n{nlog}_l0_s{sine}<R, AR>(B, v, ltab, base);")
                out.append(f"    else gen::top_{direction}_lb{LB}_lt{LT}_n{nlog}_l1_s{sine}<R, AR>(B, v, ltab, base);")
                out.append("  }")
                out.append("  template <typename R, typename AR>")
                out.append(f"  static __device__ __forceinline__ void {direction}_k(int lam, R* B, int v, const R* kk) {{")
                out.append(f"    if (lam == 0) gen::top_{direction}_lb{LB}_lt{LT}_n{nlog}_l0_s{sine}_tm<R, AR>(B, v, kk);")
                out.append(f"    else gen::top_{direction}_lb{LB}_lt{LT}_n{nlog}_l1_s{sine}_tm<R, AR>(B, v, kk);")
                out.append("  }")
            out.append("  template <typename R>")
            out.append("  static __device__ __forceinline__ void fill(R* out, int v, const R* ltab, R base) {")
            out.append(f"    gen::top_fill_lb{LB}_lt{LT}_n{nlog}<R>(out, v, ltab, base);")
            out.append("  }")
            out.append("};")
    out.append("template <int V, int HP, int NLOG> struct SmallPar;")
    for LB, nlog in FULL_SIZES:
        LT = nlog - 1 - (LB.bit_length() - 1)
        HP = 1 << LT
        for v in range(1, 9):
            fam = "smtm" if v in TM else "smhm"
            out.append(f"template <> struct SmallPar<{v}, {HP}, {nlog}> {{")
            out.append(f"  static constexpr int NCLS = {LT + 1};")
            out.append("  template <typename R, typename AR, int LOGLB, int LBV>")
            out.append("  static __device__ __forceinline__ void cls(int lam, int c, const R* T, R* F, const R* tab, R base) {")
            for lam in (0, 1):
                for cls in range(LT + 1):
                    out.append(f"    if (lam == {lam} && c == {cls}) {{ gen::{fam}_v{v}_hp{HP}_n{nlog}_l{lam}_c{cls}"
                               f"<R, AR, LOGLB, LBV>(T, F, tab, base); return; }}")
            out.append("  }")
            out.append("  template <typename R, typename AR>")
            out.append("  static __device__ __forceinline__ void serial(int lam, R* B) {")
            ser = "smtm_recomb" if v in TM else "smhm_fold"
            out.append(f"    if (lam == 0) gen::{ser}_hp{HP}_l0<R, AR>(B); else gen::{ser}_hp{HP}_l1<R, AR>(B);")
            out.append("  }")
            out.append("};")
    out.append("template <int V, int HP, int NLOG> struct SmallFull;")
    for LB, nlog in FULL_SIZES:
        LT = nlog - 1 - (LB.bit_length() - 1)
        HP = 1 << LT
        for v in range(1, 9):
            out.append(f"template <> struct SmallFull<{v}, {HP}, {nlog}> {{")
            out.append("  template <typename R, typename AR, int LOGLB, int LBV>")
            out.append("  static __device__ __forceinline__ void run(int lam, const R* T, R* F, const R* tab, R base) {")
            out.append(f"    if (lam == 0) gen::smallfull_v{v}_hp{HP}_n{nlog}_l0<R, AR, LOGLB, LBV>(T, F, tab, base);")
            out.append(f"    else gen::smallfull_v{v}_hp{HP}_n{nlog}_l1<R, AR, LOGLB, LBV>(T, F, tab, base);")
            out.append("  }")
            out.append("};")
    # Compile-time dispatch: Bottom<V, LB> and Small<V, HP>.
    out.append("template <int V, int LB> struct Bottom;")
    for LB, _ in CONFIGS:
        for v in range(1, 9):
            fam = "tmB" if v in TM else "hmB"
            out.append(f"template <> struct Bottom<{v}, {LB}> {{")
            out.append("  template <typename R, typename AR, int LOGLB, int D, int PART>")
            out.append("  static __device__ __forceinline__ void run(int rho, int lens, const R* T, R* F, int a, "
                       "const R* tab, int nmax, R base, int N, int r, int dsto) {")
            # orientation 0 only (rho is ignored): odd segments are stored
            # reversed, which is exactly the orientation-1 segment
            out.append("    (void)rho;")
            for lam in (0, 1):
                pre = f"gen::{fam}_v{v}_lb{LB}_r0_l{lam}"
                args = "<R, AR, LOGLB, D>(T, F, a, tab, nmax, base, N, r, dsto)"
                out.append(f"    if (lens == {lam}) {{ if constexpr (PART == 0) {pre}_p0{args}; "
                           f"else if constexpr (PART == 2) {pre}_p2{args}; else {pre}_p1{args}; return; }}")
            out.append("  }")
            out.append("};")
    out.append("template <int V, int HP> struct Small;")
    for v in range(1, 9):
        fam = "tmS" if v in TM else "hmS"
        for hp in hp_all:
            out.append(f"template <> struct Small<{v}, {hp}> {{")
            out.append("  template <typename R, typename AR, int LOGLB, int LBV>")
            out.append("  static __device__ __forceinline__ void run(int lam, const R* T, R* F, R base) {")
            out.append(f"    if (lam == 0) gen::{fam}_v{v}_hp{hp}_l0<R, AR, LOGLB, LBV>(T, F, base);")
            out.append(f"    else gen::{fam}_v{v}_hp{hp}_l1<R, AR, LOGLB, LBV>(T, F, base);")
            out.append("  }")
            out.append("};")
    out += ["}  // namespace amqft_b200", "#undef PH", "#undef SW", ""]
    sys.stdout.write("\n".join(out))


if __name__ == "__main__":
    main()
