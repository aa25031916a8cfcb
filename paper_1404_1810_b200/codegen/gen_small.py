#!/usr/bin/env python3
"""Generates csrc/small_gen.cuh: one whole small transform per thread.

For small N the AM-QFT recursion of one signal is a few hundred to a few
thousand scalar operations.  This generator TRACES the compiled stage
program of the plan compiler (csrc/plan.cpp via `amqft_schedule_dump`,
host-only) on symbolic cells, so every SSA node below is exactly one of the
reference's add/sub/mul on the reference's operands (elaborations.cpp and
variants.cpp, cited per case in `_item`), and emits it as straight-line code
that keeps the signal in registers.  The generated functions are
instantiated in csrc/small_kernel.cuh (one thread per row, rows staged in
shared memory by TMA bulk copies).  fp64 results are therefore bitwise those
of amqft::execute, for every variant (serial recurrences included, in the
reference order).

Shared memory is touched in 16-byte chunks only (float4 / double2): a row
slot is padded by 16 bytes, so the 8 lanes of a quarter-warp that read the
same chunk of 8 different rows hit 8 different 16-byte bank groups.  The
row is transformed in place: a chunk is stored only once all its cells are
final, and never before its input cells were loaded.

Run by csrc/Makefile at build time (the output is not committed):
  python3 codegen/gen_small.py --lib csrc/build/libamqft_plan.so --out csrc/gen
"""
from __future__ import annotations

import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

# EI opcodes (csrc/plan.hpp)
SC_F, SC_B, SR_F, SR_B, GATHER, SCATTER, SH_F_DCT, SH_F_DST, SH_F_ODD = range(1, 10)
ST_B_DCT, ST_B_DST, ST_B_ODD, AM_F, AM_B, BASE_CDFT2, BASE_PAIR2, BASE_OO8 = range(10, 18)
CHAIN_F, CHAIN_B = 18, 19
FL_DESC, FL_ADD = 4, 8

# Sizes covered per dtype (register budget: the live set of one thread).
SIZES = {"float": (2, 4, 8, 16, 32, 64), "double": (2, 4, 8, 16, 32)}
# RDFT rows (FunctionId::Rdft, N reals, packed spectrum): half the live set
RDFT_SIZES = {"float": (4, 8, 16, 32, 64, 128), "double": (2, 4, 8, 16, 32, 64)}
# DCT-0 / DST-0 rows (FunctionId::Dct/Dst; N/2 + 1 / N/2 - 1 cells)
DCT_SIZES = {"float": (4, 8, 16, 32, 64, 128, 256), "double": (4, 8, 16, 32, 64, 128)}
DST_SIZES = {"float": (8, 16, 32, 64, 128, 256), "double": (8, 16, 32, 64, 128)}
# Cooperative rows: N -> (head stages, tail stages, warp roles)
COOP = {"float": {128: (2, 2, 4), 256: (3, 3, 8), 512: (4, 4, 16)},
        "double": {64: (2, 2, 4), 128: (3, 3, 8), 256: (4, 4, 16)}}
# rows per CTA tile (lanes past it duplicate rows lane % ROWS); 32 for all
# generated instances (fp64 N = 512 would need 16-row tiles for shared memory
# and spills at 16 roles: it runs as a 16 x 32 four-step instead)
COOP_ROWS = {}


def _items(op, n):
    if op in (SC_F, SC_B):
        return 2 * n
    if op in (SR_F, SR_B, GATHER, SCATTER):
        return n
    if op in (SH_F_DCT, ST_B_DCT):
        return n // 2 + 1
    if op in (SH_F_DST, ST_B_DST):
        return n // 2 - 1
    if op in (SH_F_ODD, ST_B_ODD):
        return n // 4
    if op in (AM_F, AM_B):
        return n // 8
    return {BASE_CDFT2: 4, BASE_PAIR2: 2, BASE_OO8: 1}[op]


class Trace:
    """SSA graph: node = ('in', p) | ('add'|'sub', a, b) | ('mul', a, slot) | ('half', a)."""

    def __init__(self, cells):
        self.nodes = [("in", p) for p in range(cells)]

    def op(self, *t):
        self.nodes.append(t)
        return len(self.nodes) - 1

    def add(self, a, b):
        return self.op("add", a, b)

    def sub(self, a, b):
        return self.op("sub", a, b)

    def mul(self, a, slot):
        return self.op("mul", a, slot)

    def half(self, a):
        return self.op("half", a)


def _item(T, e, i, L, nmax):
    """Symbolic twin of eval_item (csrc/generic.cuh): node of item i of EI e."""
    op, lens, am, n, aux = e
    if op == SC_F:      # elaborations.cpp:152-155
        return L(2 * i) if i < n else L(2 * (i - n) + 1)
    if op == SC_B:      # elaborations.cpp:166-181; A at [0,n), B at [n,2n)
        k, im = i >> 1, i & 1
        if k == 0 or k == n // 2:
            return L(n + k) if im else L(k)
        if k < n // 2:
            return T.sub(L(n + k), L(n - k)) if im else T.add(L(k), L(2 * n - k))
        j = n - k
        return T.add(L(n + j), L(k)) if im else T.sub(L(j), L(n + k))
    if op == SR_F:      # elaborations.cpp:190-195
        if i == 0 or i == n // 2:
            return L(i)
        if i < n // 2:
            return T.add(L(i), L(n - i))
        m = i - n // 2
        return T.sub(L(m), L(n - m))
    if op == SR_B:      # elaborations.cpp:203-206
        return L(i) if i <= n // 2 else L(3 * n // 2 - i)
    if op == GATHER:    # elaborations.cpp:288-295
        return L(2 * i + lens) if i < aux else L(2 * (i - aux) + 1 - lens)
    if op == SCATTER:   # elaborations.cpp:268-275
        return L(i >> 1) if (i & 1) == lens else L(aux + (i >> 1))
    if op == SH_F_DCT:  # elaborations.cpp:238-255
        if i <= n // 4:
            return L(i) if i == n // 4 else T.add(L(i), L(n // 2 - i))
        j = i - (n // 4 + 1)
        return T.sub(L(j), L(n // 2 - j))
    if op == SH_F_DST:
        if i < n // 4 - 1:
            return T.sub(L(i), L(n // 2 - i - 2))
        idx = i - (n // 4 - 1) + 1
        return L(idx - 1) if idx == n // 4 else T.add(L(idx - 1), L(n // 2 - idx - 1))
    if op == SH_F_ODD:
        mc = n // 4
        if i < mc // 2:
            return T.sub(L(i), L(mc - 1 - i)) if lens else T.add(L(i), L(mc - 1 - i))
        j = i - mc // 2
        return T.add(L(j), L(mc - 1 - j)) if lens else T.sub(L(j), L(mc - 1 - j))
    if op == ST_B_DCT:  # elaborations.cpp:310-319
        o = n // 4 + 1
        if i < n // 4:
            return T.add(L(i), L(o + i))
        if i == n // 4:
            return L(i)
        j = n // 2 - i
        return T.sub(L(j), L(o + j))
    if op == ST_B_DST:  # elaborations.cpp:320-329
        o = n // 4 - 1
        k = i + 1
        if k < n // 4:
            return T.add(L(o + k - 1), L(k - 1))
        if k == n // 4:
            return L(o + n // 4 - 1)
        j = n // 2 - k
        return T.sub(L(o + j - 1), L(j - 1))
    if op == ST_B_ODD:
        mc = n // 4
        o = mc // 2
        if i < o:
            return T.add(L(o + i), L(i)) if lens else T.add(L(i), L(o + i))
        j = mc - 1 - i
        return T.sub(L(o + j), L(j)) if lens else T.sub(L(j), L(o + j))
    if op in (AM_F, AM_B):  # elaborations.cpp:359-398 (F), 460-526 (B)
        q = aux
        pointwise = am in ((1, 4, 5, 8) if op == AM_F else (2, 3, 6, 7))
        if pointwise:
            return T.mul(L(i), (2 * i + 1) * (nmax // n) - 1)
        if op == AM_F and am == 2:
            if lens == 0:
                return L(0) if i == 0 else T.add(L(i), L(i - 1))
            return L(q - 1) if i == q - 1 else T.add(L(i + 1), L(i))
        if op == AM_F:  # 6
            if lens == 0:
                return L(q - 1) if i == q - 1 else T.sub(L(i), L(i + 1))
            return L(0) if i == 0 else T.sub(L(i), L(i - 1))
        if am == 4:
            if lens == 0:
                return T.add(L(i), L(i + 1)) if i < q - 1 else L(q - 1)
            return L(0) if i == 0 else T.add(L(i - 1), L(i))
        # 8
        if lens == 0:
            return L(0) if i == 0 else T.sub(L(i), L(i - 1))
        return T.sub(L(i), L(i + 1)) if i < q - 1 else L(q - 1)
    if op == BASE_CDFT2:  # variants.cpp:360-363
        return T.add(L(i), L(i + 2)) if i < 2 else T.sub(L(i - 2), L(i))
    if op == BASE_PAIR2:  # variants.cpp:366-371
        return T.add(L(0), L(1)) if i == 0 else T.sub(L(0), L(1))
    if op == BASE_OO8:    # variants.cpp:390
        return T.mul(L(0), nmax // 4 - 1)
    raise ValueError(op)


def _chain(T, e, L):
    """Serial recurrences (generic.cuh run_chain; elaborations.cpp:402-448, 472-513)."""
    op, flags, q = e[0], e[5], e[4]
    desc, add = bool(flags & FL_DESC), bool(flags & FL_ADD)
    s, d = (q - 1, -1) if desc else (0, 1)
    f = T.add if add else T.sub
    out = {}
    if op == CHAIN_F:
        if q == 1:
            out[0] = T.half(L(0))
            return out
        prev = L(s)
        out[s] = prev
        p = s
        for _ in range(1, q - 1):
            p += d
            prev = f(L(p), prev)
            out[p] = prev
        p += d
        out[p] = T.half(f(L(p), prev))
        return out
    prev = T.half(L(s))
    out[s] = prev
    p = s
    for _ in range(1, q):
        p += d
        prev = f(L(p), prev)
        out[p] = prev
    return out


_PLANLIB = None


def _schedule_dump(v, f, n):
    """The plan compiler's single-CTA stage program.  At build time from the
    host-only library build/libamqft_plan.so (plan.cpp, no CUDA), else
    through the package."""
    if _PLANLIB is None:
        import paper_1404_1810_b200 as amqft
        return amqft.schedule_dump(v, f, n)
    import ctypes as C
    import numpy as np
    from paper_1404_1810_b200 import EI_DTYPE
    L = _PLANLIB
    cnt, nst = C.c_size_t(), C.c_size_t()
    st0 = L.amqft_schedule_dump(v, f, n, 1 << 20, None, 0, C.byref(cnt), None, 0, C.byref(nst), None)
    assert st0 == 0
    recs = np.zeros(cnt.value, dtype=EI_DTYPE)
    st = np.zeros(2 * nst.value, dtype=np.uint32)
    ops = (C.c_uint64 * 3)()
    st0 = L.amqft_schedule_dump(v, f, n, 1 << 20, C.c_void_p(recs.ctypes.data), recs.size, C.byref(cnt),
                                C.c_void_p(st.ctypes.data), nst.value, C.byref(nst), ops)
    assert st0 == 0
    return recs, st.reshape(-1, 2), tuple(int(x) for x in ops)


def trace(v, f, n):
    """(Trace, outputs): outputs[p] = node holding output cell p."""
    recs, stages, ops = _schedule_dump(v, f, n)
    nmax = max(n, 8)
    cells = {0: 2 * n, 1: n, 2: n // 2 + 1, 3: n // 2 - 1}.get(f)   # CDFT, RDFT, DCT, DST (signal.cpp:118-223)
    if cells is None:
        import paper_1404_1810_b200 as amqft
        cells = amqft.cell_count(f, n)
    T = Trace(cells)
    T.stage = [-1] * cells
    T.snap = [list(range(cells))]        # arena after each stage
    x = list(range(cells))
    for si, (b, e) in enumerate(stages):
        first = len(T.nodes)
        writes = []
        for k in range(int(b), int(e)):
            r = recs[k]
            op, off = int(r["op"]), int(r["off"])
            ei = (op, int(r["lens"]), int(r["am"]), int(r["n"]), int(r["aux"]), int(r["flags"]))
            L = (lambda base: (lambda p: x[base + p]))(off)
            if op in (CHAIN_F, CHAIN_B):
                for p, node in _chain(T, ei, L).items():
                    writes.append((off + p, node))
            else:
                for i in range(_items(op, ei[3])):
                    writes.append((off + i, _item(T, ei[:5], i, L, nmax)))
        for p, node in writes:
            x[p] = node
        T.stage += [si] * (len(T.nodes) - first)
        T.snap.append(list(x))
    return T, x, ops


def count_ops(T, outs):
    """(adds, muls, halvings) of the nodes the outputs depend on."""
    need = set()
    stack = list(outs)
    while stack:
        u = stack.pop()
        if u in need:
            continue
        need.add(u)
        nd = T.nodes[u]
        if nd[0] in ("add", "sub"):
            stack += [nd[1], nd[2]]
        elif nd[0] in ("mul", "half"):
            stack.append(nd[1])
    c = [0, 0, 0]
    for u in need:
        k = T.nodes[u][0]
        if k in ("add", "sub"):
            c[0] += 1
        elif k == "mul":
            c[1] += 1
        elif k == "half":
            c[2] += 1
    return tuple(c)


def evaluate(T, outs, x, tab):
    """numpy/Python-float evaluation of the SSA program (IEEE double, one
    rounding per op, as on the device): the CPU check of the generator."""
    val = [None] * len(T.nodes)
    for u, nd in enumerate(T.nodes):
        k = nd[0]
        if k == "in":
            val[u] = float(x[nd[1]])
        elif k == "add":
            val[u] = val[nd[1]] + val[nd[2]]
        elif k == "sub":
            val[u] = val[nd[1]] - val[nd[2]]
        elif k == "mul":
            val[u] = val[nd[1]] * float(tab[nd[2]])
        else:
            val[u] = 0.5 * val[nd[1]]
    return [val[o] for o in outs]


def schedule(T, outs, W):
    """Emission order: post-order DFS from the outputs, chunk by chunk, so
    the cone of one output chunk is finished before the next starts (the
    recursion's depth-first order).  Returns a list of instructions:
      ('ld', c) load input chunk c (W cells); ('op', u); ('st', c).
    Input chunk c is always loaded before output chunk c is stored."""
    cells = len(outs)
    nchunks = cells // W
    loaded = [False] * nchunks
    done = set()
    prog = []

    def need_input(p):
        c = p // W
        if not loaded[c]:
            loaded[c] = True
            prog.append(("ld", c))
            for q in range(c * W, c * W + W):
                done.add(q)

    def visit(u):
        stack = [(u, False)]
        while stack:
            w, expanded = stack.pop()
            if w in done:
                continue
            nd = T.nodes[w]
            if nd[0] == "in":
                need_input(nd[1])
                continue
            if expanded:
                done.add(w)
                prog.append(("op", w))
                continue
            stack.append((w, True))
            ops = [nd[1], nd[2]] if nd[0] in ("add", "sub") else [nd[1]]
            for o in reversed(ops):
                if o not in done:
                    stack.append((o, False))

    for c in range(nchunks):
        for p in range(c * W, c * W + W):
            visit(outs[p])
        if not loaded[c]:   # in place: the chunk's inputs must be read first
            need_input(c * W)
        prog.append(("st", c))
    return prog


def schedule_trace(T, outs, W):
    """Emission order = trace order (the stage program: each stage reads
    all its operands, then writes), inputs loaded at first use, an output
    chunk stored as soon as its last cell is final."""
    cells = len(outs)
    nchunks = cells // W
    need = set()
    stack = list(outs)
    while stack:
        u = stack.pop()
        if u in need:
            continue
        need.add(u)
        nd = T.nodes[u]
        if nd[0] in ("add", "sub"):
            stack += [nd[1], nd[2]]
        elif nd[0] in ("mul", "half"):
            stack.append(nd[1])
    pos_of = {}
    for p, u in enumerate(outs):
        pos_of.setdefault(u, []).append(p)
    remaining = [W] * nchunks
    loaded = [False] * nchunks
    prog = []

    def ld(c):
        if not loaded[c]:
            loaded[c] = True
            prog.append(("ld", c))

    def produced(u):
        for p in pos_of.get(u, ()):
            c = p // W
            remaining[c] -= 1
            if remaining[c] == 0:
                ld(c)
                prog.append(("st", c))

    for p, u in enumerate(outs):   # outputs that are untouched inputs
        if T.nodes[u][0] == "in":
            ld(T.nodes[u][1] // W)
    for u in sorted(need):
        nd = T.nodes[u]
        if nd[0] == "in":
            ld(nd[1] // W)
            produced(u)
            continue
        prog.append(("op", u))
        produced(u)
    return prog


def max_live(T, outs, prog, W):
    last = {}
    for t, ins in enumerate(prog):
        if ins[0] == "op":
            nd = T.nodes[ins[1]]
            for o in ([nd[1], nd[2]] if nd[0] in ("add", "sub") else [nd[1]]):
                last[o] = t
        elif ins[0] == "st":
            for p in range(ins[1] * W, ins[1] * W + W):
                last[outs[p]] = t
    live, peak = set(), 0
    for t, ins in enumerate(prog):
        if ins[0] == "ld":
            live |= set(range(ins[1] * W, ins[1] * W + W))
        elif ins[0] == "op":
            live.add(ins[1])
        peak = max(peak, len(live))
        live = {u for u in live if last.get(u, -1) > t}
    return peak


def emit_fn(v, f, n, R):
    # chunk width: 16-byte vectors for CDFT/RDFT rows; DCT/DST rows (N/2 +- 1
    # cells, odd) are scalar (their odd smem row stride is conflict-free)
    W = 1 if f in (2, 3) else (4 if R == "float" else 2)
    T, outs, ops = trace(v, f, n)
    prog = schedule_trace(T, outs, W)
    name = lambda u: (f"x{u}" if T.nodes[u][0] == "in" else f"t{u}")  # noqa: E731
    lines = [f"template <> struct SmallGen<{v}, {f}, {n.bit_length() - 1}, {R}> {{",
             f"  static constexpr int PEAK = {max_live(T, outs, prog, W)};",
             f"  static constexpr unsigned long long OPS[3] = {{{ops[0]}ull, {ops[1]}ull, {ops[2]}ull}};",
             "  template <class AR, class IO>",
             f"  static __device__ __forceinline__ void run(IO& io, const {R}* __restrict__ tab) {{"]
    for ins in prog:
        if ins[0] == "ld":
            c = ins[1]
            names = ", ".join(f"x{p}" for p in range(c * W, c * W + W))
            lines.append(f"    {R} {names}; io.ld({c}, {names});")
        elif ins[0] == "st":
            c = ins[1]
            lines.append(f"    io.st({c}, " + ", ".join(name(outs[p]) for p in range(c * W, c * W + W)) + ");")
        else:
            u = ins[1]
            nd = T.nodes[u]
            if nd[0] == "add":
                ex = f"AR::add({name(nd[1])}, {name(nd[2])})"
            elif nd[0] == "sub":
                ex = f"AR::sub({name(nd[1])}, {name(nd[2])})"
            elif nd[0] == "mul":
                ex = f"AR::mul({name(nd[1])}, tab[{nd[2]}])"
            else:
                ex = f"AR::mul({R}(0.5), {name(nd[1])})"
            lines.append(f"    const {R} t{u} = {ex};")
    lines += ["  }", "};"]
    return "\n".join(lines)


# ---------------------------------------------------------------------------
# Cooperative rows (N too large for one thread's registers): R warp roles per
# 32-row tile, lane = row.  The stage program is cut into three bands:
#   head   stages [0, hd)       SplitComplex/SplitReal (+ first splits)
#   middle stages [hd, S - td)  independent subtrees (connected components)
#   tail   stages [S - td, S)   the last recombinations
# Band B (head + middle): each role loads the input chunks of its subtrees'
# head cones, computes the head ops it needs (recomputed where two roles
# share a head value), barrier, runs its subtrees and stores the values the
# tail reads at their arena positions (the cut).  Band C (tail): each role
# loads the cut chunks its output chunks need, barrier, computes and stores
# whole output chunks.  Same nodes as the trace, so still bitwise.


class UF:
    def __init__(self):
        self.p = {}

    def find(self, a):
        self.p.setdefault(a, a)
        while self.p[a] != a:
            self.p[a] = self.p[self.p[a]]
            a = self.p[a]
        return a

    def union(self, a, b):
        ra, rb = self.find(a), self.find(b)
        if ra != rb:
            self.p[max(ra, rb)] = min(ra, rb)


def _operands(nd):
    return [nd[1], nd[2]] if nd[0] in ("add", "sub") else ([nd[1]] if nd[0] in ("mul", "half") else [])


def _cone(T, roots, stop):
    """Nodes reachable from roots through operands, not descending below
    nodes for which stop(u) is true (those are included)."""
    seen, stack = set(), list(roots)
    while stack:
        u = stack.pop()
        if u in seen:
            continue
        seen.add(u)
        if not stop(u):
            stack += _operands(T.nodes[u])
    return seen


def _pack(items, R):
    """LPT: items = [(weight, payload)] -> R bins of payloads."""
    bins = [[0, []] for _ in range(R)]
    for w, pl in sorted(items, key=lambda t: -t[0]):
        b = min(bins, key=lambda t: t[0])
        b[0] += w
        b[1].append(pl)
    return [b[1] for b in bins]


def plan_roles(T, outs, hd, td, W, R, pair=False):
    S = len(T.snap) - 1
    band = lambda u: "H" if T.stage[u] < hd else ("T" if T.stage[u] >= S - td else "M")  # noqa: E731
    need = _cone(T, outs, lambda u: False)
    cut = T.snap[S - td]
    where = {}
    for q, u in enumerate(cut):
        where.setdefault(u, q)
    # middle components
    uf = UF()
    mids = [u for u in sorted(need) if band(u) == "M"]
    for u in mids:
        uf.find(u)
        for o in _operands(T.nodes[u]):
            if band(o) == "M":
                uf.union(u, o)
    comps = {}
    for u in mids:
        comps.setdefault(uf.find(u), []).append(u)
    # tail: one unit per output chunk; tail intermediates shared by two
    # chunks are recomputed by both (unioning them chains every chunk of a
    # time-major chain recombination into one component)
    nch = len(outs) // W
    tail_units = []
    for c in range(nch):
        outs_c = [outs[p] for p in range(c * W, c * W + W)]
        cone = _cone(T, outs_c, lambda z: band(z) != "T")
        tnodes = sorted(w for w in cone if band(w) == "T")
        reads = sorted({w for w in cone if band(w) != "T"})
        tail_units.append((len(tnodes) + len(reads), ([c], tnodes, reads)))
    troles = _pack(tail_units, R)
    # cut values the tail reads -> stored by band B at position where[v]
    cut_reads = sorted({v for _, (ch, tn, rd) in tail_units for v in rd})
    for v in cut_reads:
        assert v in where, "tail operand not in the arena at the cut"
    # band-B roles: middle components (+ head/input values to be stored)
    owner = {}
    stores = [[] for _ in range(R)]
    tw = _twins(T) if pair else None
    if tw is not None:
        # Re/Im pairing: roles r < R/2 run Re components, role r + R/2 the
        # Im twins (same code, part = 1): the instruction working set halves
        par = tw["par"]
        re = [m for m in comps.values() if par[m[0]] == 1]
        im = [m for m in comps.values() if par[m[0]] == 2]
        assert len(re) == len(im) and all(len({par[u] for u in m}) == 1 for m in comps.values())
        half = _pack([(len(m), ("m", m)) for m in re], R // 2)
        broles = half + [[("m", sorted(tw["twin"][u] for u in m)) for _, m in lst] for lst in half]
        for r, lst in enumerate(broles):
            for _, m in lst:
                for u in m:
                    owner[u] = r
        load = [sum(len(m) for _, m in lst) for lst in half]
        cut_set = set(cut_reads)
        for v in cut_reads:
            if par[v] == 2:
                continue           # stored by the twin role of its Re value
            assert par[v] == 1, "a cut value mixing Re and Im"
            t = tw["twin"][v]
            assert t in cut_set and where[t] == where[v] + len(cut) // 2, "Im twin not at the shifted position"
            if band(v) == "M":
                r = owner[v]
            else:
                r = min(range(R // 2), key=lambda k: load[k])
                load[r] += 1
            stores[r].append(v)
            stores[r + R // 2].append(t)
        return dict(band=band, cut=cut, where=where, broles=broles, stores=stores, troles=troles, S=S, pair=True)
    units = [(len(m), ("m", m)) for m in comps.values()]
    broles = _pack(units, R)
    for r, lst in enumerate(broles):
        for _, m in lst:
            for u in m:
                owner[u] = r
    load = [sum(len(m) for _, m in lst) for lst in broles]
    for v in cut_reads:
        if band(v) == "M":
            r = owner[v]
        else:   # a head value / an input passing through: least-loaded role
            r = min(range(R), key=lambda k: load[k])
            load[r] += 1
        stores[r].append(v)
    return dict(band=band, cut=cut, where=where, broles=broles, stores=stores, troles=troles, S=S, pair=False)


def _twins(T):
    """Re/Im twins of a CDFT trace: nodes with the same structure over the
    even (Re) and odd (Im) input cells.  par[u]: 1 Re only, 2 Im only, 3 both.
    None when the structure does not pair up."""
    key, par, intern = {}, [], {}

    def cons(t):       # hash-consing: structurally equal nodes get one id
        return intern.setdefault(t, len(intern))

    for u, nd in enumerate(T.nodes):
        if nd[0] == "in":
            key[u] = cons(("in", nd[1] >> 1))
            par.append(1 + (nd[1] & 1))
            continue
        ops = _operands(nd)
        key[u] = cons((nd[0],) + tuple(key[o] for o in ops) + ((nd[2],) if nd[0] == "mul" else ()))
        pr = 0
        for o in ops:
            pr |= par[o]
        par.append(pr)
    groups = {}
    for u in range(len(T.nodes)):
        if par[u] in (1, 2):
            groups.setdefault((key[u], par[u]), []).append(u)
    twin = {}
    for (k, pr), lst in groups.items():
        if pr != 1:
            continue
        other = groups.get((k, 2), [])
        if len(other) != len(lst):
            return None
        for a, b in zip(lst, other):
            twin[a] = b
    return {"twin": twin, "par": par}


def emit_roles(v, n, R_t, hd, td, R, pair=True):
    W = 4 if R_t == "float" else 2
    T, outs, ops = trace(v, 0, n)
    P = plan_roles(T, outs, hd, td, W, R, pair=pair)
    pair = P["pair"]
    NB = R // 2 if pair else R        # band-B code functions
    band, where = P["band"], P["where"]
    name = lambda u: (f"x{u}" if T.nodes[u][0] == "in" else f"t{u}")  # noqa: E731

    def op_line(u):
        nd = T.nodes[u]
        if nd[0] == "add":
            ex = f"AR::add({name(nd[1])}, {name(nd[2])})"
        elif nd[0] == "sub":
            ex = f"AR::sub({name(nd[1])}, {name(nd[2])})"
        elif nd[0] == "mul":
            ex = f"AR::mul({name(nd[1])}, tab[{nd[2]}])"
        else:
            ex = f"AR::mul({R_t}(0.5), {name(nd[1])})"
        return f"    const {R_t} t{u} = {ex};"

    fns, peaks = [], []
    # position -> role that stores it (for chunk ownership)
    pos_owner = {}
    for r in range(R):
        for val in P["stores"][r]:
            pos_owner[where[val]] = r
    for r in range(NB):
        mids = sorted(u for _, m in P["broles"][r] for u in m)
        st_vals = P["stores"][r]
        head_roots = [o for u in mids for o in _operands(T.nodes[u]) if band(o) == "H"]
        head_roots += [val for val in st_vals if band(val) == "H"]
        head = sorted(_cone(T, head_roots, lambda z: band(z) != "H"))
        lines = [f"  template <class AR, class IO>",
                 f"  static __device__ __forceinline__ void b{r}(IO& io, int part, const {R_t}* __restrict__ tab) {{"]
        loaded = set()
        live = 0
        for u in head:
            nd = T.nodes[u]
            if nd[0] == "in":
                c = nd[1] // W
                if c not in loaded:
                    loaded.add(c)
                    if pair:      # the Re cells of chunk c (part 1: its Im cells)
                        nm = ", ".join(f"x{p}" for p in range(c * W, c * W + W, 2))
                        lines.append(f"    {R_t} {nm}; io.ldp({c}, part, {nm});")
                    else:
                        nm = ", ".join(f"x{p}" for p in range(c * W, c * W + W))
                        lines.append(f"    {R_t} {nm}; io.ld({c}, {nm});")
            else:
                lines.append(op_line(u))
        lines.append("    io.sync();")
        # stores: chunks owned entirely (among needed positions) -> vector
        my_pos = {where[val]: val for val in st_vals}
        chunk_vec = set()
        for q in my_pos:
            c = q // W
            if all(pos_owner.get(p, r) == r for p in range(c * W, c * W + W)):
                chunk_vec.add(c)
        pending = {c: set(p for p in range(c * W, c * W + W) if p in my_pos) for c in chunk_vec}
        ready = set(u for u in head) | set()
        emitted_st = set()

        def try_store(val):
            q = where[val]
            c = q // W
            if c in chunk_vec:
                pending[c].discard(q)
                if not pending[c] and c not in emitted_st:
                    emitted_st.add(c)
                    vals = []
                    for p in range(c * W, c * W + W):
                        vals.append(name(my_pos[p]) if p in my_pos else f"{R_t}(0)")
                    lines.append(f"    io.str({c}, part, {', '.join(vals)});")
            else:
                lines.append(f"    io.st1({q}, part, {name(val)});")

        for val in st_vals:            # head values / inputs stored as they are
            if band(val) == "H":
                try_store(val)
        sv = set(st_vals)
        for u in mids:
            lines.append(op_line(u))
            if u in sv:
                try_store(u)
        lines.append("    io.sync();")
        lines.append("  }")
        fns.append("\n".join(lines))
        peaks.append(len(mids))
    for r in range(R):
        units = P["troles"][r]
        lines = [f"  template <class AR, class IO>",
                 f"  static __device__ __forceinline__ void c{r}(IO& io, const {R_t}* __restrict__ tab) {{"]
        reads = sorted({val for chunks, tn, rd in units for val in rd})
        chunks_needed = sorted({where[val] // W for val in reads})
        for c in chunks_needed:
            nm = ", ".join(f"y{p}" for p in range(c * W, c * W + W))
            lines.append(f"    {R_t} {nm}; io.ldr({c}, {nm});")
        lines.append("    io.sync();")
        # alias: value name -> the cut register
        alias = {val: f"y{where[val]}" for val in reads}
        nm2 = lambda u: alias.get(u, name(u))  # noqa: E731
        tnodes = sorted({u for chunks, tn, rd in units for u in tn})
        for u in tnodes:
            nd = T.nodes[u]
            if nd[0] == "add":
                ex = f"AR::add({nm2(nd[1])}, {nm2(nd[2])})"
            elif nd[0] == "sub":
                ex = f"AR::sub({nm2(nd[1])}, {nm2(nd[2])})"
            elif nd[0] == "mul":
                ex = f"AR::mul({nm2(nd[1])}, tab[{nd[2]}])"
            else:
                ex = f"AR::mul({R_t}(0.5), {nm2(nd[1])})"
            lines.append(f"    const {R_t} t{u} = {ex};")
        for chunks, tn, rd in units:
            for c in chunks:
                lines.append(f"    io.st({c}, " + ", ".join(nm2(outs[p]) for p in range(c * W, c * W + W)) + ");")
        lines.append("  }")
        fns.append("\n".join(lines))
    body = [f"template <> struct SmallRoles<{v}, {n.bit_length() - 1}, {R_t}> {{",
            f"  static constexpr int R = {R};",
            f"  static constexpr int ROWS = {COOP_ROWS.get((R_t, n), 32)};",
            f"  static constexpr int HALF = {n};   // cells between a Re role's cut positions and its Im twin's",
            f"  static constexpr unsigned long long OPS[3] = {{{ops[0]}ull, {ops[1]}ull, {ops[2]}ull}};"]
    body += fns
    body.append("  template <class AR, class IO>")
    body.append(f"  static __device__ __forceinline__ void run(int role, IO& io, const {R_t}* __restrict__ tab) {{")
    body.append(f"    switch (role % {NB}) {{")
    for r in range(NB):
        body.append(f"      case {r}: b{r}<AR>(io, role / {NB}, tab); break;")
    body += ["    }", "    switch (role) {"]
    for r in range(R):
        body.append(f"      case {r}: c{r}<AR>(io, tab); break;")
    body += ["    }", "  }", "};"]
    return "\n".join(body), P, peaks


HEAD = ["#pragma once",
        "namespace amqft_b200 {",
        "namespace smallk {",
        "template <int V, int F, int LOGN, typename R> struct SmallGen;",
        "template <int V, int LOGN, typename R> struct SmallRoles;"]
TAIL = ["}  // namespace smallk", "}  // namespace amqft_b200", ""]


def main():
    """Writes <out>/small_gen_v<V>.cuh (code) and <out>/small_ops.cuh (op
    counts per instance, for the plan's meter)."""
    import argparse
    import ctypes
    ap = argparse.ArgumentParser()
    ap.add_argument("--lib", help="host-only plan library (libamqft_plan.so)")
    ap.add_argument("--out", required=True)
    a = ap.parse_args()
    global _PLANLIB
    if a.lib:
        _PLANLIB = ctypes.CDLL(a.lib)
        _PLANLIB.amqft_schedule_dump.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_size_t, ctypes.c_size_t,
                                                 ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p,
                                                 ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p,
                                                 ctypes.c_void_p]
    os.makedirs(a.out, exist_ok=True)
    ops_lines = ["// GENERATED by codegen/gen_small.py: op counts of the generated small kernels.",
                 "#pragma once", "namespace amqft_b200 {", "namespace smallk {",
                 "// {adds, muls, halvings} for CDFT variant V, log2 N, dtype (0 fp32, 1 fp64); 0 = not covered",
                 "struct SmallOps { int v, fn, logn, f64; unsigned long long a, m, b; };",
                 "static constexpr SmallOps kSmallOps[] = {"]
    for v in range(1, 9):
        out = [f"// small_gen_v{v}.cuh -- GENERATED by codegen/gen_small.py; do not edit.",
               "// Small CDFTs of AM-QFT variant %d: the traced stage program of plan.cpp as" % v,
               "// straight-line code (one reference add/sub/mul per line)."] + HEAD
        for fn, table in ((0, SIZES), (1, RDFT_SIZES), (2, DCT_SIZES), (3, DST_SIZES)):
            for R, sizes in table.items():
                for n in sizes:
                    out.append(emit_fn(v, fn, n, R))
                    _, _, ops = trace(v, fn, n)
                    ops_lines.append(f"  {{{v}, {fn}, {n.bit_length() - 1}, {int(R == 'double')}, "
                                     f"{ops[0]}ull, {ops[1]}ull, {ops[2]}ull}},")
        for R, cfg in COOP.items():
            for n, (hd, td, nr) in cfg.items():
                code, _, _ = emit_roles(v, n, R, hd, td, nr)
                out.append(code)
                _, _, ops = trace(v, 0, n)
                ops_lines.append(f"  {{{v}, 0, {n.bit_length() - 1}, {int(R == 'double')}, "
                                 f"{ops[0]}ull, {ops[1]}ull, {ops[2]}ull}},")
        out += TAIL
        with open(os.path.join(a.out, f"small_gen_v{v}.cuh"), "w") as f:
            f.write("\n".join(out))
    ops_lines += ["};", "}  // namespace smallk", "}  // namespace amqft_b200", ""]
    with open(os.path.join(a.out, "small_ops.cuh"), "w") as f:
        f.write("\n".join(ops_lines))


if __name__ == "__main__":
    main()
