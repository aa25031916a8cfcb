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

  python3 paper_1404_1810_b200/codegen/gen_small.py > paper_1404_1810_b200/csrc/small_gen.cuh
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


def trace(v, f, n):
    """(Trace, outputs): outputs[p] = node holding output cell p."""
    import paper_1404_1810_b200 as amqft
    recs, stages, ops = amqft.schedule_dump(v, f, n)
    nmax = max(n, 8)
    cells = amqft.cell_count(f, n)
    T = Trace(cells)
    x = list(range(cells))
    for b, e in stages:
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
    W = 4 if R == "float" else 2
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


def main():
    out = ["// small_gen.cuh -- GENERATED by codegen/gen_small.py; do not edit.",
           "// One whole CDFT per thread: the traced AM-QFT stage program of plan.cpp as",
           "// straight-line code (one reference add/sub/mul per line).",
           "#pragma once",
           "namespace amqft_b200 {",
           "namespace smallk {",
           "template <int V, int F, int LOGN, typename R> struct SmallGen;"]
    for R, sizes in SIZES.items():
        for n in sizes:
            for v in range(1, 9):
                out.append(emit_fn(v, 0, n, R))
    out += ["}  // namespace smallk", "}  // namespace amqft_b200", ""]
    sys.stdout.write("\n".join(out))


if __name__ == "__main__":
    main()
