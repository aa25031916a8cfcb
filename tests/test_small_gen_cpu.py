"""CPU check of codegen/gen_small.py (the one-thread-per-row kernel's code):
the traced SSA program, evaluated with IEEE doubles (one rounding per op, as
on the device), is BITWISE the oracle for every variant and size, and its
op counts are the reference meter (metering.cpp) -- the generated code runs
the AM-QFT DAG itself.  The committed small_gen.cuh is what the generator
emits now."""
import os

import numpy as np
import pytest

from paper_1404_1810_b200.codegen import gen_small as G

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("v", range(1, 9))
def test_small_trace_bitwise_and_meter(oracle, restatement, v):
    r, O = restatement, oracle
    for n in (2, 4, 8, 16, 32, 64):
        T, outs, ops = G.trace(v, 0, n)
        for trial in range(2):
            x = r.uniform(r.mix_seed(515, v, n, trial), 2 * n)
            want, meter = r.execute(v, O.F_CDFT, n, x, meter=True)
            got = np.array(G.evaluate(T, outs, x, r.trig_constants(v, max(n, 8))))
            assert got.tobytes() == want.tobytes(), (v, n, trial)
        assert G.count_ops(T, outs) == tuple(meter) == ops, (v, n)


def test_small_schedule_in_place_safe():
    """Every output chunk is stored after its input chunk was loaded, once."""
    for v in (1, 4, 7):
        for n in (16, 64):
            for W in (2, 4):
                T, outs, _ = G.trace(v, 0, n)
                prog = G.schedule_trace(T, outs, W)
                loaded, stored = set(), set()
                for ins in prog:
                    if ins[0] == "ld":
                        assert ins[1] not in stored
                        loaded.add(ins[1])
                    elif ins[0] == "st":
                        assert ins[1] in loaded and ins[1] not in stored
                        stored.add(ins[1])
                assert stored == set(range(2 * n // W))


@pytest.mark.parametrize("pair", [False, True])
@pytest.mark.parametrize("dtype", ["float", "double"])
def test_coop_roles_partition(dtype, pair):
    """Cooperative plans: every middle node belongs to exactly one role,
    every output chunk to exactly one tail role, and the tail only reads
    values the band-B roles store at the cut (so the two-band in-place
    execution computes the traced program)."""
    W = 4 if dtype == "float" else 2
    for n, (hd, td, R) in G.COOP[dtype].items():
        for v in (1, 2, 4, 7):
            T, outs, _ = G.trace(v, 0, n)
            P = G.plan_roles(T, outs, hd, td, W, R, pair=pair)
            assert P["pair"] == pair
            if pair:   # role r + R/2 runs the Im twins of role r's nodes, stored N cells further
                tw = G._twins(T)["twin"]
                for r in range(R // 2):
                    re = sorted(u for _, m in P["broles"][r] for u in m)
                    assert sorted(tw[u] for u in re) == sorted(u for _, m in P["broles"][r + R // 2] for u in m)
                    assert [P["where"][tw[x]] for x in P["stores"][r]] == \
                        [P["where"][x] + n for x in P["stores"][r + R // 2]] or \
                        [P["where"][x] for x in P["stores"][r + R // 2]] == [P["where"][x] + n for x in P["stores"][r]]
            mids = [u for lst in P["broles"] for _, m in lst for u in m]
            assert len(mids) == len(set(mids))
            chunks = sorted(c for lst in P["troles"] for ch, _, _ in lst for c in ch)
            assert chunks == list(range(2 * n // W))
            stored = {x for lst in P["stores"] for x in lst}
            for lst in P["troles"]:
                for _, _, rd in lst:
                    assert set(rd) <= stored
            assert len(stored) == sum(len(x) for x in P["stores"])


def test_coop_two_band_emulation(oracle, restatement):
    """Execute the cooperative plan band by band on a numpy arena (band B:
    head cones from the inputs, subtrees, stores at the cut; band C: reads
    of the cut, tail nodes, whole output chunks): bitwise the oracle."""
    r, O = restatement, oracle
    for dtype, W in (("float", 4), ("double", 2)):
        for n, (hd, td, R) in G.COOP[dtype].items():
            if n > 256:
                continue
            for v in (3, 4, 6):
                T, outs, _ = G.trace(v, 0, n)
                P = G.plan_roles(T, outs, hd, td, W, R, pair=True)
                x = r.uniform(r.mix_seed(99, v, n), 2 * n)
                tab = r.trig_constants(v, n)
                full = G.evaluate(T, list(range(len(T.nodes))), x, tab)
                arena = np.array(x)
                for lst in P["stores"]:
                    for val in lst:
                        arena[P["where"][val]] = full[val]
                out = np.full(2 * n, np.nan)
                for lst in P["troles"]:
                    for ch, tn, rd in lst:
                        val = {u: arena[P["where"][u]] for u in rd}
                        for u in tn:
                            nd = T.nodes[u]
                            a = val[nd[1]]
                            if nd[0] == "add":
                                val[u] = a + val[nd[2]]
                            elif nd[0] == "sub":
                                val[u] = a - val[nd[2]]
                            elif nd[0] == "mul":
                                val[u] = a * tab[nd[2]]
                            else:
                                val[u] = 0.5 * a
                        for c in ch:
                            for p in range(c * W, c * W + W):
                                out[p] = val[outs[p]]
                want = r.execute(v, O.F_CDFT, n, x)
                assert out.tobytes() == want.tobytes(), (dtype, n, v)
