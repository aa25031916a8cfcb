"""The plan compiler (paper_1404_1810_b200/csrc/plan.cpp), checked on the CPU.

The compiled stage program is run by an independent numpy restatement of
the EI semantics (tests/schedule_interp.py) and must equal the oracle
bitwise for every variant x wired function x size, with the exact op counts
of the reference meter (the schedule executes the
AM-QFT DAG, not some other FFT).
"""
import numpy as np
import pytest

import paper_1404_1810_b200 as amqft
from schedule_interp import _items, interpret


@pytest.mark.parametrize("v", range(1, 9))
def test_schedule_bitwise_equals_oracle(oracle, restatement, v):
    r, O = restatement, oracle
    for f in O.wired_functions(v):
        n = O.FUNCTION_BASE[f]
        while n <= 512:
            t = O.FUNCTION_OPERAND[f]
            x = r.uniform(r.mix_seed(3000, v, f, n), r.cell_count(t, n))
            want, meter = r.execute(v, f, n, x, meter=True)
            recs, stages, ops = amqft.schedule_dump(v, f, n)
            nmax = max(n, 8)
            got = interpret(recs, stages, x, r.trig_constants(v, nmax), nmax)
            assert got.tobytes() == want.tobytes(), (v, f, n)
            assert ops == meter, (v, f, n, ops, meter)
            n *= 2


@pytest.mark.parametrize("v", [1, 2, 5, 8])
def test_stage_writes_are_disjoint(v):
    """Within a stage every cell is written at most once (the device runs a
    stage's items in parallel), and every EI stays inside the arena."""
    n = 1024
    recs, stages, _ = amqft.schedule_dump(v, amqft.FunctionId.Cdft, n)
    cells = 2 * n
    for b, e in stages:
        seen = np.zeros(cells, dtype=np.int32)
        for k in range(b, e):
            ei = recs[k]
            items = 1 if ei["op"] in (18, 19) else _items(int(ei["op"]), int(ei["n"]))
            span = int(ei["aux"]) if ei["op"] in (18, 19) else items
            lo = int(ei["off"])
            assert lo + span <= cells
            seen[lo:lo + span] += 1
        assert seen.max() <= 1


def test_op_counts_match_closed_forms(oracle, restatement):
    """metering.cpp:85-114 closed forms, large N (schedule only)."""
    for v in (1, 2, 3, 4, 5, 6, 7, 8):
        for kind, f in ((0, 0), (1, 1), (2, 2), (3, 3)):
            for n in (1024, 4096):
                _, _, ops = amqft.schedule_dump(v, f, n)
                a, m, bt = restatement.predicted_cost(kind, n)
                assert ops == (a, m, bt if v % 2 else 0), (v, f, n)


def test_schedule_rejections():
    with pytest.raises(amqft.InvalidArgument):
        amqft.schedule_dump(9, 0, 16)
    with pytest.raises(amqft.InvalidArgument):
        amqft.schedule_dump(1, 0, 24)
    with pytest.raises(amqft.InvalidArgument):
        amqft.schedule_dump(2, amqft.FunctionId.DstOddTime, 16)
    with pytest.raises(amqft.InvalidArgument):
        amqft.schedule_dump(1, amqft.FunctionId.DctOddOdd, 4)
