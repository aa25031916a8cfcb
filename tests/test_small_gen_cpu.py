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


def test_small_gen_header_up_to_date():
    import io
    import contextlib
    buf = io.StringIO()
    with contextlib.redirect_stdout(buf):
        G.main()
    with open(os.path.join(ROOT, "paper_1404_1810_b200", "csrc", "small_gen.cuh")) as f:
        assert f.read() == buf.getvalue()
