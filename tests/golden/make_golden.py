"""Generates tests/golden/*.npz from the REFERENCE library itself
(oracle/_ref/libamqft_ref.so, compiled from /root/reference/proj/src by
oracle/Makefile).  Run here, where the reference exists; the fixtures are
committed so the GPU box (which has no /root/reference) can use them.

  python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    ref = O.reference()
    assert ref is not None, "build oracle/_ref first (make -C oracle)"
    # Config 1: CDFT N=1024, UniformSource(mix_seed(1, kind=0, n, trial=0))
    # (accuracy.cpp:20-28 seeding), all 8 variants.
    n = 1024
    x = O.seeded_signal(1, O.CDFT, n, 0, ref)
    out = {"input": x}
    for v in range(1, 9):
        y, m = ref.execute(v, O.F_CDFT, n, x, meter=True)
        out[f"v{v}"] = y
        out[f"meter_v{v}"] = np.array(m, dtype=np.uint64)
    out["naive_working"] = ref.pruned_transform(O.CDFT_FULL, n, x, extended=False)
    out["extended"] = ref.pruned_transform(O.CDFT_FULL, n, x, extended=True)
    np.savez_compressed(os.path.join(HERE, "config1_cdft1024.npz"), **out)

    # Every wired function of every variant at n = base..64, inputs as in
    # variants_test.cpp:308-327 (UniformSource(mix_seed(3000, v, f, n))).
    small = {}
    for v in range(1, 9):
        for f in O.wired_functions(v):
            nn = O.FUNCTION_BASE[f]
            while nn <= 64:
                t = O.FUNCTION_OPERAND[f]
                xi = ref.uniform(ref.mix_seed(3000, v, f, nn), ref.cell_count(t, nn))
                y, m = ref.execute(v, f, nn, xi, meter=True)
                small[f"x_{v}_{f}_{nn}"] = xi
                small[f"y_{v}_{f}_{nn}"] = y
                small[f"m_{v}_{f}_{nn}"] = np.array(m, dtype=np.uint64)
                nn *= 2
    np.savez_compressed(os.path.join(HERE, "functions_small.npz"), **small)

    # Constant tables (TrigTable::constants) at nmax = 8, 16, 1024.
    tabs = {f"v{v}_{m}": ref.trig_constants(v, m) for v in range(1, 9) for m in (8, 16, 1024)}
    # mt19937_64 stream and mix_seed values.
    tabs["uniform_seed12345"] = ref.uniform(12345, 64)
    tabs["mix_seed_1_0_1024_0"] = np.array([ref.mix_seed(1, 0, 1024, 0)], dtype=np.uint64)
    np.savez_compressed(os.path.join(HERE, "tables.npz"), **tabs)
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
