"""Per-barrier-segment summary of an ncu SASS source page (diagnostic).

  ncu -i rep.ncu-rep --page source --csv --print-source sass > /tmp/s.csv
  python tools/ncu_segments.py /tmp/s.csv ROWS
"""
import collections
import csv
import sys


def num(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


rows = list(csv.reader(open(sys.argv[1])))
R = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
h = rows[1]
ix = {k: i for i, k in enumerate(h)}
stalls = [k for k in h if k.startswith("stall_") and "(Not" not in k]
seg = 0
agg = collections.defaultdict(collections.Counter)
for r in rows[2:]:
    if len(r) < len(h):
        continue
    s = r[ix["Source"]].strip()
    c = agg[seg]
    ie = num(r[ix["Instructions Executed"]]) / R
    c["inst"] += ie
    c["wf"] += num(r[ix["L1 Wavefronts Shared"]]) / R
    c["wf_exc"] += num(r[ix["L1 Wavefronts Shared Excessive"]]) / R
    op = s.split()[1] if s.startswith("@") else s.split()[0]
    op = op.split(".")[0]
    if op in ("LDS", "STS", "LDG", "STG", "SHFL", "LDGSTS"):
        c["n_" + op] += ie
    for k in stalls:
        c[k] += num(r[ix[k]])
    if "BAR.SYNC" in s or "EXIT" in s:
        seg += 1
for sg in sorted(agg):
    c = agg[sg]
    tot = sum(c[k] for k in stalls)
    if c["inst"] < 5:
        continue
    top = sorted(((c[k], k[6:]) for k in stalls), reverse=True)[:6]
    mem = " ".join(f"{k[2:]}={c[k]:.0f}" for k in sorted(c) if k.startswith("n_"))
    print(f"seg {sg}: inst/row {c['inst']:.0f} wf/row {c['wf']:.0f} (exc {c['wf_exc']:.0f}) {mem}")
    print(f"        samples {tot:.0f}: " + " ".join(f"{n}={v:.0f}" for v, n in top))
