"""profiles/r02_ncu_c4_passes.json from the ncu CSV of one warm config-4
forward (per-launch device time and DRAM bytes of the four-step's passes):

  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
      --log-file gpurun_out/c4_passes.csv python tools/prof_fast.py --n 16777216 --batch 1 --iters 1
  python tools/ncu_c4_passes.py gpurun_out/c4_passes.csv profiles/r02_ncu_c4_passes.json
"""
import csv
import json
import re
import sys

src, dst = sys.argv[1], sys.argv[2]
rows = list(csv.reader(open(src)))
hdr = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
ix = {k: i for i, k in enumerate(rows[hdr])}
per = {}
for r in rows[hdr + 1:]:
    if len(r) < len(ix):
        continue
    name = r[ix["Kernel Name"]]
    if not re.search(r"k_slab|k_tile|k_small_col|k_transpose|k_fast", name):
        continue
    e = per.setdefault(int(r[ix["ID"]]), {"kernel": re.sub(r"\(.*", "", name).replace("amqft_b200::", "")[:90]})
    val = float(r[ix["Metric Value"]].replace(",", ""))
    unit = r[ix["Metric Unit"]]
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1.0, "ms": 1e3}.get(unit, 1.0)
    m = r[ix["Metric Name"]]
    if m == "gpu__time_duration.sum":
        e["us"] = val * scale
    elif m == "dram__bytes_read.sum":
        e["dram_read_bytes"] = val * scale
    elif m == "dram__bytes_write.sum":
        e["dram_write_bytes"] = val * scale
ids = sorted(per)
# prof_fast.py runs warm-up forwards and one timed forward: keep the last forward's launches
# (--iters 1: one warm-up forward and one timed forward, the same launches twice)
n = len(ids) // 2
last = [per[i] for i in ids[-n:]]
out = {"what": "config 4 (N = 2^24 fp32, v4): per-launch device time and DRAM bytes of one warm forward of the "
               "plan the library picks (ncu, cold caches, serialised)",
       "command": "ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none "
                  "--csv python tools/prof_fast.py --n 16777216 --batch 1 --iters 1",
       "launches": last,
       "step_dram_bytes": sum(e.get("dram_read_bytes", 0) + e.get("dram_write_bytes", 0) for e in last),
       "algorithmic_bytes": 268435456,
       "note": "writes are counted as they leave L2 during each launch; a pass's remaining dirty lines are written back "
               "during the next one"}
json.dump(out, open(dst, "w"), indent=1)
print(json.dumps(out, indent=1))
