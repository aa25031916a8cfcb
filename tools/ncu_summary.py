"""Turns the GPU-box outputs of tools/profile_round.sh into the committed
profiles/ summaries (diagnostic tooling, not part of the product).

  python tools/ncu_summary.py gpurun_out profiles r01
"""
import csv
import json
import re
import subprocess
import sys

src, dst, tag = sys.argv[1], sys.argv[2], sys.argv[3]


def short(name):
    m = re.search(r"k_tile<(.*)>(?=\(const)", name)
    if m:
        return f"k_tile<{m.group(1).replace(' ', '')}> (AM-QFT in-shared-memory four-step CDFT)"
    m = re.search(r"k_fast<(.*?)>", name)
    if m:
        return f"k_fast<{m.group(1).replace(' ', '')}> (AM-QFT fused CDFT)"
    if "k_level_table" in name:
        return "k_level_table (per-level constant table, plan creation)"
    if "randn" in name or "normal" in name or "philox" in name.lower():
        return "torch randn (input generation)"
    if "direct_copy_kernel" in name:
        return "torch copy (bench parity sample rows, after the timed region)"
    return name[:120]


# 1. launch list
rows = list(csv.reader(open(f"{src}/launches.csv")))
hdr = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
h = rows[hdr]
ix = {k: i for i, k in enumerate(h)}
launches = []
for r in rows[hdr + 1:]:
    if len(r) < len(h) or r[ix["Metric Name"]] != "gpu__time_duration.sum":
        continue
    scale = {"ns": 1.0, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6}.get(r[ix["Metric Unit"]], 1.0)
    launches.append({"id": int(r[ix["ID"]]), "kernel": short(r[ix["Kernel Name"]]), "grid": r[ix["Grid Size"]],
                     "block": r[ix["Block Size"]],
                     "duration_ns": float(r[ix["Metric Value"]].replace(",", "")) * scale})
json.dump(launches, open(f"{dst}/{tag}_launch_list.json", "w"), indent=1)

# 2. full-set summary of the fused kernel
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio",
        "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct",
        "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic"]
import os  # noqa: E402
rep = f"{src}/k_top_full.ncu-rep" if os.path.exists(f"{src}/k_top_full.ncu-rep") else f"{src}/k_fast_full.ncu-rep"
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"],
                     capture_output=True, text=True, check=True).stdout
rr = list(csv.reader(raw.splitlines()))
h, units = rr[0], rr[1]
row = next(r for r in rr[2:] if any("k_fast" in c or "k_tile" in c for c in r))
out = {"Kernel Name": short(row[h.index("Kernel Name")])}
for k in want:
    if k in h:
        out[k] = row[h.index(k)]
        out[k + " [unit]"] = units[h.index(k)]
rd = float(out["dram__bytes_read.sum"]) if "dram__bytes_read.sum" in out else None
wr = float(out["dram__bytes_write.sum"]) if "dram__bytes_write.sum" in out else None
out["_source"] = ("ncu --set full --clock-control none --import-source on -k 'regex:k_tile|k_fast' -s 3 -c 1, "
                  "python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline (B200, tools/profile_round.sh)")
kname = "k_tile" if "k_tile" in out["Kernel Name"] else "k_fast"
json.dump(out, open(f"{dst}/{tag}_ncu_{kname}_v4_n4096.json", "w"), indent=1)
print(json.dumps({k: out[k] for k in list(out)[:12]}, indent=1))
