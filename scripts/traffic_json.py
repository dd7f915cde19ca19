"""Add one config's per-launch DRAM traffic (from an ncu --set full raw CSV of the dJFA frame's
jump passes) to profiles/jump_pass_traffic.json, which bench.py reads for roofline.traffic.

  python scripts/traffic_json.py C5 gpurun_out/prof_pass_r01c5_raw.csv "<how it was captured>"
"""
import csv
import json
import sys

cfg, raw, source = sys.argv[1], sys.argv[2], sys.argv[3]
N = {"C3": 4096, "C4": 16384, "C5": 65536}[cfg]
rows = list(csv.reader(open(raw)))
h = rows[0]
col = {k: h.index(k) for k in h}


def f(r, k):
    return float(r[col[k]].replace(",", "")) if k in col else None


def scale(r, k):  # raw CSV units row (rows[1]) may say byte / Kbyte / Mbyte / Gbyte
    u = rows[1][col[k]]
    return f(r, k) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)


TIME_MS = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3}  # raw CSV time unit -> ms
launches = []
for r in rows[2:]:
    rd, wr = scale(r, "dram__bytes_read.sum"), scale(r, "dram__bytes_write.sum")
    launches.append({
        "kernel": r[col["Kernel Name"]], "dram_read_bytes": rd, "dram_write_bytes": wr, "dram_bytes": rd + wr,
        "ncu_ms": f(r, "gpu__time_duration.sum") * TIME_MS[rows[1][col["gpu__time_duration.sum"]]],
        "issue_active_pct": f(r, "smsp__issue_active.avg.pct_of_peak_sustained_active"),
        "alu_pipe_pct": f(r, "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active"),
        "fma_pipe_pct": f(r, "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"),
        "warp_instructions": f(r, "smsp__inst_executed.sum"),
    })
path = "profiles/jump_pass_traffic.json"
t = json.load(open(path))
t[cfg] = {"source": source, "algorithmic_bytes_per_launch": 8 * N * N,
          "dram_bytes_per_launch_djfa_avg": sum(x["dram_bytes"] for x in launches) / len(launches),
          "launches": launches}
json.dump(t, open(path, "w"), indent=1)
print(cfg, t[cfg]["dram_bytes_per_launch_djfa_avg"], len(launches))
