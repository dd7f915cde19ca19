"""Add one config's per-launch DRAM traffic of the dJFA frame's jump passes to
profiles/jump_pass_traffic.json, from an ncu launch list with dram__bytes_{read,write}.sum and
gpu__time_duration.sum (scripts/gpu.sh c4launch / c5launch):

  python scripts/traffic_from_launches.py C5 profiles/r02_c5_launches.csv NPASS "<how it was captured>"

The last NPASS jump-pass launches of the list (the final dJFA frame's passes) are averaged."""
import csv
import json
import sys

cfg, path, npass, source = sys.argv[1], sys.argv[2], int(sys.argv[3]), sys.argv[4]
N = {"C3": 4096, "C4": 16384, "C5": 65536}[cfg]
rows = list(csv.reader(open(path)))
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr]
ki, ii, mi, ui, vi = (h.index(x) for x in ("Kernel Name", "ID", "Metric Name", "Metric Unit", "Metric Value"))
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "ns": 1e-6, "us": 1e-3, "ms": 1.0,
        "second": 1e3}
per = {}
for r in rows[hdr + 1:]:
    if len(r) > vi:
        per.setdefault(int(r[ii]), {"kernel": r[ki]})[r[mi]] = float(r[vi].replace(",", "")) * UNIT.get(r[ui], 1)
passes = [v for _, v in sorted(per.items()) if "jump_pass" in v["kernel"]][-npass:]
launches = [{"kernel": p["kernel"].split("(")[0], "dram_read_bytes": p["dram__bytes_read.sum"],
             "dram_write_bytes": p["dram__bytes_write.sum"],
             "dram_bytes": p["dram__bytes_read.sum"] + p["dram__bytes_write.sum"], "ncu_ms": p["gpu__time_duration.sum"]}
            for p in passes]
out = "profiles/jump_pass_traffic.json"
t = json.load(open(out))
t[cfg] = {"source": source, "algorithmic_bytes_per_launch": 8 * N * N,
          "dram_bytes_per_launch_djfa_avg": sum(x["dram_bytes"] for x in launches) / len(launches),
          "launches": launches}
json.dump(t, open(out, "w"), indent=1)
print(cfg, t[cfg]["dram_bytes_per_launch_djfa_avg"], len(launches))
