"""Print key metrics + stall breakdown + top stalled SASS lines of a captured jump pass."""
import csv
import sys

tag = sys.argv[1]
rows = list(csv.reader(open(f"gpurun_out/prof_pass_{tag}_raw.csv")))
h = rows[0]
keys = ["gpu__time_duration.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__inst_executed.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct",
        "launch__grid_size", "launch__registers_per_thread", "lts__throughput.avg.pct_of_peak_sustained_elapsed"]
for r in rows[2:3 if len(sys.argv) < 3 else 2 + int(sys.argv[2])]:
    print(r[h.index("Kernel Name")][:60])
    for k in keys:
        if k in h:
            print(f"   {k} = {r[h.index(k)]}")
    st = sorted(((float(r[i]), h[i][len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")])
                 for i in range(len(h)) if h[i].startswith("smsp__average_warps_issue_stalled")
                 and h[i].endswith("per_issue_active.ratio")), reverse=True)
    print("   stalls: " + " ".join(f"{n}={v:.2f}" for v, n in st[:9]))
try:
    rows = list(csv.reader(open(f"gpurun_out/prof_pass_{tag}_src.csv")))
    hi = next(i for i, r in enumerate(rows) if "Address" in r and "Source" in r)
    h = rows[hi]
    si, wi = h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
    data = []
    for r in rows[hi + 1:]:
        try:
            data.append((int(r[wi]), r[si].strip()))
        except (ValueError, IndexError):
            pass
    tot = sum(d[0] for d in data) or 1
    print(f"   SASS lines {len(data)}, samples {tot}")
    for w, src in sorted(set(data), reverse=True)[:10]:
        print(f"   {w:7d} {100 * w / tot:5.1f}%  {src[:80]}")
except FileNotFoundError:
    pass
