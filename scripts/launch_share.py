"""Share of the jump-pass kernels in a dJFA step from an ncu launch list of bench.py
(ncu --metrics gpu__time_duration.sum --clock-control none --csv).

  python scripts/launch_share.py gpurun_out/launches_bench_r01.csv [first_step last_step]

A dJFA step is the run of launches from one move_fwd to the next launch that is not part of
the step (the next move_fwd, move_clamp, fill_value, or a reduction)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr]
ki, ii, mi, vi = h.index("Kernel Name"), h.index("ID"), h.index("Metric Name"), h.index("Metric Value")
launches = []
for r in rows[hdr + 1:]:
    if len(r) > vi and r[mi] == "gpu__time_duration.sum":
        launches.append((r[ki].split("(")[0], float(r[vi].replace(",", ""))))
STEP = ("move_fwd", "stamp_flagged", "jump_pass_sk_remap", "fwd_reset", "remap", "remap_lanes", "reset_stamp",
        "jump_pass_fast", "jump_pass_sk")
steps, cur = [], None
for name, t in launches:
    base = name.replace("void ", "").split("<")[0]
    if base == "move_fwd":
        cur = []
        steps.append(cur)
    elif cur is not None and base not in STEP:
        cur = None
    if cur is not None:
        cur.append((base, t))
a, b = (int(sys.argv[2]), int(sys.argv[3])) if len(sys.argv) > 3 else (3, min(len(steps), 8))
sel = steps[a:b]
tot = sum(t for s in sel for _, t in s)
jp = sum(t for s in sel for n, t in s if n.startswith("jump_pass"))
print(f"{len(launches)} launches, {len(steps)} dJFA steps; steps {a + 1}..{b}:")
print(f"  jump-pass kernels' share of the step = {jp / tot:.3f}")
print(f"  serialized per-step kernel time   = {tot / len(sel) / 1e6:.3f} ms (ncu, cold cache, serialised)")
for n in STEP:
    ts = [t for s in sel for nn, t in s if nn == n]
    if ts:
        print(f"  {n:16s} {len(ts) / len(sel):4.1f} launches/step, {sum(ts) / len(sel) / 1e6:.3f} ms/step")
