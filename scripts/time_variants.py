"""Time the dJFA frame and its jump passes for each libvd variant in build/variants/ (C4)."""
import glob
import json
import os
import subprocess
import sys

CHILD = r'''
import json, os, sys
sys.path.insert(0, os.getcwd())
import torch, synth
import paper_2209_00117_b200 as vd
if os.environ.get('VARIANT_LIB'):
    vd._load_variant(os.environ['VARIANT_LIB'])
N, s = {"C4": (16384, 1 << 20), "C3": (4096, 65536), "C5": (65536, 1 << 24)}[os.environ.get("VD_CFG", "C4")]
xy = synth.uniform_seeds(N, s, rng_seed=2209)
st = torch.cuda.Stream()
d = vd.VoronoiDiagram(N, xy, device=0, stream=st.cuda_stream)
d.jfa()
for f in range(3):
    d.djfa_step(synth.displacements(s, 1, f, rng_seed=2209), 1)
h = d.label_hash()
disp = torch.from_numpy(__import__("numpy").stack([synth.displacements(s, 1, f, rng_seed=2209) for f in range(3, 23)])).cuda()
d.synchronize()
d.set_pass_timing(True)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
with torch.cuda.stream(st):
    e0.record(st)
    for f in range(20):
        d.djfa_step(disp[f], 1)
    e1.record(st)
torch.cuda.synchronize()
pt = d.pass_times()
ms, n, px = d.pass_timing()
d.set_pass_timing(False)
j0, j1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
d.set_pass_timing(True)
j0.record(st)
for f in range(5):
    d.jfa()
j1.record(st)
torch.cuda.synchronize()
jpt = d.pass_times()
jms, jn, jpx = d.pass_timing()
def perk(v):
    out = {}
    for k, t in v:
        out.setdefault(k, []).append(t)
    return {k: round(sum(t) / len(t), 4) for k, t in sorted(out.items(), reverse=True)}
print(json.dumps({"djfa_k": perk(pt), "jfa_k": perk(jpt), "frame_ms": e0.elapsed_time(e1) / 20, "pass_ms": ms / n, "pass_GBps": 8 * px / n / (ms / n * 1e-3) / 1e9,
                  "jfa_frame_ms": j0.elapsed_time(j1) / 5, "jfa_pass_ms": jms / jn, "hash3": hex(h)}))
'''
# Usage: time_variants.py                      every build/variants/*.so + the in-tree libvd.so
#        time_variants.py VAR=v1,v2,...         the in-tree libvd.so under each value of env VAR
runs = []
if len(sys.argv) > 1 and "=" in sys.argv[1]:
    var, vals = sys.argv[1].split("=", 1)
    runs = [(f"{var}={v}", "", {var: v}) for v in vals.split(",")]
else:
    runs = [(os.path.basename(l), l, {}) for l in sorted(glob.glob("build/variants/*.so")) + ["paper_2209_00117_b200/libvd.so"]]
for name, lib, extra in runs:
    env = dict(os.environ, VARIANT_LIB=os.path.abspath(lib) if lib else "", **extra)
    r = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True, timeout=600)
    out = r.stdout.strip().splitlines()[-1] if r.stdout.strip() else r.stderr[-400:]
    print(f"{name:45s} {out}", flush=True)
