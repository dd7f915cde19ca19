"""C4 JFA + 3 dJFA frames with the separate remap (VD_NO_FUSE=1), optionally on another build of
libvd, for ncu -k regex:remap:   python scripts/profile_remap.py [path/to/libvd.so]"""
import os
import sys

os.environ["VD_NO_FUSE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_2209_00117_b200 as vd  # noqa: E402

if len(sys.argv) > 1:
    vd._load_variant(sys.argv[1])
N, s = 16384, 1 << 20
xy = synth.uniform_seeds(N, s, rng_seed=2209)
d = vd.VoronoiDiagram(N, xy)
d.jfa()
for f in range(3):
    d.djfa_step(synth.displacements(s, 1, f, rng_seed=2209), 1)
print("hash", hex(d.label_hash()))
