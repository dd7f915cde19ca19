"""Small JFA + dJFA run for compute-sanitizer (no oracle needed)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_2209_00117_b200 as vd  # noqa: E402

for N, s, G in ((64, 16, 0), (1024, 1024, 0), (1031, 200, 0), (256, 100, 4)):
    xy = synth.uniform_seeds(N, s, rng_seed=1)
    d = vd.VoronoiDiagram(N, xy, virtual_shards=G)
    d.jfa()
    for f in range(2):
        d.djfa_step(synth.displacements(s, 2, f, rng_seed=1), 2)
    print(N, s, G, hex(d.label_hash()), flush=True)
    d.close()
