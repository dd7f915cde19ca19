"""One wide exact pass (jump_pass_wsk) on a random far-label map, for ncu:
   ncu --set full -k regex:jump_pass_wsk python scripts/profile_wsk.py [N] [k] [empty_frac]"""
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_2209_00117_b200 as vd  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 33280
k = int(sys.argv[2]) if len(sys.argv) > 2 else 512
ef = float(sys.argv[3]) if len(sys.argv) > 3 else 0.0
rng = np.random.default_rng(1)
G = ((rng.integers(0, N, (N, N)) << 16) | rng.integers(0, N, (N, N))).astype(np.uint32)
if ef > 0:
    G[rng.random((N, N), dtype=np.float32) < ef] = 0xFFFFFFFF
vd.load_library()
d = vd.VoronoiDiagram(N, np.array([0, 0], dtype=np.uint16))
d.set_labels(G)
for _ in range(2):
    d.jump_pass(k)
d.labels()
d.close()
print("ok", N, k, ef)
