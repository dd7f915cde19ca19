import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, oracle, synth
import paper_2209_00117_b200 as vd
EMPTY = 0xFFFFFFFF
for N, k in ((1024, 512), (1024, 256), (1024, 1024), (2048, 512), (1024, 2)):
    s = 40
    xy = synth.uniform_seeds(N, s, rng_seed=N)
    labels = np.array([oracle.pack(int(xy[2*i]), int(xy[2*i+1])) for i in range(s)] + [EMPTY], dtype=np.uint32)
    rng = np.random.default_rng(0)
    G = labels[rng.integers(0, len(labels) - 1, size=(N, N))]  # no EMPTY
    d = vd.VoronoiDiagram(N, xy)
    d.set_labels(G); d.jump_pass(k)
    A = d.labels(); B = oracle.jump_pass(G, k)
    bad = np.argwhere(A != B)
    print(N, k, "mismatches", len(bad), bad[:5].tolist(), flush=True)
    if len(bad):
        y, x = bad[0]
        print("  got", hex(A[y, x]), "want", hex(B[y, x]), "cands", [hex(G[yy, xx]) for yy in (y-k, y, y+k) for xx in (x-k, x, x+k) if 0 <= yy < N and 0 <= xx < N])
