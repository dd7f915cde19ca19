"""Run the wide exact pass under a debug build (-DVD_CHECK=1: device-side checks that every decoded
label lies in the grid and reproduces its winning key) and compare with the oracle.
   python scripts/check_wsk_variant.py build/variants/libvd_-DVD_CHECK-1.so"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import oracle  # noqa: E402
import synth  # noqa: E402
import paper_2209_00117_b200 as vd  # noqa: E402

vd._load_variant(sys.argv[1])
os.environ["VD_FORCE_WSK"] = "1"
for N in (1024, 1536, 2048, 33280):
    rng = np.random.default_rng(N)
    G = ((rng.integers(0, N, (N, N)) << 16) | rng.integers(0, N, (N, N))).astype(np.uint32)
    H = G.copy()
    H[rng.random((N, N), dtype=np.float32) < 0.6] = 0xFFFFFFFF
    d = vd.VoronoiDiagram(N, np.array([0, 0], dtype=np.uint16))
    for M in (G, H):
        for k in (256, 512, 1024, 2048, 8192):
            if 4 * k <= N:
                d.set_labels(M)
                d.jump_pass(k)
                assert np.array_equal(d.labels(), oracle.jump_pass(M, k)), (N, k)
    if N <= 2048:
        xy = synth.uniform_seeds(N, N * N // 256, rng_seed=N)
        e = vd.VoronoiDiagram(N, xy)
        e.jfa()
        assert np.array_equal(e.labels(), oracle.jfa(N, xy)), N
        e.close()
    d.close()
    print("checked", N, flush=True)
print("VD_CHECK wide pass ok")
