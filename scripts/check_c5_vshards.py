"""JFA at C5 (65536^2, 2^24 seeds) on two virtual row bands -- the banded lattice walks, with halo
rows from the other band -- against the oracle, every pixel (too slow for the test suite: ~5 min).
   python scripts/check_c5_vshards.py [env=value ...]   (VSHARDS=n: n bands, default 2)"""
import os
import sys
import time

for kv in sys.argv[1:]:
    k, v = kv.split("=")
    os.environ[k] = v
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import oracle  # noqa: E402
import synth  # noqa: E402
import paper_2209_00117_b200 as vd  # noqa: E402

N, s = 65536, 1 << 24
xy = synth.uniform_seeds(N, s, rng_seed=2209)
t0 = time.time()
G_bands = int(os.environ.get("VSHARDS", "2"))
d = vd.VoronoiDiagram(N, xy, virtual_shards=G_bands)
d.jfa()
L = d.labels()
d.close()
t1 = time.time()
G = oracle.jfa(N, xy)
t2 = time.time()
ok = np.array_equal(L, G)
print(f"C5 JFA, {G_bands} virtual bands {sys.argv[1:]}: gpu+download {t1 - t0:.1f} s, oracle {t2 - t1:.1f} s, equal: {ok}", flush=True)
sys.exit(0 if ok else 1)
