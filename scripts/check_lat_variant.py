"""JFA under a debug build (-DVD_CHECK=1): the lattice walk traps if an input label is not congruent
to its pixel mod k, and the wide pass re-verifies its decoded labels; results against the oracle.
   python scripts/check_lat_variant.py build/variants/libvd_-DVD_CHECK-1.so"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import synth  # noqa: E402
import paper_2209_00117_b200 as vd  # noqa: E402
import numpy as np  # noqa: E402

vd._load_variant(sys.argv[1])
for N, s in ((512, 1000), (1024, 4096), (1536, 9000), (2048, 50), (4096, 65536), (16384, 1 << 20), (33280, 1 << 22)):
    xy = synth.uniform_seeds(N, s, rng_seed=N)
    d = vd.VoronoiDiagram(N, xy)
    d.jfa()
    assert np.array_equal(d.labels(), oracle.jfa(N, xy)), N
    d.close()
    print("checked JFA", N, s, flush=True)
print("VD_CHECK lattice walk ok")
