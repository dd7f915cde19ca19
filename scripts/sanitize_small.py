"""Small JFA / dJFA / StF / variant runs for compute-sanitizer (no oracle needed)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import synth  # noqa: E402
import paper_2209_00117_b200 as vd  # noqa: E402

cases = [
    (64, 16, {}), (1031, 200, {}), (1024, 1024, {}), (256, 100, {"virtual_shards": 4}),
    (300, 50, {"metric": "manhattan", "vn_waves": 2}), (128, 30, {"jfa_vn_waves": 99}),
    (1024, 1024, {"virtual_shards": 4, "peer_halos": True}), (512, 300, {"virtual_shards": 2, "peer_halos": True}),
    # dense (L_avg = 16): the dJFA passes take the packed-key walk, one band and sharded
    (1024, 4096, {}), (1024, 4096, {"virtual_shards": 4}), (1000, 3906, {}),
]
for N, s, cfg in cases:
    xy = synth.uniform_seeds(N, s, rng_seed=1)
    d = vd.VoronoiDiagram(N, xy, **cfg)
    d.jfa()
    for f in range(2):
        try:
            d.djfa_step(synth.displacements(s, 2, f, rng_seed=1), 2)
        except vd.VDError:
            pass  # Von Neumann-only JFA may be incomplete: dJFA is refused (VD_ERR_STATE)
    e = vd.VoronoiDiagram(N, xy, **{k: v for k, v in cfg.items() if k != "jfa_vn_waves"})
    e.stf()
    e.set_labels(d.labels())
    e.jump_pass(3)
    print(N, s, cfg, hex(d.label_hash()), d.match_count(d), "packed", d.last_packed_passes(), flush=True)
    d.close()
    e.close()

# the windowed kernel (forced at small N) on a complete map, including its exact recomputation
os.environ["VD_FORCE_WINDOWED"] = "1"
N, s = 1031, 300
xy = synth.uniform_seeds(N, s, rng_seed=2)
d = vd.VoronoiDiagram(N, xy)
d.jfa()
for f in range(2):
    d.djfa_step(synth.displacements(s, 3, f, rng_seed=2), 3)
G = d.labels()
rng = np.random.default_rng(0)
for k in (1, 2, 4, 16, 512):
    d.set_labels(G)
    d.jump_pass(k)
print("windowed", hex(d.label_hash()), flush=True)
d.close()

# the wide exact pass (forced at small N by its test hook): JFA and passes with EMPTY, partial groups
os.environ["VD_FORCE_WINDOWED"] = "0"
os.environ["VD_FORCE_WSK"] = "1"
for N in (1536, 2048):
    xy = synth.uniform_seeds(N, N * N // 256, rng_seed=3)
    d = vd.VoronoiDiagram(N, xy)
    d.jfa()
    rng = np.random.default_rng(N)
    G = ((rng.integers(0, N, (N, N)) << 16) | rng.integers(0, N, (N, N))).astype(np.uint32)
    G[rng.random((N, N)) < 0.5] = 0xFFFFFFFF
    for k in (256, 512):
        if 4 * k <= N:
            d.set_labels(G)
            d.jump_pass(k)
    print("wide", N, hex(d.label_hash()), flush=True)
    d.close()
