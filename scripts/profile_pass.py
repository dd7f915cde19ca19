"""Small driver for ncu: JFA bootstrap + a few dJFA frames through the C ABI (VD_CFG = C2..C5)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
import paper_2209_00117_b200 as vd  # noqa: E402

cfg = {"C3": (4096, 65536), "C4": (16384, 1 << 20), "C2": (1024, 1024), "C5": (65536, 1 << 24)}[os.environ.get("VD_CFG", "C4")]
frames = int(os.environ.get("VD_FRAMES", "3"))
N, s = cfg
xy = synth.uniform_seeds(N, s, rng_seed=2209)
st = torch.cuda.Stream()
d = vd.VoronoiDiagram(N, xy, device=0, stream=st.cuda_stream)
d.jfa()
for f in range(frames):
    d.djfa_step(synth.displacements(s, 1, f, rng_seed=2209), 1)
d.synchronize()
print("passes/frame", d.last_passes(), "hash", hex(d.label_hash()))
