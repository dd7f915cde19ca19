"""Per-launch breakdown driver (run under ncu --metrics gpu__time_duration.sum): one JFA and
two dJFA frames at VD_CFG (C4 / C5) through the C ABI."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
import paper_2209_00117_b200 as vd  # noqa: E402

N, s = {"C4": (16384, 1 << 20), "C5": (65536, 1 << 24), "C3": (4096, 65536)}[os.environ.get("VD_CFG", "C5")]
xy = synth.uniform_seeds(N, s, rng_seed=2209)
st = torch.cuda.Stream()
d = vd.VoronoiDiagram(N, xy, device=0, stream=st.cuda_stream)
d.jfa()
d.synchronize()
for f in range(2):
    d.djfa_step(synth.displacements(s, 1, f, rng_seed=2209), 1)
d.synchronize()
print("passes/frame", d.last_passes())
