"""ncu driver: C4 JFA, then one label_hash and one match_count launch."""
import os, sys
sys.path.insert(0, os.getcwd())
import torch, synth
import paper_2209_00117_b200 as vd
N, s = 16384, 1 << 20
xy = synth.uniform_seeds(N, s, rng_seed=2209)
st = torch.cuda.Stream()
d = vd.VoronoiDiagram(N, xy, device=0, stream=st.cuda_stream)
d.jfa()
print(hex(d.label_hash()), d.similarity(d))
