#!/usr/bin/env python
"""dJFA vs JFA sweeps on one B200 (BASELINE.json configs[2]; the paper's Figs. 7-9 axes).

  python scripts/sweep.py --kind radius   # 4096^2, 65,536 seeds, d_max = 1 .. 2048
  python scripts/sweep.py --kind density  # 4096^2, s = 2^8 .. 2^20, d_max = 2

For each point: dJFA passes (Eq. 4), dJFA and JFA frames/s (CUDA events, device-resident
displacements, frames = move + full step), Eq. 6 speedup, and Eq. 5 similarity of dJFA vs
the same-frame JFA (mean over frames) -- Euclidean (dJFAe) and Manhattan (dJFAm).
One JSON object per line on stdout.
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import synth  # noqa: E402


def point(vd, torch, N, s, d, frames, warm, metric):
    st = torch.cuda.Stream()
    torch.cuda.set_stream(st)
    xy = synth.uniform_seeds(N, s, rng_seed=synth.RNG_SEED)
    disp = torch.from_numpy(np.stack([synth.displacements(s, d, f, rng_seed=synth.RNG_SEED)
                                      for f in range(warm + frames)])).cuda()
    dj = vd.VoronoiDiagram(N, xy, stream=st.cuda_stream, metric=metric)
    jf = vd.VoronoiDiagram(N, xy, stream=st.cuda_stream)
    dj.jfa()
    for f in range(warm):
        dj.djfa_step(disp[f], d)
        jf.move_seeds(disp[f])
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    tdj = tjf = 0.0
    sims = []
    for f in range(warm, warm + frames):
        a, b, c = ev(), ev(), ev()
        a.record(st)
        dj.djfa_step(disp[f], d)
        b.record(st)
        jf.move_seeds(disp[f])
        jf.jfa()
        c.record(st)
        torch.cuda.synchronize()
        tdj += a.elapsed_time(b)
        tjf += b.elapsed_time(c)
        sims.append(dj.similarity(jf))
    out = {"N": N, "seeds": s, "d_max": d, "metric": metric, "djfa_passes": dj.last_passes(),
           "jfa_passes": jf.last_passes(), "djfa_fps": frames / (tdj / 1e3), "jfa_fps": frames / (tjf / 1e3),
           "speedup": tjf / tdj, "similarity_vs_jfa_mean": float(np.mean(sims)),
           "similarity_vs_jfa_min": float(np.min(sims)), "frames": frames}
    dj.close()
    jf.close()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--kind", choices=["radius", "density"], default="radius")
    ap.add_argument("--frames", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--N", type=int, default=4096)
    args = ap.parse_args()
    import torch
    import paper_2209_00117_b200 as vd
    vd.load_library()
    N = args.N
    if args.kind == "radius":
        pts = [(65536, d) for d in (1, 2, 4, 8, 16, 32, 64, 128, 256, 512, 1024, 2048)]
    else:
        pts = [(2 ** e, 2) for e in range(8, 21, 2)]
    for s, d in pts:
        for metric in ("euclid", "manhattan"):
            print(json.dumps(point(vd, torch, N, s, d, args.frames, args.warmup, metric)), flush=True)


if __name__ == "__main__":
    main()
