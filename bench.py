#!/usr/bin/env python
"""bench.py -- dJFA frames/s on B200 (BASELINE.json metric), JSON line on rank 0.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C4] [--impl reference]

A step is one dJFA time step (Alg. 1 body) of the whole hot path over the
grid: seed move + forward map + remap + re-stamp + the delta_1..1 jump passes, through
the C ABI (vd_djfa_step) with the displacement stream already resident in HBM.  At N=1
the workload is BASELINE.json configs[3] (16384^2 grid, 2^20 uniform seeds, +-1 px
uniform moves): the largest config that fits one GPU and is inside the metric's
N = 4096..65536 range; its two 1-GiB ping-pong buffers exceed the 126 MB L2, so no
flush is needed between steps.  With N > 1 GPUs (torchrun) the same grid is split into
row bands, one per rank, with NCCL halo exchange per pass (strong scaling; value =
whole-job frames/s, time = max over ranks).

Also reported: the JFA baseline on the same frames (vs JFA, Eq. 6 speedup),
Gpix.pass/s, Eq. 5 similarity of dJFA vs the same-frame JFA and vs the exact diagram
on sampled pixels, the jump-pass roofline (algorithmic 8 B/px/pass vs measured HBM
peak), end-to-end (host displacements in, 8-byte label hash out per step), the CPU
oracle on a bounded sample, clocks during the timed region, and kernel launch counts.

--impl reference: the CPU oracle (oracle/, plain C + OpenMP) on a bounded sample of the
same workload, on the host cores (rank 0 only).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

CONFIGS = {
    # name: (N, seeds, d_max, description)            -- BASELINE.json configs
    "C2": (1024, 1024, 1, "1024x1024 grid, 1,024 uniform seeds, +-1 px uniform moves"),
    "C3": (4096, 65536, 1, "4096x4096 grid, 65,536 uniform seeds, +-1 px uniform moves"),
    "C4": (16384, 1 << 20, 1, "16384x16384 grid, 2^20 uniform seeds, +-1 px uniform moves"),
    "C5": (65536, 1 << 24, 1, "65536x65536 grid, 2^24 uniform seeds, +-1 px uniform moves"),
}
RNG = synth.RNG_SEED
# bounded CPU sample: same seed density (L_avg = 16) and move radius, 4096^2 grid
CPU_SAMPLE = (4096, 65536, 1)


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def _traffic_per_launch(cfg_name):
    """dram bytes per jump-pass launch from the committed ncu --set full capture."""
    path = os.path.join(ROOT, "profiles", "jump_pass_traffic.json")
    try:
        with open(path) as f:
            t = json.load(f)
        e = t.get(cfg_name)
        return None if e is None else float(e["dram_bytes_per_launch_djfa_avg"])
    except Exception:
        return None


class ClockSampler:
    """NVML clocks + throttle reasons sampled while the timed region runs."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
        0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
        0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
    }

    def __init__(self, device_index: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.005)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv:
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unavailable"]}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "samples": len(self.samples), "reasons": sorted(self.reasons)}


# ---------------------------------------------------------------------- CPU oracle leg

def cpu_oracle_sample(steps: int, warmup: int, budget_s: float | None, target_n: int):
    """Time the oracle's literal dJFA on the bounded sample.  Returns (frames/s scaled to
    the target grid, Gpix.pass/s, description, threads, frames timed)."""
    import oracle
    n, s, d = CPU_SAMPLE
    xy = synth.uniform_seeds(n, s, rng_seed=RNG)
    G = oracle.jfa(n, xy)
    passes = len(oracle.djfa_schedule(n, s, d))
    for f in range(warmup):
        G, xy, _ = oracle.djfa_step(n, xy, synth.displacements(s, d, f, rng_seed=RNG), d, G)
    frames, t0 = 0, time.perf_counter()
    while frames < steps:
        G, xy, _ = oracle.djfa_step(n, xy, synth.displacements(s, d, warmup + frames, rng_seed=RNG), d, G)
        frames += 1
        if budget_s is not None and time.perf_counter() - t0 > budget_s:
            break
    dt = time.perf_counter() - t0
    fps_sample = frames / dt
    scale = (n * n) / float(target_n * target_n)
    desc = (f"oracle dJFA (fwd map + remap + stamp + {passes} passes) on a {n}x{n} grid with {s} seeds "
            f"(same density L_avg=16 and +-{d} px moves as the bench grid), {frames} frames in {dt:.1f} s; "
            f"frames/s scaled by pixel ratio {n}^2/{target_n}^2")
    return fps_sample * scale, n * n * passes * fps_sample / 1e9, desc, oracle.num_threads(), frames


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    N, s, d, _ = CONFIGS[args.config]
    fps, gpps, desc, threads, frames = cpu_oracle_sample(args.steps, args.warmup, None, N)
    line = {
        "impl": "reference", "metric": "dJFA frames/s", "value": fps, "unit": "frames/s",
        "n_gpus": args.gpus, "steps": frames, "warmup": args.warmup, "ms_per_step": 1000.0 / fps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u32",
        "data": "synthetic", "gpix_pass_per_s": gpps,
        "config": {"workload": f"{args.config}: {CONFIGS[args.config][3]} (bounded CPU sample, see cpu_baseline)",
                   "N": N, "seeds": s, "d_max": d},
        "cpu_baseline": {"value": fps, "unit": "frames/s", "cores": threads, "kind": "oracle", "sample": desc},
        "e2e": {"value": fps, "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------- GPU leg

def run_gpu(args):
    import torch
    import torch.distributed as dist

    import paper_2209_00117_b200 as vd

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}; launch N>1 with torchrun")
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    vd.load_library()
    # a real (non-default) stream shared by torch and libvd: events recorded on it bracket
    # exactly the library's kernels
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    N, s, d, cdesc = CONFIGS[args.config]

    def handle_cfg():
        # every libvd handle gets its own NCCL communicator, hence its own unique id
        nccl_id = None
        if world > 1:
            idt = torch.zeros(128, dtype=torch.uint8, device="cuda")
            if rank == 0:
                idt.copy_(torch.frombuffer(bytearray(vd.vd_nccl_unique_id()), dtype=torch.uint8))
            dist.broadcast(idt, 0)
            nccl_id = bytes(idt.cpu().numpy().tobytes())
        return dict(device=local, stream=stream.cuda_stream, rank=rank, world=world, nccl_id=nccl_id,
                    peer_halos=world > 1 and args.halo == "peer")

    halo_mode = ["nccl" if world > 1 else None]

    def make(**extra):
        h = vd.VoronoiDiagram(N, xy0, **handle_cfg(), **extra)
        if world > 1 and args.halo == "peer":
            # fused peer-memory halo push (NEXT-3); NCCL stays for steps with 2k >= band rows
            try:
                h.attach_peers()
                halo_mode[0] = "peer (fused push, NVLink P2P) + nccl for 2k >= band"
            except Exception as e:  # noqa: BLE001 -- fall back to the NCCL exchange, say so
                print(f"peer halos unavailable ({e}); using NCCL", file=sys.stderr)
        return h

    xy0 = synth.uniform_seeds(N, s, rng_seed=RNG)
    W, K = args.warmup, args.steps
    KE = max(3, min(K, args.e2e_steps))
    nframes = W + K + KE
    disp_host = [synth.displacements(s, d, f, rng_seed=RNG) for f in range(nframes)]
    disp_dev = torch.from_numpy(np.stack(disp_host[: W + K])).to("cuda")  # resident in HBM
    disp_pin = [torch.from_numpy(a).pin_memory() for a in disp_host[W + K:]]

    def ev():
        return torch.cuda.Event(enable_timing=True)

    # ---------------- dJFA: bootstrap (untimed), warmup, timed region
    dj = make()
    jf = make()
    dj.jfa()
    for f in range(W):
        dj.djfa_step(disp_dev[f], d)
    passes = dj.last_passes()
    packed = dj.last_packed_passes()  # passes of the last warm-up frame on the packed-key kernel
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    launches0 = dj.launch_count()
    dj.set_pass_timing(True)
    e0, e1 = ev(), ev()
    with ClockSampler(local) as clk:
        e0.record(stream)
        for f in range(W, W + K):
            dj.djfa_step(disp_dev[f], d)
        e1.record(stream)
        torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    ms = max_over_ranks(e0.elapsed_time(e1))
    dj.set_pass_timing(False)
    pass_ms, pass_launches, pass_px = dj.pass_timing()
    launches = dj.launch_count() - launches0
    fps = K / (ms / 1000.0)
    gpps = N * N * passes * K / (ms / 1000.0) / 1e9

    # ---------------- JFA baseline on the same frames (move + full JFA each frame)
    for f in range(W):
        jf.move_seeds(disp_dev[f])
        jf.jfa()
    jpasses = None
    torch.cuda.synchronize()
    barrier()
    j0, j1 = ev(), ev()
    j0.record(stream)
    for f in range(W, W + K):
        jf.move_seeds(disp_dev[f])
        jf.jfa()
    j1.record(stream)
    torch.cuda.synchronize()
    barrier()
    jms = max_over_ranks(j0.elapsed_time(j1))
    jpasses = jf.last_passes()
    jpacked = jf.last_packed_passes()
    jfps = K / (jms / 1000.0)
    sim_vs_jfa = dj.similarity(jf)  # Eq. 5, same frame, dJFA vs JFA

    # ---------------- dJFAm (Manhattan) on the same frames: speed + similarity
    djm = None
    if not args.no_variants:
        dm = make(metric="manhattan")
        dm.jfa()
        for f in range(W):
            dm.djfa_step(disp_dev[f], d)
        torch.cuda.synchronize()
        barrier()
        m0, m1 = ev(), ev()
        m0.record(stream)
        for f in range(W, W + K):
            dm.djfa_step(disp_dev[f], d)
        m1.record(stream)
        torch.cuda.synchronize()
        barrier()
        mms = max_over_ranks(m0.elapsed_time(m1))
        djm = {"value": K / (mms / 1000.0), "unit": "frames/s", "ms_per_frame": mms / K,
               "similarity_vs_jfa_pct": dm.similarity(jf),
               "speedup_vs_jfa": (K / (mms / 1000.0)) / jfps,
               "paper": "dJFAm ~5x over JFA at 88-92% similarity (P:268, P:296; A100)"}
        dm.close()

    # similarity vs the exact diagram on sampled pixels (Eq. 1 by brute force per pixel)
    sim_exact = None
    if rank == 0 and world == 1 and not args.no_exact_sample:
        L = dj.labels()
        cur = dj.seeds()
        lx, ly = cur[0::2].astype(np.int64), cur[1::2].astype(np.int64)
        lab = (ly.astype(np.uint64) << np.uint64(16)) | lx.astype(np.uint64)
        rng = np.random.default_rng(1)
        good, n_s = 0, 200
        for y, x in zip(rng.integers(0, N, n_s), rng.integers(0, N, n_s)):
            d2 = (lx - x) ** 2 + (ly - y) ** 2
            good += int(L[y, x] == lab[d2 == d2.min()].min())
        sim_exact = {"pct": 100.0 * good / n_s, "pixels": n_s}

    # ---------------- end to end: host (pinned) displacements in, 8-byte hash out
    barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    x0, x1 = ev(), ev()
    hashes = torch.zeros(len(disp_pin), dtype=torch.int64).pin_memory()  # each step's result
    x0.record(stream)
    for i, a in enumerate(disp_pin):
        vd.vd_djfa_step(dj.h, a, d, s)
        vd.vd_label_hash_async(dj.h, hashes[i].data_ptr())  # D2H without a host round trip
    x1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = max_over_ranks(x0.elapsed_time(x1))
    assert int(hashes[-1]) & 0xFFFFFFFFFFFFFFFF == dj.label_hash(), "async checksum mismatch"
    e2e_fps = len(disp_pin) / (e2e_ms / 1000.0)

    # ---------------- roofline of the dominant kernel (the jump pass)
    peak, peak_src = _peaks()
    alg_bytes = 8.0 * pass_px / max(pass_launches, 1)
    pass_avg_ms = pass_ms / max(pass_launches, 1)
    achieved = alg_bytes / (pass_avg_ms / 1000.0) / 1e9
    frame_share = pass_ms / (ms if world == 1 else pass_ms + 1e-9)
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "traffic": _traffic_per_launch(args.config), "kernel": "jump_pass_fast",
                "alg_bytes_per_launch": alg_bytes, "avg_launch_ms": pass_avg_ms,
                "launches_timed": pass_launches, "share_of_step": frame_share if world == 1 else None,
                "peak_source": peak_src}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cfps, cgpps, cdesc2, threads, _ = cpu_oracle_sample(10**6, 1, args.cpu_seconds, N)
        cpu = {"value": cfps, "unit": "frames/s", "cores": threads, "kind": "oracle", "sample": cdesc2,
               "gpix_pass_per_s": cgpps}

    if rank == 0:
        line = {
            "metric": "dJFA frames/s", "value": fps, "unit": "frames/s", "n_gpus": world, "steps": K, "warmup": W,
            "ms_per_step": ms / K, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "u32", "data": "synthetic",
            "config": {"workload": f"{args.config}: {cdesc}, dJFA time steps", "N": N, "seeds": s, "d_max": d,
                       "passes_per_frame": passes, "packed_passes_per_frame": packed, "parallelism": f"rowband{world}", "halo": halo_mode[0],
                       "l2": (f"inputs larger than L2 (two {4 * N * N / 2**30:g}-GiB ping-pong label buffers vs 126 MB L2)"
                              if 8 * N * N > 126e6 else "inputs fit in L2, no flush: a parity config, not the headline")},
            "gpix_pass_per_s": gpps,
            "jfa": {"value": jfps, "unit": "frames/s", "ms_per_frame": jms / K, "passes_per_frame": jpasses,
                    "packed_passes_per_frame": jpacked,
                    "gpix_pass_per_s": N * N * jpasses * K / (jms / 1000.0) / 1e9},
            "speedup_vs_jfa": jfps and fps / jfps,
            "similarity_vs_jfa_pct": sim_vs_jfa,
            "similarity_vs_exact_sampled": sim_exact,
            "djfam": djm,
            "paper_context": "A100 40GB (P:222-240): dJFA up to ~5.3x over JFA, similarity >= 88% (P:25)",
            "roofline": roofline,
            "e2e": {"value": e2e_fps, "unit": "frames/s", "h2d_bytes_per_step": 4 * s, "d2h_bytes_per_step": 8,
                    "steps": len(disp_pin),
                    "what": "vd_djfa_step with pinned host displacements + vd_label_hash_async (8-byte D2H into pinned memory, no per-step host round trip) per step"},
            "gpu_launches": launches,
            "clocks": clk.summary(),
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    dj.close()
    jf.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="C4", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=30)
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-exact", "--no-exact-sample", dest="no_exact_sample", action="store_true")
    ap.add_argument("--no-variants", action="store_true", help="skip the dJFAm (Manhattan) measurement")
    ap.add_argument("--halo", default="peer", choices=["peer", "nccl"],
                    help="N > 1: halo rows pushed by the pass kernels over peer memory, or NCCL send/recv")
    args = ap.parse_args()
    if args.warmup < 3:
        raise SystemExit("--warmup must be >= 3")
    if args.impl == "reference":
        return run_reference(args)
    return run_gpu(args)


if __name__ == "__main__":
    sys.exit(main())
