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
NOMINAL_HBM_GBS = 8000.0  # the north star's "B200 peak of about 8 TB/s"
CPU_FRAMES = 3            # timed oracle frames for cpu_baseline (after the untimed bootstrap)


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
        if e is None:
            return None
        plain = [x["dram_bytes"] for x in e["launches"] if "remap" not in x["kernel"]]  # the dominant kernel's
        return sum(plain) / len(plain) if plain else float(e["dram_bytes_per_launch_djfa_avg"])
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

def cpu_model() -> str:
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def oracle_run(N: int, xy0, disps, d: int, warmup: int, check=None):
    """The CPU oracle on the bench workload itself (the same grid, seeds and displacement
    stream as the GPU): JFA bootstrap (untimed), `warmup` untimed dJFA frames, then one
    timed dJFA frame (oracle.djfa_step: move + fwd map + remap + re-stamp + passes, the same
    region the GPU step covers) per remaining entry of `disps`.  check(stage, G) is called on
    the bootstrap (stage 0) and after every frame (stage f + 1), untimed.
    Returns (ms per timed frame, passes per frame, threads)."""
    import oracle
    G = oracle.jfa(N, xy0)
    if check:
        check(0, G)
    xy = xy0
    times, passes = [], 0
    for f, disp in enumerate(disps):
        t0 = time.perf_counter()
        G, xy, passes = oracle.djfa_step(N, xy, disp, d, G, inplace=True)
        dt = time.perf_counter() - t0
        if f >= warmup:
            times.append(dt)
        if check:
            check(f + 1, G)
    return [1000.0 * t for t in times], passes, oracle.num_threads()


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    N, s, d, cdesc = CONFIGS[args.config]
    xy0 = synth.uniform_seeds(N, s, rng_seed=RNG)
    W, K = args.warmup, args.steps
    disps = [synth.displacements(s, d, f, rng_seed=RNG) for f in range(W + K)]
    ms, passes, threads = oracle_run(N, xy0, disps, d, W)
    mean_ms = sum(ms) / len(ms)
    fps = 1000.0 / mean_ms
    sample = (f"oracle/ (plain C + OpenMP, uint64 keys) on the bench workload itself: {N}x{N} grid, {s} seeds, "
              f"+-{d} px moves; JFA bootstrap and {W} warm-up frames untimed, then {K} dJFA frames timed one by one "
              f"(move + fwd map + remap + re-stamp + {passes} passes each); CPU: {cpu_model()}")
    line = {
        "impl": "reference", "metric": "dJFA frames/s", "value": fps, "unit": "frames/s",
        "n_gpus": args.gpus, "steps": K, "warmup": W, "ms_per_step": mean_ms,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u32",
        "data": "synthetic", "gpix_pass_per_s": N * N * passes / (mean_ms / 1000.0) / 1e9,
        "config": {"workload": f"{args.config}: {cdesc}, dJFA time steps", "N": N, "seeds": s, "d_max": d},
        "cpu_baseline": {"value": fps, "unit": "frames/s", "cores": threads, "kind": "oracle", "sample": sample,
                         "cpu_model": cpu_model()},
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

    def gather(obj):
        if world == 1:
            return [obj]
        out = [None] * world
        dist.all_gather_object(out, obj)
        return out

    N, s, d, cdesc = CONFIGS[args.config]
    B = N // world

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
    peak, peak_src = _peaks()

    def ev():
        return torch.cuda.Event(enable_timing=True)

    def roofline(times, kernel):
        """times: [(k, ms)] of timed jump passes (all launches of a pass); 8 B/px/pass algorithmic."""
        tot_ms = sum(t for _, t in times)
        n = max(len(times), 1)
        alg = 8.0 * B * N  # bytes per pass per rank (one band)
        ach = alg * n / (tot_ms / 1000.0) / 1e9 if tot_ms else 0.0
        per_k = {}
        for k, t in times:
            per_k.setdefault(k, []).append(t)
        return {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
                "frac_nominal": ach / NOMINAL_HBM_GBS, "kernel": kernel, "alg_bytes_per_launch": alg,
                "avg_launch_ms": tot_ms / n, "launches_timed": len(times), "peak_source": peak_src,
                "per_k": {str(k): {"ms": statistics.mean(v), "frac": alg / (statistics.mean(v) / 1000.0) / 1e9 / peak}
                          for k, v in sorted(per_k.items(), reverse=True)}}

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
        fev = [ev() for _ in range(K)] if args.frames_csv else None  # per-frame boundaries (optional CSV)
        for f in range(W, W + K):
            dj.djfa_step(disp_dev[f], d)
            if fev:
                fev[f - W].record(stream)
        e1.record(stream)
        torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    own_ms = e0.elapsed_time(e1)
    ms = max_over_ranks(own_ms)
    dj.set_pass_timing(False)
    dj_times = dj.pass_times()
    pass_ms, pass_launches, pass_px = dj.pass_timing()
    launches = dj.launch_count() - launches0
    if world > 1:
        assert not dj.peer_timed_out(), "a peer-halo wait timed out during the timed region"
    fps = K / (ms / 1000.0)
    gpps = N * N * passes * K / (ms / 1000.0) / 1e9
    per_rank = gather({"rank": rank, "frame_ms": own_ms / K, "pass_ms": pass_ms / K,
                       "other_ms": (own_ms - pass_ms) / K})

    # ---------------- JFA baseline on the same frames (move + full JFA each frame)
    for f in range(W):
        jf.move_seeds(disp_dev[f])
        jf.jfa()
    torch.cuda.synchronize()
    barrier()
    jf.set_pass_timing(True)
    j0, j1 = ev(), ev()
    j0.record(stream)
    jev = [ev() for _ in range(K)] if args.frames_csv else None
    for f in range(W, W + K):
        jf.move_seeds(disp_dev[f])
        jf.jfa()
        if jev:
            jev[f - W].record(stream)
    j1.record(stream)
    torch.cuda.synchronize()
    barrier()
    jms = max_over_ranks(j0.elapsed_time(j1))
    jf.set_pass_timing(False)
    jf_times = jf.pass_times()
    jf.pass_timing()
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

    # ---------------- Eq. 5 similarity of each method vs the exact diagram (Eq. 1), whole grid
    # (untimed; the exact diagram is the oracle's bucketed brute force on this frame's seeds)
    sim_exact = None
    if rank == 0 and world == 1 and not args.no_exact:
        import oracle
        t0 = time.perf_counter()
        E = oracle.exact(N, dj.seeds())
        sim_exact = {"djfa_pct": dj.similarity_host(E), "jfa_pct": jf.similarity_host(E), "pixels": N * N,
                     "frame": W + K, "exact": f"oracle.exact (bucketed brute force, Eq. 1), {time.perf_counter() - t0:.1f} s"}
        if djm is not None:
            sim_exact["note"] = "dJFAm is compared with the Euclidean JFA only (R-23)"
        del E

    # ---------------- end to end: host (pinned) displacements in, 8-byte hash out
    barrier()
    torch.cuda.synchronize()
    x0, x1 = ev(), ev()
    hashes = torch.zeros(len(disp_pin), dtype=torch.int64).pin_memory()  # each step's result
    x0.record(stream)
    for i, a in enumerate(disp_pin):
        # the step's last pass also sums the checksum; 8-byte D2H without a host round trip
        vd.vd_djfa_step_hash(dj.h, a, d, s, hashes[i].data_ptr())
    x1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = max_over_ranks(x0.elapsed_time(x1))
    assert int(hashes[-1]) & 0xFFFFFFFFFFFFFFFF == dj.label_hash(), "async checksum mismatch"
    e2e_fps = len(disp_pin) / (e2e_ms / 1000.0)
    # ... and with the whole label map (this rank's band) copied to pinned host memory each step
    e2e_full = None
    if not args.no_e2e_full:
        out = torch.empty((B, N), dtype=torch.int32).pin_memory()
        barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for a in disp_pin:
            vd.vd_djfa_step(dj.h, a, d, s)
            vd.vd_get_labels_into(dj.h, out.data_ptr())
        full_s = max_over_ranks(time.perf_counter() - t0)
        e2e_full = {"value": len(disp_pin) / full_s, "unit": "frames/s", "h2d_bytes_per_step": 4 * s,
                    "d2h_bytes_per_step": 4 * B * N, "steps": len(disp_pin),
                    "what": "vd_djfa_step with pinned host displacements + vd_get_labels of the whole label map "
                            "into pinned host memory (synchronous) per step; host wall clock"}

    # ---------------- parity of the timed path (untimed): the JFA bootstrap and the first
    # CPU_FRAMES dJFA frames of this workload, GPU vs the CPU oracle.  One GPU: every pixel
    # (np.array_equal); N > 1: the all-reduced whole-diagram label hash on rank 0.
    pv = make()
    pv.jfa()
    gpu_stages = [(pv.label_hash(), pv.labels() if world == 1 else None)]
    for f in range(CPU_FRAMES):
        pv.djfa_step(disp_host[f], d)
        gpu_stages.append((pv.label_hash(), pv.labels() if world == 1 else None))
    pv.close()
    cpu, parity = None, None
    if rank == 0 and not args.no_cpu_baseline:
        import oracle
        ok = []

        def check(stage, G):
            h, L = gpu_stages[stage]
            ok.append(bool(np.array_equal(L, G)) if L is not None else h == oracle.label_hash(G))

        cms, cpasses, threads = oracle_run(N, xy0, disp_host[:CPU_FRAMES], d, 0, check)
        cmean = sum(cms) / len(cms)
        parity = {"ok": all(ok), "stages": ok,
                  "what": ("JFA bootstrap + dJFA frames 1..%d of this workload: GPU %s vs the CPU oracle"
                           % (CPU_FRAMES, "label map == oracle map (every pixel)" if world == 1
                              else "all-reduced label hash == oracle label hash"))}
        if world == 1:
            cpu = {"value": 1000.0 / cmean, "unit": "frames/s", "cores": threads, "kind": "oracle",
                   "sample": (f"the bench workload itself ({N}x{N}, {s} seeds, +-{d} px): oracle JFA bootstrap "
                              f"untimed, then {CPU_FRAMES} dJFA frames timed one by one (move + fwd map + remap + "
                              f"re-stamp + {cpasses} passes), {cmean / 1000.0:.2f} s per frame"),
                   "cpu_model": cpu_model(), "gpix_pass_per_s": N * N * cpasses / (cmean / 1000.0) / 1e9,
                   "ms_per_frame": cmean}
    barrier()

    remap_ms = [t for k, t in dj_times if k == 0]
    # The dominant kernel: jump_pass_sk's packed passes.  On one band the frame's first pass is
    # jump_pass_sk_remap (the remap fused in, NEXT-1): it is reported beside them, not averaged in.
    pass_times = [(k, t) for k, t in dj_times if k != 0]
    fused = world == 1 and not remap_ms and pass_times
    first_k = pass_times[0][0] if fused else None
    if args.frames_csv and rank == 0:  # one row per frame
        import csv
        with open(args.frames_csv, "w", newline="") as fh:
            w = csv.writer(fh)
            w.writerow(["config", "n_gpus", "algorithm", "frame", "passes", "ms", "gpix_pass_per_s", "frac_hbm_measured",
                        "frac_hbm_nominal"])
            for name, starts, evs, npass in (("dJFA", e0, fev, passes), ("JFA", j0, jev, jpasses)):
                prev = starts
                for i, e in enumerate(evs):
                    t = prev.elapsed_time(e)
                    gbs = 8.0 * N * N * npass / (t / 1000.0) / 1e9
                    w.writerow([args.config, world, name, W + i, npass, f"{t:.4f}",
                                f"{N * N * npass / (t / 1000.0) / 1e9:.2f}", f"{gbs / peak:.4f}",
                                f"{gbs / NOMINAL_HBM_GBS:.4f}"])
                    prev = e

    dj_roof = roofline([(k, t) for k, t in pass_times if not fused or k != first_k], "jump_pass_sk (packed-key walk)")
    dj_roof["all_passes"] = {k: v for k, v in roofline(pass_times, "all jump passes of the frame").items()
                             if k in ("achieved", "frac", "frac_nominal", "avg_launch_ms", "launches_timed")}
    if fused:
        fm = statistics.mean([t for k, t in pass_times if k == first_k])
        dj_roof["first_pass_fused_remap"] = {
            "kernel": "jump_pass_sk_remap", "k": first_k, "avg_launch_ms": fm,
            "achieved": 8.0 * B * N / (fm / 1000.0) / 1e9, "frac": 8.0 * B * N / (fm / 1000.0) / 1e9 / peak,
            "note": "pass k = delta_1 with the remap of the previous diagram fused in: 8 B/px algorithmic (the "
                    "separate remap's 8 B/px never happen); it replaces a remap + pass pair"}
    if remap_ms:  # the frame's second kernel: 8 B/px algorithmic (read + write every label)
        rm = statistics.mean(remap_ms)
        dj_roof["remap"] = {"kernel": "remap_lanes", "avg_launch_ms": rm,
                            "achieved": 8.0 * B * N / (rm / 1000.0) / 1e9,
                            "frac": 8.0 * B * N / (rm / 1000.0) / 1e9 / peak}
    dj_roof["traffic"] = _traffic_per_launch(args.config)
    dj_roof["share_of_step"] = pass_ms / own_ms
    jf_roof = roofline(jf_times, "jump_pass_sk (exact walk)")
    jf_roof["note"] = ("JFA's first pass (k_1) is fused with the initialisation (jfa_first_pass, a seed scatter) "
                       "and is not a timed pass; its time is in jfa.ms_per_frame")
    if rank == 0:
        line = {
            "metric": "dJFA frames/s", "value": fps, "unit": "frames/s", "n_gpus": world, "steps": K, "warmup": W,
            "ms_per_step": ms / K, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "u32", "data": "synthetic",
            "config": {"workload": f"{args.config}: {cdesc}, dJFA time steps", "N": N, "seeds": s, "d_max": d,
                       "passes_per_frame": passes, "packed_passes_per_frame": packed, "parallelism": f"rowband{world}",
                       "halo": halo_mode[0],
                       "l2": (f"inputs larger than L2 (two {4 * N * N / 2**30:g}-GiB ping-pong label buffers vs 126 MB L2)"
                              if 8 * N * N > 126e6 else "inputs fit in L2, no flush: a parity config, not the headline")},
            "gpix_pass_per_s": gpps,
            "jfa": {"value": jfps, "unit": "frames/s", "ms_per_frame": jms / K, "passes_per_frame": jpasses,
                    "packed_passes_per_frame": jpacked,
                    "gpix_pass_per_s": N * N * jpasses * K / (jms / 1000.0) / 1e9, "roofline": jf_roof},
            "speedup_vs_jfa": jfps and fps / jfps,
            "similarity_vs_jfa_pct": sim_vs_jfa,
            "similarity_vs_exact": sim_exact,
            "djfam": djm,
            "paper_context": "A100 40GB (P:222-240): dJFA up to ~5.3x over JFA, similarity >= 88% (P:25)",
            "roofline": dj_roof,
            "parity": parity,
            "e2e": {"value": e2e_fps, "unit": "frames/s", "h2d_bytes_per_step": 4 * s, "d2h_bytes_per_step": 8,
                    "steps": len(disp_pin),
                    "what": ("vd_djfa_step_hash with pinned host displacements per step: the dJFA step, whose last "
                             "pass also sums the new diagram's checksum; the result read back is that 8-byte checksum "
                             "of the whole label map (a consumer of the map itself: see e2e_full_map)")},
            "e2e_full_map": e2e_full,
            "gpu_launches": launches,
            "clocks": clk.summary(),
            "cpu_baseline": cpu,
        }
        if world > 1:
            line["per_rank"] = per_rank
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
    ap.add_argument("--no-e2e-full", action="store_true", help="skip the e2e run that copies the whole map out")
    ap.add_argument("--frames-csv", default=None, help="also write one CSV row per timed frame (dJFA and JFA)")
    ap.add_argument("--no-cpu-baseline", action="store_true", help="skip the CPU oracle (cpu_baseline and parity)")
    ap.add_argument("--no-exact", action="store_true", help="skip the whole-grid similarity vs the exact diagram")
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
