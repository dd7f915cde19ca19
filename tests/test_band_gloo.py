"""Row-band sharding on CPU: world_size 2 and 4 `gloo` process groups.

Each rank holds only its band of rows.  Before every pass it exchanges halos exactly as
libvd's vd_halo_plan says (the same plan libvd's NCCL path and virtual-shard path use),
with torch.distributed point-to-point send/recv, then computes its band with the oracle's
pass on a grid whose rows it does NOT hold are poisoned.  The gathered result must be
bit-identical to the unsharded oracle JFA / dJFA ("CPU band
simulation").  Only the plan is product code here; the arithmetic is the oracle's.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

POISON_SEED = 977


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _band_pass(G_band, k, N, world, rank, plan_fn, oracle):
    B = N // world
    p = plan_fn(N, world, rank, k)
    h = p["halo_rows"]
    reqs = []
    top = np.empty((h, N), dtype=np.uint32)
    bot = np.empty((h, N), dtype=np.uint32)
    t_top, t_bot = torch.from_numpy(top), torch.from_numpy(bot)
    ops = []
    if p["recv_top_rank"] >= 0:
        ops.append(dist.P2POp(dist.irecv, t_top, p["recv_top_rank"]))
        ops.append(dist.P2POp(dist.isend, torch.from_numpy(G_band[p["send_top_row0"]:p["send_top_row0"] + h].copy()),
                              p["recv_top_rank"]))
    if p["recv_bot_rank"] >= 0:
        ops.append(dist.P2POp(dist.irecv, t_bot, p["recv_bot_rank"]))
        ops.append(dist.P2POp(dist.isend, torch.from_numpy(G_band[p["send_bot_row0"]:p["send_bot_row0"] + h].copy()),
                              p["recv_bot_rank"]))
    if ops:
        reqs = dist.batch_isend_irecv(ops)
        for r in reqs:
            r.wait()
    # A full-size grid holding only what this rank has; other rows are poison labels
    # (real-looking seeds next to every pixel, so using one changes the result).
    rng = np.random.default_rng(POISON_SEED + rank)
    yy, xx = np.mgrid[0:N, 0:N]
    poison = ((np.clip(yy + rng.integers(-1, 2, size=(N, N)), 0, N - 1).astype(np.uint32) << 16)
              | np.clip(xx + rng.integers(-1, 2, size=(N, N)), 0, N - 1).astype(np.uint32))
    full = poison.astype(np.uint32)
    full[rank * B:(rank + 1) * B] = G_band
    if p["recv_top_rank"] >= 0:
        full[p["top_row0"]:p["top_row0"] + h] = top
    if p["recv_bot_rank"] >= 0:
        full[p["bot_row0"]:p["bot_row0"] + h] = bot
    out = oracle.jump_pass(full, k)
    return out[rank * B:(rank + 1) * B].copy()


def _worker(rank, world, port, N, s, frames, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        import synth
        import paper_2209_00117_b200 as vd
        B = N // world
        xy = synth.uniform_seeds(N, s, rng_seed=31)
        G = oracle.init(N, xy)[rank * B:(rank + 1) * B].copy()
        for k in vd.vd_schedule_jfa(N):
            G = _band_pass(G, k, N, world, rank, vd.vd_halo_plan, oracle)
        hashes = [G]
        for f in range(frames):  # dJFA: remap/stamp are per-pixel, only the passes exchange
            disp = synth.displacements(s, 2, f, rng_seed=31)
            new = oracle.move(N, xy, disp)
            old_l = (xy[1::2].astype(np.uint32) << 16) | xy[0::2]
            new_l = (new[1::2].astype(np.uint32) << 16) | new[0::2]
            fwd = {}
            for o, n_ in zip(old_l.tolist(), new_l.tolist()):
                fwd[o] = min(fwd.get(o, 0xFFFFFFFF), n_)
            G = np.vectorize(lambda c: fwd[int(c)], otypes=[np.uint32])(G)
            for c in new_l.tolist():
                y, x = c >> 16, c & 0xFFFF
                if rank * B <= y < (rank + 1) * B:
                    G[y - rank * B, x] = c
            for k in vd.vd_schedule_djfa(N, s, 2):
                G = _band_pass(G, k, N, world, rank, vd.vd_halo_plan, oracle)
            xy = new
            hashes.append(G)
        q.put((rank, [h.copy() for h in hashes]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_band_sharded_jfa_djfa_equals_unsharded(world):
    import oracle
    import synth
    from paper_2209_00117_b200 import build
    build.build()
    N, s, frames = 32, 12, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, N, s, frames, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    xy = synth.uniform_seeds(N, s, rng_seed=31)
    ref = [oracle.jfa(N, xy)]
    G = ref[0]
    for f in range(frames):
        disp = synth.displacements(s, 2, f, rng_seed=31)
        G, xy, _ = oracle.djfa_step(N, xy, disp, 2, G)
        ref.append(G)
    for i, R in enumerate(ref):
        assembled = np.concatenate([got[r][i] for r in range(world)], axis=0)
        assert np.array_equal(assembled, R), i
