"""Multi-GPU row bands across processes: one process per GPU,
each holding one band of N/world rows, halos exchanged per pass over NCCL send/recv or
pushed by the pass kernels into the neighbours' halo buffers (CUDA IPC peer memory across
devices).  Every rank's band must equal the same rows of the CPU oracle, every frame, and
the all-reduced label hash must equal the oracle's hash of the whole diagram.

The paper's waves are pixel-parallel ("parallel GPU threads ... mapped to the VD
pixels"), so a band split cannot change any pixel's result; these tests check that the
transport delivers exactly the rows the passes need.

They need >= 2 visible GPUs: NCCL refuses two ranks of one communicator on one device.
(The one-GPU stand-ins are the virtual-shard and same-device IPC tests in
test_gpu_parity.py and the gloo band test in test_band_gloo.py.)
"""
import multiprocessing as mp
import socket

import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _need_two_gpus():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    if torch.cuda.device_count() < 2:
        pytest.skip(f"needs >= 2 GPUs (found {torch.cuda.device_count()}); NCCL cannot put two ranks on one device")


def _free_port():
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def _band_worker(rank, world, port, N, s, dmax, frames, halo, q):
    import os
    import torch.distributed as dist
    os.environ["MASTER_ADDR"], os.environ["MASTER_PORT"] = "127.0.0.1", str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2209_00117_b200 as m
    m.load_library()
    dev = rank % torch.cuda.device_count()
    torch.cuda.set_device(dev)
    ids = [m.vd_nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(ids, src=0)
    xy = synth.uniform_seeds(N, s, rng_seed=11)
    B = N // world
    rows = slice(rank * B, (rank + 1) * B)
    d = m.VoronoiDiagram(N, xy, device=dev, rank=rank, world=world, nccl_id=ids[0], peer_halos=halo == "peer")
    if halo == "peer":
        d.attach_peers()
    d.jfa()
    ref = oracle.jfa(N, xy)
    res = [bool(np.array_equal(d.labels(), ref[rows])), d.label_hash() == oracle.label_hash(ref)]
    for f in range(frames):
        disp = synth.displacements(s, dmax, f, rng_seed=11)
        d.djfa_step(disp, dmax)
        ref, xy, _ = oracle.djfa_step(N, xy, disp, dmax, ref)
        res += [bool(np.array_equal(d.labels(), ref[rows])), d.label_hash() == oracle.label_hash(ref)]
    q.put((rank, res, d.peer_timed_out()))
    dist.barrier()
    d.close()
    dist.destroy_process_group()


def _run(world, halo, N=1024, s=4096, dmax=2, frames=3):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_band_worker, args=(r, world, port, N, s, dmax, frames, halo, q)) for r in range(world)]
    for p in ps:
        p.start()
    try:
        out = sorted(q.get(timeout=600) for _ in ps)
    finally:
        for p in ps:
            p.join(timeout=120)
            if p.is_alive():
                p.kill()
    assert [r for r, _, _ in out] == list(range(world))
    for r, res, timed_out in out:
        assert all(res), (r, res)
        assert not timed_out, r


@pytest.mark.parametrize("world", [2, 4, 8])
def test_nccl_bands_bit_exact(world):
    _need_two_gpus()
    if torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs")
    _run(world, "nccl")


@pytest.mark.parametrize("world", [2, 4, 8])
def test_peer_halos_across_devices_bit_exact(world):
    # fused halo push into the neighbours' buffers over NVLink (cross-device IPC), with
    # release/acquire flags; NCCL only for JFA's steps with 2k >= band rows
    _need_two_gpus()
    if torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs")
    _run(world, "peer")
