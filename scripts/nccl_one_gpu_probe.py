"""Probe: can two ranks of one NCCL communicator share one GPU?  (NCCL normally refuses with
"Duplicate GPU detected".)  Runs libvd's world-2 NCCL halo path on cuda:0 from two processes and
compares every rank's band with the oracle.  Prints one line per rank and exits 0 either way."""
import multiprocessing as mp
import os
import socket
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def worker(rank, world, port, q):
    import numpy as np
    import torch.distributed as dist
    import oracle
    import synth
    os.environ["MASTER_ADDR"], os.environ["MASTER_PORT"] = "127.0.0.1", str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2209_00117_b200 as m
    m.load_library()
    ids = [m.vd_nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(ids, src=0)
    N, s = 512, 1024
    xy = synth.uniform_seeds(N, s, rng_seed=3)
    B = N // world
    try:
        d = m.VoronoiDiagram(N, xy, device=0, rank=rank, world=world, nccl_id=ids[0])
        d.jfa()
        ref = oracle.jfa(N, xy)
        ok = [bool(np.array_equal(d.labels(), ref[rank * B:(rank + 1) * B]))]
        for f in range(2):
            disp = synth.displacements(s, 2, f, rng_seed=3)
            d.djfa_step(disp, 2)
            ref, xy, _ = oracle.djfa_step(N, xy, disp, 2, ref)
            ok.append(bool(np.array_equal(d.labels(), ref[rank * B:(rank + 1) * B])))
        q.put((rank, "ran", ok))
        d.close()
    except Exception as e:  # noqa: BLE001
        q.put((rank, "error", str(e)[:300]))


if __name__ == "__main__":
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    try:
        for _ in ps:
            print(q.get(timeout=180), flush=True)
    except Exception as e:  # noqa: BLE001
        print("timeout / no result:", e, flush=True)
    for p in ps:
        p.join(timeout=30)
        if p.is_alive():
            p.kill()
