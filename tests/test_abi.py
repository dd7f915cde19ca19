"""C-ABI checks that need no GPU: libvd loads, exports every symbol include/vd.h declares,
its host-only helpers (schedules, halo plan) agree with the oracle / with the geometry,
and argument errors are reported before any device work."""
import os
import re

import numpy as np
import pytest

import oracle
import paper_2209_00117_b200 as vd

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_2209_00117_b200 import build
    build.build()
    return vd.load_library()


def _declared_functions():
    text = open(os.path.join(ROOT, "include", "vd.h"), encoding="utf-8").read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(vd_[a-z_0-9]+)\s*\(", text)))


def test_exports_every_declared_symbol(lib):
    names = _declared_functions()
    assert len(names) >= 20
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(vd.EXPORTED_SYMBOLS)


@pytest.mark.parametrize("N", [2, 3, 5, 8, 13, 64, 100, 1000, 1024, 4096, 16384, 65536])
def test_jfa_schedule_matches_oracle(lib, N):
    for extras in (0, 1, 2):
        assert vd.vd_schedule_jfa(N, extras) == oracle.jfa_schedule(N, extras)


def test_djfa_schedule_matches_oracle(lib):
    rng = np.random.default_rng(5)
    for _ in range(3000):
        N = int(rng.integers(2, 65537))
        s = int(rng.integers(1, min(N * N, 2**30) + 1))
        d = int(rng.integers(0, 5000))
        e = int(rng.integers(0, 3))
        assert vd.vd_schedule_djfa(N, s, d, e) == oracle.djfa_schedule(N, s, d, e), (N, s, d, e)
    for N, s, d in ((1000, 100, 5), (1024, 4096, 4), (64, 1, 1), (16384, 2**20, 1), (65536, 2**24, 1)):
        assert vd.vd_schedule_djfa(N, s, d) == oracle.djfa_schedule(N, s, d)


@pytest.mark.parametrize("N,G", [(64, 2), (64, 4), (64, 8), (1024, 8), (16384, 8), (65536, 8)])
def test_halo_plan_covers_exactly_the_needed_rows(lib, N, G):
    # For each rank and every step k of JFA: the rows a band needs (y +- k inside the grid,
    # outside the band) are exactly the halo rows, and they come from the ranks that own
    # them, at the row offsets the plan sends.
    B = N // G
    for k in oracle.jfa_schedule(N):
        for g in range(G):
            p = vd.vd_halo_plan(N, G, g, k)
            need = set()
            for y in range(g * B, (g + 1) * B):
                for r in (y - k, y + k):
                    if 0 <= r < N and not (g * B <= r < (g + 1) * B):
                        need.add(r)
            have = set()
            if p["recv_top_rank"] >= 0:
                src = p["recv_top_rank"]
                rows = range(p["top_row0"], p["top_row0"] + p["halo_rows"])
                have |= set(rows)
                # the sender's rows [B-h, B) are these global rows
                assert list(rows) == [src * B + r for r in range(B - p["halo_rows"], B)]
                q = vd.vd_halo_plan(N, G, src, k)
                assert q["recv_bot_rank"] == g and q["send_bot_row0"] == B - p["halo_rows"]
            if p["recv_bot_rank"] >= 0:
                src = p["recv_bot_rank"]
                rows = range(p["bot_row0"], p["bot_row0"] + p["halo_rows"])
                have |= set(rows)
                assert list(rows) == [src * B + r for r in range(0, p["halo_rows"])]
                q = vd.vd_halo_plan(N, G, src, k)
                assert q["recv_top_rank"] == g and q["send_top_row0"] == 0
            assert need <= have, (k, g)
            # nothing superfluous beyond the h rows per side
            assert len(have) <= 2 * min(k, B)


def test_create_argument_errors_need_no_gpu(lib):
    with pytest.raises(vd.VDError) as e:
        vd.vd_create(1, np.array([0, 0], dtype=np.uint16))
    assert e.value.status == vd.VD_ERR_ARG
    with pytest.raises(vd.VDError) as e:
        vd.vd_create(8, np.array([8, 0], dtype=np.uint16))  # x = N: outside the grid
    assert e.value.status == vd.VD_ERR_RANGE
    with pytest.raises(vd.VDError) as e:
        vd.vd_create(65536, np.array([65535, 65535], dtype=np.uint16))  # reserved pixel (R-4)
    assert e.value.status == vd.VD_ERR_RANGE
    with pytest.raises(vd.VDError) as e:  # sharding needs a power-of-two N
        vd.vd_create(1000, np.array([1, 1], dtype=np.uint16), virtual_shards=2)
    assert e.value.status == vd.VD_ERR_ARG
    with pytest.raises(vd.VDError) as e:  # world > 1 needs an NCCL id
        vd.vd_create(64, np.array([1, 1], dtype=np.uint16), rank=0, world=2)
    assert e.value.status == vd.VD_ERR_ARG


def test_null_handle_calls_are_errors(lib):
    assert lib.vd_jfa(None) == vd.VD_ERR_ARG
    assert lib.vd_synchronize(None) == vd.VD_ERR_ARG
    lib.vd_destroy(None)  # NULL-safe
    assert vd.vd_status_str(vd.VD_ERR_STATE) == "VD_ERR_STATE"
