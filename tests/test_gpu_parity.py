"""GPU parity: libvd (CUDA, through the C ABI) against the CPU oracle, bit-exact.

Labels are integers, so the bar is element-by-element equality (north star: "GPU
JFA/dJFA label maps must match the CPU JFA/dJFA bit-exactly on the same host-generated
seeds and displacement streams").  Inputs: synth (seeded, shared by both sides).
"""
import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

EMPTY = 0xFFFFFFFF


@pytest.fixture(scope="module")
def vd():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    import paper_2209_00117_b200 as m
    from paper_2209_00117_b200 import build
    build.build()
    m.load_library()
    return m


def _jfa_gpu(vd, N, xy, **cfg):
    d = vd.VoronoiDiagram(N, xy, **cfg)
    d.jfa()
    return d


SMALL = [(2, 1), (2, 3), (3, 2), (4, 2), (5, 3), (8, 5), (13, 7), (16, 16), (31, 9), (64, 16), (100, 40),
         (127, 300), (128, 128), (257, 50), (1000, 50), (1024, 1024), (1031, 2000)]


@pytest.mark.parametrize("N,s", SMALL)
def test_jfa_bit_exact(vd, N, s):
    xy = synth.uniform_seeds(N, s, rng_seed=N + s)
    d = _jfa_gpu(vd, N, xy)
    G = d.labels()
    assert np.array_equal(G, oracle.jfa(N, xy))
    assert d.last_passes() == len(oracle.jfa_schedule(N))


# Multiples of 512 that 4k does not divide for some k >= 256: the shared-term kernel's last group
# of 4k columns is partial (outputs beyond the grid not stored, slots beyond it duplicated), and
# where k does not divide N the rows are staged span by span instead of by one tensor copy.
@pytest.mark.parametrize("N,s", [(1536, 300), (2560, 700), (3584, 1000), (6656, 5000)])
def test_jfa_partial_span_groups_bit_exact(vd, N, s):
    xy = synth.uniform_seeds(N, s, rng_seed=N + 7)
    d = _jfa_gpu(vd, N, xy)
    assert np.array_equal(d.labels(), oracle.jfa(N, xy))
    rng = np.random.default_rng(N)
    G = ((rng.integers(0, N, (N, N)) << 16) | rng.integers(0, N, (N, N))).astype(np.uint32)
    for k in (256, 512, 1024):
        if 4 * k <= N:
            d.set_labels(G)
            d.jump_pass(k)
            assert np.array_equal(d.labels(), oracle.jump_pass(G, k)), k
    d.close()


@pytest.mark.parametrize("extras", [1, 2])
def test_jfa_extras_bit_exact(vd, extras):
    N, s = 200, 60
    xy = synth.uniform_seeds(N, s, rng_seed=3)
    d = _jfa_gpu(vd, N, xy, extra_passes=extras)
    assert np.array_equal(d.labels(), oracle.jfa(N, xy, extras))


@pytest.mark.parametrize("N", [2, 3, 5, 8, 13, 64, 100, 257, 1024, 1031, 2048, 2051])
def test_single_pass_random_states_bit_exact(vd, N):
    # One pass from arbitrary label maps (seeds and EMPTY mixed, not only reachable
    # states), for every k regime: 1, 2, multiples of 4, >= 512 and non-powers of two
    # (generic kernel).  N = 1024 / 2048: the shared-term kernel (jump_pass_sk) at every step
    # it takes -- adjacent (k <= 2), compile-time stride (4 .. 128), staged spans (>= 256) and
    # whole residue classes per CTA (N/k rows fit the stage).
    rng = np.random.default_rng(N)
    s = min(N * N, 40)
    xy = synth.uniform_seeds(N, s, rng_seed=N)
    labels = np.array([oracle.pack(int(xy[2 * i]), int(xy[2 * i + 1])) for i in range(s)] + [EMPTY], dtype=np.uint32)
    d = vd.VoronoiDiagram(N, xy)
    for trial in range(3):
        G = labels[rng.integers(0, len(labels), size=(N, N))]
        for k in sorted({1, 2, 3, 4, 5, 8, 16, 32, 64, 128, 256, 512, 1024} | {max(1, N // 2)}):
            d.set_labels(G)
            d.jump_pass(k)
            assert np.array_equal(d.labels(), oracle.jump_pass(G, k)), (trial, k)


@pytest.mark.parametrize("case", ["one_seed_corner", "all_colocated", "corners", "every_pixel", "row", "diag"])
def test_jfa_edge_cases(vd, case):
    N = 37
    if case == "one_seed_corner":
        xy = np.array([N - 1, N - 1], dtype=np.uint16)
    elif case == "all_colocated":
        xy = np.array([5, 7] * 20, dtype=np.uint16)
    elif case == "corners":
        xy = np.array([0, 0, N - 1, 0, 0, N - 1, N - 1, N - 1], dtype=np.uint16)
    elif case == "every_pixel":
        yy, xx = np.mgrid[0:N, 0:N]
        xy = np.stack([xx.ravel(), yy.ravel()], 1).astype(np.uint16).ravel()
    elif case == "row":
        xy = np.array([[x, 3] for x in range(0, N, 3)], dtype=np.uint16).ravel()
    else:
        xy = np.array([[i, i] for i in range(N)], dtype=np.uint16).ravel()
    d = _jfa_gpu(vd, N, xy)
    assert np.array_equal(d.labels(), oracle.jfa(N, xy))


def _djfa_run(vd, N, s, dmax, frames, seed, **cfg):
    xy = synth.uniform_seeds(N, s, rng_seed=seed)
    d = _jfa_gpu(vd, N, xy, **cfg)
    G = oracle.jfa(N, xy)
    assert np.array_equal(d.labels(), G)
    for f in range(frames):
        disp = synth.displacements(s, dmax, f, rng_seed=seed)
        d.djfa_step(disp, dmax)
        G, xy, n = oracle.djfa_step(N, xy, disp, dmax, G)
        assert d.last_passes() == n
        assert np.array_equal(d.seeds(), xy), f
        assert np.array_equal(d.labels(), G), f
    return d, G, xy


def test_djfa_c1_all_frames(vd):
    # BASELINE.json configs[0]: 64x64, 16 uniform seeds, 10 dJFA time steps
    _djfa_run(vd, 64, 16, 1, 10, 2209)


@pytest.mark.parametrize("N,s,dmax", [(256, 256, 1), (256, 256, 4), (300, 100, 7), (1024, 1024, 1),
                                      (1024, 4096, 64), (512, 2048, 300), (64, 4096, 2)])
def test_djfa_bit_exact(vd, N, s, dmax):
    _djfa_run(vd, N, s, dmax, 4, N * 7 + s)


def test_djfa_c2_all_frames(vd):
    # BASELINE.json configs[1]: 1024x1024, 1024 seeds, +-1 px moves, all 100 steps, every
    # pixel of every frame compared
    _djfa_run(vd, 1024, 1024, 1, 100, 2209)


def test_djfa_colocated_split_golden(vd):
    # tests/golden/djfa_colocated_split.txt (hand-worked; pins R-9's co-location rule in the
    # oracle): the GPU step from the same previous diagram gives the fixture's labels and
    # the oracle's whole diagram.
    import golden_io
    fx = golden_io.load_seed_runs("djfa_colocated_split.txt")
    N, old, disp = fx["N"], fx["old_xy"], fx["disp_xy"]
    prev = oracle.exact_brute(N, old)
    d = vd.VoronoiDiagram(N, old)
    d.set_labels(prev)
    d.djfa_step(disp, fx["d_max"])
    L = d.labels()
    G, _, _ = oracle.djfa_step(N, old, disp, fx["d_max"], prev)
    assert np.array_equal(L, G)
    for px, py, lab in fx["expect"]:
        assert int(L[py, px]) == lab, (px, py)


def test_djfa_clamp_at_borders(vd):
    # displacements far larger than the grid: every seed is clamped to an edge
    N, s = 64, 40
    xy = synth.uniform_seeds(N, s, rng_seed=1)
    d = _jfa_gpu(vd, N, xy)
    G = oracle.jfa(N, xy)
    for f in range(3):
        disp = synth.displacements(s, 200, f, rng_seed=1)
        d.djfa_step(disp, 200)
        G, xy, _ = oracle.djfa_step(N, xy, disp, 200, G)
        assert np.array_equal(d.labels(), G)


def test_djfa_device_displacements(vd):
    N, s = 512, 512
    xy = synth.uniform_seeds(N, s, rng_seed=4)
    d = _jfa_gpu(vd, N, xy)
    G = oracle.jfa(N, xy)
    for f in range(3):
        disp = synth.displacements(s, 3, f, rng_seed=4)
        d.djfa_step(torch.from_numpy(disp).cuda(), 3)
        G, xy, _ = oracle.djfa_step(N, xy, disp, 3, G)
        assert np.array_equal(d.labels(), G)


def test_djfa_before_jfa_is_state_error(vd):
    d = vd.VoronoiDiagram(16, np.array([1, 1, 9, 9], dtype=np.uint16))
    with pytest.raises(vd.VDError) as e:
        d.djfa_step(np.zeros(4, dtype=np.int16), 1)
    assert e.value.status == vd.VD_ERR_STATE
    d.jfa()
    d.move_seeds(np.array([1, 0, 0, 1], dtype=np.int16))  # diagram now stale
    with pytest.raises(vd.VDError):
        d.djfa_step(np.zeros(4, dtype=np.int16), 1)


@pytest.mark.parametrize("G", [2, 4, 8])
def test_virtual_shards_bit_identical(vd, G):
    # The row-band path (halo plan + banded kernel) on one GPU: identical to 1 band and to
    # the oracle, for JFA (k up to N/2 >= band height) and dJFA.
    N, s, dmax = 256, 200, 3
    xy = synth.uniform_seeds(N, s, rng_seed=G)
    one = _jfa_gpu(vd, N, xy)
    many = _jfa_gpu(vd, N, xy, virtual_shards=G)
    ref = oracle.jfa(N, xy)
    assert np.array_equal(many.labels(), ref) and np.array_equal(one.labels(), ref)
    assert many.label_hash() == one.label_hash() == oracle.label_hash(ref)
    for f in range(3):
        disp = synth.displacements(s, dmax, f, rng_seed=G)
        one.djfa_step(disp, dmax)
        many.djfa_step(disp, dmax)
        ref, xy, _ = oracle.djfa_step(N, xy, disp, dmax, ref)
        assert np.array_equal(many.labels(), ref), f
        assert many.label_hash() == one.label_hash() == oracle.label_hash(ref)
        assert many.match_count(many) == N * N


def test_similarity_and_hash_match_oracle(vd):
    N, s = 300, 77
    xy = synth.uniform_seeds(N, s, rng_seed=12)
    a = _jfa_gpu(vd, N, xy)
    b = vd.VoronoiDiagram(N, xy)
    b.jfa()
    disp = synth.displacements(s, 5, 0, rng_seed=12)
    b.djfa_step(disp, 5)
    A, B = a.labels(), b.labels()
    pct, m = vd.vd_similarity(a.h, b.h)
    assert m == oracle.match_count(A, B)
    assert pct == pytest.approx(100.0 * m / (N * N), abs=1e-12)
    E = oracle.exact(N, xy)
    pct_h, m_h = vd.vd_similarity_host(a.h, E)
    assert m_h == oracle.match_count(A, E)
    assert a.label_hash() == oracle.label_hash(A)
    assert b.label_hash() == oracle.label_hash(B)


@pytest.mark.parametrize("dmax", [1, 64])
def test_c3_full_size_bit_exact(vd, dmax):
    # BASELINE.json configs[2]: 4096x4096, 65,536 seeds; JFA + 10 dJFA frames at move radius
    # 1 (6 passes) and 64 (7 passes: d_max sets delta_1), every pixel of every frame
    # compared.
    _djfa_run(vd, 4096, 65536, dmax, 10, 2209 + dmax)


def test_c3_move_radius_sweep_bit_exact(vd):
    # configs[2]'s sweep over the move radius: the delta schedule grows with d_max
    N, s = 4096, 65536
    for dmax in (8, 64, 512):
        d, G, xy = _djfa_run(vd, N, s, dmax, 1, 100 + dmax)
        assert d.last_passes() == len(oracle.djfa_schedule(N, s, dmax))


@pytest.mark.slow
def test_c4_bench_config_full_grid(vd):
    # BASELINE.json configs[3] at the size bench.py times (16384^2, 2^20 seeds, +-1 px), in
    # the same launch configuration: JFA bootstrap + 3 dJFA frames, every pixel of every frame
    # compared with the oracle (np.array_equal on the host), plus properties that hold at any
    # size.
    N, s = 16384, 1 << 20
    xy = synth.uniform_seeds(N, s, rng_seed=2209)
    d = _jfa_gpu(vd, N, xy)
    G = oracle.jfa(N, xy)
    assert np.array_equal(d.labels(), G), "JFA bootstrap"
    for f in range(3):
        disp = synth.displacements(s, 1, f, rng_seed=2209)
        d.djfa_step(disp, 1)
        G, xy, n = oracle.djfa_step(N, xy, disp, 1, G, inplace=True)
        assert d.last_passes() == n == 6
        assert d.last_packed_passes() == 6  # the bench's regime: every delta pass on the packed walk
        L = d.labels()
        assert np.array_equal(L, G), f
    assert d.label_hash() == oracle.label_hash(G)
    # every seed pixel holds its own label
    lx, ly = xy[0::2].astype(np.int64), xy[1::2].astype(np.int64)
    assert np.array_equal(L[ly, lx], (ly.astype(np.uint32) << 16) | lx.astype(np.uint32))


@pytest.mark.slow
def test_c5_jfa_and_djfa_frames_full_grid(vd):
    # BASELINE.json configs[4]: 65536^2 grid, 2^24 uniform seeds, +-1 px moves, one GPU, the
    # launch configuration bench.py --config C5 times: JFA (64-bit kernel while EMPTY remains,
    # then the large-step and windowed kernels) + 2 dJFA frames (move_fwd with a 16-GiB fwd
    # map, remap, reset_stamp, windowed packed passes), every pixel compared with the oracle.
    # Host memory: the oracle's map (16 GiB) + its fwd and pass buffers (32 GiB) + the GPU
    # map (16 GiB).
    import time
    N, s = 65536, 1 << 24
    xy = synth.uniform_seeds(N, s, rng_seed=2209)
    t0 = time.perf_counter()
    d = _jfa_gpu(vd, N, xy)
    L = d.labels()
    t1 = time.perf_counter()
    G = oracle.jfa(N, xy)
    t2 = time.perf_counter()
    assert np.array_equal(L, G), "JFA bootstrap"
    print(f"C5 JFA: gpu+download {t1 - t0:.1f} s, oracle {t2 - t1:.1f} s, equal", flush=True)
    del L
    for f in range(2):
        disp = synth.displacements(s, 1, f, rng_seed=2209)
        t0 = time.perf_counter()
        d.djfa_step(disp, 1)
        L = d.labels()
        t1 = time.perf_counter()
        G, xy, n = oracle.djfa_step(N, xy, disp, 1, G, inplace=True)
        t2 = time.perf_counter()
        assert d.last_passes() == n == 6
        assert np.array_equal(d.seeds(), xy), f
        assert np.array_equal(L, G), f
        print(f"C5 dJFA frame {f}: gpu+download {t1 - t0:.1f} s, oracle {t2 - t1:.1f} s, equal, "
              f"packed passes {d.last_packed_passes()}", flush=True)
        del L
    d.close()


@pytest.mark.parametrize("N", [16384, 20000])
def test_empty_never_wins_at_large_n(vd, N):
    # R-21 / R-4: a single seed in the far corner; every JFA pass compares EMPTY (key +inf)
    # against that seed at the largest distances the grid allows.  One-seed JFA is exact,
    # so every pixel must end with the seed.  16384 is the largest N of the fast kernel's
    # EMPTY variant (virtual far seed), 20000 runs the 64-bit kernel.
    xy = np.array([N - 1, N - 1], dtype=np.uint16)
    d = _jfa_gpu(vd, N, xy)
    L = d.labels()
    assert (L == oracle.pack(N - 1, N - 1)).all()
    xy = np.array([0, 0], dtype=np.uint16)
    d2 = _jfa_gpu(vd, N, xy)
    assert d2.match_count(d2) == N * N
    assert (d2.labels() == 0).all()


# ---------------------------------------------------------------- NEXT-2 variants
# dJFAm (Manhattan) and Von Neumann waves, bit-exact
# against the oracle's variant functions (pinned in tests/test_oracle_variants.py).

@pytest.mark.parametrize("N", [5, 64, 257, 1024, 1031])
@pytest.mark.parametrize("metric,vn", [("manhattan", False), ("euclid", True), ("manhattan", True)])
def test_single_pass_variants_bit_exact(vd, N, metric, vn):
    rng = np.random.default_rng(N + 7)
    s = min(N * N, 40)
    xy = synth.uniform_seeds(N, s, rng_seed=N)
    labels = np.array([oracle.pack(int(xy[2 * i]), int(xy[2 * i + 1])) for i in range(s)] + [EMPTY], dtype=np.uint32)
    d = vd.VoronoiDiagram(N, xy, metric=metric)
    G = labels[rng.integers(0, len(labels), size=(N, N))]
    for k in sorted({1, 2, 3, 4, 8, 64, 512} | {max(1, N // 2)}):
        d.set_labels(G)
        d.jump_pass(k, von_neumann=vn)
        assert np.array_equal(d.labels(), oracle.jump_pass(G, k, metric=metric, vn=vn)), k


@pytest.mark.parametrize("N,s", [(64, 16), (300, 100), (1024, 1024)])
def test_jfa_variants_bit_exact(vd, N, s):
    xy = synth.uniform_seeds(N, s, rng_seed=N * 3)
    m = _jfa_gpu(vd, N, xy, metric="manhattan")
    assert np.array_equal(m.labels(), oracle.jfa(N, xy, metric="manhattan"))
    v = _jfa_gpu(vd, N, xy, jfa_vn_waves=99)  # Von Neumann-only JFA (Fig. 5): may stay incomplete
    assert np.array_equal(v.labels(), oracle.jfa(N, xy, vn_waves=99))


@pytest.mark.parametrize("metric,vn_waves", [("manhattan", 0), ("euclid", 2), ("manhattan", 2)])
@pytest.mark.parametrize("N,s,dmax,G", [(64, 16, 1, 0), (1024, 1024, 2, 0), (512, 2048, 3, 4)])
def test_djfa_variants_bit_exact(vd, metric, vn_waves, N, s, dmax, G):
    xy = synth.uniform_seeds(N, s, rng_seed=N + s)
    d = _jfa_gpu(vd, N, xy, metric=metric, vn_waves=vn_waves, virtual_shards=G)
    ref = oracle.jfa(N, xy, metric=metric)
    assert np.array_equal(d.labels(), ref)
    for f in range(3):
        disp = synth.displacements(s, dmax, f, rng_seed=N)
        d.djfa_step(disp, dmax)
        ref, xy, _ = oracle.djfa_step(N, xy, disp, dmax, ref, metric=metric, vn_waves=vn_waves)
        assert np.array_equal(d.labels(), ref), f


# ---------------------------------------------------------------- NEXT-4

@pytest.mark.parametrize("N,s,metric", [(11, 1, "euclid"), (64, 16, "euclid"), (100, 7, "manhattan"), (257, 60, "euclid")])
def test_stf_bit_exact(vd, N, s, metric):
    # Standard Flooding: k = 1 passes until the grid is fully flooded (R-22)
    xy = np.array([5, 5], dtype=np.uint16) if N == 11 else synth.uniform_seeds(N, s, rng_seed=N)
    d = vd.VoronoiDiagram(N, xy, metric=metric)
    n = d.stf()
    G, n_ref = oracle.stf(N, xy, metric=metric)
    assert n == n_ref and np.array_equal(d.labels(), G)
    if N == 11:
        assert n == 5  # P:76 "StF fulfills its purpose in 5 iterations"


def test_paper_sample_run_1000x1000_50_seeds(vd):
    # Fig. 6: "A 100 step simulation of 50 seeds on a grid of 1000x1000 pixels".
    # Non-power-of-two grid; sparse seeds make delta_1 = k_1 ("behave very much like
    # JFA").  All 100 frames bit-exact against the oracle.
    N, s, dmax = 1000, 50, 4
    xy = synth.uniform_seeds(N, s, rng_seed=6)
    d = _jfa_gpu(vd, N, xy)
    G = oracle.jfa(N, xy)
    for f in range(100):
        disp = synth.displacements(s, dmax, f, rng_seed=6)
        d.djfa_step(disp, dmax)
        G, xy, n = oracle.djfa_step(N, xy, disp, dmax, G)
        assert n == len(oracle.jfa_schedule(N))
        if f % 10 == 9:
            assert d.label_hash() == oracle.label_hash(G), f
    assert np.array_equal(d.labels(), G)


# ---------------------------------------------------------------- windowed fast pass (REL)
# For 32768 < N <= 65536 the fast kernel works in 16-bit coordinates relative to a
# 32768-wide window around each walk; a walk that meets a label outside its window is
# recomputed with 64-bit keys.  Both halves are checked against the oracle over the whole
# grid: jittered maps (labels near their pixel, the converged-dJFA case) sprinkled with
# far labels (forcing the exact recomputation), and fully random maps (every walk falls back).

def _jittered_map(N, jitter, far, seed):
    rng = np.random.default_rng(seed)
    G = np.empty((N, N), dtype=np.uint32)
    x = np.arange(N, dtype=np.int64)
    for y0 in range(0, N, 2048):
        y1 = min(N, y0 + 2048)
        ys = np.arange(y0, y1, dtype=np.int64)[:, None]
        lx = np.clip(x[None, :] + rng.integers(-jitter, jitter + 1, size=(y1 - y0, N)), 0, N - 1)
        ly = np.clip(ys + rng.integers(-jitter, jitter + 1, size=(y1 - y0, N)), 0, N - 1)
        G[y0:y1] = ((ly << 16) | lx).astype(np.uint32)
    n = far
    py, px = rng.integers(0, N, n), rng.integers(0, N, n)
    G[py, px] = ((rng.integers(0, N, n) << 16) | rng.integers(0, N, n)).astype(np.uint32)
    return G


@pytest.fixture(scope="module")
def rel_grid():
    N = 36000  # > 32768 (windowed path), ragged against the 512-column CTA tile
    return N, _jittered_map(N, 40, 3000, 77)


@pytest.mark.slow
@pytest.mark.parametrize("k,metric,vn", [(1, "euclid", False), (2, "euclid", False), (4, "euclid", False),
                                         (64, "euclid", False), (4096, "euclid", False),
                                         (8, "manhattan", False), (16, "euclid", True)])
def test_windowed_pass_bit_exact(vd, rel_grid, k, metric, vn):
    N, G = rel_grid
    d = vd.VoronoiDiagram(N, np.array([0, 0], dtype=np.uint16), metric=metric)
    d.set_labels(G)
    d.jump_pass(k, von_neumann=vn)
    got = d.labels()
    d.close()
    want = oracle.jump_pass(G, k, metric=metric, vn=vn)
    bad = np.argwhere(got != want)
    assert bad.size == 0, (k, bad[:5].tolist(), len(bad))


@pytest.mark.slow
def test_windowed_pass_all_far_labels(vd):
    N, k = 33000, 8
    rng = np.random.default_rng(5)
    G = ((rng.integers(0, N, (N, N), dtype=np.uint32) << 16) | rng.integers(0, N, (N, N), dtype=np.uint32))
    d = vd.VoronoiDiagram(N, np.array([0, 0], dtype=np.uint16))
    d.set_labels(G)
    d.jump_pass(k)
    got = d.labels()
    d.close()
    assert np.array_equal(got, oracle.jump_pass(G, k))


@pytest.mark.slow
@pytest.mark.parametrize("k", [1, 16, 2048])
def test_windowed_pass_with_empty_bit_exact(vd, rel_grid, k):
    # Maps with EMPTY beyond N = 16384 take the 64-bit kernel (any k).
    N, G0 = rel_grid
    G = G0.copy()
    rng = np.random.default_rng(k)
    G[rng.integers(0, N, 5000), rng.integers(0, N, 5000)] = EMPTY
    G[1000:1003] = EMPTY  # whole empty rows
    d = vd.VoronoiDiagram(N, np.array([0, 0], dtype=np.uint16))
    d.set_labels(G)
    d.jump_pass(k)
    got = d.labels()
    d.close()
    assert np.array_equal(got, oracle.jump_pass(G, k))


@pytest.mark.slow
def test_djfa_beyond_32768_sparse_seeds_bit_exact(vd):
    # A dJFA frame on a grid beyond 32768 (33280 = 65 * 512) with sparse seeds: the labels are far
    # from their pixels, so the shared-term kernel's small steps take its exact 64-bit walk (X64),
    # and the large steps the windowed / 64-bit kernels.  Every pixel against the oracle.
    N, s, dmax = 33280, 2000, 3
    xy = synth.uniform_seeds(N, s, rng_seed=33)
    d = _jfa_gpu(vd, N, xy)
    G = oracle.jfa(N, xy)
    assert np.array_equal(d.labels(), G)
    disp = synth.displacements(s, dmax, 0, rng_seed=33)
    d.djfa_step(disp, dmax)
    G, xy, n = oracle.djfa_step(N, xy, disp, dmax, G, inplace=True)
    assert d.last_passes() == n and d.last_packed_passes() == 0
    assert np.array_equal(d.labels(), G)
    d.close()


@pytest.mark.slow
@pytest.mark.parametrize("s,packed", [(1 << 22, False), (1 << 23, True)])
def test_djfa_fused_remap_beyond_32768_bit_exact(vd, s, packed):
    # dJFA frames beyond N = 32768 with the remap fused into the first pass (the new seed pixels
    # marked EMPTY by move_fwd, labels 32 bits wide): delta_1 = 64 takes the fused pass's exact
    # 64-bit walk (X64), delta_1 = 32 its packed walk.  Every pixel against the oracle.
    N, dmax = 33280, 1
    xy = synth.uniform_seeds(N, s, rng_seed=s)
    d = _jfa_gpu(vd, N, xy)
    G = oracle.jfa(N, xy)
    assert np.array_equal(d.labels(), G)
    for f in range(2):
        disp = synth.displacements(s, dmax, f, rng_seed=s)
        d.djfa_step(disp, dmax)
        G, xy, n = oracle.djfa_step(N, xy, disp, dmax, G, inplace=True)
        assert d.last_passes() == n
        if packed and f == 1:  # (frame 0 follows JFA, whose last passes may not report locality)
            assert d.last_packed_passes() == n
        assert np.array_equal(d.labels(), G), f
    d.close()


@pytest.mark.slow
@pytest.mark.parametrize("N,s", [(20000, 25000), (33000, 4000)])
def test_jfa_large_grid_bit_exact(vd, N, s):
    # JFA beyond the plain fast kernel's range: the 64-bit kernel while EMPTY remains, then
    # the EMPTY-free kernels (windowed beyond N = 32768).
    xy = synth.uniform_seeds(N, s, rng_seed=N)
    d = _jfa_gpu(vd, N, xy)
    got = d.labels()
    d.close()
    assert np.array_equal(got, oracle.jfa(N, xy))


@pytest.mark.parametrize("N", [5, 64, 257, 1024, 1031, 2051])
@pytest.mark.parametrize("metric,vn", [("euclid", False), ("manhattan", False), ("euclid", True)])
def test_single_pass_windowed_forced_bit_exact(vd, monkeypatch, N, metric, vn):
    # The windowed kernel forced at small N (test hook) on complete maps; maps with EMPTY
    # keep the EMPTY-aware kernels (the windowed one takes complete diagrams only).
    monkeypatch.setenv("VD_FORCE_WINDOWED", "1")
    rng = np.random.default_rng(N + 11)
    s = min(N * N, 40)
    xy = synth.uniform_seeds(N, s, rng_seed=N)
    labels = np.array([oracle.pack(int(xy[2 * i]), int(xy[2 * i + 1])) for i in range(s)], dtype=np.uint32)
    d = vd.VoronoiDiagram(N, xy, metric=metric)
    full = labels[rng.integers(0, len(labels), size=(N, N))]
    holes = full.copy()
    holes[rng.random((N, N)) < 0.002] = EMPTY
    for G in (full, holes):
        for k in sorted({1, 2, 4, 8, 64, 512} | {max(1, N // 2)}):
            d.set_labels(G)
            d.jump_pass(k, von_neumann=vn)
            assert np.array_equal(d.labels(), oracle.jump_pass(G, k, metric=metric, vn=vn)), (k, (G == EMPTY).any())


# The wide exact pass (jump_pass_wsk, the kernel of JFA's large steps beyond N = 32768) forced at
# small N by its test hook: its key arithmetic holds for any N <= 65536.  JFA (the virtual far
# seed of N <= 16384 included), single passes on random maps with and without EMPTY, planted ties,
# partial groups of 4k columns (1536, 2560) and ragged tensor-map cases (k not dividing N).
@pytest.mark.parametrize("N", [1024, 1536, 2048, 2560, 4096])
def test_wide_pass_forced_small_n_bit_exact(vd, monkeypatch, N):
    monkeypatch.setenv("VD_FORCE_WSK", "1")
    s = max(4, N * N // 256)
    xy = synth.uniform_seeds(N, s, rng_seed=N + 3)
    d = vd.VoronoiDiagram(N, xy)
    d.jfa()
    assert np.array_equal(d.labels(), oracle.jfa(N, xy))
    rng = np.random.default_rng(N)
    far = ((rng.integers(0, N, (N, N)) << 16) | rng.integers(0, N, (N, N))).astype(np.uint32)
    ties = far.copy()
    for y, x in rng.integers(300, N - 300, (2000, 2)):
        a = int(rng.integers(0, 40))
        ties[y, x] = far[0, 0]
        ties[y, x - 256] = oracle.pack(x + a, y + 7)   # mirror labels about column x (same cy)
        ties[y, x + 256] = oracle.pack(x - a, y + 7)
        ties[y - 256, x] = oracle.pack(x + 3, y + 4)   # d2 = 25 vs 26 with the smaller cy
        ties[y + 256, x] = oracle.pack(x + 1, y - 5)
    holes = far.copy()
    holes[rng.random((N, N)) < 0.7] = EMPTY
    holes[: N // 3, : N // 3] = EMPTY
    for G in (far, ties, holes):
        for k in (256, 512, 1024):
            if 4 * k <= N:
                d.set_labels(G)
                d.jump_pass(k)
                assert np.array_equal(d.labels(), oracle.jump_pass(G, k)), (N, k, (G == EMPTY).any())
    d.close()


@pytest.mark.parametrize("G,metric,vn", [(4, "euclid", False), (8, "manhattan", False), (2, "euclid", True)])
def test_virtual_shards_single_pass_bit_exact(vd, G, metric, vn):
    # Sharded passes with the halo exchange overlapped (interior rows, then the two edge
    # strips once the halos landed; 2k < band) and not (2k >= band), on arbitrary maps with
    # EMPTY: fast kernel for powers of two, the 64-bit one otherwise.
    N = 2048
    rng = np.random.default_rng(G)
    s = 60
    xy = synth.uniform_seeds(N, s, rng_seed=G)
    labels = np.array([oracle.pack(int(xy[2 * i]), int(xy[2 * i + 1])) for i in range(s)] + [EMPTY], dtype=np.uint32)
    G_map = labels[rng.integers(0, len(labels), size=(N, N))]
    d = vd.VoronoiDiagram(N, xy, metric=metric, virtual_shards=G)
    B = N // G
    for k in sorted({1, 2, 3, 4, 8, 64, B // 2 - 1, B // 2, B - 1, B, 2 * B} & set(range(1, N))):
        if k > B and k % B:
            continue
        d.set_labels(G_map)
        d.jump_pass(k, von_neumann=vn)
        assert np.array_equal(d.labels(), oracle.jump_pass(G_map, k, metric=metric, vn=vn)), k


@pytest.mark.slow
def test_windowed_pass_full_c5_size_bit_exact(vd):
    # BASELINE configs[4] size (65536^2, the reserved pixel included) in the launch
    # configuration bench.py times: one windowed pass per dJFA step regime (k = 32, 4, 1) on a
    # jittered complete map, the whole grid against the oracle.
    N = 65536
    G = _jittered_map(N, 24, 20000, 2209)
    G[G == EMPTY] = oracle.pack(N - 2, N - 1)  # label (65535, 65535) is EMPTY itself (R-4)
    d = vd.VoronoiDiagram(N, np.array([0, 0], dtype=np.uint16))
    for k in (32, 4, 1):
        d.set_labels(G)
        d.jump_pass(k)
        got = d.labels()
        want = oracle.jump_pass(G, k)
        assert np.array_equal(got, want), k
        del got, want
    d.close()


# ---------------------------------------------------------------- peer halos (NEXT-3)

@pytest.mark.parametrize("G,metric,vn_waves", [(2, "euclid", 0), (4, "euclid", 2), (8, "manhattan", 0)])
def test_peer_halos_virtual_shards_bit_exact(vd, G, metric, vn_waves):
    # Halo rows pushed by the pass kernels into the neighbouring bands' (double-buffered)
    # halo buffers instead of exchanged before each pass: JFA + dJFA identical to the oracle.
    N, s, dmax = 1024, 1024, 2
    xy = synth.uniform_seeds(N, s, rng_seed=G + 40)
    d = _jfa_gpu(vd, N, xy, metric=metric, vn_waves=vn_waves, virtual_shards=G, peer_halos=True)
    ref = oracle.jfa(N, xy, metric=metric)
    assert np.array_equal(d.labels(), ref)
    for f in range(4):
        disp = synth.displacements(s, dmax, f, rng_seed=G)
        d.djfa_step(disp, dmax)
        ref, xy, _ = oracle.djfa_step(N, xy, disp, dmax, ref, metric=metric, vn_waves=vn_waves)
        assert np.array_equal(d.labels(), ref), f


def _peer_worker(rank, world, port, N, s, dmax, frames, q):
    import os
    import torch.distributed as dist
    os.environ["MASTER_ADDR"], os.environ["MASTER_PORT"] = "127.0.0.1", str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2209_00117_b200 as m
    m.load_library()
    xy = synth.uniform_seeds(N, s, rng_seed=5)
    ref = oracle.jfa(N, xy)
    B = N // world
    d = m.VoronoiDiagram(N, xy, device=0, rank=rank, world=world, peer_halos=True)  # no NCCL id
    d.attach_peers()
    d.set_labels(ref[rank * B:(rank + 1) * B])
    ok = True
    for f in range(frames):
        disp = synth.displacements(s, dmax, f, rng_seed=5)
        d.djfa_step(disp, dmax)
        ref, xy, _ = oracle.djfa_step(N, xy, disp, dmax, ref)
        ok &= bool(np.array_equal(d.labels(), ref[rank * B:(rank + 1) * B]))
    q.put((rank, ok, d.peer_timed_out()))
    dist.barrier()
    d.close()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_peer_halos_two_processes_one_gpu(vd, world):
    # The cross-process path: each rank a process (here all on cuda:0), IPC-mapped halo buffers
    # and flag words, fused pushes + release/acquire flags, no NCCL communicator at all.
    import multiprocessing as mp
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_peer_worker, args=(r, world, port, 512, 1024, 2, 3, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = sorted(q.get(timeout=600) for _ in ps)
    for p in ps:
        p.join(timeout=120)
    assert [r for r, _, _ in res] == list(range(world))
    assert all(ok for _, ok, _ in res), res
    assert not any(t for _, _, t in res), res


def test_label_hash_async_matches(vd):
    N, s = 512, 300
    xy = synth.uniform_seeds(N, s, rng_seed=9)
    d = _jfa_gpu(vd, N, xy, virtual_shards=2)
    out = torch.zeros(3, dtype=torch.int64).pin_memory()
    ref = oracle.jfa(N, xy)
    want = []
    for f in range(3):
        disp = synth.displacements(s, 2, f, rng_seed=9)
        d.djfa_step(disp, 2)
        vd.vd_label_hash_async(d.h, out[f].data_ptr())
        ref, xy, _ = oracle.djfa_step(N, xy, disp, 2, ref)
        want.append(oracle.label_hash(ref))
    d.synchronize()
    assert [int(v) & 0xFFFFFFFFFFFFFFFF for v in out] == want


@pytest.mark.parametrize("N,s,G", [(1024, 4096, 0), (1024, 4096, 4), (1000, 3906, 0), (512, 100, 0)])
def test_djfa_step_hash_matches(vd, N, s, G):
    # vd_djfa_step_hash: the checksum summed by the last pass (jump_pass_sk, N % 512 == 0, one band
    # or banded) or by label_hash (N = 1000), equal to the oracle's label_hash of the new diagram
    xy = synth.uniform_seeds(N, s, rng_seed=N + s)
    d = _jfa_gpu(vd, N, xy, virtual_shards=G)
    ref = oracle.jfa(N, xy)
    out = torch.zeros(3, dtype=torch.int64).pin_memory()
    want = []
    for f in range(3):
        disp = synth.displacements(s, 2, f, rng_seed=N)
        vd.vd_djfa_step_hash(d.h, disp, 2, s, out[f].data_ptr())
        ref, xy, _ = oracle.djfa_step(N, xy, disp, 2, ref)
        want.append(oracle.label_hash(ref))
    d.synchronize()
    assert [int(v) & 0xFFFFFFFFFFFFFFFF for v in out] == want
    assert np.array_equal(d.labels(), ref)


# ---- packed-key passes (labels local to their pixels; vd_kernels.cuh row_packed) ---------
# The kernel switches to the one-key evaluation when the kernel that wrote its input found
# every label within distance 63 of its pixel (and k <= 64).  The result must not change:
# bit-exact against the same oracle, whichever path ran.


def _djfa_frames_packed(vd, N, s, dmax, frames, seed, **cfg):
    xy = synth.uniform_seeds(N, s, rng_seed=seed)
    d = _jfa_gpu(vd, N, xy, **cfg)
    G = oracle.jfa(N, xy)
    assert np.array_equal(d.labels(), G)
    packed = []
    for f in range(frames):
        disp = synth.displacements(s, dmax, f, rng_seed=seed)
        d.djfa_step(disp, dmax)
        G, xy, n = oracle.djfa_step(N, xy, disp, dmax, G)
        packed.append(d.last_packed_passes())
        assert np.array_equal(d.labels(), G), (f, packed)
    return d, packed


def test_packed_passes_taken_on_dense_seeds(vd):
    # L_avg = 16 (the C3-C5 density): the remapped diagram is local, every delta pass
    # (32 ... 1) takes the packed kernel
    d, packed = _djfa_frames_packed(vd, 1024, 4096, 1, 4, 77)
    assert packed == [d.last_passes()] * 4


@pytest.mark.parametrize("s,dmax", [(16, 1), (64, 2), (128, 1), (256, 3), (512, 1), (2048, 5), (4096, 40)])
def test_packed_passes_density_sweep_bit_exact(vd, s, dmax):
    # From sparse (every remap far: exact kernel throughout) to dense (all packed), with
    # densities in between where single frames or single passes switch paths.
    d, packed = _djfa_frames_packed(vd, 512, s, dmax, 4, 1000 + s)
    if s == 16:
        assert packed == [0] * 4
    if s >= 2048:
        assert min(packed) > 0


@pytest.mark.parametrize("N", [1000, 1031])
def test_packed_passes_ragged_grid_bit_exact(vd, N):
    # N not a multiple of 512 (edge CTAs) / of 4 (partial vectors)
    d, packed = _djfa_frames_packed(vd, N, N * N // 256, 1, 3, N)
    assert max(packed) > 0


@pytest.mark.parametrize("env", ["VD_NO_FIRST_SCATTER=1", "VD_FIRST_GATHER=1", "VD_NO_SK=1", "VD_NO_FULL=1",
                                 "VD_ORDER=1", "VD_NO_FUSE=1", "VD_REMAP=1", "VD_NO_TMAP=1", "VD_NO_FIVE=1",
                                 "VD_FUSE_PF=0", "VD_NO_RST_FOLD=1", "VD_LAT_ALL=1", "VD_FULL_MIN=4"])
def test_kernel_variant_switches_bit_exact(vd, env):
    # The A/B switches (read once per process) select the r01 kernels: JFA's init + gather
    # first pass instead of the seed scatter, jump_pass_fast instead of jump_pass_sk, segment
    # walks instead of whole residue classes, the other grid order, the separate remap kernel
    # instead of the remap fused into the first dJFA pass (and the lanes variant of it), six
    # bulk copies instead of one tensor copy per staged row, the seed scatter instead of the bitmap
    # gather for JFA's first pass, the separate fwd reset, the lattice walk below N = 32768 (the
    # packed form with unclaimed labels), one residue class per FULL walk.  Same labels either way.
    import subprocess, sys, os
    code = (
        "import numpy as np, synth, oracle, paper_2209_00117_b200 as vd\n"
        "for N, s, G in ((1024, 4096, 0), (2048, 300, 0), (1024, 1024, 4)):\n"
        "    xy = synth.uniform_seeds(N, s, rng_seed=N + s)\n"
        "    d = vd.VoronoiDiagram(N, xy, virtual_shards=G); d.jfa(); ref = oracle.jfa(N, xy)\n"
        "    assert np.array_equal(d.labels(), ref), (N, s, G)\n"
        "    for f in range(2):\n"
        "        disp = synth.displacements(s, 2, f, rng_seed=N)\n"
        "        d.djfa_step(disp, 2); ref, xy, _ = oracle.djfa_step(N, xy, disp, 2, ref)\n"
        "        assert np.array_equal(d.labels(), ref), (N, s, G, f)\n"
    )
    name, val = env.split("=")
    e = dict(os.environ, **{name: val})
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], env=e, cwd=root, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]


def test_packed_passes_disabled_env(vd, tmp_path):
    # VD_NO_PACK=1 (read once per process): the exact kernel only, same labels
    import subprocess, sys, os
    code = (
        "import numpy as np, synth, oracle, paper_2209_00117_b200 as vd\n"
        "N, s = 512, 1024\n"
        "xy = synth.uniform_seeds(N, s, rng_seed=5)\n"
        "d = vd.VoronoiDiagram(N, xy); d.jfa(); G = oracle.jfa(N, xy)\n"
        "disp = synth.displacements(s, 1, 0, rng_seed=5)\n"
        "d.djfa_step(disp, 1); G, xy, n = oracle.djfa_step(N, xy, disp, 1, G)\n"
        "assert d.last_packed_passes() == 0\n"
        "assert np.array_equal(d.labels(), G)\n"
    )
    env = dict(os.environ, VD_NO_PACK="1")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], env=env, cwd=root, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]


def test_packed_passes_windowed_kernel_forced(vd, monkeypatch):
    # The windowed kernel (grids beyond 32768) carries the packed path too; forced at small N
    monkeypatch.setenv("VD_FORCE_WINDOWED", "1")
    d, packed = _djfa_frames_packed(vd, 1024, 4096, 2, 3, 91)
    assert min(packed) > 0


@pytest.mark.parametrize("G,peer", [(2, False), (4, False), (4, True), (8, True)])
def test_packed_passes_sharded_bit_exact(vd, G, peer):
    # Row bands: the interior launch of an overlapped pass (rows that read no halo) takes the
    # packed walk when the band's own flag is clear; edge strips and non-overlapped passes
    # (2k >= band height) stay exact.  Identical to the oracle and to one band.
    N, s, dmax = 1024, 4096, 2
    d, packed = _djfa_frames_packed(vd, N, s, dmax, 3, 300 + G, virtual_shards=G, peer_halos=peer)
    assert min(packed) > 0


def test_packed_passes_sharded_counts_only_overlapped_passes(vd):
    # G = 8 bands of 32 rows: the k = 32 and 16 passes (2k >= B) read halos in every launch and
    # stay exact; only k = 8 ... 1 can pack
    d, packed = _djfa_frames_packed(vd, 256, 256, 1, 3, 8, virtual_shards=8)
    assert d.last_passes() == 6
    assert 0 < min(packed) and max(packed) <= 4


@pytest.mark.parametrize("N,s,dmax,G", [(1024, 4096, 1, 1), (1000, 3906, 3, 1), (512, 1024, 2, 1), (1024, 4096, 2, 4)])
def test_packed_passes_manhattan_bit_exact(vd, N, s, dmax, G):
    # dJFAm: the packed key with d = |dx| + |dy| (one VABSDIFF per candidate)
    xy = synth.uniform_seeds(N, s, rng_seed=N + s)
    d = vd.VoronoiDiagram(N, xy, metric="manhattan", virtual_shards=G)
    d.jfa()
    G_ = oracle.jfa(N, xy, metric="manhattan")
    assert np.array_equal(d.labels(), G_)
    packed = []
    for f in range(3):
        disp = synth.displacements(s, dmax, f, rng_seed=N)
        d.djfa_step(disp, dmax)
        G_, xy, _ = oracle.djfa_step(N, xy, disp, dmax, G_, metric="manhattan")
        packed.append(d.last_packed_passes())
        assert np.array_equal(d.labels(), G_), (f, packed)
    if s * 256 >= N * N:
        assert min(packed) > 0
