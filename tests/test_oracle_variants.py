"""Pins for the paper's variants (NEXT-2): the Manhattan metric of dJFAm and
the Von Neumann neighbourhood, alone (Fig. 5) or for the first waves of a
dJFA step followed by Moore.

Independent references: scipy's exact taxicab distance transform, a hand-worked fixture,
the Algorithm-1 scatter form (re-derived below), closed-form reachability, and the
paper's qualitative claims (VN alone is worse than Moore; dJFAm similarity to JFA is at
least ~88%).
"""
import numpy as np
import pytest
from scipy import ndimage

import golden_io
import oracle
import synth

EMPTY = 0xFFFFFFFF


def _l1_of_labels(G):
    N = G.shape[0]
    y, x = np.mgrid[0:N, 0:N]
    return np.abs(x - (G & 0xFFFF).astype(np.int64)) + np.abs(y - (G >> 16).astype(np.int64))


@pytest.mark.parametrize("N,s,seed", [(5, 1, 0), (9, 4, 1), (31, 12, 2), (64, 30, 3), (100, 77, 4)])
def test_manhattan_exact_matches_scipy_taxicab(N, s, seed):
    xy = synth.uniform_seeds(N, s, rng_seed=seed)
    E = oracle.exact_brute(N, xy, metric="manhattan")
    img = np.ones((N, N), dtype=np.uint8)
    img[xy[1::2].astype(int), xy[0::2].astype(int)] = 0
    ref = ndimage.distance_transform_cdt(img, metric="taxicab").astype(np.int64)
    assert np.array_equal(_l1_of_labels(E), ref)
    seeds = {oracle.pack(int(xy[2 * i]), int(xy[2 * i + 1])) for i in range(s)}
    assert set(np.unique(E).tolist()) <= seeds


def test_golden_manhattan_fixture():
    fx = golden_io.load("manhattan_4x4_two_seeds.txt")
    N = fx["N"]
    xy = golden_io.seeds_xy(fx)
    assert np.array_equal(oracle.exact_brute(N, xy, metric="manhattan"), golden_io.grid(fx, "exact"))
    G = oracle.jump_pass(oracle.init(N, xy), 2, metric="manhattan")
    assert np.array_equal(G, golden_io.grid(fx, "after_k2"))
    G = oracle.jump_pass(G, 1, metric="manhattan")
    assert np.array_equal(G, golden_io.grid(fx, "final"))
    assert np.array_equal(oracle.jfa(N, xy, metric="manhattan"), golden_io.grid(fx, "final"))


def _key(x, y, c, metric):
    if c == EMPTY:
        return (float("inf"), 0)
    cx, cy = c & 0xFFFF, c >> 16
    d = abs(x - cx) + abs(y - cy) if metric == "manhattan" else (x - cx) ** 2 + (y - cy) ** 2
    return (d, c)


def _scatter_pass(G, k, metric, vn):
    """Algorithm 1's body, double-buffered: every pixel pushes its seed to its
    neighbours (Table 1's 8, or the 4 axis ones for Von Neumann) -- re-derived here."""
    N = G.shape[0]
    out = G.copy()
    offs = [(k, 0), (0, k), (-k, 0), (0, -k)]
    if not vn:
        offs += [(k, k), (-k, k), (-k, -k), (k, -k)]
    for py in range(N):
        for px in range(N):
            sp = int(G[py, px])
            for dx, dy in offs:
                qx, qy = px + dx, py + dy
                if 0 <= qx < N and 0 <= qy < N and _key(qx, qy, sp, metric) < _key(qx, qy, int(out[qy, qx]), metric):
                    out[qy, qx] = sp
    return out


@pytest.mark.parametrize("metric,vn", [("manhattan", False), ("euclid", True), ("manhattan", True)])
def test_gather_equals_scatter_variants(metric, vn):
    rng = np.random.default_rng(5)
    for trial in range(30):
        N = int(rng.integers(2, 10))
        s = int(rng.integers(1, min(5, N * N) + 1))
        xy = synth.uniform_seeds(N, s, rng_seed=trial)
        labels = np.array([oracle.pack(int(xy[2 * i]), int(xy[2 * i + 1])) for i in range(s)] + [EMPTY],
                          dtype=np.uint32)
        G = labels[rng.integers(0, len(labels), size=(N, N))]
        for k in (1, 2, 3, 4):
            assert np.array_equal(oracle.jump_pass(G, k, metric=metric, vn=vn), _scatter_pass(G, k, metric, vn))


def test_von_neumann_offsets():
    # the 4 axis offsets of Table 1 (neighbours 1, 3, 5, 7) at range k, plus the pixel
    N, k = 9, 3
    G = np.full((N, N), EMPTY, dtype=np.uint32)
    G[4, 4] = oracle.pack(4, 4)
    H = oracle.jump_pass(G, k, vn=True)
    got = {(int(x) - 4, int(y) - 4) for y, x in zip(*np.nonzero(H != EMPTY))}
    assert got == {(0, 0), (k, 0), (-k, 0), (0, k), (0, -k)}


def test_von_neumann_alone_can_leave_pixels_unreached():
    # Closed form: on a 2x2 grid JFA has the single pass k = 1; with Von Neumann only, a
    # seed at (0,0) reaches (1,0) and (0,1) but not the diagonal (1,1) (Von
    # Neumann alone "generates an incorrect VD even for JFA").
    G = oracle.jfa(2, np.array([0, 0], dtype=np.uint16), vn_waves=99)
    assert G[1, 1] == EMPTY and G[0, 1] == 0 and G[1, 0] == 0


def test_von_neumann_jfa_worse_than_moore():
    # regions become concave / saw-toothed with Von Neumann alone.
    worse = 0
    for r in range(12):
        xy = synth.uniform_seeds(64, 16, rng_seed=300 + r)
        E = oracle.exact_brute(64, xy)
        moore = oracle.similarity(oracle.jfa(64, xy), E)
        vn = oracle.similarity(oracle.jfa(64, xy, vn_waves=99), E)
        assert vn <= moore
        worse += vn < moore
    assert worse >= 10


def _djfa_run(N, s, d, frames, seed, metric="euclid", vn_waves=0):
    xy = synth.uniform_seeds(N, s, rng_seed=seed)
    G = oracle.jfa(N, xy, metric=metric)
    out = []
    for f in range(frames):
        disp = synth.displacements(s, d, f, rng_seed=seed)
        G, xy, _ = oracle.djfa_step(N, xy, disp, d, G, metric=metric, vn_waves=vn_waves)
        out.append((G.copy(), xy.copy()))
    return out


def test_djfam_similarity_band():
    # dJFAm reaches "88% to 92%" similarity to (Euclidean) JFA; the abstract says
    # "at least 88%".  At desk scale we accept [80, 97] and require it to differ
    # from the Euclidean diagram (a different metric cannot be ~100% equal).
    sims = []
    for G, xy in _djfa_run(256, 512, 2, 4, 17, metric="manhattan"):
        assert (G != EMPTY).all()
        sims.append(oracle.similarity(G, oracle.jfa(256, xy)))
        # and it is close to the exact Manhattan diagram
        assert oracle.similarity(G, oracle.exact_brute(256, xy, metric="manhattan")) >= 97.0
    assert 80.0 <= np.mean(sims) <= 97.0


def test_djfa_with_von_neumann_waves_stays_complete_and_close():
    # P:170 / P:204: Von Neumann for the first two waves, Moore for the rest.
    for G, xy in _djfa_run(128, 128, 2, 4, 23, vn_waves=2):
        assert (G != EMPTY).all()
        assert oracle.similarity(G, oracle.jfa(128, xy)) >= 95.0


def test_zero_motion_manhattan_exact_is_identity():
    N, s = 40, 9
    xy = synth.uniform_seeds(N, s, rng_seed=2)
    E = oracle.exact_brute(N, xy, metric="manhattan")
    G, _, _ = oracle.djfa_step(N, xy, np.zeros(2 * s, dtype=np.int16), 1, E, metric="manhattan", vn_waves=2)
    assert np.array_equal(G, E)


# ---------------------------------------------------------------- Standard Flooding (NEXT-4)

def test_stf_paper_example_five_iterations():
    # P:76 / Fig. 2(a): "StF fulfills its purpose in 5 iterations" for one seed; a seed at
    # the centre of an 11x11 grid is at Chebyshev distance 5 from the corners.
    G, n = oracle.stf(11, np.array([5, 5], dtype=np.uint16))
    assert n == 5 and (G == oracle.pack(5, 5)).all()


@pytest.mark.parametrize("N,x,y", [(2, 0, 0), (7, 0, 0), (9, 2, 6), (16, 15, 3)])
def test_stf_one_seed_passes_equal_chebyshev_radius(N, x, y):
    # one seed floods the grid in max Chebyshev distance to a corner passes (closed form)
    G, n = oracle.stf(N, np.array([x, y], dtype=np.uint16))
    assert n == max(x, N - 1 - x, y, N - 1 - y)
    assert (G == oracle.pack(x, y)).all()


def test_stf_complete_and_close_to_exact():
    # StF propagates claims one ring at a time; the result is complete and, like JFA,
    # close to Eq. 1 (each pass is the same gather, R-12).
    for r in range(6):
        xy = synth.uniform_seeds(48, 10, rng_seed=40 + r)
        G, n = oracle.stf(48, xy)
        assert (G != EMPTY).all()
        assert n <= 47
        assert oracle.similarity(G, oracle.exact_brute(48, xy)) >= 97.0
