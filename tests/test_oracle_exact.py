"""Pins for the exact diagram (Eq. 1): or_exact_brute and or_exact_bucketed.

Independent references: scipy's exact Euclidean distance transform (a library routine
with a different algorithm; it fixes the nearest distance, which is unique), hand-worked
fixtures (tests/golden/), and closed-form special cases.
"""
import numpy as np
import pytest
from scipy import ndimage

import golden_io
import oracle
import synth


def _d2_of_labels(G):
    N = G.shape[0]
    y, x = np.mgrid[0:N, 0:N]
    cx = (G & 0xFFFF).astype(np.int64)
    cy = (G >> 16).astype(np.int64)
    return (x - cx) ** 2 + (y - cy) ** 2


def _edt_d2(N, xy):
    img = np.ones((N, N), dtype=np.uint8)
    img[xy[1::2].astype(int), xy[0::2].astype(int)] = 0
    d = ndimage.distance_transform_edt(img)
    return np.rint(d * d).astype(np.int64)


@pytest.mark.parametrize("N,s,seed", [(5, 1, 0), (8, 3, 1), (13, 7, 2), (32, 20, 3), (64, 16, 4),
                                      (100, 50, 5), (127, 300, 6)])
def test_exact_distance_matches_scipy_edt(N, s, seed):
    xy = synth.uniform_seeds(N, s, rng_seed=seed)
    E = oracle.exact_brute(N, xy)
    assert np.array_equal(_d2_of_labels(E), _edt_d2(N, xy))
    # every label is one of the seeds
    seeds = set(int(v) for v in (xy[1::2].astype(np.uint32) << 16) | xy[0::2].astype(np.uint32))
    assert set(np.unique(E).tolist()) <= seeds


def test_golden_exact_fixtures():
    for name in ("jfa_4x4_two_seeds.txt", "djfa_4x4_step.txt", "exact_3x3_tie.txt"):
        fx = golden_io.load(name)
        xy = golden_io.seeds_xy(fx)
        assert np.array_equal(oracle.exact_brute(fx["N"], xy), golden_io.grid(fx, "exact")), name
        assert np.array_equal(oracle.exact(fx["N"], xy, bucket=1), golden_io.grid(fx, "exact")), name


def test_one_seed_labels_everything():
    # 1 seed -> every pixel claimed by it
    for N, x, y in ((2, 1, 0), (7, 3, 5), (33, 0, 32)):
        E = oracle.exact_brute(N, np.array([x, y], dtype=np.uint16))
        assert (E == oracle.pack(x, y)).all()


@pytest.mark.parametrize("N", [4, 5, 9, 10])
def test_two_seeds_split_left_right(N):
    # seeds (0,y) and (N-1,y) split the grid into halves; for odd N the midline
    # column is equidistant and goes to the left seed (smaller packed label, R-3).
    y0 = N // 2
    xy = np.array([0, y0, N - 1, y0], dtype=np.uint16)
    E = oracle.exact_brute(N, xy)
    left, right = oracle.pack(0, y0), oracle.pack(N - 1, y0)
    for x in range(N):
        want = left if 2 * x <= N - 1 else right
        assert (E[:, x] == want).all(), x


def test_exhaustive_two_seed_placements_small():
    # All ordered placements of 2 distinct seeds on 4x4: the label's distance equals
    # the minimum of the two closed-form distances, and ties go to the smaller label.
    N = 4
    y, x = np.mgrid[0:N, 0:N]
    for a in range(N * N):
        for b in range(N * N):
            if a == b:
                continue
            ax, ay, bx, by = a % N, a // N, b % N, b // N
            xy = np.array([ax, ay, bx, by], dtype=np.uint16)
            E = oracle.exact_brute(N, xy)
            da = (x - ax) ** 2 + (y - ay) ** 2
            db = (x - bx) ** 2 + (y - by) ** 2
            la, lb = oracle.pack(ax, ay), oracle.pack(bx, by)
            want = np.where(da < db, la, np.where(db < da, lb, min(la, lb)))
            assert np.array_equal(E, want.astype(np.uint32))


@pytest.mark.parametrize("N,s,seed", [(16, 5, 0), (64, 64, 1), (100, 7, 2), (256, 256, 3),
                                      (300, 1000, 4), (512, 128, 5)])
def test_bucketed_equals_brute(N, s, seed):
    xy = synth.uniform_seeds(N, s, rng_seed=seed)
    B = oracle.exact_brute(N, xy)
    for bs in (1, 3, 16, None):
        assert np.array_equal(oracle.exact(N, xy, bucket=bs), B)


def test_colocated_seeds():
    # co-located seeds are allowed; they share one label.
    xy = np.array([3, 3, 3, 3, 0, 0], dtype=np.uint16)
    E = oracle.exact_brute(8, xy)
    assert set(np.unique(E).tolist()) == {oracle.pack(3, 3), oracle.pack(0, 0)}
