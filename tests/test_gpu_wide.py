"""GPU parity of the wide exact pass (jump_pass_wsk): grids beyond N = 32768, whose squared
distances need 33 bits, with labels anywhere and EMPTY allowed (JFA's large steps at C5).

Every test compares one pass over the whole grid with the oracle's Alg. 1 pass (oracle.jump_pass,
key (d2, c) lexicographically: Eq. 1, reading R-3), element by element.  The maps
are built to reach the kernel's corner cases:
  * uniform random labels over the whole grid (|dx|, |dy| up to N - 1: at N = 65536 squared
    distances up to 2^33, the range the kernel's split key D >> 2 / D & 3 exists for);
  * EMPTY sprinkled and in whole rows / columns (the MAY_EMPTY variant, all-EMPTY neighbourhoods);
  * planted exact ties: mirror labels about the pixel's column (same cy, dx = -a / +a), equal d2 with
    different cy ((3s, 4s) vs (4s, 3s)), and d2 values in one group of four (25 vs 26, decided by
    d2 & 3 before cy) -- the three levels of the key's low word;
  * grid edges (the out-of-grid neighbour substitution) on every side.
"""
import numpy as np
import pytest

import oracle

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu, pytest.mark.slow]

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


def _pack(y, x):
    return ((np.asarray(y, dtype=np.int64) << 16) | np.asarray(x, dtype=np.int64)).astype(np.uint32)


def _random_map(N, seed):
    rng = np.random.default_rng(seed)
    G = np.empty((N, N), dtype=np.uint32)
    for y0 in range(0, N, 4096):
        y1 = min(N, y0 + 4096)
        G[y0:y1] = _pack(rng.integers(0, N, (y1 - y0, N)), rng.integers(0, N, (y1 - y0, N)))
    if N == 65536:
        G[G == EMPTY] = 0  # (65535, 65535) is the reserved pixel, never a label (R-4)
    return G


def _plant_ties(G, k, seed, count=20000):
    """Plant exact and near ties among the candidates of random pixels of pass k."""
    N = G.shape[0]
    rng = np.random.default_rng(seed)
    m = 8 * 64
    for kind in range(3):
        s = rng.integers(1, 64, count)
        X = rng.integers(k + m, N - k - m, count)
        y = rng.integers(k + m, N - k - m, count)
        G[y, X] = _pack(rng.integers(0, N, count), rng.integers(0, N, count))  # own label: usually far
        if kind == 0:    # mirror images about the pixel's column (same cy): smaller cx (dx < 0) wins
            a, dy = rng.integers(0, m, count), rng.integers(-m, m, count)
            G[y, X - k] = _pack(y + dy, X + a)
            G[y, X + k] = _pack(y + dy, X - a)
        elif kind == 1:  # (3s, 4s) vs (4s, 3s): equal d2, smaller cy wins
            G[y - k, X] = _pack(y + 4 * s, X + 3 * s)
            G[y + k, X] = _pack(y + 3 * s, X + 4 * s)
        else:            # 25 vs 26 (one group of four of D >> 2): d2 & 3 decides before cy
            G[y - k, X - k] = _pack(y - 5, X + 1)   # d2 = 26, smaller cy
            G[y + k, X + k] = _pack(y + 4, X + 3)   # d2 = 25: wins
    return G


def _one_pass(vd, G, k):
    N = G.shape[0]
    d = vd.VoronoiDiagram(N, np.array([0, 0], dtype=np.uint16))
    try:
        d.set_labels(G)
        d.jump_pass(k)
        return d.labels()
    finally:
        d.close()


def _check(vd, G, k):
    got = _one_pass(vd, G, k)
    want = oracle.jump_pass(G, k)
    bad = np.argwhere(got != want)
    assert bad.size == 0, (k, bad[:5].tolist(), len(bad),
                           [(int(got[tuple(b)]), int(want[tuple(b)])) for b in bad[:3]])


@pytest.fixture(scope="module")
def grid_33280():
    return _random_map(33280, 11)  # 65 * 512: the smallest CTA-tiled grid beyond 32768


@pytest.mark.parametrize("k", [256, 512, 1024, 4096, 8192])
def test_wide_pass_random_labels(vd, grid_33280, k):
    _check(vd, _plant_ties(grid_33280.copy(), k, k), k)


@pytest.mark.parametrize("k", [256, 2048, 8192])
def test_wide_pass_with_empty(vd, grid_33280, k):
    G = _plant_ties(grid_33280.copy(), k, k + 1)
    rng = np.random.default_rng(k)
    G[rng.random(G.shape) < 0.6] = EMPTY   # EMPTY-dominated, as JFA's first passes
    G[4000:4004] = EMPTY                    # whole rows
    G[:, 17000:17003] = EMPTY               # whole columns
    G[:k, :k] = EMPTY                       # all-EMPTY neighbourhoods (outputs stay EMPTY)
    _check(vd, G, k)


def test_wide_pass_full_walks_c5(vd):
    # BASELINE configs[4] size: d2 up to 2 * 65535^2 (33 bits), k = 16384 runs whole residue
    # classes per CTA (FULL walks), k = 512 segment walks; with EMPTY in the second pass.
    N = 65536
    G = _random_map(N, 12)
    for k in (16384, 512):
        G2 = _plant_ties(G.copy(), k, 3 * k, count=50000)
        if k == 16384:
            G2[np.random.default_rng(1).random((N, N), dtype=np.float32) < 0.9] = EMPTY
        _check(vd, G2, k)
        del G2
