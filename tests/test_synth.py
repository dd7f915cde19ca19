"""The shared seeded input generators (no method arithmetic here)."""
import numpy as np

import synth


def test_splitmix64_known_values():
    # Reference outputs of SplitMix64 for state 0 (Vigna's splitmix64.c): the first call
    # advances the state by the golden gamma and mixes it.
    assert int(synth.splitmix64(np.array([0], dtype=np.uint64))[0]) == 0xE220A8397B1DCDAF
    assert int(synth.splitmix64(np.array([0x9E3779B97F4A7C15], dtype=np.uint64))[0]) == 0x6E789E6AA1B965F4


def test_seeds_in_range_and_deterministic():
    for N in (2, 3, 64, 1000, 65536):
        xy = synth.uniform_seeds(N, min(5000, N * N), rng_seed=1)
        assert xy.dtype == np.uint16 and xy.size == 2 * min(5000, N * N)
        assert int(xy.max()) < N
        assert np.array_equal(xy, synth.uniform_seeds(N, min(5000, N * N), rng_seed=1))
    assert not np.array_equal(synth.uniform_seeds(64, 100, 1), synth.uniform_seeds(64, 100, 2))


def test_seeds_roughly_uniform():
    xy = synth.uniform_seeds(400, 160000, rng_seed=3)
    counts = np.bincount(xy[0::2].astype(int) // 25, minlength=16)
    assert counts.min() > 9000 and counts.max() < 11000


def test_displacements_support():
    for d in (0, 1, 4):
        v = synth.displacements(10000, d, frame=3)
        assert v.dtype == np.int16 and v.min() >= -d and v.max() <= d
        if d:
            assert set(np.unique(v).tolist()) == set(range(-d, d + 1))
    assert not np.array_equal(synth.displacements(100, 2, 0), synth.displacements(100, 2, 1))
