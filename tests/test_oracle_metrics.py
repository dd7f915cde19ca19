"""Pins for Eq. 5 similarity / match count and the label hash."""
import numpy as np

import oracle
import synth

EMPTY = 0xFFFFFFFF


def test_similarity_spec_examples():
    # identical -> 100; all different -> 0; 8x8 with 16 different -> 75.
    rng = np.random.default_rng(0)
    a = rng.integers(0, 2**31, size=(8, 8)).astype(np.uint32)
    assert oracle.similarity(a, a) == 100.0
    assert oracle.similarity(a, a ^ np.uint32(1)) == 0.0
    b = a.copy()
    idx = rng.choice(64, size=16, replace=False)
    b.reshape(-1)[idx] ^= np.uint32(7)
    assert oracle.similarity(a, b) == 75.0
    assert oracle.match_count(a, b) == 48


def test_similarity_symmetric_and_empty_matches_empty():
    a = np.array([[EMPTY, 1], [2, EMPTY]], dtype=np.uint32)
    b = np.array([[EMPTY, 1], [EMPTY, 3]], dtype=np.uint32)
    assert oracle.match_count(a, b) == oracle.match_count(b, a) == 2


def test_label_hash_order_independent_and_sensitive():
    G = oracle.jfa(32, synth.uniform_seeds(32, 9, rng_seed=1))
    h = oracle.label_hash(G)
    # a permutation of the rows changes positions -> changes the hash
    assert oracle.label_hash(G[::-1].copy()) != h or (G == G[::-1]).all()
    H = G.copy()
    H[5, 5] ^= 1
    assert oracle.label_hash(H) != h
    # closed form on a tiny map: MurmurHash3's fmix32 reference vectors, then the sum
    def fmix32(h):
        h ^= h >> 16
        h = (h * 0x85EBCA6B) & 0xFFFFFFFF
        h ^= h >> 13
        h = (h * 0xC2B2AE35) & 0xFFFFFFFF
        return h ^ (h >> 16)
    assert fmix32(0) == 0 and fmix32(1) == 0x514E28B7  # smhasher's fmix32(1)
    g = np.array([[7, 9]], dtype=np.uint32)
    want = fmix32((0 * 0x9E3779B9) & 0xFFFFFFFF ^ 7) + fmix32((1 * 0x9E3779B9) & 0xFFFFFFFF ^ 9)
    assert oracle.label_hash(g) == want
