"""Pins for the oracle's schedule functions (Eq. 2 and Eq. 3-4).

Sources of truth: the paper's printed example, direct evaluation of the printed
equations in floating point (a different computation from the oracle's integer form),
and SPEC.md's worked examples.
"""
import math
import random

import pytest

import oracle


def test_eq2_paper_example_8x8():
    # "for a 8 x 8 grid, there are three iterations with the values of {4,2,1}"
    assert oracle.jfa_schedule(8) == [4, 2, 1]


@pytest.mark.parametrize("N,k1,n", [(1024, 512, 10), (1000, 512, 10), (2, 1, 1), (3, 2, 2),
                                    (64, 32, 6), (16384, 8192, 14), (65536, 32768, 16)])
def test_eq2_values(N, k1, n):
    # S:128-130 examples and Eq. 2 evaluated by hand: k1 = 2^(ceil(log2 N) - 1)
    ks = oracle.jfa_schedule(N)
    assert ks[0] == k1 and len(ks) == n and ks[-1] == 1


def test_eq2_float_evaluation():
    # Eq. 2 evaluated literally with floating-point log2 for every N it is
    # unambiguous on, then halving "until k_i = 1 (inclusive)".
    for N in range(2, 5000):
        k1 = 2 ** (math.ceil(math.log2(N)) - 1)
        expect = []
        i = 1
        while True:
            k = k1 / 2 ** (i - 1)
            expect.append(int(k))
            if k == 1:
                break
            i += 1
        assert oracle.jfa_schedule(N) == expect, N
        # P:81 "JFA does log2(k)+1 steps"
        assert len(expect) == int(math.log2(k1)) + 1


def test_extras_append_unit_passes():
    # P:114 JFA+1 / JFA+2 (reading R-6: trailing k = 1 passes)
    assert oracle.jfa_schedule(8, extras=2) == [4, 2, 1, 1, 1]
    assert oracle.djfa_schedule(1024, 4096, 4, extras=1) == [32, 16, 8, 4, 2, 1, 1]


@pytest.mark.parametrize("N,s,d,delta1,waves", [
    (1000, 100, 5, 256, 9),    # S:221 (2 L_avg = 200 -> 2^8)
    (1024, 4096, 4, 32, 6),    # S:222 (2 L_avg = 32)
    (64, 1, 1, 32, 6),         # S:223 capped at k_1 = 32 ("behaves very much like JFA")
    (16384, 2**20, 1, 32, 6),  # config C4 of BASELINE.json (L_avg = 16)
    (65536, 2**24, 1, 32, 6),  # config C5
    (1024, 1024, 1, 64, 7),    # config C2 (L_avg = 32)
    (4096, 65536, 64, 64, 7),  # d_max dominates ("it will trigger the usage of d_max")
    (4096, 65536, 2048, 2048, 12),
])
def test_eq4_examples(N, s, d, delta1, waves):
    ks = oracle.djfa_schedule(N, s, d)
    assert ks[0] == delta1 and len(ks) == waves
    assert ks == [delta1 >> i for i in range(waves)]


def _eq4_float(N, s, d):
    L = math.sqrt(N * N / s)                       # Eq. 3
    e = math.ceil(math.log2(max(2 * L, d)))        # Eq. 4 exponent
    return e


def test_eq4_against_float_evaluation():
    # Random (N, s, d_max): the oracle's integer form must equal Eq. 4 evaluated in
    # floating point whenever the float exponent is not within rounding of an integer.
    rng = random.Random(7)
    checked = 0
    for _ in range(20000):
        N = rng.randint(2, 70000) if rng.random() < 0.5 else 2 ** rng.randint(1, 16)
        N = min(N, 65536)
        s = rng.randint(1, min(N * N, 2**26))
        d = rng.randint(0, 3000)
        L = math.sqrt(N * N / s)
        x = math.log2(max(2 * L, d, 1e-300))
        if abs(x - round(x)) < 1e-9:
            continue
        e = max(_eq4_float(N, s, d), 0)
        e = min(e, math.ceil(math.log2(N)) - 1)
        assert oracle.djfa_schedule(N, s, d)[0] == 2 ** e, (N, s, d)
        checked += 1
    assert checked > 15000


def test_eq4_exact_powers_of_two():
    # At exact powers of two the float form can round either way; the integer form must
    # give the mathematically exact ceil: 2 L_avg = 32 exactly -> delta_1 = 32, not 64.
    assert oracle.djfa_schedule(4096, 65536, 1)[0] == 32
    assert oracle.djfa_schedule(4096, 65536, 32)[0] == 32
    assert oracle.djfa_schedule(4096, 65536, 33)[0] == 64
    # one seed fewer than the exact case: 2 L_avg slightly above 32 -> 64
    assert oracle.djfa_schedule(4096, 65535, 1)[0] == 64


def test_eq4_staircase_monotone():
    # S:245-247 / P:285 staircase: waves non-increasing in s, non-decreasing in N.
    for N in (256, 1000, 4096):
        prev = 99
        for s in [2 ** i for i in range(0, 20)]:
            if s > N * N:
                break
            n = len(oracle.djfa_schedule(N, s, 2))
            assert n <= prev
            prev = n
    for s in (16, 1000, 65536):
        prev = 0
        for N in range(64, 5000, 61):
            if s > N * N:
                continue
            n = len(oracle.djfa_schedule(N, s, 2))
            assert n >= prev
            prev = n


def test_djfa_never_longer_than_jfa():
    for N in (2, 3, 64, 1000, 4096):
        for s in (1, 7, 100):
            if s > N * N:
                continue
            assert len(oracle.djfa_schedule(N, s, 5)) <= len(oracle.jfa_schedule(N))
