"""The packed-key evaluation of the jump pass (vd_kernels.cuh: row_packed / min9_packed), its
arithmetic restated in numpy uint32 and checked against the lexicographic key of R-3 by brute
force.  No GPU: this pins the DESIGN of the kernel's fast path (which operands, which modular
identities, which comparison kind per row), so that a wrong constant or sign fails here before
any GPU run.  The GPU path itself is checked against the oracle in test_gpu_parity.py.

Claim: for a pixel (X, y) and candidates c = (cy << 16) | cx with
|cx - X|, |cy - y| <= 127, the nine values Qk + cy * M_y (mod 2^32), minimised as unsigned when
-C_y <= 2^31 and as signed otherwise, give min over i of key_i - C_y, where
key = d2 * 2^16 + (dy + 128) * 2^8 + (dx + 128); and the label is recovered from the key.
"""
import numpy as np

M32 = np.uint64(0xFFFFFFFF)


def _u32(a):
    return (np.asarray(a, dtype=np.int64) & 0xFFFFFFFF).astype(np.uint64)


def packed_label(X, y, c):
    """Kernel arithmetic for one pixel; c: uint32 labels (9 candidates)."""
    c = _u32(c)
    cy = c >> np.uint64(16)
    D1 = (c * np.uint64(65536) + _u32(1 - (X << 16))) & M32          # (cx - X) << 16 | 1
    dx = _u32(((D1.astype(np.int64) ^ 0x80000000) - 0x80000000) >> 16)  # arithmetic shift of int32
    chi = c & np.uint64(0xFFFF0000)
    Qk = (dx * D1 + cy * chi) & M32
    My = _u32(256 - (y << 17))
    Cy = _u32(y * y * 65536 - 256 * y + 32896)
    k = (Qk + cy * My) & M32
    if (-int(Cy)) % 2**32 <= 2**31:
        m = int(k.min())
    else:
        ks = k.astype(np.int64)
        ks = np.where(ks >= 2**31, ks - 2**32, ks)
        m = int(ks.min()) % 2**32
    s = (m + int(Cy)) % 2**32
    prmt = ((s >> 8) & 0xFF) << 16 | (s & 0xFF)
    return (prmt + (((y - 128) << 16) % 2**32) + (X - 128)) % 2**32, s


def lexi_label(X, y, c):
    c = np.asarray(c, dtype=np.int64)
    cx, cy = c & 0xFFFF, c >> 16
    d2 = (cx - X) ** 2 + (cy - y) ** 2
    order = np.lexsort((c, d2))
    return int(c[order[0]]), int(d2[order[0]])


def test_random_candidates_match_lexicographic_key():
    rng = np.random.default_rng(2209)
    for _ in range(4000):
        X, y = int(rng.integers(127, 65536 - 127)), int(rng.integers(127, 65536 - 128))
        d = rng.integers(-127, 128, size=(9, 2))
        c = ((y + d[:, 1]) << 16) | (X + d[:, 0])
        got, s = packed_label(X, y, c)
        want, d2 = lexi_label(X, y, c)
        assert got == want, (X, y, d.tolist())
        assert s >> 16 == d2  # the key's high half is d2


def test_ties_resolved_by_smaller_label():
    # equidistant candidates (symmetric offsets): the smaller packed label (smaller y, then x)
    rng = np.random.default_rng(5)
    for _ in range(2000):
        X, y = int(rng.integers(127, 60000)), int(rng.integers(127, 60000))
        a, b = int(rng.integers(0, 90)), int(rng.integers(0, 90))
        offs = [(a, b), (-a, b), (a, -b), (-a, -b), (b, a), (-b, a), (b, -a), (-b, -a), (a, b)]
        c = [((y + dy) << 16) | (X + dx) for dx, dy in offs]
        assert packed_label(X, y, c)[0] == lexi_label(X, y, c)[0]


def test_every_row_kind_and_extreme_offsets():
    # both comparison kinds occur, and the extreme |dx| = |dy| = 127 corners keep d2 < 2^15
    kinds = set()
    for y in list(range(127, 2000, 7)) + [32767, 32768, 40000, 65535 - 127]:
        Cy = (y * y * 65536 - 256 * y + 32896) % 2**32
        kinds.add((-Cy) % 2**32 <= 2**31)
        X = 1000
        for sx, sy in [(127, 127), (-127, -127), (127, -127), (-127, 127), (0, 0)]:
            c = [((y + sy) << 16) | (X + sx)] * 8 + [((y - sy) << 16) | (X - sx)]
            assert packed_label(X, y, c)[0] == lexi_label(X, y, c)[0]
    assert kinds == {True, False}


def test_locality_radius_bounds_the_key():
    # kLocR = 63 and k <= 64: candidate offsets <= 127 per axis, d2 <= 2 * 127^2 < 2^15
    assert 63 + 64 == 127 and 2 * 127 ** 2 < 2 ** 15
    # remap's Chebyshev 44 implies Euclidean <= 63
    assert 2 * 44 ** 2 <= 63 ** 2


def packed_label_manhattan(X, y, c):
    """Manhattan (METRIC 1) form: per label chi = cy << 16, Qm = |dx| << 16 + dx + 256 cy; per
    candidate |chi - (y << 16)| + Qm = key - C'_y with C'_y = 32896 - 256 y."""
    c = [int(v) for v in c]
    k = []
    for v in c:
        chi = v & 0xFFFF0000
        D = (v * 65536 - (X << 16)) % 2**32
        Ds = D - 2**32 if D >= 2**31 else D
        dx = Ds >> 16
        Qm = (abs(Ds) + dx + (chi >> 8)) % 2**32
        k.append((abs(chi - ((y << 16) % 2**32)) + Qm) % 2**32)
    Cy = (32896 - 256 * y) % 2**32
    if (-Cy) % 2**32 <= 2**31:
        m = min(k)
    else:
        m = min((v - 2**32 if v >= 2**31 else v) for v in k) % 2**32
    s = (m + Cy) % 2**32
    prmt = ((s >> 8) & 0xFF) << 16 | (s & 0xFF)
    return (prmt + (((y - 128) << 16) % 2**32) + (X - 128)) % 2**32, s


def test_manhattan_packed_key_matches_lexicographic_key():
    rng = np.random.default_rng(173)
    for _ in range(3000):
        X, y = int(rng.integers(127, 65536 - 127)), int(rng.integers(127, 65536 - 128))
        if rng.random() < 0.5:  # equidistant offsets (ties in d = |dx| + |dy|)
            a, b = int(rng.integers(0, 64)), int(rng.integers(0, 64))
            d = np.array([(a, b), (-a, b), (a, -b), (-a, -b), (b, a), (-b, a), (b, -a), (-b, -a), (a + b, 0)])
        else:
            d = rng.integers(-127, 128, size=(9, 2))
        c = ((y + d[:, 1]) << 16) | (X + d[:, 0])
        cx, cy = c & 0xFFFF, c >> 16
        dist = np.abs(cx - X) + np.abs(cy - y)
        want = int(c[np.lexsort((c, dist))[0]])
        got, s = packed_label_manhattan(X, y, c)
        assert got == want, (X, y, d.tolist())
        assert s >> 16 == int(dist.min())
