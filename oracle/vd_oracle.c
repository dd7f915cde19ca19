/*
 * vd_oracle.c -- plain, slow, obviously correct CPU oracle for the dJFA hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no code,
 * header, table or constant with the CUDA path (paper_2209_00117_b200/), and the
 * CUDA path never loads it.
 *
 * Source: /root/reference/PAPER.md ("P:n" = line n), arXiv 2209.00117.
 * Readings of ambiguous passages are the R-n entries of DESIGN.md §3.
 *
 * Conventions:
 *   pixel p = (x, y), 0 <= x, y < N, stored row-major at index y*N + x;
 *   a label is the packed position of the claimed seed, P(x, y) = (y << 16) | x (R-1);
 *   EMPTY = 0xFFFFFFFF (R-4);
 *   d2(p, c) = (x - cx)^2 + (y - cy)^2 computed in uint64 (R-2, exact for all N <= 65536);
 *   key(p, c) = (d2(p, c), c) compared lexicographically; key(p, EMPTY) = +infinity (R-3).
 *
 * Every loop is the literal definition.  OpenMP only splits independent output pixels
 * across threads ("parallel GPU threads ... mapped to the VD pixels using a
 * one-to-one correspondence"); the result does not depend on the split.
 */
#include "vd_oracle.h"

#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------- labels */

uint32_t or_pack(uint32_t x, uint32_t y) { return (y << 16) | x; }
static uint32_t label_x(uint32_t c) { return c & 0xFFFFu; }
static uint32_t label_y(uint32_t c) { return c >> 16; }

/* squared Euclidean distance between pixel (x, y) and the seed packed in label c,
 * in uint64 (Euclidean is the default metric). */
static uint64_t dist2(uint32_t x, uint32_t y, uint32_t c) {
    int64_t dx = (int64_t)x - (int64_t)label_x(c);
    int64_t dy = (int64_t)y - (int64_t)label_y(c);
    return (uint64_t)(dx * dx) + (uint64_t)(dy * dy);
}

/* Manhattan distance |dx| + |dy| (dJFAm: "not having square roots neither
 * squared values"). */
static uint64_t dist1(uint32_t x, uint32_t y, uint32_t c) {
    int64_t dx = (int64_t)x - (int64_t)label_x(c);
    int64_t dy = (int64_t)y - (int64_t)label_y(c);
    return (uint64_t)(dx < 0 ? -dx : dx) + (uint64_t)(dy < 0 ? -dy : dy);
}

/* The distance a metric compares: OR_EUCLID -> squared Euclidean (same order as the
 * Euclidean distance), OR_MANHATTAN -> Manhattan. */
static uint64_t dist_m(uint32_t x, uint32_t y, uint32_t c, int metric) {
    return metric == OR_MANHATTAN ? dist1(x, y, c) : dist2(x, y, c);
}

/* Does candidate label c beat the current best label b at pixel (x, y)?
 * key(p, c) < key(p, b) lexicographically on (distance, label); EMPTY is +infinity (R-3, R-4).
 * "the distance function is used as a criterion to check which flood carries
 * the closest seed". */
static int better_m(uint32_t x, uint32_t y, uint32_t c, uint32_t b, int metric) {
    if (c == OR_EMPTY) return 0;
    if (b == OR_EMPTY) return 1;
    uint64_t dc = dist_m(x, y, c, metric), db = dist_m(x, y, b, metric);
    if (dc != db) return dc < db;
    return c < b;
}
static int better(uint32_t x, uint32_t y, uint32_t c, uint32_t b) { return better_m(x, y, c, b, OR_EUCLID); }

/* ---------------------------------------------------------------- schedules */

/* ceil(log2(N)) for N >= 1, by counting. */
static uint32_t ceil_log2(uint64_t n) {
    uint32_t e = 0;
    while (((uint64_t)1 << e) < n) e++;
    return e;
}

/* Eq. 2: k_i(N) = 2^(ceil(log2 N) - 1) / 2^(i-1), i = 1 .. until k_i = 1.
 * Reading R-5: N is the grid side.  Then `extras` trailing k = 1 passes (R-6). */
int or_jfa_schedule(uint32_t N, uint32_t extras, uint32_t* ks, int cap) {
    if (N < 2) return -1;
    uint32_t k1 = 1u << (ceil_log2(N) - 1);
    int n = 0;
    for (uint32_t k = k1; k >= 1; k /= 2) {
        if (n >= cap) return -1;
        ks[n++] = k;
    }
    for (uint32_t e = 0; e < extras; e++) {
        if (n >= cap) return -1;
        ks[n++] = 1;
    }
    return n;
}

/* Eq. 3-4, exact integer form (reading R-7):
 *   L_avg = sqrt(N*N/s);  delta_1 = 2^ceil(log2(max(2 L_avg, d_max)))
 *   2^e >= 2 L_avg  <=>  4^e >= 4 N^2 / s  <=>  s * 4^e >= 4 N^2   (all integers)
 *   e_L = min{ e >= 0 : s * 4^e >= 4 N^2 }
 *   e_d = ceil(log2 d_max)   (0 when d_max <= 1)
 *   e   = min(max(e_L, e_d), log2 k_1)   (cap at the JFA k_1: "never exceed the static schedule")
 * then delta_1 = 2^e halving to 1: e + 1 passes ("log2(delta_1)+1 generational steps"),
 * plus `extras` k = 1 passes ("An extra step may be included"). */
int or_djfa_schedule(uint32_t N, uint64_t s, uint32_t d_max, uint32_t extras, uint32_t* ks,
                     int cap) {
    if (N < 2 || s == 0) return -1;
    uint64_t four_n2 = 4ull * (uint64_t)N * (uint64_t)N; /* <= 2^34 */
    uint32_t e_L = 0;
    while (1) {
        /* s * 4^e_L >= 4 N^2 ?  (compare without overflow: 4^e_L <= 2^36 before stopping) */
        unsigned __int128 lhs = (unsigned __int128)s << (2 * e_L);
        if (lhs >= four_n2) break;
        e_L++;
    }
    uint32_t e_d = (d_max <= 1) ? 0 : ceil_log2(d_max);
    uint32_t e = e_L > e_d ? e_L : e_d;
    uint32_t log2_k1 = ceil_log2(N) - 1;
    if (e > log2_k1) e = log2_k1;
    int n = 0;
    for (int32_t i = (int32_t)e; i >= 0; i--) {
        if (n >= cap) return -1;
        ks[n++] = 1u << i;
    }
    for (uint32_t x = 0; x < extras; x++) {
        if (n >= cap) return -1;
        ks[n++] = 1;
    }
    return n;
}

/* ---------------------------------------------------------------- exact diagram */

/* Eq. 1: R_k = {x : d(x, P_k) <= d(x, P_j) for all j}.  Brute force: every
 * pixel scans every seed and keeps the minimum key (R-3 picks one region on ties). */
void or_exact_brute_m(uint32_t N, uint64_t s, const uint16_t* xy, int metric, uint32_t* out) {
#pragma omp parallel for schedule(static)
    for (int64_t y = 0; y < (int64_t)N; y++) {
        for (uint32_t x = 0; x < N; x++) {
            uint32_t best = OR_EMPTY;
            for (uint64_t i = 0; i < s; i++) {
                uint32_t c = or_pack(xy[2 * i], xy[2 * i + 1]);
                if (better_m(x, (uint32_t)y, c, best, metric)) best = c;
            }
            out[(uint64_t)y * N + x] = best;
        }
    }
}
void or_exact_brute(uint32_t N, uint64_t s, const uint16_t* xy, uint32_t* out) {
    or_exact_brute_m(N, s, xy, OR_EUCLID, out);
}

/* Same result as or_exact_brute (tests check equality), found faster: seeds are put in
 * square buckets of side bs; a pixel scans rings of buckets around its own bucket.  Every
 * seed in ring r >= 1 is at least (r-1)*bs + 1 pixels away along one axis, so once
 * ((r-1)*bs + 1)^2 > best d2 no farther ring can hold a key <= the best (ties included,
 * since the bound is strict). */
int or_exact_bucketed(uint32_t N, uint64_t s, const uint16_t* xy, uint32_t bs, uint32_t* out) {
    if (bs == 0) return -1;
    uint32_t nb = (N + bs - 1) / bs;
    uint64_t nbk = (uint64_t)nb * nb;
    uint64_t* start = (uint64_t*)calloc(nbk + 1, sizeof(uint64_t));
    uint32_t* items = (uint32_t*)malloc((s ? s : 1) * sizeof(uint32_t));
    uint64_t* fill = (uint64_t*)calloc(nbk, sizeof(uint64_t));
    if (!start || !items || !fill) { free(start); free(items); free(fill); return -2; }
    for (uint64_t i = 0; i < s; i++) start[(uint64_t)(xy[2 * i + 1] / bs) * nb + xy[2 * i] / bs + 1]++;
    for (uint64_t b = 0; b < nbk; b++) start[b + 1] += start[b];
    for (uint64_t i = 0; i < s; i++) {
        uint64_t b = (uint64_t)(xy[2 * i + 1] / bs) * nb + xy[2 * i] / bs;
        items[start[b] + fill[b]++] = or_pack(xy[2 * i], xy[2 * i + 1]);
    }
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t y = 0; y < (int64_t)N; y++) {
        for (uint32_t x = 0; x < N; x++) {
            int64_t bx = x / bs, by = y / bs;
            uint32_t best = OR_EMPTY;
            uint64_t bestd = 0;
            for (int64_t r = 0; r <= (int64_t)nb; r++) {
                if (best != OR_EMPTY && r >= 1) {
                    uint64_t lb = (uint64_t)(r - 1) * bs + 1;
                    if (lb * lb > bestd) break;
                }
                for (int64_t qy = by - r; qy <= by + r; qy++) {
                    if (qy < 0 || qy >= (int64_t)nb) continue;
                    for (int64_t qx = bx - r; qx <= bx + r; qx++) {
                        if (qx < 0 || qx >= (int64_t)nb) continue;
                        int64_t cheb = llabs(qx - bx) > llabs(qy - by) ? llabs(qx - bx) : llabs(qy - by);
                        if (cheb != r) continue; /* only the ring */
                        uint64_t b = (uint64_t)qy * nb + (uint64_t)qx;
                        for (uint64_t j = start[b]; j < start[b + 1]; j++) {
                            uint32_t c = items[j];
                            if (better(x, (uint32_t)y, c, best)) { best = c; bestd = dist2(x, (uint32_t)y, c); }
                        }
                    }
                }
            }
            out[(uint64_t)y * N + x] = best;
        }
    }
    free(start); free(items); free(fill);
    return 0;
}

/* ---------------------------------------------------------------- JFA */

/* Initial grid: every pixel EMPTY, then each seed's pixel holds its own packed position
 * ("StF works by defining the positions as the starting points for each flood";
 * JFA starts the same way).  Co-located seeds write the same value. */
void or_init(uint32_t N, uint64_t s, const uint16_t* xy, uint32_t* G) {
    for (uint64_t p = 0; p < (uint64_t)N * N; p++) G[p] = OR_EMPTY;
    for (uint64_t i = 0; i < s; i++)
        G[(uint64_t)xy[2 * i + 1] * N + xy[2 * i]] = or_pack(xy[2 * i], xy[2 * i + 1]);
}

/* Table 1: the 8 Moore neighbours at range k, in the table's order. */
static const int MOORE[8][2] = {{+1, 0}, {+1, +1}, {0, +1}, {-1, +1},
                                {-1, 0}, {-1, -1}, {0, -1}, {+1, -1}};

/* One jump-flooding pass with step k, gather form on two buffers (reading R-12):
 *   out[p] = argmin_key over {in[p]} U {in[p + o*k] : o in Table 1, p + o*k inside the grid}
 * Out-of-grid neighbours are skipped (R-11).  This is Alg. 1's per-pixel body
 * with the roles of p and q exchanged: pixel p takes the closest seed among
 * the seeds its neighbours carry (S:177 proves the equivalence; tests check it).
 * vn != 0: Von Neumann neighbourhood, the 4 axis offsets of Table 1 (neighbours 1, 3, 5,
 * 7; "explore half the neighbors compared to Moore").  metric: OR_EUCLID or
 * OR_MANHATTAN. */
void or_pass_v(uint32_t N, uint32_t k, int metric, int vn, const uint32_t* in, uint32_t* out) {
#pragma omp parallel for schedule(static)
    for (int64_t y = 0; y < (int64_t)N; y++) {
        for (int64_t x = 0; x < (int64_t)N; x++) {
            uint32_t best = in[(uint64_t)y * N + (uint64_t)x];
            for (int j = 0; j < 8; j++) {
                if (vn && (j & 1)) continue; /* Table 1 neighbours 2, 4, 6, 8 are diagonal */
                int64_t qx = x + (int64_t)MOORE[j][0] * k;
                int64_t qy = y + (int64_t)MOORE[j][1] * k;
                if (qx < 0 || qy < 0 || qx >= (int64_t)N || qy >= (int64_t)N) continue;
                uint32_t c = in[(uint64_t)qy * N + (uint64_t)qx];
                if (better_m((uint32_t)x, (uint32_t)y, c, best, metric)) best = c;
            }
            out[(uint64_t)y * N + (uint64_t)x] = best;
        }
    }
}
void or_pass(uint32_t N, uint32_t k, const uint32_t* in, uint32_t* out) { or_pass_v(N, k, OR_EUCLID, 0, in, out); }

/* Run the passes of ks[0..n) on G (in place, using `tmp` as the other buffer); the first
 * vn_waves passes use the Von Neumann neighbourhood, the rest Moore (P:170, P:188,
 * P:204 "Von Neumann for the first two waves, Moore for the rest"). */
static void run_passes_v(uint32_t N, const uint32_t* ks, int n, int metric, int vn_waves, uint32_t* G,
                         uint32_t* tmp) {
    uint64_t np = (uint64_t)N * N;
    for (int i = 0; i < n; i++) {
        or_pass_v(N, ks[i], metric, i < vn_waves, G, tmp);
        memcpy(G, tmp, np * sizeof(uint32_t));
    }
}

/* Full JFA: init, then passes k_1, ..., 1 (+ extras).  Returns #passes.
 * metric / vn_waves as in run_passes_v (Euclidean Moore JFA: OR_EUCLID, 0). */
int or_jfa_v(uint32_t N, uint64_t s, const uint16_t* xy, uint32_t extras, int metric, int vn_waves, uint32_t* G) {
    uint32_t ks[64];
    int n = or_jfa_schedule(N, extras, ks, 64);
    if (n < 0 || s == 0) return -1;
    uint32_t* tmp = (uint32_t*)malloc((uint64_t)N * N * sizeof(uint32_t));
    if (!tmp) return -2;
    or_init(N, s, xy, G);
    run_passes_v(N, ks, n, metric, vn_waves, G, tmp);
    free(tmp);
    return n;
}
int or_jfa(uint32_t N, uint64_t s, const uint16_t* xy, uint32_t extras, uint32_t* G) {
    return or_jfa_v(N, s, xy, extras, OR_EUCLID, 0, G);
}

/* Standard Flooding (Fig. 2a): from the seed pixels, flood the neighbours at
 * Chebyshev distance 1 (Moore, k = 1) in parallel, pass after pass, "until the grid is
 * fully flooded" -- i.e. stop after the first pass that leaves no EMPTY pixel (reading
 * R-22).  Returns the number of passes (0 if the seeds already cover the grid). */
int or_stf(uint32_t N, uint64_t s, const uint16_t* xy, int metric, uint32_t* G) {
    if (s == 0) return -1;
    uint64_t np = (uint64_t)N * N;
    uint32_t* tmp = (uint32_t*)malloc(np * sizeof(uint32_t));
    if (!tmp) return -2;
    or_init(N, s, xy, G);
    int passes = 0;
    while (1) {
        uint64_t empty = 0;
        for (uint64_t p = 0; p < np; p++) empty += (G[p] == OR_EMPTY);
        if (empty == 0) break;
        or_pass_v(N, 1, metric, 0, G, tmp);
        memcpy(G, tmp, np * sizeof(uint32_t));
        passes++;
    }
    free(tmp);
    return passes;
}

/* ---------------------------------------------------------------- dJFA */

/* SimulateParticles (Alg. 1): new = old + disp, clamped to the grid per axis
 * (reading R-10: P:145 bounds moves by d_max; clamp, not wrap).  At N = 65536 the pixel
 * (65535, 65535) is the EMPTY sentinel and is reserved: a seed landing there goes to
 * (65534, 65535) (reading R-4). */
void or_move(uint32_t N, uint64_t s, const uint16_t* xy_old, const int16_t* disp, uint16_t* xy_new) {
    for (uint64_t i = 0; i < s; i++) {
        int64_t x = (int64_t)xy_old[2 * i] + disp[2 * i];
        int64_t y = (int64_t)xy_old[2 * i + 1] + disp[2 * i + 1];
        if (x < 0) x = 0;
        if (y < 0) y = 0;
        if (x > (int64_t)N - 1) x = (int64_t)N - 1;
        if (y > (int64_t)N - 1) y = (int64_t)N - 1;
        if (N == 65536 && x == 65535 && y == 65535) x = 65534;
        xy_new[2 * i] = (uint16_t)x;
        xy_new[2 * i + 1] = (uint16_t)y;
    }
}

/* One dJFA time step (Alg. 1 body P:185-199; state reuse P:117-122; reading R-9):
 *   1. move the seeds (or_move);
 *   2. fwd[P(old_i)] = min over {j : old_j = old_i} of P(new_j)      (labels follow seeds)
 *   3. G[p] <- fwd[G[p]] for every pixel (G must be complete: every label an old seed)
 *   4. G[P(new_i)] <- P(new_i)                                         (re-stamp)
 *   5. passes delta_1, ..., 1 (+ extras) from Eq. 4, as or_pass_v (metric; the first
 *      vn_waves of them Von Neumann).
 * Returns the number of passes, or -3 if G held a label that is not an old seed position
 * ("rejects incomplete prev"). */
int or_djfa_step_v(uint32_t N, uint64_t s, const uint16_t* xy_old, const int16_t* disp, uint32_t d_max,
                   uint32_t extras, int metric, int vn_waves, uint32_t* G, uint16_t* xy_new) {
    uint32_t ks[64];
    int n = or_djfa_schedule(N, s, d_max, extras, ks, 64);
    if (n < 0) return -1;
    uint64_t np = (uint64_t)N * N;
    uint32_t* fwd = (uint32_t*)malloc(np * sizeof(uint32_t));
    uint32_t* tmp = (uint32_t*)malloc(np * sizeof(uint32_t));
    if (!fwd || !tmp) { free(fwd); free(tmp); return -2; }

    or_move(N, s, xy_old, disp, xy_new);

    for (uint64_t p = 0; p < np; p++) fwd[p] = OR_EMPTY;
    for (uint64_t i = 0; i < s; i++) {
        uint32_t o = or_pack(xy_old[2 * i], xy_old[2 * i + 1]);
        uint32_t nw = or_pack(xy_new[2 * i], xy_new[2 * i + 1]);
        uint64_t at = (uint64_t)label_y(o) * N + label_x(o);
        if (nw < fwd[at]) fwd[at] = nw;
    }

    int bad = 0;
    for (uint64_t p = 0; p < np; p++) {
        uint32_t c = G[p];
        uint32_t f = OR_EMPTY;
        if (c != OR_EMPTY && label_x(c) < N && label_y(c) < N)
            f = fwd[(uint64_t)label_y(c) * N + label_x(c)];
        if (f == OR_EMPTY) bad = 1;
        G[p] = f;
    }
    if (bad) { free(fwd); free(tmp); return -3; }

    for (uint64_t i = 0; i < s; i++)
        G[(uint64_t)xy_new[2 * i + 1] * N + xy_new[2 * i]] = or_pack(xy_new[2 * i], xy_new[2 * i + 1]);

    run_passes_v(N, ks, n, metric, vn_waves, G, tmp);
    free(fwd); free(tmp);
    return n;
}

int or_djfa_step(uint32_t N, uint64_t s, const uint16_t* xy_old, const int16_t* disp,
                 uint32_t d_max, uint32_t extras, uint32_t* G, uint16_t* xy_new) {
    return or_djfa_step_v(N, s, xy_old, disp, d_max, extras, OR_EUCLID, 0, G, xy_new);
}

/* ---------------------------------------------------------------- metrics */

/* Eq. 5 numerator: number of pixels whose labels are equal. */
uint64_t or_match_count(uint64_t np, const uint32_t* a, const uint32_t* b) {
    uint64_t m = 0;
    for (uint64_t p = 0; p < np; p++) m += (a[p] == b[p]);
    return m;
}

/* Order-independent checksum of a label map (not from the paper; used to compare whole
 * diagrams by one number): sum over p of fmix32((uint32)(p * 0x9E3779B9) ^ label[p])
 * in uint64, with fmix32 the MurmurHash3 32-bit finaliser. */
static uint32_t fmix32(uint32_t h) {
    h ^= h >> 16;
    h *= 0x85EBCA6Bu;
    h ^= h >> 13;
    h *= 0xC2B2AE35u;
    h ^= h >> 16;
    return h;
}
uint64_t or_label_hash(uint64_t np, const uint32_t* g) {
    uint64_t h = 0;
    for (uint64_t p = 0; p < np; p++) h += fmix32((uint32_t)(p * 0x9E3779B9u) ^ g[p]);
    return h;
}

int or_num_threads(void) {
#ifdef _OPENMP
    extern int omp_get_max_threads(void);
    return omp_get_max_threads();
#else
    return 1;
#endif
}
