/* vd_oracle.h -- CPU oracle for the dJFA hot path.  TEST INFRASTRUCTURE ONLY.
 * Private to oracle/; the CUDA path (paper_2209_00117_b200/, include/vd.h) never includes it.
 * Semantics and citations: see vd_oracle.c. */
#ifndef VD_ORACLE_H
#define VD_ORACLE_H
#include <stdint.h>

#define OR_EMPTY 0xFFFFFFFFu
#define OR_EUCLID 0
#define OR_MANHATTAN 1

uint32_t or_pack(uint32_t x, uint32_t y);
int or_jfa_schedule(uint32_t N, uint32_t extras, uint32_t* ks, int cap);
int or_djfa_schedule(uint32_t N, uint64_t s, uint32_t d_max, uint32_t extras, uint32_t* ks, int cap);
void or_exact_brute(uint32_t N, uint64_t s, const uint16_t* xy, uint32_t* out);
int or_exact_bucketed(uint32_t N, uint64_t s, const uint16_t* xy, uint32_t bs, uint32_t* out);
void or_init(uint32_t N, uint64_t s, const uint16_t* xy, uint32_t* G);
void or_pass(uint32_t N, uint32_t k, const uint32_t* in, uint32_t* out);
void or_pass_v(uint32_t N, uint32_t k, int metric, int vn, const uint32_t* in, uint32_t* out);
void or_exact_brute_m(uint32_t N, uint64_t s, const uint16_t* xy, int metric, uint32_t* out);
int or_jfa_v(uint32_t N, uint64_t s, const uint16_t* xy, uint32_t extras, int metric, int vn_waves, uint32_t* G);
int or_djfa_step_v(uint32_t N, uint64_t s, const uint16_t* xy_old, const int16_t* disp, uint32_t d_max,
                   uint32_t extras, int metric, int vn_waves, uint32_t* G, uint16_t* xy_new);
int or_jfa(uint32_t N, uint64_t s, const uint16_t* xy, uint32_t extras, uint32_t* G);
void or_move(uint32_t N, uint64_t s, const uint16_t* xy_old, const int16_t* disp, uint16_t* xy_new);
int or_djfa_step(uint32_t N, uint64_t s, const uint16_t* xy_old, const int16_t* disp,
                 uint32_t d_max, uint32_t extras, uint32_t* G, uint16_t* xy_new);
uint64_t or_match_count(uint64_t np, const uint32_t* a, const uint32_t* b);
uint64_t or_label_hash(uint64_t np, const uint32_t* g);
int or_stf(uint32_t N, uint64_t s, const uint16_t* xy, int metric, uint32_t* G);
int or_num_threads(void);

#endif
