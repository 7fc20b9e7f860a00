/* fhp_oracle.h — TEST INFRASTRUCTURE ONLY: plain-C restatement of the
 * reference FHP path used as the parity checker. See fhp_oracle.c. */
#ifndef FHP_ORACLE_H
#define FHP_ORACLE_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

uint64_t fo_mix64(uint64_t z);
uint64_t fo_node_random(uint64_t seed, uint64_t purpose, uint64_t step, uint64_t x, uint64_t y);
uint64_t fo_bernoulli_threshold(double p);
int fo_bernoulli(uint64_t word, uint64_t threshold);
void fo_build_default_table(uint8_t* t512);
int fo_validate_table(const uint8_t* t512);
void fo_init(int W, int H, uint64_t seed, double density, const uint8_t* mask, uint8_t* out);
uint64_t fo_advance(int W, int H, uint8_t* state, const uint8_t* mask, const uint8_t* table,
                    uint64_t seed, uint64_t force_thr, int64_t first_step, int64_t step_count);
uint64_t fo_digest(int W, int H, const uint8_t* state);
void fo_global(int W, int H, const uint8_t* state, int64_t* mass, int64_t* px, int64_t* py);
void fo_cells(int W, int H, const uint8_t* state, int B, int32_t* nodes, int32_t* particles,
              int64_t* px, int64_t* py);
void fo_rows(int W, int H, const uint8_t* state, int64_t* px, int32_t* fluid);
void fo_scramble(int W, int H, uint64_t seed, uint8_t* state, uint8_t* mask);
void fo_cylinder(int W, int H, double cx, double cy, double R, uint8_t* mask);
uint64_t fo_step_strip(int W, int H, int row0, int nrows, const uint8_t* src, const uint8_t* mask,
                       const uint8_t* table, uint64_t seed, uint64_t thr, uint64_t step,
                       uint8_t* dst);

#ifdef __cplusplus
}
#endif
#endif
