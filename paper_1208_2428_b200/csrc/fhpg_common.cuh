// fhpg_common.cuh — node encoding and the counter RNG, bit-exact with the
// reference (proj/core/include/fhp/node_state.hpp, rng.hpp), usable from host
// and device code.
#pragma once
#include <cstdint>

#if defined(__CUDACC__)
#define FHPG_HD __host__ __device__ __forceinline__
#else
#define FHPG_HD inline
#endif

namespace fhpg {

// node_state.hpp:13-15
constexpr uint32_t kMovingMask = 0x3F;
constexpr uint32_t kRestBit = 0x40;
constexpr uint32_t kObstacleBit = 0x80;

// rng.hpp:11, :13
enum Purpose : uint64_t { kInit = 0, kForcing = 1, kChirality = 2 };
constexpr uint64_t kGamma = 0x9E3779B97F4A7C15ull;
constexpr uint64_t kC1 = 0xBF58476D1CE4E5B9ull;
constexpr uint64_t kC2 = 0x94D049BB133111EBull;

// rng.hpp:15-23 — splitmix64 finaliser, split as mix64(z) = fin64(z + gamma)
// so the "+ gamma" can be folded into per-column precomputed keys.
FHPG_HD uint64_t fin64(uint64_t z) {
  z ^= z >> 30;
  z *= kC1;
  z ^= z >> 27;
  z *= kC2;
  z ^= z >> 31;
  return z;
}
FHPG_HD uint64_t mix64(uint64_t z) { return fin64(z + kGamma); }

// rng.hpp:25-33
FHPG_HD uint64_t node_random(uint64_t seed, uint64_t purpose, uint64_t step, uint64_t x,
                             uint64_t y) {
  uint64_t z = mix64(seed + kGamma * purpose);
  z = mix64(z + step);
  z = mix64(z + x);
  return mix64(z + y);
}

// Per-(purpose, step) prefix of node_random: mix64(mix64(seed+g*p)+step).
FHPG_HD uint64_t step_key(uint64_t seed, uint64_t purpose, uint64_t step) {
  return mix64(mix64(seed + kGamma * purpose) + step);
}

// Per-column key: node_random(seed,p,step,x,y) == fin64(column_key + y).
FHPG_HD uint64_t column_key(uint64_t step_key_value, uint64_t x) {
  return mix64(step_key_value + x) + kGamma;
}

// Bit 0 of fin64(z), computing only what that bit depends on: bit 0 of the
// result is bit0 ^ bit31 of z2 = z1' * C2, whose low 32 bits depend only on
// the low 32 bits of z1' = z1 ^ (z1 >> 27).
FHPG_HD uint32_t fin64_bit0(uint64_t z) {
  z ^= z >> 30;
  z *= kC1;
  const uint32_t lo = static_cast<uint32_t>(z) ^ static_cast<uint32_t>(z >> 27);
  const uint32_t p = lo * static_cast<uint32_t>(kC2);
  return (p ^ (p >> 31)) & 1u;
}

// The same bit with fewer ALU-pipe instructions (the step kernel's
// bottleneck). With lo, hi the words of z:
//   lo32(z ^ z >> 30) = lo ^ (lo >> 30) ^ (hi << 2)
//   hi32(z ^ z >> 30) = hi ^ (hi >> 30),
// z1 = (z ^ z >> 30) * C1 is one IMAD.WIDE of the low word plus two IMADs
// into its high word, and bit0(p) ^ bit31(p) of p = lo32(z1 ^ z1 >> 27) *
// lo32(C2) is the sign bit of p * (1 + 2^31) = lo32(z1 ^ z1 >> 27) * kC2s.
// `four` = 4, passed at run time, keeps hi << 2 an IMAD (FMA pipe).
constexpr uint32_t kC2s = static_cast<uint32_t>(kC2) * 0x80000001u;
FHPG_HD uint32_t chir_bit(uint64_t z, uint32_t four) {
  const uint32_t lo = static_cast<uint32_t>(z), hi = static_cast<uint32_t>(z >> 32);
  const uint32_t zl = lo ^ (lo >> 30) ^ (hi * four);
  const uint32_t g = (hi ^ (hi >> 30)) * static_cast<uint32_t>(kC1);
  const uint64_t w = static_cast<uint64_t>(zl) * static_cast<uint32_t>(kC1) +
                     (static_cast<uint64_t>(g) << 32);
  const uint32_t z1lo = static_cast<uint32_t>(w);
  const uint32_t z1hi = static_cast<uint32_t>(w >> 32) + zl * static_cast<uint32_t>(kC1 >> 32);
  const uint32_t lo2 = z1lo ^ ((z1lo >> 27) | (z1hi << 5));
  return (lo2 * kC2s) >> 31;
}
// The same bit as a mask: 0 or ~0u (arithmetic shift of the sign).
FHPG_HD uint32_t chir_mask(uint64_t z, uint32_t four) {
  const uint32_t lo = static_cast<uint32_t>(z), hi = static_cast<uint32_t>(z >> 32);
  const uint32_t zl = lo ^ (lo >> 30) ^ (hi * four);
  const uint32_t g = (hi ^ (hi >> 30)) * static_cast<uint32_t>(kC1);
  const uint64_t w = static_cast<uint64_t>(zl) * static_cast<uint32_t>(kC1) +
                     (static_cast<uint64_t>(g) << 32);
  const uint32_t z1lo = static_cast<uint32_t>(w);
  const uint32_t z1hi = static_cast<uint32_t>(w >> 32) + zl * static_cast<uint32_t>(kC1 >> 32);
  const uint32_t lo2 = z1lo ^ ((z1lo >> 27) | (z1hi << 5));
  return static_cast<uint32_t>(static_cast<int32_t>(lo2 * kC2s) >> 31);
}

// Column terms precomputed per (column, key base row b): with K = column key
// + b, lo/hi its words, a site at row b + dy has z = K + dy. While lo + dy
// stays inside the same 2^30-aligned block as lo (no carry into the high
// word, same lo >> 30), the hash inputs that depend on the column alone fold
// into two words:
//   t2 = (hi << 2) ^ (lo >> 30)          so lo32(z ^ z >> 30) = (lo + dy) ^ t2
//   g  = lo32((hi ^ hi >> 30) * C1)      the high word's share of z1's high word
// (dy < colkey_span(lo) guarantees it; other rows take the full hash).
struct ColKey {
  uint32_t lo, t2, g;
};
FHPG_HD ColKey col_key_terms(uint64_t K) {
  const uint32_t lo = static_cast<uint32_t>(K), hi = static_cast<uint32_t>(K >> 32);
  return {lo, (hi << 2) ^ (lo >> 30), (hi ^ (hi >> 30)) * static_cast<uint32_t>(kC1)};
}
// Rows dy in [0, span) keep lo + dy inside lo's 2^30-aligned block.
FHPG_HD uint32_t colkey_span(uint32_t lo) { return (1u << 30) - (lo & ((1u << 30) - 1u)); }
// z1 = (z ^ z >> 30) * C1 from the folded terms: (low word, high word).
FHPG_HD void colkey_z1(uint32_t l, uint32_t t2, uint32_t g, uint32_t& z1lo, uint32_t& z1hi) {
  const uint32_t zl = l ^ t2;
  const uint64_t w = static_cast<uint64_t>(zl) * static_cast<uint32_t>(kC1);
  z1lo = static_cast<uint32_t>(w);
  z1hi = static_cast<uint32_t>(w >> 32) + zl * static_cast<uint32_t>(kC1 >> 32) + g;
}
// Chirality mask (0 or ~0u) of the site at dy: bit 0 of fin64(K + dy).
FHPG_HD uint32_t chir_mask_pre(uint32_t l, uint32_t t2, uint32_t g) {
  uint32_t z1lo, z1hi;
  colkey_z1(l, t2, g, z1lo, z1hi);
  const uint32_t lo2 = z1lo ^ ((z1lo >> 27) | (z1hi << 5));
  return static_cast<uint32_t>(static_cast<int32_t>(lo2 * kC2s) >> 31);
}
// High word of z2 = (z1 ^ z1 >> 27) * C2, the last product of fin64(K + dy).
FHPG_HD uint32_t fin64_z2hi_pre(uint32_t l, uint32_t t2, uint32_t g) {
  uint32_t z1lo, z1hi;
  colkey_z1(l, t2, g, z1lo, z1hi);
  const uint32_t ulo = z1lo ^ ((z1lo >> 27) | (z1hi << 5));
  const uint32_t uhi = z1hi ^ (z1hi >> 27);
  return static_cast<uint32_t>((static_cast<uint64_t>(ulo) * static_cast<uint32_t>(kC2)) >> 32) +
         ulo * static_cast<uint32_t>(kC2 >> 32) + uhi * static_cast<uint32_t>(kC2);
}
// High word of fin64(K + dy) (the forcing draw, rng.hpp:37-42). For a
// bernoulli threshold thr <= 2^31, (hi < thr) == (z2hi < thr): z2hi >= 2^31
// gives hi >= 2^31 >= thr, else hi = z2hi.
FHPG_HD uint32_t fin64_hi_pre(uint32_t l, uint32_t t2, uint32_t g) {
  const uint32_t z2hi = fin64_z2hi_pre(l, t2, g);
  return z2hi ^ (z2hi >> 31);
}

// rng.hpp:37-42: bernoulli(word, p) == (word >> 32) < threshold(p).
inline uint64_t bernoulli_threshold(double p) {
  return p >= 1.0 ? (1ull << 32) : static_cast<uint64_t>(p * 4294967296.0);
}

}  // namespace fhpg
