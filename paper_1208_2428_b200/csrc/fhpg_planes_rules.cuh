// fhpg_planes_rules.cuh — collision rules as bit-sliced logic for the
// bit-plane step kernel (fhpg_step_planes.cu): every word holds one bit of 32
// sites, one word per direction plane.
//
// Each rule is split in two phases because chirality is drawn lazily:
//   classify(a, r, solid) -> per-site class masks and `dep`, the sites whose
//                           outcome depends on the chirality bit;
//   apply(class, c)       -> the outgoing movers and rest, given the chirality
//                           word c (only bits set in dep are read).
// tests/test_planes_rules (tools/planes_rules_check.cpp) checks every rule
// exhaustively (all 2^9 (movers, rest, obstacle) states x both chiralities)
// against the 512-entry table the engine would otherwise use.
//
// FHP-III (definition: fhpg_fhp3_logic.cuh) written for a small circuit:
//  * The rule is particle-hole self-dual with the same chirality,
//    f(s, c) = ~f(~s, c) (checked by the tool), so sites holding 4 or more of
//    the 7 particles are complemented on the way in and out (D below) and the
//    rest of the circuit only distinguishes states of mass <= 3.
//  * With mass <= 3 and axis signals O_k (odd axis) the classes are: no odd
//    axis (head-on pair, +-60 deg rotation by chirality); symmetric triple or
//    obstacle (bounce-back, o_k = a_{k+3}); one odd axis + a pair (X states:
//    either the pair moves to the empty axis, o_k = ~a_{k+3}, or the state
//    goes to Y); one mover + rest (B -> A); two movers 120 deg apart without
//    rest (A -> B) or with rest (Y -> X); anything else is kept.
//  * Outcomes per plane k, in terms of neighbouring planes:
//      rotation  rot_k = c ? a_{k-1} : a_{k+1}
//      A -> B    a_{k-1} & a_{k+1}
//      B -> A and X -> Y   v_{k-1} | v_{k+1},  v_j = a_j & ~a_{j+3} (the odd mover)
//      Y -> X    a_{k-1} & a_{k+1} | a_k & rot_{k+3} | a_{k+3} & rot_k
#pragma once
#include <cstdint>

#include "fhpg_common.cuh"

namespace fhpg {

// Three-input boolean function as one LOP3; LUT = f(0xF0, 0xCC, 0xAA) & 0xFF.
constexpr uint32_t kLA = 0xF0, kLB = 0xCC, kLC = 0xAA;
#define FHPG_LUT(expr) ((expr) & 0xFFu)
template <uint32_t LUT>
FHPG_HD uint32_t lop3(uint32_t a, uint32_t b, uint32_t c) {
#if defined(__CUDA_ARCH__)
  uint32_t d;
  asm("lop3.b32 %0, %1, %2, %3, %4;" : "=r"(d) : "r"(a), "r"(b), "r"(c), "n"(LUT));
  return d;
#else
  uint32_t d = 0;
  for (int m = 0; m < 8; ++m)
    if ((LUT >> m) & 1u) d |= ((m & 4) ? a : ~a) & ((m & 2) ? b : ~b) & ((m & 1) ? c : ~c);
  return d;
#endif
}
constexpr uint32_t kMaj = FHPG_LUT((kLA & kLB) | (kLA & kLC) | (kLB & kLC));
constexpr uint32_t kXor3 = FHPG_LUT(kLA ^ kLB ^ kLC);
constexpr uint32_t kOr3 = FHPG_LUT(kLA | kLB | kLC);
constexpr uint32_t kNor3 = FHPG_LUT(~(kLA | kLB | kLC));
constexpr uint32_t kAndOr = FHPG_LUT((kLA & kLB) | kLC);          // (a & b) | c
constexpr uint32_t kMux = FHPG_LUT((kLA & kLB) | (~kLA & kLC));   // a ? b : c
// Reduced pair / reduced a_i & a_j: c ? ~(a | b) : a & b (c = D).
constexpr uint32_t kRedAnd = FHPG_LUT((kLC & ~(kLA | kLB)) | (~kLC & kLA & kLB));
// Reduced single: c ? ~a & b : a & ~b.
constexpr uint32_t kRedSingle = FHPG_LUT((kLC & ~kLA & kLB) | (~kLC & kLA & ~kLB));

// FHP-III, phase 1 output: class masks kept across the chirality walk.
struct Fhp3Class {
  uint32_t D;      // sites with mass >= 4 (complemented)
  uint32_t ROT, BB, X, B, AY, xp;  // (keep = none of them: the apply muxes' default)
  uint32_t YE[3];  // Y sites whose axis m is empty (no odd mover)
  uint32_t dep;
};

FHPG_HD Fhp3Class fhp3_classify(const uint32_t a[6], uint32_t r, uint32_t s) {
  Fhp3Class k;
  // mass >= 4 of the 7 bits: carries of three full adders, then a majority.
  const uint32_t c1 = lop3<kMaj>(a[0], a[1], a[2]), c2 = lop3<kMaj>(a[3], a[4], a[5]);
  const uint32_t s1 = lop3<kXor3>(a[0], a[1], a[2]), s2 = lop3<kXor3>(a[3], a[4], a[5]);
  const uint32_t c3 = lop3<kMaj>(s1, s2, r);
  const uint32_t D = lop3<kMaj>(c1, c2, c3);
  k.D = D;
  // Axis signals: O (odd axis) is unchanged by the reduction; a pair of the
  // reduced state is a pair (D = 0) or an empty axis (D = 1) of the original.
  // Obstacle sites count every axis as odd (O_k |= s): no fluid class
  // (ROT, X, B, AY: none or one or two odd axes) then needs its own ~s.
  constexpr uint32_t kOddOrS = FHPG_LUT((kLA ^ kLB) | kLC);
  const uint32_t O0 = lop3<kOddOrS>(a[0], a[3], s), O1 = lop3<kOddOrS>(a[1], a[4], s),
                 O2 = lop3<kOddOrS>(a[2], a[5], s);
  const uint32_t P0 = lop3<kRedAnd>(a[0], a[3], D);
  const uint32_t P1 = lop3<kRedAnd>(a[1], a[4], D);
  const uint32_t P2 = lop3<kRedAnd>(a[2], a[5], D);
  const uint32_t anyP = lop3<kOr3>(P0, P1, P2);
  k.ROT = lop3<kNor3>(O0, O1, O2);
  const uint32_t ex1 = lop3<FHPG_LUT((kLA ^ kLB ^ kLC) & ~(kLA & kLB & kLC))>(O0, O1, O2);
  const uint32_t ex2 = lop3<FHPG_LUT(((kLA & kLB) | (kLA & kLC) | (kLB & kLC)) & ~(kLA & kLB & kLC))>(O0, O1, O2);
  const uint32_t O3 = lop3<FHPG_LUT(kLA & kLB & kLC)>(O0, O1, O2);
  // Three odd axes (3 movers, no rest): a symmetric triple iff a0 == a2 == a4
  // (invariant under the reduction). Obstacles bounce back too.
  const uint32_t eqv = lop3<FHPG_LUT((kLA & kLB & kLC) | (~kLA & ~kLB & ~kLC))>(a[0], a[2], a[4]);
  k.BB = lop3<FHPG_LUT(kLB & (kLA | kLC))>(s, O3, eqv);  // O3 & (eqv | s)
  // One odd axis, fluid: with a pair X, without one B (B needs the reduced
  // rest, r ^ D).
  k.X = ex1 & anyP;
  const uint32_t exn = ex1 & ~anyP;
  k.B = lop3<FHPG_LUT(kLA & (kLB ^ kLC))>(exn, r, D);
  // Two odd axes with movers 120 deg apart <=> both on directions of the
  // same parity <=> an even number of singles on odd directions. With two
  // odd axes the third axis is empty (reduced), i.e. a pair when D = 1, so
  // that parity is a1 ^ a3 ^ a5 ^ D.
  const uint32_t pi = lop3<kXor3>(a[1], a[3], a[5]);
  k.AY = lop3<FHPG_LUT(kLA & ~(kLB ^ kLC))>(ex2, pi, D);
  const uint32_t Y = lop3<FHPG_LUT(kLA & (kLB ^ kLC))>(k.AY, r, D);
  k.YE[0] = Y & ~O0;
  k.YE[1] = Y & ~O1;
  k.YE[2] = Y & ~O2;
  // X states (one odd axis o, one pair): the pair's axis is o + 1 (X+) or
  // o - 1 (X-).
  k.xp = lop3<kMux>(O0, P1, lop3<kMux>(O1, P2, P0));
  const uint32_t d1 = lop3<kAndOr>(k.ROT, anyP, k.X);
  k.dep = d1 | Y;
  return k;
}

// a: the original movers (as passed to fhp3_classify), r: the original rest.
FHPG_HD void fhp3_apply(const Fhp3Class& k, uint32_t c, uint32_t r, const uint32_t a[6],
                        uint32_t o[6], uint32_t& o_r) {
  // X -> Y for X+ with c = 1 and X- with c = 0; otherwise the pair moves.
  const uint32_t NX = lop3<FHPG_LUT(kLA & (kLB ^ kLC))>(k.X, k.xp, c);
  const uint32_t U = lop3<FHPG_LUT((kLA & ~kLB) | kLC)>(k.X, NX, k.B);
  const uint32_t UAY = U | k.AY;
  // Permutation classes act on the original movers (the reduction cancels):
  // rotation (c ? a_{k-1} : a_{k+1}), bounce-back / pair move (a_{k+3}, NX
  // complemented by DN), keep (a_k). U / AY classes use reduced movers and
  // are complemented back with D.
  const uint32_t S3 = k.BB | NX;
  const uint32_t DN = lop3<FHPG_LUT(kLA | (kLB & kLC))>(NX, k.D, UAY);
  uint32_t v[6];
#pragma unroll
  for (int i = 0; i < 6; ++i)
    v[i] = lop3<kRedSingle>(a[i], a[(i + 3) % 6], k.D);  // reduced: odd mover of its axis
  // Y = {j-1, j+1} + R -> X: the pair lands on the axis of j+1 (c = 0) or
  // j-1 (c = 1), i.e. one (c = 0: two) axes after the empty axis j.
  uint32_t PA[3];
#pragma unroll
  for (int m = 0; m < 3; ++m) PA[m] = lop3<kMux>(c, k.YE[(m + 1) % 3], k.YE[(m + 2) % 3]);
  // The permutation classes as three muxes per direction: keep (a_i) or
  // bounce-back / pair move (a_{i+3}) by S3, the rotation by the chirality
  // (c ? a_{i-1} : a_{i+1}), one of the two by ROT; U / AY sites override.
#pragma unroll
  for (int i = 0; i < 6; ++i) {
    const uint32_t m1 = lop3<kMux>(S3, a[(i + 3) % 6], a[i]);
    const uint32_t rot = lop3<kMux>(c, a[(i + 5) % 6], a[(i + 1) % 6]);
    const uint32_t m = lop3<kMux>(k.ROT, rot, m1);
    // B -> A, X -> Y: v_{i-1} | v_{i+1}; A -> B (and Y's single): v_{i-1} & v_{i+1}
    const uint32_t q = lop3<FHPG_LUT((kLC & kLA & kLB) | (~kLC & (kLA | kLB)))>(
        v[(i + 5) % 6], v[(i + 1) % 6], k.AY);
    const uint32_t x = lop3<kMux>(UAY, q, m);
    o[i] = lop3<FHPG_LUT((kLA | kLB) ^ kLC)>(x, PA[i % 3], DN);
  }
  // The rest flips exactly for B -> A, X -> Y, A -> B, Y -> X (unchanged by D).
  o_r = lop3<FHPG_LUT(kLA ^ (kLB | kLC))>(r, U, k.AY);
}

// The reference's own rule (RuleVariant::Default, collision.cpp:22-72) as a
// circuit, ~63 LOP3 per 32 sites. Fluid classes by axis signals O_k = a_k ^
// a_{k+3} (odd axis) and P_k = a_k & a_{k+3} (pair):
//   HO head-on pair, no rest (no odd axis, exactly one pair): rotate by 1
//      (chirality 1) or 2 (chirality 0)                      collision.cpp:29-31
//   TB symmetric triple, no rest (three odd axes, a0 == a2 == a4): complement
//                                                            collision.cpp:33-35
//   RA one mover + rest (one odd axis, no pair): {i}+R -> {i-1, i+1}  :37-41
//   RC two movers 120 deg apart, no rest (two odd axes, no pair, an even
//      number of them on odd directions): {i, i+2} -> {i+1}+R        :43-51
//   obstacles bounce back, rest kept                                   :59-63
// Only HO depends on the chirality. A symmetric triple has a_{i+3} = ~a_i on
// every axis, so TB and the obstacles share one selector S3 (out_i =
// a_{i+3}); keep is the muxes' default.
struct DefClass {
  uint32_t HO, S3, RA, RC, RARC;
  uint32_t dep;
};

FHPG_HD DefClass def_classify(const uint32_t a[6], uint32_t r, uint32_t s) {
  DefClass k;
  const uint32_t O0 = a[0] ^ a[3], O1 = a[1] ^ a[4], O2 = a[2] ^ a[5];
  const uint32_t P0 = a[0] & a[3], P1 = a[1] & a[4], P2 = a[2] & a[5];
  const uint32_t rs = r | s;
  constexpr uint32_t kOne = FHPG_LUT((kLA ^ kLB ^ kLC) & ~(kLA & kLB & kLC));
  constexpr uint32_t kTwo = FHPG_LUT(((kLA & kLB) | (kLA & kLC) | (kLB & kLC)) & ~(kLA & kLB & kLC));
  const uint32_t noO = lop3<kNor3>(O0, O1, O2);
  const uint32_t oneP = lop3<kOne>(P0, P1, P2);
  const uint32_t anyP = lop3<kOr3>(P0, P1, P2);
  const uint32_t ex1 = lop3<kOne>(O0, O1, O2);
  const uint32_t ex2 = lop3<kTwo>(O0, O1, O2);
  const uint32_t O3 = lop3<FHPG_LUT(kLA & kLB & kLC)>(O0, O1, O2);
  const uint32_t eqv = lop3<FHPG_LUT((kLA & kLB & kLC) | (~kLA & ~kLB & ~kLC))>(a[0], a[2], a[4]);
  const uint32_t pi = lop3<kXor3>(a[1], a[3], a[5]);
  constexpr uint32_t kAnB_nC = FHPG_LUT(kLA & kLB & ~kLC);
  k.HO = lop3<kAnB_nC>(noO, oneP, rs);
  k.S3 = lop3<kAnB_nC>(O3, eqv, rs) | s;
  k.RA = lop3<FHPG_LUT(kLA & ~kLB & kLC)>(ex1, anyP, r) & ~s;
  k.RC = lop3<FHPG_LUT(kLA & ~kLB & ~kLC)>(ex2, anyP, rs) & ~pi;
  k.RARC = k.RA | k.RC;
  k.dep = k.HO;
  return k;
}

FHPG_HD void def_apply(const DefClass& k, uint32_t c, uint32_t r, const uint32_t a[6],
                       uint32_t o[6], uint32_t& o_r, uint32_t s) {
  (void)s;
#pragma unroll
  for (int i = 0; i < 6; ++i) {
    const uint32_t am1 = a[(i + 5) % 6], ap1 = a[(i + 1) % 6];
    const uint32_t m1 = lop3<kMux>(k.S3, a[(i + 3) % 6], a[i]);  // bounce / triple, or keep
    const uint32_t rot = lop3<kMux>(c, am1, a[(i + 4) % 6]);     // c ? a_{i-1} : a_{i-2}
    const uint32_t m = lop3<kMux>(k.HO, rot, m1);
    // RA: a_{i-1} | a_{i+1}; RC: a_{i-1} & a_{i+1}
    const uint32_t q = lop3<FHPG_LUT((kLC & kLA & kLB) | (~kLC & (kLA | kLB)))>(am1, ap1, k.RC);
    o[i] = lop3<kMux>(k.RARC, q, m);
  }
  o_r = lop3<FHPG_LUT((kLA & ~kLB) | kLC)>(r, k.RA, k.RC);
}

// FHP-I (fhpg_tables.cpp build_fhp1): head-on pairs without rest rotate by
// +60 (chirality 1) or -60 degrees (chirality 0), symmetric triples without
// rest complement, obstacles bounce back (one selector S3, out_i = a_{i+3});
// ~25 LOP3 per 32 sites.
struct Fhp1Class {
  uint32_t HO, S3;
  uint32_t dep;
};

FHPG_HD Fhp1Class fhp1_classify(const uint32_t a[6], uint32_t r, uint32_t s) {
  Fhp1Class k;
  const uint32_t O0 = a[0] ^ a[3], O1 = a[1] ^ a[4], O2 = a[2] ^ a[5];
  const uint32_t P0 = a[0] & a[3], P1 = a[1] & a[4], P2 = a[2] & a[5];
  const uint32_t rs = r | s;
  constexpr uint32_t kOne = FHPG_LUT((kLA ^ kLB ^ kLC) & ~(kLA & kLB & kLC));
  const uint32_t noO = lop3<kNor3>(O0, O1, O2);
  const uint32_t oneP = lop3<kOne>(P0, P1, P2);
  const uint32_t O3 = lop3<FHPG_LUT(kLA & kLB & kLC)>(O0, O1, O2);
  const uint32_t eqv = lop3<FHPG_LUT((kLA & kLB & kLC) | (~kLA & ~kLB & ~kLC))>(a[0], a[2], a[4]);
  constexpr uint32_t kAnB_nC = FHPG_LUT(kLA & kLB & ~kLC);
  k.HO = lop3<kAnB_nC>(noO, oneP, rs);
  k.S3 = lop3<kAnB_nC>(O3, eqv, rs) | s;
  k.dep = k.HO;
  return k;
}

FHPG_HD void fhp1_apply(const Fhp1Class& k, uint32_t c, uint32_t r, const uint32_t a[6],
                        uint32_t o[6], uint32_t& o_r, uint32_t s) {
  (void)s;
#pragma unroll
  for (int i = 0; i < 6; ++i) {
    const uint32_t rot = lop3<kMux>(c, a[(i + 5) % 6], a[(i + 1) % 6]);  // c ? a_{i-1} : a_{i+1}
    const uint32_t m1 = lop3<kMux>(k.S3, a[(i + 3) % 6], a[i]);
    o[i] = lop3<kMux>(k.HO, rot, m1);
  }
  o_r = r;
}

}  // namespace fhpg
