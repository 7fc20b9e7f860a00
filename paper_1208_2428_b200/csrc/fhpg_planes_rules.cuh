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

// FHP-III, phase 1 output.
struct Fhp3Class {
  uint32_t ap[6];  // movers after the particle-hole reduction
  uint32_t rp;     // rest after the reduction
  uint32_t D;      // sites with mass >= 4 (complemented)
  uint32_t ROT, BB, X, B, AY, KEEP, xp;
  uint32_t dep;
};

FHPG_HD uint32_t maj3(uint32_t a, uint32_t b, uint32_t c) { return (a & b) | (a & c) | (b & c); }

FHPG_HD Fhp3Class fhp3_classify(const uint32_t a[6], uint32_t r, uint32_t solid) {
  Fhp3Class k;
  // mass >= 4 of the 7 bits: carries of three full adders, then a majority.
  const uint32_t c1 = maj3(a[0], a[1], a[2]), c2 = maj3(a[3], a[4], a[5]);
  const uint32_t s1 = a[0] ^ a[1] ^ a[2], s2 = a[3] ^ a[4] ^ a[5];
  const uint32_t c3 = maj3(s1, s2, r);
  const uint32_t D = maj3(c1, c2, c3);
  k.D = D;
#pragma unroll
  for (int i = 0; i < 6; ++i) k.ap[i] = a[i] ^ D;
  k.rp = r ^ D;
  const uint32_t fl = ~solid;
  // Axis signals (O is unchanged by the reduction).
  const uint32_t O0 = a[0] ^ a[3], O1 = a[1] ^ a[4], O2 = a[2] ^ a[5];
  const uint32_t P0 = k.ap[0] & k.ap[3], P1 = k.ap[1] & k.ap[4], P2 = k.ap[2] & k.ap[5];
  const uint32_t anyP = P0 | P1 | P2;
  const uint32_t no0 = ~(O0 | O1 | O2);
  const uint32_t ex1 = (O0 ^ O1 ^ O2) & ~(O0 & O1 & O2);
  const uint32_t ex2 = maj3(O0, O1, O2) & ~(O0 & O1 & O2);
  const uint32_t O3 = O0 & O1 & O2;
  // Three odd axes (3 movers, no rest): a symmetric triple iff a0 == a2 == a4.
  const uint32_t eqv = ~((k.ap[0] ^ k.ap[2]) | (k.ap[2] ^ k.ap[4]));
  k.BB = solid | (O3 & eqv);
  k.ROT = no0 & fl;
  k.X = ex1 & anyP & fl;
  k.B = ex1 & ~anyP & k.rp & fl;
  // Two odd axes, movers 120 deg apart <=> both on the same sublattice.
  const uint32_t ev = k.ap[0] | k.ap[2] | k.ap[4], od = k.ap[1] | k.ap[3] | k.ap[5];
  k.AY = ex2 & (ev ^ od) & fl;
  k.KEEP = fl & ~(k.ROT | k.BB | k.X | k.B | k.AY);
  // X states: the pair's axis follows the odd axis (X+) or precedes it (X-).
  k.xp = (O0 & P1) | (O1 & P2) | (O2 & P0);
  k.dep = (k.ROT & anyP) | k.X | (k.AY & k.rp);
  return k;
}

FHPG_HD void fhp3_apply(const Fhp3Class& k, uint32_t c, uint32_t r, uint32_t o[6],
                        uint32_t& o_r) {
  const uint32_t* a = k.ap;
  // X -> Y for X+ with c = 1 and X- with c = 0; otherwise the pair moves.
  const uint32_t toY = ~(k.xp ^ c);
  const uint32_t NX = k.X & ~toY;
  const uint32_t U = (k.X & toY) | k.B;
  const uint32_t BNX = k.BB | NX;
  uint32_t rot[6], v[6];
#pragma unroll
  for (int i = 0; i < 6; ++i) {
    rot[i] = (c & a[(i + 5) % 6]) | (~c & a[(i + 1) % 6]);
    v[i] = a[i] & ~a[(i + 3) % 6];
  }
#pragma unroll
  for (int i = 0; i < 6; ++i) {
    const uint32_t am = a[(i + 5) % 6], apl = a[(i + 1) % 6], opp = a[(i + 3) % 6];
    const uint32_t t = am & apl;
    const uint32_t pp = (a[i] & rot[(i + 3) % 6]) | (opp & rot[i]);
    const uint32_t ay = t | (k.rp & pp);
    const uint32_t u = v[(i + 5) % 6] | v[(i + 1) % 6];
    const uint32_t acc = (k.ROT & rot[i]) | (BNX & (opp ^ NX)) | (U & u) | (k.AY & ay) |
                         (k.KEEP & a[i]);
    o[i] = acc ^ k.D;
  }
  // The rest flips exactly for B -> A, X -> Y, A -> B, Y -> X (unchanged by D).
  o_r = r ^ (U | k.AY);
}

}  // namespace fhpg
