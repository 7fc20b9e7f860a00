// fhpg_tables.cpp — collision-table generation and validation (host side).
//
// The reference ships one rule set, RuleVariant::Default (collision.hpp:12,
// collision.cpp:22-72): an FHP-II-like table. BASELINE's configs also name
// FHP-I and FHP-III; the reference has no such variants ("reserved for future
// variants"), so they are defined here in the reference's own
// 512-entry format (index (chirality << 8) | state) and enter the engine and
// the oracle as plain tables:
//
//  * FHP-I  — six movers, no rest particle: head-on pairs rotate by +-60
//             degrees by chirality, symmetric triples go to their complement
//             (the two original FHP collisions); every state with the rest
//             bit is left unchanged.
//  * FHP-III — collision-saturated with rest particle: every fluid state whose
//             (mass, momentum) class has another member moves to another
//             member, by the bit-sliced circuit of fhpg_fhp3_logic.cuh (the
//             table is that circuit evaluated per state). The rule commutes
//             with lattice rotations, and a mirror maps the chirality-0 rule
//             onto the chirality-1 rule.
//
// All variants use the reference's obstacle rule: full bounce-back keeping
// the rest and obstacle bits (collision.cpp:62-66).
#include <cstdint>

#include "../../include/fhpg_tables.h"
#include "fhpg_fhp3_logic.cuh"

namespace {

// node_state.hpp:54-61 integer momentum of each direction.
constexpr int kPx[6] = {-1, 1, 2, 1, -1, -2};
constexpr int kPy[6] = {1, 1, 0, -1, -1, 0};

unsigned rot(unsigned s, int by) {  // rotate the moving bits by `by` sixths, keep bit 6/7
  by = ((by % 6) + 6) % 6;
  const unsigned m = s & 0x3Fu;
  return (s & 0xC0u) | (((m << by) | (m >> (6 - by))) & 0x3Fu);
}

unsigned reverse6(unsigned m) { return rot(m & 0x3Fu, 3); }

int popc7(unsigned s) { return __builtin_popcount(s & 0x7Fu); }

void momentum(unsigned s, int& px, int& py) {
  px = py = 0;
  for (int k = 0; k < 6; ++k)
    if (s & (1u << k)) {
      px += kPx[k];
      py += kPy[k];
    }
}

uint8_t bounce(unsigned s) { return static_cast<uint8_t>((s & 0xC0u) | reverse6(s & 0x3Fu)); }

void build_fhp1(uint8_t* t) {
  for (int ch = 0; ch < 2; ++ch)
    for (unsigned s = 0; s < 256; ++s) {
      unsigned out = s;
      if (s & 0x80u) {
        out = bounce(s);
      } else if (!(s & 0x40u)) {
        const unsigned m = s & 0x3Fu;
        const int n = __builtin_popcount(m);
        if (n == 2 && reverse6(m) == m) out = rot(m, ch ? 1 : -1);
        else if (n == 3 && (m == 0x15u || m == 0x2Au)) out = m ^ 0x3Fu;
      }
      t[(ch << 8) | s] = static_cast<uint8_t>(out);
    }
}

// FHP-III: the bit-sliced rule of fhpg_fhp3_logic.cuh evaluated per state
// (bit 0 of each word), so the table and the bit-plane kernel are one rule.
void build_fhp3(uint8_t* t) {
  for (int ch = 0; ch < 2; ++ch)
    for (unsigned s = 0; s < 256; ++s) {
      uint32_t a[6], o[6], orr, dep;
      for (int k = 0; k < 6; ++k) a[k] = (s >> k) & 1u;
      fhpg::fhp3_collide<uint32_t>(a, (s >> 6) & 1u, (s >> 7) & 1u, static_cast<uint32_t>(ch), o,
                                   orr, dep);
      unsigned out = s & 0x80u;
      for (int k = 0; k < 6; ++k) out |= (o[k] & 1u) << k;
      out |= (orr & 1u) << 6;
      t[(ch << 8) | s] = static_cast<uint8_t>(out);
    }
}

// collision.cpp:22-51 (the reference's DEFAULT rules), restated.
unsigned default_fluid(unsigned s, int ch) {
  const unsigned m = s & 0x3Fu;
  const bool rest = (s & 0x40u) != 0;
  const int n = __builtin_popcount(m);
  if (n == 2 && !rest && reverse6(m) == m) return rot(m, ch ? 1 : 2);
  if (n == 3 && !rest && (m == 0x15u || m == 0x2Au)) return m ^ 0x3Fu;
  if (n == 1 && rest) {
    const int i = __builtin_ctz(m);
    return (1u << ((i + 5) % 6)) | (1u << ((i + 1) % 6));
  }
  if (n == 2 && !rest)
    for (int i = 0; i < 6; ++i)
      if (m == ((1u << i) | (1u << ((i + 2) % 6)))) return (1u << ((i + 1) % 6)) | 0x40u;
  return s;
}

void build_default(uint8_t* t) {
  for (int ch = 0; ch < 2; ++ch)
    for (unsigned s = 0; s < 256; ++s)
      t[(ch << 8) | s] = static_cast<uint8_t>((s & 0x80u) ? bounce(s) : default_fluid(s, ch));
}

}  // namespace

extern "C" {

int fhpg_build_table(int variant, uint8_t* out512) {
  if (!out512) return 2;
  switch (variant) {
    case FHPG_RULES_DEFAULT: build_default(out512); return 0;
    case FHPG_RULES_FHP_I: build_fhp1(out512); return 0;
    case FHPG_RULES_FHP_III: build_fhp3(out512); return 0;
    default: return 2;
  }
}

// collision.cpp:74-101: counts violations (obstacle bit, bounce-back, mass,
// momentum), the same checks and order as validate_table.
int fhpg_validate_table(const uint8_t* t, int* issues) {
  if (!t || !issues) return 2;
  int n = 0;
  for (int idx = 0; idx < 512; ++idx) {
    const unsigned s = static_cast<unsigned>(idx) & 0xFFu, o = t[idx];
    if ((o & 0x80u) != (s & 0x80u)) {
      ++n;
      continue;
    }
    if (s & 0x80u) {
      if (o != bounce(s)) ++n;
      continue;
    }
    if (popc7(o) != popc7(s)) ++n;
    int a, b, c, d;
    momentum(o, a, b);
    momentum(s, c, d);
    if (a != c || b != d) ++n;
  }
  *issues = n;
  return 0;
}

}  // extern "C"
