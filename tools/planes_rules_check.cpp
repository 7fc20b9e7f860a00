// Exhaustive check of the bit-sliced collision circuits used by the bit-plane
// kernel (paper_1208_2428_b200/csrc/fhpg_planes_rules.cuh) against the
// 512-entry tables (fhpg_tables.cpp): all 256 states (bit 7 = obstacle) x
// both chiralities, 32 sites per word. Also checks that sites outside `dep`
// do not read the chirality word and that `dep` is exactly "table outcome
// depends on chirality". Exit status 0 = all rules match.
//   g++ -std=c++17 -O1 -I include -I paper_1208_2428_b200/csrc \
//       tools/planes_rules_check.cpp paper_1208_2428_b200/csrc/fhpg_tables.cpp
#include <cstdint>
#include <cstdio>

#include "fhpg_planes_rules.cuh"
#include "fhpg_tables.h"

using namespace fhpg;

struct Words {
  uint32_t a[6], r, solid;
};

// Sites i = 32 w + j, state s = i & 255 (the word covers 32 consecutive states).
static Words pack(int w) {
  Words x{};
  for (int j = 0; j < 32; ++j) {
    const unsigned s = static_cast<unsigned>(w * 32 + j) & 255u;
    for (int k = 0; k < 6; ++k) x.a[k] |= ((s >> k) & 1u) << j;
    x.r |= ((s >> 6) & 1u) << j;
    x.solid |= ((s >> 7) & 1u) << j;
  }
  return x;
}

template <typename Classify, typename Apply>
static int check(const char* name, int variant, Classify classify, Apply apply) {
  uint8_t t[512];
  fhpg_build_table(variant, t);
  int bad = 0, deps = 0;
  for (int w = 0; w < 8; ++w) {
    const Words x = pack(w);
    const auto k = classify(x.a, x.r, x.solid);
    uint32_t o0[6], o1[6], r0, r1;
    apply(k, 0u, x.r, x.a, o0, r0);
    apply(k, ~0u, x.r, x.a, o1, r1);
    for (int j = 0; j < 32; ++j) {
      const unsigned s = static_cast<unsigned>(w * 32 + j);
      for (int c = 0; c < 2; ++c) {
        const uint32_t* o = c ? o1 : o0;
        const uint32_t rr = c ? r1 : r0;
        unsigned got = ((rr >> j) & 1u) << 6 | (s & 0x80u);
        for (int q = 0; q < 6; ++q) got |= ((o[q] >> j) & 1u) << q;
        if (got != t[(c << 8) | s]) {
          if (bad < 10) printf("%s: state %02x c=%d: got %02x want %02x\n", name, s, c, got, t[(c << 8) | s]);
          ++bad;
        }
      }
      const bool dep_t = t[s] != t[256 + s];
      const bool dep_k = (k.dep >> j) & 1u;
      deps += dep_k;
      if (dep_t != dep_k) {
        if (bad < 10) printf("%s: state %02x dep got %d want %d\n", name, s, dep_k, dep_t);
        ++bad;
      }
    }
  }
  printf("%s: %s (%d dep states)\n", name, bad ? "MISMATCH" : "ok", deps);
  return bad;
}

int main() {
  int bad = 0;
  bad += check("fhp3", FHPG_RULES_FHP_III,
               [](const uint32_t* a, uint32_t r, uint32_t s) { return fhp3_classify(a, r, s); },
               [](const Fhp3Class& k, uint32_t c, uint32_t r, const uint32_t* x_a, uint32_t* o, uint32_t& orr) {
                 fhp3_apply(k, c, r, x_a, o, orr);
               });
  bad += check("default", FHPG_RULES_DEFAULT,
               [](const uint32_t* a, uint32_t r, uint32_t s) {
                 struct K : DefClass { uint32_t solid; };
                 K k;
                 static_cast<DefClass&>(k) = def_classify(a, r, s);
                 k.solid = s;
                 return k;
               },
               [](const auto& k, uint32_t c, uint32_t r, const uint32_t* x_a, uint32_t* o, uint32_t& orr) {
                 def_apply(k, c, r, x_a, o, orr, k.solid);
               });
  bad += check("fhp1", FHPG_RULES_FHP_I,
               [](const uint32_t* a, uint32_t r, uint32_t s) {
                 struct K : Fhp1Class { uint32_t solid; };
                 K k;
                 static_cast<Fhp1Class&>(k) = fhp1_classify(a, r, s);
                 k.solid = s;
                 return k;
               },
               [](const auto& k, uint32_t c, uint32_t r, const uint32_t* x_a, uint32_t* o, uint32_t& orr) {
                 fhp1_apply(k, c, r, x_a, o, orr, k.solid);
               });
  // chir_bit (fhpg_common.cuh) == bit 0 of fin64(z): random keys, and keys
  // whose low word is at the carry boundary.
  {
    uint64_t st = 0x243F6A8885A308D3ull;
    long n = 0, wrong = 0;
    for (int i = 0; i < 2000000; ++i) {
      st = mix64(st);
      uint64_t K = st;
      const uint32_t y = static_cast<uint32_t>(mix64(st ^ 1) >> 40);  // < 2^24
      if (i % 4 == 1) K = (K & ~0xFFFFFFFFull) | (0xFFFFFFFFull - (y & 0xFF));
      if (i % 4 == 2) K = (K & ~0xFFFFFFFFull) | (0x100000000ull - y + (st & 0xFF));
      ++n;
      if (chir_bit(K + y, 4u) != (fin64(K + y) & 1u) || fin64_bit0(K + y) != (fin64(K + y) & 1u))
        ++wrong;
    }
    std::printf("chir_bit: %s (%ld keys)\n", wrong ? "MISMATCH" : "ok", n);
    bad += wrong != 0;
  }
  // Folded column terms (col_key_terms / chir_mask_pre / fin64_hi_pre) ==
  // fin64(K + dy) for every dy inside colkey_span: random keys, and keys at
  // the end of a 2^30 block (span 1 .. 256).
  {
    uint64_t st = 0x13198A2E03707344ull;
    long n = 0, wrong = 0;
    for (int i = 0; i < 1000000; ++i) {
      st = mix64(st);
      uint64_t K = st;
      if (i % 2) K = (K & ~0x3FFFFFFFull) | (0x3FFFFFFFull - (mix64(st ^ 7) & 0xFF));
      const ColKey c = col_key_terms(K);
      const uint32_t span = colkey_span(c.lo);
      uint32_t dy = static_cast<uint32_t>(mix64(st ^ 3) >> 44);  // < 2^20
      if (i % 2 || dy >= span) dy = span - 1 - (dy % (span < 64 ? span : 64));
      const uint64_t f = fin64(K + dy);
      ++n;
      if (chir_mask_pre(c.lo + dy, c.t2, c.g) != ((f & 1u) ? ~0u : 0u) ||
          fin64_hi_pre(c.lo + dy, c.t2, c.g) != static_cast<uint32_t>(f >> 32))
        ++wrong;
      // thresholds <= 2^31: z2's high word decides the forcing draw alike
      // (random thresholds, 2^31 itself, and thresholds next to the value)
      const uint32_t z2hi = fin64_z2hi_pre(c.lo + dy, c.t2, c.g);
      const uint64_t near = (z2hi & 0x7FFFFFFFu) + (i & 1);
      const uint64_t thr = i % 3 == 0 ? (1ull << 31) : i % 3 == 1 ? (mix64(st ^ 11) >> 33) : near;
      if ((z2hi < thr) != ((f >> 32) < thr)) ++wrong;
    }
    std::printf("col_key_terms: %s (%ld keys)\n", wrong ? "MISMATCH" : "ok", n);
    bad += wrong != 0;
  }
  return bad ? 1 : 0;
}
