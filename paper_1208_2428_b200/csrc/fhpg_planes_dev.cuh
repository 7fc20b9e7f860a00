// fhpg_planes_dev.cuh — device helpers shared by the bit-plane kernels
// (fhpg_step_planes.cu: the streaming ring kernels; fhpg_step_resident.cu:
// the shared-memory-resident kernel for small lattices): shared-memory and
// TMA / mbarrier primitives, the rule dispatch, the plane reads of the
// hexagonal pull and the per-lane chirality walk. Included inside an
// anonymous namespace of namespace fhpg.
#pragma once
constexpr unsigned kFull = 0xFFFFFFFFu;

// Collision circuits the bit-plane kernels evaluate (fhpg_planes_rules.cuh):
// RULE 2 = FHP-III, 1 = FHP-I, 0 = the reference's DEFAULT rule.
template <int RULE>
struct PlaneRule;
template <>
struct PlaneRule<2> {
  using Class = Fhp3Class;
  static __device__ __forceinline__ Class classify(const uint32_t a[6], uint32_t r, uint32_t s) {
    return fhp3_classify(a, r, s);
  }
  static __device__ __forceinline__ void apply(const Class& k, uint32_t c, uint32_t r,
                                               const uint32_t a[6], uint32_t o[6], uint32_t& o_r,
                                               uint32_t) {
    fhp3_apply(k, c, r, a, o, o_r);
  }
};
template <>
struct PlaneRule<1> {
  using Class = Fhp1Class;
  static __device__ __forceinline__ Class classify(const uint32_t a[6], uint32_t r, uint32_t s) {
    return fhp1_classify(a, r, s);
  }
  static __device__ __forceinline__ void apply(const Class& k, uint32_t c, uint32_t r,
                                               const uint32_t a[6], uint32_t o[6], uint32_t& o_r,
                                               uint32_t s) {
    fhp1_apply(k, c, r, a, o, o_r, s);
  }
};
template <>
struct PlaneRule<0> {
  using Class = DefClass;
  static __device__ __forceinline__ Class classify(const uint32_t a[6], uint32_t r, uint32_t s) {
    return def_classify(a, r, s);
  }
  static __device__ __forceinline__ void apply(const Class& k, uint32_t c, uint32_t r,
                                               const uint32_t a[6], uint32_t o[6], uint32_t& o_r,
                                               uint32_t s) {
    def_apply(k, c, r, a, o, o_r, s);
  }
};
// Warps per CTA (one CTA per SM): 16 with 2 words per lane, 8 with 4.
// Programmatic dependent launch of the step kernels: the next step's grid is
// launched while this one runs (griddepcontrol.wait orders its reads).
#ifndef FHPG_PDL
#define FHPG_PDL 1
#endif
#ifndef FHPG_STREAM_ONLY
#define FHPG_STREAM_ONLY 0  // timing experiments (wrong results): 1 memory pipeline only,
                            // 2 loads only, 3 stores only, 4 loads + shared reads,
                            // 5 compute + stores (no loads), 6 compute only
#endif

#ifndef FHPG_PLANES_RING
#define FHPG_PLANES_RING 1
#endif
#ifndef FHPG_PLANES_WARPS
#define FHPG_PLANES_WARPS 16
#endif
#ifndef FHPG_PLANES_SLOTS
#define FHPG_PLANES_SLOTS 4
#endif
template <int NW>
constexpr int kPWarps = NW == 4 ? 8 : FHPG_PLANES_WARPS;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint32_t lds32(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ uint2 lds64v(uint32_t a) {
  uint2 v;
  asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(a));
  return v;
}
__device__ __forceinline__ uint64_t lds64(uint32_t a) {
  uint64_t v;
  asm volatile("ld.shared.u64 %0, [%1];" : "=l"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ uint4 lds128(uint32_t a) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts32(uint32_t a, uint32_t v) {
  asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(v));
}
__device__ __forceinline__ void sts64(uint32_t a, uint64_t v) {
  asm volatile("st.shared.u64 [%0], %1;" ::"r"(a), "l"(v));
}
__device__ __forceinline__ void sts128(uint32_t a, uint32_t x, uint32_t y, uint32_t z, uint32_t w) {
  asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(a), "r"(x), "r"(y), "r"(z), "r"(w));
}
__device__ __forceinline__ void red_or(uint32_t a, uint32_t v) {
  asm volatile("red.shared.or.b32 [%0], %1;" ::"r"(a), "r"(v));
}
__device__ __forceinline__ uint32_t top_bit(uint32_t m) {
  uint32_t p;
  asm("bfind.u32 %0, %1;" : "=r"(p) : "r"(m));
  return p;
}

// mbarrier + bulk async copy (TMA engine, non-tensor form).
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}
// Suspend-time hint (ns) of the ring waits: a waiting warp sleeps in the
// barrier until the phase completes instead of re-polling (0: no hint).
#ifndef FHPG_WAIT_HINT
#define FHPG_WAIT_HINT 0
#endif
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  uint32_t done;
  do {
#if FHPG_WAIT_HINT
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3; selp.u32 %0, 1, 0, p; }"
        : "=r"(done) : "r"(bar), "r"(parity), "n"(FHPG_WAIT_HINT) : "memory");
#else
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(done) : "r"(bar), "r"(parity) : "memory");
#endif
  } while (!done);
}
// One TMA box {72 words, 8 planes, 1 row} of the plane tensor.
__device__ __forceinline__ void tma_row(uint32_t dst, const CUtensorMap* map, int word, int row,
                                        uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];"
      ::"r"(dst), "l"(map), "r"(word), "r"(0), "r"(row), "r"(bar) : "memory");
}

// TMA store of a dense smem box (the 7 outgoing planes of a band row, or
// the 4 pad words of each plane) into the plane tensor; bulk-group tracked.
__device__ __forceinline__ void tma_store(const CUtensorMap* map, int word, int row, uint32_t src) {
  asm volatile(
      "cp.async.bulk.tensor.3d.global.shared::cta.tile.bulk_group [%0, {%1, %2, %3}], [%4];"
      ::"l"(map), "r"(word), "r"(0), "r"(row), "r"(src) : "memory");
}
__device__ __forceinline__ void bulk_commit() {
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}

__device__ __forceinline__ void bulk_wait_all() {
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
__device__ __forceinline__ void fence_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
template <int NW>
__device__ __forceinline__ void stsv(uint32_t a, const uint32_t (&v)[NW]) {
  if constexpr (NW == 4) {
    sts128(a, v[0], v[1], v[2], v[3]);
  } else if constexpr (NW == 2) {
    asm volatile("st.shared.v2.u32 [%0], {%1,%2};" ::"r"(a), "r"(v[0]), "r"(v[1]));
  } else {
    sts32(a, v[0]);
  }
}

template <int NW>
__device__ __forceinline__ void stv(uint32_t* p, const uint32_t (&v)[NW]) {
  if constexpr (NW == 4) {
    __stcs(reinterpret_cast<uint4*>(p), make_uint4(v[0], v[1], v[2], v[3]));
  } else if constexpr (NW == 2) {
    __stcs(reinterpret_cast<uint2*>(p), make_uint2(v[0], v[1]));
  } else {
    __stcs(p, v[0]);
  }
}

// Geometry of a warp's smem: a ring of kSlots source rows. A slot holds the
// 8 planes of the band, each as [kSlotPad words left of the band | band
// words | kSlotPad words right of it] (one TMA box), so the +-1 column funnel shifts read the
// neighbouring lane's (or band's) word straight from shared memory.
// Words a ring slot holds on either side of the band (the +-1 column moves
// read one): 4, because a TMA box must start on a 16-byte boundary of the
// row (a 2-word pad faults with an illegal instruction).
constexpr int kSlotPad = 4;
template <int NW, bool FORCE>
struct Geo {
  static constexpr int kBandWords = 32 * NW;
  static constexpr int kBandCols = 1024 * NW;
  static constexpr int kPlane = 4 * (2 * kSlotPad + kBandWords);
  static constexpr int kSlot = 8 * kPlane;
  static constexpr int kSlots = FHPG_PLANES_SLOTS;
  // Output staging (7 planes x band words, the TMA store source) followed by
  // the edge bands' wrap-sector box (7 planes x kPlaneWrap words). The
  // walk's list and result words reuse the staging area: they are dead
  // before the row's outputs land.
  static constexpr int kStage = 7 * 4 * kBandWords;
  static constexpr int kPad = kStage;             // TMA source: 128 B aligned
  static constexpr int kList = 16 * kBandWords;   // walk list entries (uint4), inside the stage
  static constexpr int kOut = 4 * kBandWords;     // walk result words, after the list
  static_assert(kList + kOut <= kStage, "walk scratch must fit the staging area");
  static_assert(kStage % 128 == 0, "TMA store sources are 128 B aligned");
  static_assert(7 * 4 * kPlaneWrap <= 256, "wrap box");
  static constexpr int kStageAll = kStage + 256;
  static constexpr int kWarp = (kSlots * kSlot + kStageAll + 8 * kSlots + 127) / 128 * 128;
  static constexpr uint32_t kRowBytes = kSlot;
};

struct Lanes {
  int lane;
  int WW;           // words per plane row (W / 32)
  int PW;           // words per plane row (plane_stride_words)
  int w0;           // first word of the band
  int padx;         // bit 0: last band (left wrap sector), bit 1: first band (right wrap
                    // sector), padx >> 2 = WW
};

// Plane words of this lane from a slot: aligned, or shifted by one column.
template <int NW>
__device__ __forceinline__ void rd_al(uint32_t a, uint32_t (&o)[NW]) {
  if constexpr (NW == 4) {
    const uint4 v = lds128(a);
    o[0] = v.x;
    o[1] = v.y;
    o[2] = v.z;
    o[3] = v.w;
  } else if constexpr (NW == 2) {
    const uint2 v = lds64v(a);
    o[0] = v.x;
    o[1] = v.y;
  } else {
    o[0] = lds32(a);
  }
}
// L: out bit j = column x-1 (funnel with the previous word).
template <int NW>
__device__ __forceinline__ void rd_shl(uint32_t a, uint32_t (&o)[NW]) {
  uint32_t v[NW];
  rd_al<NW>(a, v);
  const uint32_t prev = lds32(a - 4);
  o[0] = __funnelshift_l(prev, v[0], 1);
#pragma unroll
  for (int i = 1; i < NW; ++i) o[i] = __funnelshift_l(v[i - 1], v[i], 1);
}
// R: out bit j = column x+1 (funnel with the next word).
template <int NW>
__device__ __forceinline__ void rd_shr(uint32_t a, uint32_t (&o)[NW]) {
  uint32_t v[NW];
  rd_al<NW>(a, v);
  const uint32_t next = lds32(a + 4 * NW);
#pragma unroll
  for (int i = 0; i < NW - 1; ++i) o[i] = __funnelshift_r(v[i], v[i + 1], 1);
  o[NW - 1] = __funnelshift_r(v[NW - 1], next, 1);
}

// The same reads for the lanes at a lattice edge (E: 0 = interior band;
// 1 = band 0 of several, lane 0's previous word is the periodic wrap, read
// from the side buffer at `wp`; 2 = the last band of several, lane 31's
// next word, from `wp`; 3 = a single band, both wraps inside the slot).
template <int NW, int E>
__device__ __forceinline__ void rd_shl_e(uint32_t a, uint32_t wp, int lane, uint32_t (&o)[NW]) {
  uint32_t v[NW];
  rd_al<NW>(a, v);
  uint32_t pa = a - 4;
  if constexpr (E == 1) pa = lane == 0 ? wp : pa;
  if constexpr (E == 3) pa = lane == 0 ? a + (32 * NW - 1) * 4 : pa;
  const uint32_t prev = lds32(pa);
  o[0] = __funnelshift_l(prev, v[0], 1);
#pragma unroll
  for (int i = 1; i < NW; ++i) o[i] = __funnelshift_l(v[i - 1], v[i], 1);
}
template <int NW, int E>
__device__ __forceinline__ void rd_shr_e(uint32_t a, uint32_t wp, int lane, uint32_t (&o)[NW]) {
  uint32_t v[NW];
  rd_al<NW>(a, v);
  uint32_t na = a + 4 * NW;
  if constexpr (E == 2) na = lane == 31 ? wp : na;
  if constexpr (E == 3) na = lane == 31 ? a - 31 * NW * 4 : na;
  const uint32_t next = lds32(na);
#pragma unroll
  for (int i = 0; i < NW - 1; ++i) o[i] = __funnelshift_r(v[i], v[i + 1], 1);
  o[NW - 1] = __funnelshift_r(v[NW - 1], next, 1);
}

// The step kernels' chirality / forcing walk: every lane visits the set bits
// of its own NW dep words, one word after the other, highest bit first, and
// keeps the result bits in registers (no list, no prefix sums, no slice
// search, no shared-memory results; a balanced warp walk — a list of the
// nonzero words, prefix sums, equal slices per lane — costs ~90
// instructions per lane-row of setup and measured slower, see git history). The warp waits
// for its busiest lane. (Rotating the key table per lane against shared-
// memory bank conflicts measured 1.6% slower: two more shifts per word.)
#ifndef FHPG_LOP3P
#define FHPG_LOP3P 1
#endif
// a ^ b and whether it is nonzero, from one LOP3 with a predicate output
// (PTX lop3.or.b32 d|p): the walk's mask update doubles as its loop test
// (no separate ISETP per visited site).
__device__ __forceinline__ uint32_t xor_nonzero(uint32_t a, uint32_t b, bool& nonzero) {
  uint32_t d, nz;
  asm("{\n\t.reg .pred p;\n\tlop3.or.b32 %0|p, %2, %3, 0, 0x3c, 0;\n\tselp.u32 %1, 1, 0, p;\n\t}"
      : "=r"(d), "=r"(nz) : "r"(a), "r"(b));
  nonzero = nz != 0u;
  return d;
}
// step(acc, bit, band column) folds one visited site's result bit into acc.
template <int NW, typename Step>
__device__ __forceinline__ void walk_core(const uint32_t (&m)[NW], int lane, uint32_t (&c)[NW],
                                          Step&& step) {
  auto visit = [&](uint32_t mask, uint32_t k0) {
    uint32_t acc = 0u;
#if FHPG_LOP3P
    if (mask) {
      bool more;
      do {
        const uint32_t j = top_bit(mask);
        const uint32_t bit = 1u << j;
        mask = xor_nonzero(mask, bit, more);
        acc = step(acc, bit, k0 + j);
      } while (more);
    }
#else
    while (mask) {
      const uint32_t j = top_bit(mask);
      const uint32_t bit = 1u << j;
      mask ^= bit;
      acc = step(acc, bit, k0 + j);
    }
#endif
    return acc;
  };
  if constexpr (NW == 2) {
    // One loop per word: every lane takes its fuller word first, so the
    // first loop's maximum is over the fuller words and the second's over
    // the emptier ones (expected 15.0 instead of 16.6 iterations at 12.6%
    // dep sites).
    const bool sw = __popc(m[1]) > __popc(m[0]);
    const uint32_t kw = static_cast<uint32_t>(lane * 2) * 32u;
    const uint32_t acc0 = visit(sw ? m[1] : m[0], kw + (sw ? 32u : 0u));
    const uint32_t acc1 = visit(sw ? m[0] : m[1], kw + (sw ? 0u : 32u));
    c[0] = sw ? acc1 : acc0;
    c[1] = sw ? acc0 : acc1;
    return;
  }
#pragma unroll
  for (int w = 0; w < NW; ++w) c[w] = visit(m[w], static_cast<uint32_t>(lane * NW + w) * 32u);
}
// fn(band column) returns the site's result as a mask (0 or ~0u).
template <int NW, typename Fn>
__device__ __forceinline__ void walk_own(const uint32_t (&m)[NW], int lane, uint32_t (&c)[NW],
                                         Fn&& fn) {
  walk_core<NW>(m, lane, c,
                [&](uint32_t acc, uint32_t bit, uint32_t col) { return acc | (fn(col) & bit); });
}
#ifndef FHPG_WALK_PRED
#define FHPG_WALK_PRED 1
#endif
// The same walk for a result "h(column) < thr" (the forcing draw): the
// compare's predicate guards the OR directly (ISETP + @P LOP3 instead of
// ISETP + SEL + LOP3: one ALU-pipe instruction less per visited site).
template <int NW, typename Fn>
__device__ __forceinline__ void walk_own_lt(const uint32_t (&m)[NW], int lane, uint32_t (&c)[NW],
                                            uint32_t thr, Fn&& h) {
  walk_core<NW>(m, lane, c, [&](uint32_t acc, uint32_t bit, uint32_t col) {
#if FHPG_WALK_PRED
    asm("{\n\t.reg .pred q;\n\tsetp.lt.u32 q, %1, %2;\n\t@q or.b32 %0, %0, %3;\n\t}"
        : "+r"(acc) : "r"(h(col)), "r"(thr), "r"(bit));
    return acc;
#else
    return acc | (h(col) < thr ? bit : 0u);
#endif
  });
}

template <int NW, bool FORCE>
struct Ctx {
  // Column keys of the band (fhpg_common.cuh ColKey, key base row ybase):
  // {lo, t2, g, 0} per column (one 16-byte load), chirality and forcing.
  uint32_t kc;
  uint32_t kf;
  uint32_t ybase;   // global row the band's column keys were made for
  uint32_t span;    // rows ybase .. ybase + span - 1 use them; later rows hash
                    // from the step keys (kcur, kfcur)
  uint32_t x1;      // 1-based lattice column of band column 0
  uint64_t kcur, kfcur;
  uint32_t four;    // 4, passed at run time (chir_bit)
  uint32_t lsm;     // smem: walk list
  uint32_t osm;     // smem: walk result words
  uint32_t stage;   // smem: output staging (the TMA store source)
  uint64_t thr;
};

// Builds the band's column keys for columns c0, c0 + dc, ... < ncols (a
// thread's share) at key base row ybase (global); returns the smallest
// span among them (every thread of the CTA takes part; the caller reduces).
template <bool FORCE>
__device__ __forceinline__ uint32_t make_col_keys(uint32_t kc, uint32_t kf, uint64_t kcur,
                                                  uint64_t kfcur, uint32_t x1, uint32_t ybase,
                                                  int c0, int dc, int ncols) {
  uint32_t span = 0xFFFFFFFFu;
  for (int c = c0; c < ncols; c += dc) {
    const uint64_t x = static_cast<uint64_t>(x1) + c;
    const uint32_t pos = static_cast<uint32_t>(c);
    const ColKey k = col_key_terms(column_key(kcur, x) + ybase);
    sts128(kc + pos * 16, k.lo, k.t2, k.g, 0u);
    span = min(span, colkey_span(k.lo));
    if (FORCE) {
      const ColKey f = col_key_terms(column_key(kfcur, x) + ybase);
      sts128(kf + pos * 16, f.lo, f.t2, f.g, 0u);
      span = min(span, colkey_span(f.lo));
    }
  }
  return span;
}
// CTA-wide minimum of the per-thread spans through one slot per warp
// (slots: 32 words): each warp's lane 0 writes its minimum; after a barrier
// every thread reads the minimum over the CTA's warps' slots.
__device__ __forceinline__ void span_put(uint32_t slots, uint32_t span) {
  const uint32_t m = __reduce_min_sync(kFull, span);
  if ((threadIdx.x & 31) == 0) sts32(slots + (threadIdx.x >> 5) * 4, m);
}
__device__ __forceinline__ uint32_t span_get(uint32_t slots) {
  // (only the slots of the CTA's warps hold values)
  const uint32_t l = threadIdx.x & 31;
  return __reduce_min_sync(kFull, l < (blockDim.x >> 5) ? lds32(slots + l * 4) : 0xFFFFFFFFu);
}

// One destination row. sm, sc, sn: this lane's word address inside plane 0
// of the slots of rows r-1, r, r+1; Q = global parity of r.
// `released()` is called once the source rows have been read into
// registers (the ring slots may be refilled from then on).
