// fhpg_step_planes.cu — the hot path on a bit-plane lattice: one fused FHP
// time step (motion -> collision with lazy chirality -> forcing) for rules
// that have a bit-sliced circuit (fhpg_planes_rules.cuh), plus the
// byte <-> plane converters.
//
// Replaces, per step, sync_ghost_columns (lattice.cpp:32-39), motion_step
// (step.cpp:40-61, pull offsets backends.cpp:64-73), swap_buffers and
// collide_rows with its counter-RNG chirality and forcing (step.cpp:63-93),
// bit-exactly.
//
// Layout. A lattice row keeps its W bytes but holds 8 bit planes of W/8 bytes:
// plane p (0-5 movers NW..W, 6 rest, 7 obstacle), bit j of word i = column
// 32 i + j. Row pitch, halo rows and spare rows are those of the byte layout,
// so halo exchange, row strips and buffer sizes do not change. The obstacle
// plane is static: it is written into both ping-pong buffers by the pack
// kernel and never by the step, so a step moves exactly the algorithmic
// 15 bits per site (8 planes read, 7 written).
//
// Work decomposition. A warp owns a band of 32 * NW words (1024 NW columns)
// and a segment of rows that it streams top to bottom; lane l holds words
// [l NW, l NW + NW) of every plane. Each source row is loaded once (one
// NW-word vector load per plane and lane, two rows in flight) and turned on
// arrival into the shifted planes the three destination rows need: the
// +-1 column moves of the hexagonal pull are funnel shifts with the
// neighbour lane's edge word (SHFL) or, at band edges, the neighbour band's
// word (one scalar load per shifted plane, periodic wrap).
//
// Collision: bit-sliced circuit on 32 sites per instruction. Chirality is
// drawn only where the outcome depends on it: the dep masks of the warp's
// row go to shared memory, the warp splits the dep sites evenly over its
// lanes (prefix sum), each lane evaluates fin64_bit0(column key + row) for
// its slice (keys staged in shared memory) and sets the chirality bits with
// shared-memory ORs. Forcing (thr > 0) is resolved the same way on the
// post-collision candidates (fluid, W set, E clear).
#include <cstdint>
#include <type_traits>

#include "fhpg_common.cuh"
#include "fhpg_kernels.cuh"
#include "fhpg_planes_rules.cuh"

namespace fhpg {
namespace {

constexpr unsigned kFull = 0xFFFFFFFFu;
constexpr int kPWarps = 16;
constexpr int kPThreads = kPWarps * 32;

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
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  uint32_t done;
  do {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(done) : "r"(bar), "r"(parity) : "memory");
  } while (!done);
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes,
                                         uint32_t bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
      ::"r"(dst), "l"(src), "r"(bytes), "r"(bar) : "memory");
}

template <int NW>
__device__ __forceinline__ void stv(uint32_t* p, const uint32_t (&v)[NW]) {
  if constexpr (NW == 2) {
    __stcs(reinterpret_cast<uint2*>(p), make_uint2(v[0], v[1]));
  } else {
    __stcs(p, v[0]);
  }
}

// Geometry of a warp's smem: a ring of kSlots source rows. A slot holds the
// 8 planes of the band, each as [16 B left edge chunk | band words | 16 B
// right edge chunk] so that the +-1 column funnel shifts read the
// neighbouring lane's (or band's) word straight from shared memory.
template <int NW, bool FORCE>
struct Geo {
  static constexpr int kBandWords = 32 * NW;
  static constexpr int kBandCols = 1024 * NW;
  static constexpr int kPlane = 32 + 4 * kBandWords;
  static constexpr int kSlot = 8 * kPlane;
  static constexpr int kSlots = FORCE ? 4 : 5;
  static constexpr int kList = 16 * kBandWords;   // walk list entries (uint4)
  static constexpr int kOut = 4 * kBandWords;     // walk result words
  static constexpr int kWarp = (kSlots * kSlot + kList + kOut + 8 * kSlots + 127) / 128 * 128;
  static constexpr uint32_t kRowBytes = 8u * 4u * kBandWords + 4u * 16u;
};

struct Lanes {
  int lane;
  int WW;           // words per plane row (W / 32)
  int w0;           // first word of the band
  int wl, wr;       // first word of the left / right edge chunks (periodic)
};

// Planes that shift for a source row of global parity PS (pull offsets,
// backends.cpp:64-73, with the destination row's parity q):
//   PS = 0: plane 0 R (dest s-1, q=1), 2 L, 4 R (dest s+1, q=1), 5 R
//   PS = 1: plane 1 L (dest s-1, q=0), 2 L, 3 L (dest s+1, q=0), 5 R
// Issue the bulk copies of source row `row` (local index) into `slot`
// (called by one lane).
template <int NW, bool FORCE>
__device__ __forceinline__ void issue_row(const uint8_t* src, long long pitch, long long row,
                                          int ps, const Lanes& L, uint32_t slot, uint32_t bar) {
  using G = Geo<NW, FORCE>;
  const uint8_t* r = src + row * pitch;
  const size_t pb = static_cast<size_t>(L.WW) * 4;  // bytes per plane row
  mbar_expect_tx(bar, G::kRowBytes);
#pragma unroll
  for (int p = 0; p < 8; ++p)
    bulk_g2s(slot + p * G::kPlane + 16, r + p * pb + L.w0 * 4, 4 * G::kBandWords, bar);
  const int pl0 = ps ? 1 : 0, pl3 = ps ? 3 : 4;
  // left chunks for L shifts, right chunks for R shifts
  if (ps) {
    bulk_g2s(slot + pl0 * G::kPlane, r + pl0 * pb + L.wl * 4, 16, bar);
    bulk_g2s(slot + pl3 * G::kPlane, r + pl3 * pb + L.wl * 4, 16, bar);
  } else {
    bulk_g2s(slot + pl0 * G::kPlane + 16 + 4 * G::kBandWords, r + pl0 * pb + L.wr * 4, 16, bar);
    bulk_g2s(slot + pl3 * G::kPlane + 16 + 4 * G::kBandWords, r + pl3 * pb + L.wr * 4, 16, bar);
  }
  bulk_g2s(slot + 2 * G::kPlane, r + 2 * pb + L.wl * 4, 16, bar);
  bulk_g2s(slot + 5 * G::kPlane + 16 + 4 * G::kBandWords, r + 5 * pb + L.wr * 4, 16, bar);
}

// Plane words of this lane from a slot: aligned, or shifted by one column.
template <int NW>
__device__ __forceinline__ void rd_al(uint32_t a, uint32_t (&o)[NW]) {
  if constexpr (NW == 2) {
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

// Balanced walk over the set bits of the warp's NW * 32 mask words (word
// i = lane * NW + w <-> band word i, bit j <-> column 32 i + j of the band).
// The warp's nonzero words go to a list {mask, word, sites before it}; the
// T sites are split into 32 equal contiguous slices; each lane finds its
// first word (binary search over the lanes' counts), skips the sites before
// its slice and visits its sites two at a time, advancing through the list
// (no empty words on it). fn(col0, col1, has1) returns the two result bits,
// ORed into the result words (osm) bit by bit. Returns T.
template <int NW, typename Fn>
__device__ __forceinline__ int walk(const uint32_t (&m)[NW], uint32_t lsm, uint32_t osm, int lane,
                                    Fn&& fn) {
  int cnt = 0, nz = 0;
#pragma unroll
  for (int w = 0; w < NW; ++w) {
    cnt += __popc(m[w]);
    nz += m[w] != 0u;
  }
  const int packed = cnt | (nz << 16);
  int incl = packed;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const int v = __shfl_up_sync(kFull, incl, d);
    if (lane >= d) incl += v;
  }
  const int T = __shfl_sync(kFull, incl, 31) & 0xFFFF;
  if (T == 0) return 0;
  const int excl = incl - packed;
  {
    int q = excl >> 16, c = excl & 0xFFFF;
#pragma unroll
    for (int w = 0; w < NW; ++w) {
      if (m[w]) {
        sts128(lsm + q * 16, m[w], static_cast<uint32_t>(lane * NW + w), static_cast<uint32_t>(c), 0u);
        ++q;
        c += __popc(m[w]);
      }
      sts32(osm + (lane * NW + w) * 4, 0u);
    }
  }
  __syncwarp();
  const int s = (lane * T) >> 5;
  const int e = ((lane + 1) * T) >> 5;
  // owner lane of site s: last lane whose exclusive count is <= s
  const int icnt = incl & 0xFFFF;
  int o = 0;
#pragma unroll
  for (int step = 16; step; step >>= 1) {
    const int v = __shfl_sync(kFull, icnt, o + step - 1);
    if (v <= s) o += step;
  }
  const int o_excl = __shfl_sync(kFull, excl, o);
  if (s < e) {
    int q = o_excl >> 16;
    uint4 en = lds128(lsm + q * 16);
    if (NW > 1 && s >= static_cast<int>(en.z) + __popc(en.x)) {
      ++q;
      en = lds128(lsm + q * 16);
    }
    uint32_t mask = en.x;
    uint32_t base = en.y * 32u;
    for (int k = s - static_cast<int>(en.z); k > 0; --k) mask ^= 1u << top_bit(mask);
    auto next = [&](uint32_t& col) {
      if (mask == 0u) {
        ++q;
        const uint4 n = lds128(lsm + q * 16);
        mask = n.x;
        base = n.y * 32u;
      }
      const uint32_t j = top_bit(mask);
      mask ^= 1u << j;
      col = base + j;
    };
    for (int it = s; it < e; it += 2) {
      uint32_t c0, c1 = 0;
      next(c0);
      const bool has1 = it + 1 < e;
      if (has1) next(c1);
      uint32_t b0, b1;
      fn(c0, c1, has1, b0, b1);
      red_or(osm + (c0 >> 5) * 4u, b0 << (c0 & 31u));
      red_or(osm + (c1 >> 5) * 4u, b1 << (c1 & 31u));
    }
  }
  __syncwarp();
  return T;
}

template <int NW, bool FORCE>
struct Ctx {
  uint32_t kc;      // smem: chirality keys of the band (8 B per column)
  uint32_t kf;      // smem: forcing keys of the band
  uint32_t lsm;     // smem: walk list
  uint32_t osm;     // smem: walk result words
  uint64_t thr;
};

// One destination row. sm, sc, sn: this lane's word address inside plane 0
// of the slots of rows r-1, r, r+1; Q = global parity of r.
template <int NW, bool FORCE, int Q>
__device__ __forceinline__ void dest_row(uint32_t sm, uint32_t sc, uint32_t sn,
                                         const Ctx<NW, FORCE>& cx, int lane, uint32_t y,
                                         uint32_t* out_row, int plane_words, unsigned& swaps) {
  using G = Geo<NW, FORCE>;
  constexpr int P = G::kPlane;
  uint32_t a0[NW], a1[NW], a2[NW], a3[NW], a4[NW], a5[NW], rr[NW], so[NW];
  // Pull sources (backends.cpp:64-73): k0 (x+q, r+1), k1 (x+q-1, r+1),
  // k2 (x-1, r), k3 (x+q-1, r-1), k4 (x+q, r-1), k5 (x+1, r).
  if (Q) rd_shr<NW>(sn + 0 * P, a0); else rd_al<NW>(sn + 0 * P, a0);
  if (Q) rd_al<NW>(sn + 1 * P, a1); else rd_shl<NW>(sn + 1 * P, a1);
  rd_shl<NW>(sc + 2 * P, a2);
  if (Q) rd_al<NW>(sm + 3 * P, a3); else rd_shl<NW>(sm + 3 * P, a3);
  if (Q) rd_shr<NW>(sm + 4 * P, a4); else rd_al<NW>(sm + 4 * P, a4);
  rd_shr<NW>(sc + 5 * P, a5);
  rd_al<NW>(sc + 6 * P, rr);
  rd_al<NW>(sc + 7 * P, so);
  Fhp3Class K[NW];
  uint32_t dep[NW];
#pragma unroll
  for (int w = 0; w < NW; ++w) {
    const uint32_t a[6] = {a0[w], a1[w], a2[w], a3[w], a4[w], a5[w]};
    K[w] = fhp3_classify(a, rr[w], so[w]);
    dep[w] = K[w].dep;
  }
  // Chirality: bit 0 of node_random(seed, Chirality, step, x + 1, y)
  // = fin64(key[x] + y) (rng.hpp:25-33, step.cpp:73-76).
  const int T = walk<NW>(dep, cx.lsm, cx.osm, lane,
                         [&](uint32_t c0, uint32_t c1, bool has1, uint32_t& b0, uint32_t& b1) {
    const uint64_t k0 = lds64(cx.kc + c0 * 8u);
    const uint64_t k1 = lds64(cx.kc + c1 * 8u);
    b0 = fin64_bit0(k0 + y);
    b1 = fin64_bit0(k1 + y) & (has1 ? 1u : 0u);
  });
  uint32_t o[NW][7];
  const uint32_t mine = cx.osm + lane * NW * 4;
#pragma unroll
  for (int w = 0; w < NW; ++w) {
    const uint32_t c = T ? lds32(mine + w * 4) : 0u;
    uint32_t oo[6], orr;
    fhp3_apply(K[w], c, rr[w], oo, orr);
#pragma unroll
    for (int p = 0; p < 6; ++p) o[w][p] = oo[p];
    o[w][6] = orr;
  }
  if constexpr (FORCE) {
    // step.cpp:79-88: fluid, W (bit 5) set, E (bit 2) clear after collision.
    uint32_t f[NW];
#pragma unroll
    for (int w = 0; w < NW; ++w) f[w] = ~so[w] & o[w][5] & ~o[w][2];
    const int TF = walk<NW>(f, cx.lsm, cx.osm, lane,
                            [&](uint32_t c0, uint32_t c1, bool has1, uint32_t& b0, uint32_t& b1) {
      const uint64_t k0 = lds64(cx.kf + c0 * 8u);
      const uint64_t k1 = lds64(cx.kf + c1 * 8u);
      b0 = (fin64(k0 + y) >> 32) < cx.thr ? 1u : 0u;
      b1 = has1 && (fin64(k1 + y) >> 32) < cx.thr ? 1u : 0u;
    });
    if (TF) {
#pragma unroll
      for (int w = 0; w < NW; ++w) {
        const uint32_t acc = lds32(mine + w * 4);
        o[w][5] ^= acc;
        o[w][2] ^= acc;
        swaps += __popc(acc);
      }
    }
  }
#pragma unroll
  for (int p = 0; p < 7; ++p) {
    uint32_t v[NW];
#pragma unroll
    for (int w = 0; w < NW; ++w) v[w] = o[w][p];
    stv<NW>(out_row + p * plane_words, v);
  }
}

template <int NW, bool FORCE, int Q0>
__device__ __forceinline__ void run_segment(const StepArgs& a, const Lanes& L, uint32_t ring,
                                            uint32_t bars, const Ctx<NW, FORCE>& cx, int r_begin,
                                            int r_end, unsigned& swaps) {
  using G = Geo<NW, FORCE>;
  const long long pitch = static_cast<long long>(a.pitch);
  const int first = r_begin - 1;          // source rows first .. r_end
  const int last = r_end;
  const uint32_t lane_off = 16u + L.lane * NW * 4u;
  auto slot_of = [&](int row) { return static_cast<uint32_t>((row - first) % G::kSlots); };
  auto issue = [&](int row) {
    if (L.lane == 0) {
      const uint32_t k = slot_of(row);
      issue_row<NW, FORCE>(a.src, pitch, row, static_cast<int>((a.row0 + row) & 1), L,
                           ring + k * G::kSlot, bars + k * 8u);
    }
  };
  auto wait = [&](int row) {
    const uint32_t k = slot_of(row);
    mbar_wait(bars + k * 8u, static_cast<uint32_t>(((row - first) / G::kSlots) & 1));
  };
  const int pro = min(last, first + G::kSlots - 1);
  for (int row = first; row <= pro; ++row) issue(row);
  wait(first);
  wait(first + 1);
  const uint32_t y0 = static_cast<uint32_t>(a.row0);  // global rows < 2^31
  uint32_t* out = reinterpret_cast<uint32_t*>(a.dst + r_begin * pitch) + L.w0 + L.lane * NW;
  const long long pw = pitch / 4;
  auto one = [&](int r, auto qc) {
    constexpr int Q = decltype(qc)::value;
    wait(r + 1);
    dest_row<NW, FORCE, Q>(ring + slot_of(r - 1) * G::kSlot + lane_off,
                           ring + slot_of(r) * G::kSlot + lane_off,
                           ring + slot_of(r + 1) * G::kSlot + lane_off, cx, L.lane, y0 + r, out,
                           L.WW, swaps);
    out += pw;
    // Slot of row r-1 is free once every lane has read it.
    __syncwarp();
    if (r - 1 + G::kSlots <= last) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(r - 1 + G::kSlots);
    }
  };
  int r = r_begin;
  for (; r + 2 <= r_end; r += 2) {
    one(r, std::integral_constant<int, Q0>{});
    one(r + 1, std::integral_constant<int, Q0 ^ 1>{});
  }
  if (r < r_end) one(r, std::integral_constant<int, Q0>{});
}

template <int NW, bool FORCE>
__global__ void __launch_bounds__(kPThreads, 1) step_planes_kernel(StepArgs a) {
  using G = Geo<NW, FORCE>;
  extern __shared__ __align__(128) uint8_t smem[];
  const uint32_t sbase = smem_u32(smem);
  const int warp = threadIdx.x >> 5;
  const int band_group = blockIdx.x % a.nbands_groups;
  const int seg_group = blockIdx.x / a.nbands_groups;
  const int cta_cols = a.bpc * G::kBandCols;
  const int cta_x0 = band_group * cta_cols;
  // smem: chirality keys [cta_cols], forcing keys [cta_cols], then per warp
  // the row ring, the walk list and results, the ring's mbarriers.
  const uint32_t kc_base = sbase;
  const uint32_t kf_base = sbase + cta_cols * 8;
  const uint32_t wbase = sbase + (FORCE ? 2 : 1) * cta_cols * 8 + warp * G::kWarp;
  const uint32_t ring = wbase;
  const uint32_t lsm = ring + G::kSlots * G::kSlot;
  const uint32_t osm = lsm + G::kList;
  const uint32_t bars = osm + G::kOut;
  if ((threadIdx.x & 31) == 0) {
    for (int k = 0; k < G::kSlots; ++k) mbar_init(bars + k * 8, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int c = threadIdx.x; c < cta_cols; c += blockDim.x) {
    sts64(kc_base + c * 8, a.zc[cta_x0 + c]);
    if (FORCE) sts64(kf_base + c * 8, a.zf[cta_x0 + c]);
  }
  // Next step's column keys (read by the next launch only).
  if (a.zc_next) {
    const int n = gridDim.x * blockDim.x;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < a.W; i += n) {
      a.zc_next[i] = column_key(a.kc_next, static_cast<uint64_t>(i) + 1);
      if (a.zf_next) a.zf_next[i] = column_key(a.kf_next, static_cast<uint64_t>(i) + 1);
    }
  }
  __syncthreads();

  const int bic = warp % a.bpc;
  const int band = band_group * a.bpc + bic;
  const int seg = seg_group * a.spc + warp / a.bpc;
  const int r_begin = a.row_lo + seg * a.seg_rows;
  if (warp >= a.bpc * a.spc || band >= a.nbands || r_begin >= a.row_hi) return;  // whole warp
  const int r_end = min(a.row_hi, r_begin + a.seg_rows);

  Lanes L;
  L.lane = threadIdx.x & 31;
  L.WW = a.W >> 5;
  L.w0 = band * G::kBandWords;
  L.wl = L.w0 == 0 ? L.WW - 4 : L.w0 - 4;
  L.wr = L.w0 + G::kBandWords == L.WW ? 0 : L.w0 + G::kBandWords;
  Ctx<NW, FORCE> cx;
  cx.kc = kc_base + bic * G::kBandCols * 8;
  cx.kf = kf_base + bic * G::kBandCols * 8;
  cx.lsm = lsm;
  cx.osm = osm;
  cx.thr = a.thr;
  unsigned swaps = 0;
  if ((a.row0 + r_begin) & 1)
    run_segment<NW, FORCE, 1>(a, L, ring, bars, cx, r_begin, r_end, swaps);
  else
    run_segment<NW, FORCE, 0>(a, L, ring, bars, cx, r_begin, r_end, swaps);
  if (FORCE) {
    unsigned long long s = swaps;
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(kFull, s, o);
    if (L.lane == 0 && s) atomicAdd(a.swaps, s);
  }
}

template <int NW, bool FORCE>
int smem_bytes(int bpc) {
  using G = Geo<NW, FORCE>;
  return (FORCE ? 2 : 1) * bpc * G::kBandCols * 8 + kPWarps * G::kWarp;
}

template <int NW, bool FORCE>
void launch_nw(StepArgs a, int num_sms, cudaStream_t st) {
  using G = Geo<NW, FORCE>;
  const int rows = a.row_hi - a.row_lo;
  a.nbands = a.W / G::kBandCols;
  // Bands per CTA: as many as the shared-memory budget allows (the column
  // keys of every band a CTA covers are staged).
  int bpc = a.nbands < kPWarps ? a.nbands : kPWarps;
  while (bpc > 1 && smem_bytes<NW, FORCE>(bpc) > 227 * 1024) bpc >>= 1;
  while (kPWarps % bpc) --bpc;
  a.bpc = bpc;
  a.spc = kPWarps / bpc;
  a.nbands_groups = (a.nbands + bpc - 1) / bpc;
  int seg_groups = num_sms / a.nbands_groups;
  if (seg_groups < 1) seg_groups = 1;
  int seg = (rows + seg_groups * a.spc - 1) / (seg_groups * a.spc);
  if (seg < 1) seg = 1;
  a.seg_rows = seg;
  const int nseg = (rows + seg - 1) / seg;
  seg_groups = (nseg + a.spc - 1) / a.spc;
  const int grid = a.nbands_groups * seg_groups;
  const int smem = smem_bytes<NW, FORCE>(bpc);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(step_planes_kernel<NW, FORCE>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    attr = true;
  }
  step_planes_kernel<NW, FORCE><<<grid, kPThreads, smem, st>>>(a);
}

// ---------------------------------------------------------------------------
// Converters. One thread per (row, word): 32 sites.
// ---------------------------------------------------------------------------
// Planes 0-6 from the node bytes, plane 7 from the obstacle mask (nonzero =
// solid) into both buffers: the planes are always "normalised" (bit 7 = mask,
// what the reference's motion pass derives, step.cpp:50).
__global__ void pack_kernel(const uint8_t* src, const uint8_t* mask, uint8_t* dst,
                            uint8_t* dst_obst, size_t pitch, int W, int nrows) {
  const int WW = W >> 5;
  const long long n = static_cast<long long>(nrows) * WW;
  for (long long t = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; t < n;
       t += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long r = t / WW;
    const int i = static_cast<int>(t % WW);
    const long long off = r * static_cast<long long>(pitch) + i * 32;
    const uint4* s = reinterpret_cast<const uint4*>(src + off);
    const uint4* m = reinterpret_cast<const uint4*>(mask + off);
    const uint4 lo = s[0], hi = s[1], mlo = m[0], mhi = m[1];
    uint32_t v[8] = {lo.x, lo.y, lo.z, lo.w, hi.x, hi.y, hi.z, hi.w};
    const uint32_t mv[8] = {mlo.x, mlo.y, mlo.z, mlo.w, mhi.x, mhi.y, mhi.z, mhi.w};
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      // nonzero mask byte -> bit 7 of the node byte
      const uint32_t nz = (mv[k] | (mv[k] >> 4)) & 0x0F0F0F0Fu;
      const uint32_t nz2 = (nz | (nz >> 2)) & 0x03030303u;
      const uint32_t nz1 = (nz2 | (nz2 >> 1)) & 0x01010101u;
      v[k] = (v[k] & 0x7F7F7F7Fu) | (nz1 << 7);
    }
    uint32_t* d = reinterpret_cast<uint32_t*>(dst + r * static_cast<long long>(pitch)) + i;
#pragma unroll
    for (int p = 0; p < 8; ++p) {
      uint32_t w = 0;
#pragma unroll
      for (int k = 0; k < 8; ++k)  // bytes 4k..4k+3: bit p of each -> 4 bits
        w |= ((((v[k] >> p) & 0x01010101u) * 0x01020408u) >> 24 & 0xFu) << (4 * k);
      d[p * WW] = w;
      if (p == 7)
        reinterpret_cast<uint32_t*>(dst_obst + r * static_cast<long long>(pitch))[7 * WW + i] = w;
    }
  }
}

__global__ void unpack_kernel(const uint8_t* src, uint8_t* dst, size_t pitch, int W, int nrows) {
  const int WW = W >> 5;
  const long long n = static_cast<long long>(nrows) * WW;
  for (long long t = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; t < n;
       t += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long r = t / WW;
    const int i = static_cast<int>(t % WW);
    const uint32_t* s = reinterpret_cast<const uint32_t*>(src + r * static_cast<long long>(pitch)) + i;
    uint32_t p[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) p[q] = s[q * WW];
    uint32_t v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      uint32_t b = 0;
#pragma unroll
      for (int q = 0; q < 8; ++q) b |= ((((p[q] >> (4 * k)) & 0xFu) * 0x00204081u) & 0x01010101u) << q;
      v[k] = b;
    }
    uint4* d = reinterpret_cast<uint4*>(dst + r * static_cast<long long>(pitch) + i * 32);
    d[0] = make_uint4(v[0], v[1], v[2], v[3]);
    d[1] = make_uint4(v[4], v[5], v[6], v[7]);
  }
}

int grid_for(long long n, int num_sms) {
  const long long g = (n + 255) / 256;
  return static_cast<int>(g < num_sms * 8LL ? (g > 0 ? g : 1) : num_sms * 8LL);
}

}  // namespace

int planes_words_per_lane(int W) {
  if (W <= 0 || W % 1024) return 0;
  const int bands1 = W / 1024;
  if (bands1 % 2 == 0) return 2;
  return 1;
}

bool planes_ok(int W) { return planes_words_per_lane(W) != 0; }

int launch_step_planes(const StepArgs& a, int num_sms, cudaStream_t st) {
  const int nw = planes_words_per_lane(a.W);
  const bool force = a.thr != 0;
  if (nw == 2) {
    if (force) launch_nw<2, true>(a, num_sms, st);
    else launch_nw<2, false>(a, num_sms, st);
  } else {
    if (force) launch_nw<1, true>(a, num_sms, st);
    else launch_nw<1, false>(a, num_sms, st);
  }
  return 1;
}

void launch_pack_planes(const uint8_t* src, const uint8_t* mask, uint8_t* dst, uint8_t* dst_obst,
                        size_t pitch, int W, int nrows, int num_sms, cudaStream_t st) {
  const long long n = static_cast<long long>(nrows) * (W >> 5);
  if (n <= 0) return;
  pack_kernel<<<grid_for(n, num_sms), 256, 0, st>>>(src, mask, dst, dst_obst, pitch, W, nrows);
}

void launch_unpack_planes(const uint8_t* src, uint8_t* dst, size_t pitch, int W, int nrows,
                          int num_sms, cudaStream_t st) {
  const long long n = static_cast<long long>(nrows) * (W >> 5);
  if (n <= 0) return;
  unpack_kernel<<<grid_for(n, num_sms), 256, 0, st>>>(src, dst, pitch, W, nrows);
}

}  // namespace fhpg
