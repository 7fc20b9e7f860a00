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

#include "fhpg_common.cuh"
#include "fhpg_kernels.cuh"
#include "fhpg_planes_rules.cuh"

namespace fhpg {
namespace {

constexpr unsigned kFull = 0xFFFFFFFFu;
constexpr int kPWarps = 8;
constexpr int kPThreads = kPWarps * 32;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint32_t lds32(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ uint64_t lds64(uint32_t a) {
  uint64_t v;
  asm volatile("ld.shared.u64 %0, [%1];" : "=l"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts32(uint32_t a, uint32_t v) {
  asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(v));
}
__device__ __forceinline__ void sts64(uint32_t a, uint64_t v) {
  asm volatile("st.shared.u64 [%0], %1;" ::"r"(a), "l"(v));
}
__device__ __forceinline__ void red_or(uint32_t a, uint32_t v) {
  asm volatile("red.shared.or.b32 [%0], %1;" ::"r"(a), "r"(v));
}
__device__ __forceinline__ uint32_t top_bit(uint32_t m) {
  uint32_t p;
  asm("bfind.u32 %0, %1;" : "=r"(p) : "r"(m));
  return p;
}

// NW consecutive words: vector loads / stores.
template <int NW>
__device__ __forceinline__ void ldv(const uint32_t* p, uint32_t (&v)[NW]) {
  if constexpr (NW == 4) {
    const uint4 t = __ldg(reinterpret_cast<const uint4*>(p));
    v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w;
  } else if constexpr (NW == 2) {
    const uint2 t = __ldg(reinterpret_cast<const uint2*>(p));
    v[0] = t.x; v[1] = t.y;
  } else {
    v[0] = __ldg(p);
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

// A source row as loaded: 8 planes of NW words, plus 4 band-edge words for
// the planes that shift (lane 0: word left of the band, lane 31: word right
// of it).
template <int NW>
struct Raw {
  uint32_t v[8][NW];
  uint32_t e[4];
};

// A source row after arrival processing: the planes as its three
// destination rows pull them (rows s-1: n0, n1; s: c2, c5, c6, c7; s+1: p3, p4).
template <int NW>
struct Src {
  uint32_t n0[NW], n1[NW], c2[NW], c5[NW], c6[NW], c7[NW], p3[NW], p4[NW];
};

struct Band {
  int lane;
  int WW;                 // words per plane row
  int plane_words;        // = WW (offset between planes, in words)
  int wlane;              // first word of this lane
  int wedge;              // edge word this lane loads (lane 0: left, 31: right)
};

// Shifted planes. L: out bit j = column x-1 (funnel with the previous word);
// R: out bit j = column x+1 (funnel with the next word).
template <int NW>
__device__ __forceinline__ void shift_l(const uint32_t (&v)[NW], uint32_t edge, int lane,
                                        uint32_t (&o)[NW]) {
  const uint32_t up = __shfl_up_sync(kFull, v[NW - 1], 1);
  const uint32_t prev = lane == 0 ? edge : up;
  o[0] = __funnelshift_l(prev, v[0], 1);
#pragma unroll
  for (int i = 1; i < NW; ++i) o[i] = __funnelshift_l(v[i - 1], v[i], 1);
}
template <int NW>
__device__ __forceinline__ void shift_r(const uint32_t (&v)[NW], uint32_t edge, int lane,
                                        uint32_t (&o)[NW]) {
  const uint32_t dn = __shfl_down_sync(kFull, v[0], 1);
  const uint32_t next = lane == 31 ? edge : dn;
#pragma unroll
  for (int i = 0; i < NW - 1; ++i) o[i] = __funnelshift_r(v[i], v[i + 1], 1);
  o[NW - 1] = __funnelshift_r(v[NW - 1], next, 1);
}
template <int NW>
__device__ __forceinline__ void copy(const uint32_t (&v)[NW], uint32_t (&o)[NW]) {
#pragma unroll
  for (int i = 0; i < NW; ++i) o[i] = v[i];
}

// Planes that shift for a source row of global parity PS (pull offsets,
// backends.cpp:64-73, with the destination row's parity q):
//   PS = 0: plane 0 R (dest s-1, q=1), 2 L, 4 R (dest s+1, q=1), 5 R
//   PS = 1: plane 1 L (dest s-1, q=0), 2 L, 3 L (dest s+1, q=0), 5 R
template <int PS>
__device__ __forceinline__ constexpr int edge_plane(int slot) {
  return PS == 0 ? (slot == 0 ? 0 : slot == 1 ? 2 : slot == 2 ? 4 : 5)
                 : (slot == 0 ? 1 : slot == 1 ? 2 : slot == 2 ? 3 : 5);
}

template <int NW, int PS>
__device__ __forceinline__ void load_row(const uint8_t* row, const Band& b, Raw<NW>& r) {
  const uint32_t* base = reinterpret_cast<const uint32_t*>(row);
#pragma unroll
  for (int p = 0; p < 8; ++p) ldv<NW>(base + p * b.plane_words + b.wlane, r.v[p]);
#pragma unroll
  for (int s = 0; s < 4; ++s) r.e[s] = __ldg(base + edge_plane<PS>(s) * b.plane_words + b.wedge);
}

template <int NW, int PS>
__device__ __forceinline__ void arrive(const Raw<NW>& r, int lane, Src<NW>& s) {
  if constexpr (PS == 0) {
    shift_r<NW>(r.v[0], r.e[0], lane, s.n0);
    copy<NW>(r.v[1], s.n1);
    shift_l<NW>(r.v[2], r.e[1], lane, s.c2);
    copy<NW>(r.v[3], s.p3);
    shift_r<NW>(r.v[4], r.e[2], lane, s.p4);
    shift_r<NW>(r.v[5], r.e[3], lane, s.c5);
  } else {
    copy<NW>(r.v[0], s.n0);
    shift_l<NW>(r.v[1], r.e[0], lane, s.n1);
    shift_l<NW>(r.v[2], r.e[1], lane, s.c2);
    shift_l<NW>(r.v[3], r.e[2], lane, s.p3);
    copy<NW>(r.v[4], s.p4);
    shift_r<NW>(r.v[5], r.e[3], lane, s.c5);
  }
  copy<NW>(r.v[6], s.c6);
  copy<NW>(r.v[7], s.c7);
}

// Balanced walk over the set bits of the warp's NW * 32 mask words (word
// i = lane * NW + w <-> band word i). The total T is split into 32 equal
// contiguous slices; each lane finds the start of its slice (binary search
// over the lanes' inclusive counts, then a popcount scan) and visits its
// sites two at a time. fn(i0, j0, i1, j1, has1) handles two sites (word
// index, bit) and returns the bits to OR into out[i] as (b0, b1).
template <int NW, typename Fn>
__device__ __forceinline__ void balanced_walk(const uint32_t (&m)[NW], uint32_t msm, int lane,
                                              Fn&& fn) {
  int cnt = 0;
#pragma unroll
  for (int w = 0; w < NW; ++w) cnt += __popc(m[w]);
  int incl = cnt;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const int v = __shfl_up_sync(kFull, incl, d);
    if (lane >= d) incl += v;
  }
  const int T = __shfl_sync(kFull, incl, 31);
  if (T == 0) return;
  const int s = (lane * T) >> 5;
  const int e = ((lane + 1) * T) >> 5;
  int o = 0;
#pragma unroll
  for (int step = 16; step; step >>= 1) {
    const int v = __shfl_sync(kFull, incl, o + step - 1);
    if (v <= s) o += step;
  }
  const int excl_o = __shfl_sync(kFull, incl - cnt, o);
  if (s >= e) return;
  int k = s - excl_o;
  uint32_t i = static_cast<uint32_t>(o * NW);
  uint32_t mask = lds32(msm + i * 4);
  for (;;) {
    const int c = __popc(mask);
    if (k < c) break;
    k -= c;
    ++i;
    mask = lds32(msm + i * 4);
  }
  for (; k > 0; --k) mask ^= 1u << top_bit(mask);
  auto next = [&](uint32_t& wi, uint32_t& bj) {
    while (mask == 0u) {
      ++i;
      mask = lds32(msm + i * 4);
    }
    bj = top_bit(mask);
    mask ^= 1u << bj;
    wi = i;
  };
  for (int it = s; it < e; it += 2) {
    uint32_t i0, j0, i1 = 0, j1 = 0;
    next(i0, j0);
    const bool has1 = it + 1 < e;
    if (has1) next(i1, j1);
    fn(i0, j0, i1, j1, has1);
  }
}

template <int NW, bool FORCE>
struct Ctx {
  uint32_t kc;      // smem: chirality keys of the band (8 B per column)
  uint32_t kf;      // smem: forcing keys of the band
  uint32_t msm;     // smem: warp's mask words [32 * NW]
  uint32_t osm;     // smem: warp's result words [32 * NW]
  uint64_t thr;
};

// One destination row r (global parity Q is implicit in the Src planes).
template <int NW, bool FORCE>
__device__ __forceinline__ void dest_row(const Src<NW>& Pm, const Src<NW>& Pc, const Src<NW>& Pn,
                                         const Ctx<NW, FORCE>& cx, int lane, uint32_t y,
                                         uint32_t* out_row, int plane_words, unsigned& swaps) {
  Fhp3Class K[NW];
  uint32_t dep[NW];
#pragma unroll
  for (int w = 0; w < NW; ++w) {
    const uint32_t a[6] = {Pn.n0[w], Pn.n1[w], Pc.c2[w], Pm.p3[w], Pm.p4[w], Pc.c5[w]};
    K[w] = fhp3_classify(a, Pc.c6[w], Pc.c7[w]);
    dep[w] = K[w].dep;
  }
  // Stage masks, clear results.
  const uint32_t mine = static_cast<uint32_t>(lane * NW) * 4u;
#pragma unroll
  for (int w = 0; w < NW; ++w) {
    sts32(cx.msm + mine + w * 4, dep[w]);
    sts32(cx.osm + mine + w * 4, 0u);
  }
  __syncwarp();
  // Chirality: bit 0 of node_random(seed, Chirality, step, x + 1, y)
  // = fin64(key[x] + y) (rng.hpp:25-33, step.cpp:73-76).
  balanced_walk<NW>(dep, cx.msm, lane, [&](uint32_t i0, uint32_t j0, uint32_t i1, uint32_t j1,
                                           bool has1) {
    const uint64_t k0 = lds64(cx.kc + (i0 * 32u + j0) * 8u);
    const uint64_t k1 = lds64(cx.kc + (i1 * 32u + j1) * 8u);
    const uint32_t b0 = fin64_bit0(k0 + y);
    const uint32_t b1 = fin64_bit0(k1 + y) & (has1 ? 1u : 0u);
    red_or(cx.osm + i0 * 4u, b0 << j0);
    red_or(cx.osm + i1 * 4u, b1 << j1);
  });
  __syncwarp();
  uint32_t o[NW][7];
#pragma unroll
  for (int w = 0; w < NW; ++w) {
    const uint32_t c = lds32(cx.osm + mine + w * 4);
    uint32_t oo[6], orr;
    fhp3_apply(K[w], c, Pc.c6[w], oo, orr);
#pragma unroll
    for (int p = 0; p < 6; ++p) o[w][p] = oo[p];
    o[w][6] = orr;
  }
  if constexpr (FORCE) {
    // step.cpp:79-88: fluid, W (bit 5) set, E (bit 2) clear after collision.
    uint32_t f[NW];
#pragma unroll
    for (int w = 0; w < NW; ++w) f[w] = ~Pc.c7[w] & o[w][5] & ~o[w][2];
    __syncwarp();
#pragma unroll
    for (int w = 0; w < NW; ++w) {
      sts32(cx.msm + mine + w * 4, f[w]);
      sts32(cx.osm + mine + w * 4, 0u);
    }
    __syncwarp();
    balanced_walk<NW>(f, cx.msm, lane, [&](uint32_t i0, uint32_t j0, uint32_t i1, uint32_t j1,
                                           bool has1) {
      const uint64_t k0 = lds64(cx.kf + (i0 * 32u + j0) * 8u);
      const uint64_t k1 = lds64(cx.kf + (i1 * 32u + j1) * 8u);
      const uint32_t b0 = (fin64(k0 + y) >> 32) < cx.thr ? 1u : 0u;
      const uint32_t b1 = has1 && (fin64(k1 + y) >> 32) < cx.thr ? 1u : 0u;
      red_or(cx.osm + i0 * 4u, b0 << j0);
      red_or(cx.osm + i1 * 4u, b1 << j1);
    });
    __syncwarp();
#pragma unroll
    for (int w = 0; w < NW; ++w) {
      const uint32_t acc = lds32(cx.osm + mine + w * 4);
      o[w][5] ^= acc;
      o[w][2] ^= acc;
      swaps += __popc(acc);
    }
  }
  __syncwarp();  // the next row restages msm / osm
#pragma unroll
  for (int p = 0; p < 7; ++p) {
    uint32_t v[NW];
#pragma unroll
    for (int w = 0; w < NW; ++w) v[w] = o[w][p];
    stv<NW>(out_row + p * plane_words, v);
  }
}

template <int NW, bool FORCE, int Q0>
__device__ __forceinline__ void run_segment(const StepArgs& a, const Band& b,
                                            const Ctx<NW, FORCE>& cx, int r_begin, int r_end,
                                            unsigned& swaps) {
  constexpr int Q1 = Q0 ^ 1;
  const long long pitch = static_cast<long long>(a.pitch);
  const uint8_t* src = a.src;
  // Rows r-1 (parity Q1), r (Q0), r+1 (Q1) arrive; r+2 (Q0), r+3 (Q1) in flight.
  Src<NW> Sm, Sc, Sn;
  {
    Raw<NW> t;
    load_row<NW, Q1>(src + (r_begin - 1) * pitch, b, t);
    arrive<NW, Q1>(t, b.lane, Sm);
    load_row<NW, Q0>(src + r_begin * pitch, b, t);
    arrive<NW, Q0>(t, b.lane, Sc);
    load_row<NW, Q1>(src + (r_begin + 1) * pitch, b, t);
    arrive<NW, Q1>(t, b.lane, Sn);
  }
  Raw<NW> R0, R1;  // rows r+2 (parity Q0) and r+3 (parity Q1)
  // Only rows up to r_end are needed (a spare zero row follows the bottom halo).
  if (r_begin + 2 <= r_end + 1) load_row<NW, Q0>(src + (r_begin + 2) * pitch, b, R0);
  if (r_begin + 3 <= r_end) load_row<NW, Q1>(src + (r_begin + 3) * pitch, b, R1);
  const uint32_t y0 = static_cast<uint32_t>(a.row0);  // global rows < 2^31
  uint32_t* out = reinterpret_cast<uint32_t*>(a.dst + r_begin * pitch) + b.wlane;
  const long long pw = pitch / 4;
  int r = r_begin;
  // Two rows per iteration so that every parity is a compile-time constant.
  // Spare zero rows below the bottom halo make the over-prefetch safe.
  for (; r + 2 <= r_end; r += 2) {
    dest_row<NW, FORCE>(Sm, Sc, Sn, cx, b.lane, y0 + r, out, b.plane_words, swaps);
    out += pw;
    Sm = Sc;
    Sc = Sn;
    arrive<NW, Q0>(R0, b.lane, Sn);
    if (r + 4 <= r_end) load_row<NW, Q0>(src + (r + 4) * pitch, b, R0);
    dest_row<NW, FORCE>(Sm, Sc, Sn, cx, b.lane, y0 + r + 1, out, b.plane_words, swaps);
    out += pw;
    Sm = Sc;
    Sc = Sn;
    arrive<NW, Q1>(R1, b.lane, Sn);
    if (r + 5 <= r_end) load_row<NW, Q1>(src + (r + 5) * pitch, b, R1);
  }
  if (r < r_end) dest_row<NW, FORCE>(Sm, Sc, Sn, cx, b.lane, y0 + r, out, b.plane_words, swaps);
}

template <int NW, bool FORCE>
__global__ void __launch_bounds__(kPThreads, 1) step_planes_kernel(StepArgs a) {
  extern __shared__ __align__(16) uint8_t smem[];
  const uint32_t sbase = smem_u32(smem);
  constexpr int kBandCols = NW * 1024;
  const int warp = threadIdx.x >> 5;
  const int band_group = blockIdx.x % a.nbands_groups;
  const int seg_group = blockIdx.x / a.nbands_groups;
  const int cta_cols = a.bpc * kBandCols;
  const int cta_x0 = band_group * cta_cols;
  // smem: chirality keys [cta_cols], forcing keys [cta_cols], per warp 2 x 32 NW words.
  const uint32_t kc_base = sbase;
  const uint32_t kf_base = sbase + cta_cols * 8;
  const uint32_t warp_base = sbase + (FORCE ? 2 : 1) * cta_cols * 8 + warp * (2 * 32 * NW * 4);
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

  Band b;
  b.lane = threadIdx.x & 31;
  b.WW = a.W >> 5;
  b.plane_words = a.W >> 5;
  const int w0 = band * 32 * NW;
  b.wlane = w0 + b.lane * NW;
  b.wedge = b.lane == 0 ? (w0 == 0 ? b.WW - 1 : w0 - 1)
                        : (b.lane == 31 ? (w0 + 32 * NW == b.WW ? 0 : w0 + 32 * NW) : b.wlane);
  Ctx<NW, FORCE> cx;
  cx.kc = kc_base + bic * kBandCols * 8;
  cx.kf = kf_base + bic * kBandCols * 8;
  cx.msm = warp_base;
  cx.osm = warp_base + 32 * NW * 4;
  cx.thr = a.thr;
  unsigned swaps = 0;
  if ((a.row0 + r_begin) & 1)
    run_segment<NW, FORCE, 1>(a, b, cx, r_begin, r_end, swaps);
  else
    run_segment<NW, FORCE, 0>(a, b, cx, r_begin, r_end, swaps);
  if (FORCE) {
    unsigned long long s = swaps;
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(kFull, s, o);
    if (b.lane == 0 && s) atomicAdd(a.swaps, s);
  }
}

template <int NW, bool FORCE>
int smem_bytes(int bpc) {
  return (FORCE ? 2 : 1) * bpc * NW * 1024 * 8 + kPWarps * 2 * 32 * NW * 4;
}

template <int NW, bool FORCE>
void launch_nw(StepArgs a, int num_sms, cudaStream_t st) {
  constexpr int kBandCols = NW * 1024;
  const int rows = a.row_hi - a.row_lo;
  a.nbands = a.W / kBandCols;
  // Bands per CTA: all of a row's bands when they fit (edge words then come
  // from the same SM's recent loads), within the shared-memory budget.
  int bpc = a.nbands < kPWarps ? a.nbands : kPWarps;
  while (bpc > 1 && smem_bytes<NW, FORCE>(bpc) > 200 * 1024) bpc >>= 1;
  while (kPWarps % bpc) --bpc;
  a.bpc = bpc;
  a.spc = kPWarps / bpc;
  a.nbands_groups = (a.nbands + bpc - 1) / bpc;
  int seg_groups = num_sms / a.nbands_groups;
  if (seg_groups < 1) seg_groups = 1;
  int seg = (rows + seg_groups * a.spc - 1) / (seg_groups * a.spc);
  if (seg < 2) seg = 2;
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
