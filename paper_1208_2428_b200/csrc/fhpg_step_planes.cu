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
// Layout. A lattice row holds 8 bit planes (0-5 movers NW..W, 6 rest, 7
// obstacle); bit j of word i of a plane = column 32 i + j. Each plane row is
// W/32 words plus 4 pad words on either side holding the periodic wrap
// (words W/32-4 .. W/32-1 on the left, 0 .. 3 on the right), so a row is
// W + 256 bytes and every band's row, edges included, is one rectangular
// TMA box. Pitch, halo rows and spare rows follow the byte layout. The
// obstacle plane is static: the pack kernel writes it into both ping-pong
// buffers and the step never does, so a step moves the algorithmic 15 bits
// per site (8 planes read, 7 written) plus the pad words.
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

#include <cuda.h>
#include <cudaTypedefs.h>

#include "fhpg_common.cuh"
#include "fhpg_kernels.cuh"
#include "fhpg_planes_rules.cuh"

// 4 words per lane (8 warps per SM) measured slower than 2 (16 warps):
// 1368 vs 1646 GSUPS on cfg4; build with -DFHPG_PLANES_NW4=4 to select it.
#ifndef FHPG_PLANES_NW4
#define FHPG_PLANES_NW4 2
#endif

namespace fhpg {
namespace {

#include "fhpg_planes_dev.cuh"  // shared device helpers (in this anonymous namespace)
template <int NW, bool FORCE, int RULE, int Q, typename Rel>
__device__ __forceinline__ void dest_row(uint32_t sm, uint32_t sc, uint32_t sn,
                                         const Ctx<NW, FORCE>& cx, int lane, uint32_t y,
                                         const CUtensorMap* stmap, const CUtensorMap* padmap,
                                         int w0, int trow, int pad, int padx,
                                         bool pad_band, unsigned& swaps, Rel&& released) {
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
  released();
#if FHPG_STREAM_ONLY && FHPG_STREAM_ONLY < 5
  // Timing experiment only (wrong results): the memory pipeline without the
  // collision and the chirality walk.
  if (lane == 0) bulk_wait_read();
  __syncwarp();
#pragma unroll
  for (int p = 0; p < 7; ++p) {
    uint32_t v[NW];
#pragma unroll
    for (int w = 0; w < NW; ++w)
      v[w] = (p == 0 ? a0[w] : p == 1 ? a1[w] : p == 2 ? a2[w] : p == 3 ? a3[w] : p == 4 ? a4[w]
              : p == 5 ? a5[w] : rr[w]) ^ so[w];
    stsv<NW>(cx.stage + p * (4 * 32 * NW) + lane * NW * 4, v);
  }
#if FHPG_STREAM_ONLY == 4  // timing experiment: loads + shared reads only
  (void)swaps; (void)y; (void)pad; (void)padx; (void)pad_band; (void)padmap; (void)stmap;
  return;
#endif
  fence_async_smem();
  __syncwarp();
  if (lane == 0 && FHPG_STREAM_ONLY != 2) {  // 2: loads only
    tma_store(stmap, w0 + 4, trow, cx.stage);
    bulk_commit();
  }
  (void)swaps; (void)y; (void)pad; (void)padx; (void)pad_band; (void)padmap;
  return;
#endif
  typename PlaneRule<RULE>::Class K[NW];
  uint32_t dep[NW];
#pragma unroll
  for (int w = 0; w < NW; ++w) {
    const uint32_t a[6] = {a0[w], a1[w], a2[w], a3[w], a4[w], a5[w]};
    K[w] = PlaneRule<RULE>::classify(a, rr[w], so[w]);
    dep[w] = K[w].dep;
  }
  // The previous row's TMA store must have read the staging area (which
  // also holds the walk scratch) before it is rewritten.
  if (lane == 0) bulk_wait_read();
  __syncwarp();
  // Chirality: bit 0 of node_random(seed, Chirality, step, x + 1, y)
  // = fin64(key[x] + y) (rng.hpp:25-33, step.cpp:73-76).
  // (chir_bit: fin64 bit 0 with fewer ALU-pipe instructions.)
  const int T = walk<NW>(dep, cx.lsm, cx.osm, cx.kc, lane,
                         [&](uint32_t ka) { return chir_bit(lds64(ka) + y, cx.four); });
  uint32_t o[NW][7];
  const uint32_t mine = cx.osm + lane * NW * 4;
#pragma unroll
  for (int w = 0; w < NW; ++w) {
    const uint32_t c = T ? lds32(mine + w * 4) : 0u;
    uint32_t oo[6], orr;
    const uint32_t a[6] = {a0[w], a1[w], a2[w], a3[w], a4[w], a5[w]};
    PlaneRule<RULE>::apply(K[w], c, rr[w], a, oo, orr, so[w]);
#pragma unroll
    for (int p = 0; p < 6; ++p) o[w][p] = oo[p];
    o[w][6] = orr;
  }
  if constexpr (FORCE) {
    // step.cpp:79-88: fluid, W (bit 5) set, E (bit 2) clear after collision.
    uint32_t f[NW];
#pragma unroll
    for (int w = 0; w < NW; ++w) f[w] = ~so[w] & o[w][5] & ~o[w][2];
    const int TF = walk<NW>(f, cx.lsm, cx.osm, cx.kf, lane, [&](uint32_t ka) {
      return (fin64(lds64(ka) + y) >> 32) < cx.thr ? 1u : 0u;
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
    stsv<NW>(cx.stage + p * (4 * 32 * NW) + lane * NW * 4, v);
    // periodic wrap copies: lanes holding words 0..3 / WW-4..WW-1
    if (pad_band && pad >= 0) stsv<NW>(cx.stage + pad + p * 16, v);
  }
  fence_async_smem();
  __syncwarp();
  if (lane == 0) {
#if FHPG_STREAM_ONLY != 6  // 6: no stores (timing experiment)
    tma_store(stmap, w0 + 4, trow, cx.stage);
    if (pad_band) {
      if (padx & 1) tma_store(padmap, 0, trow, cx.stage + Geo<NW, FORCE>::kPadL);
      if (padx & 2) tma_store(padmap, (padx >> 2) + 4, trow, cx.stage + Geo<NW, FORCE>::kPadR);
    }
#endif
    bulk_commit();
  }
}

template <int NW, bool FORCE, int RULE, int Q0>
__device__ __forceinline__ void run_segment(const StepArgs& a, const CUtensorMap* map,
                                            const CUtensorMap* stmap, const CUtensorMap* padmap,
                                            const Lanes& L, uint32_t ring, uint32_t bars,
                                            const Ctx<NW, FORCE>& cx, int r_begin, int r_end,
                                            unsigned& swaps) {
  using G = Geo<NW, FORCE>;
  const long long pitch = static_cast<long long>(a.pitch);
  const int first = r_begin - 1;  // source rows first .. r_end (local; tensor row = local + 1)
  const int last = r_end;
  const uint32_t lane_off = 16u + L.lane * NW * 4u;
  // Ring position of the next row to issue / of rows r-1, r, r+1, and the
  // mbarrier phase of each slot, tracked incrementally.
  uint32_t phase = 0;  // bit k: phase of slot k's next completion
  int issue_row = first, issue_slot = 0;
  auto issue = [&]() {
    if (L.lane == 0) {
      const uint32_t bar = bars + issue_slot * 8u;
      mbar_expect_tx(bar, G::kRowBytes);
      tma_row(ring + issue_slot * G::kSlot, map, L.w0, issue_row + 1, bar);
    }
    ++issue_row;
    issue_slot = issue_slot + 1 == G::kSlots ? 0 : issue_slot + 1;
  };
  auto wait = [&](int slot) {
    mbar_wait(bars + slot * 8u, (phase >> slot) & 1u);
    phase ^= 1u << slot;
  };
  while (issue_row <= last && issue_row < first + G::kSlots) issue();
  int sm = 0, sc = 1, sn = 2;  // slots of rows r-1, r, r+1
  wait(sm);
  wait(sc);
  const uint32_t y0 = static_cast<uint32_t>(a.row0);  // global rows < 2^31
  (void)pitch;
  auto one = [&](int r, auto qc) {
    constexpr int Q = decltype(qc)::value;
    wait(sn);
    dest_row<NW, FORCE, RULE, Q>(ring + sm * G::kSlot + lane_off, ring + sc * G::kSlot + lane_off,
                           ring + sn * G::kSlot + lane_off, cx, L.lane, y0 + r, stmap, padmap,
                           L.w0, r + 1, L.pad, L.padx, L.pad_band, swaps, [] {});
    // The slot of row r-1 is free once every lane has read it.
    __syncwarp();
    if (issue_row <= last) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue();
    }
    sm = sc;
    sc = sn;
    sn = sn + 1 == G::kSlots ? 0 : sn + 1;
  };
  int r = r_begin;
  for (; r + 2 <= r_end; r += 2) {
    one(r, std::integral_constant<int, Q0>{});
    one(r + 1, std::integral_constant<int, Q0 ^ 1>{});
  }
  if (r < r_end) one(r, std::integral_constant<int, Q0>{});
  if (L.lane == 0) bulk_wait_all();  // the stores have landed before the kernel ends
}

template <int NW, bool FORCE, int RULE>
__global__ void __launch_bounds__(kPWarps<NW> * 32, 1)
    step_planes_kernel(StepArgs a, const __grid_constant__ CUtensorMap map,
                       const __grid_constant__ CUtensorMap stmap,
                       const __grid_constant__ CUtensorMap padmap) {
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
  const uint32_t stage = ring + G::kSlots * G::kSlot;
  const uint32_t lsm = stage;
  const uint32_t osm = lsm + G::kList;
  const uint32_t bars = stage + G::kStageAll;
  if ((threadIdx.x & 31) == 0) {
    for (int k = 0; k < G::kSlots; ++k) mbar_init(bars + k * 8, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // Column keys from the step keys (independent of the previous step, so
  // this overlaps its tail under PDL), then wait for the previous grid.
  for (int c = threadIdx.x; c < cta_cols; c += blockDim.x) {
    const uint64_t x = static_cast<uint64_t>(cta_x0 + c) + 1;
    sts64(kc_base + c * 8, column_key(a.kc_cur, x));
    if (FORCE) sts64(kf_base + c * 8, column_key(a.kf_cur, x));
  }
#if FHPG_PDL
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
#endif
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
  L.PW = L.WW + 8;
  L.w0 = band * G::kBandWords;
  // Lanes holding words 0..3 / WW-4..WW-1 also stage the right / left pad
  // box (periodic wrap copies): words 0..3 go to padded words WW+4..WW+7,
  // words WW-4..WW-1 to padded words 0..3.
  const int wl = L.w0 + L.lane * NW;
  L.pad = wl < 4 ? G::kPadR + wl * 4 : (wl >= L.WW - 4 ? G::kPadL + (wl - (L.WW - 4)) * 4 : -1);
  L.padx = (L.w0 + G::kBandWords == L.WW ? 1 : 0) | (L.w0 == 0 ? 2 : 0) | (L.WW << 2);
  L.pad_band = L.w0 == 0 || L.w0 + G::kBandWords == L.WW;
  Ctx<NW, FORCE> cx;
  cx.kc = kc_base + bic * G::kBandCols * 8;
  cx.kf = kf_base + bic * G::kBandCols * 8;
  cx.lsm = lsm;
  cx.osm = osm;
  cx.stage = stage;
  cx.thr = a.thr;
  cx.four = a.k4;
  unsigned swaps = 0;
  if ((a.row0 + r_begin) & 1)
    run_segment<NW, FORCE, RULE, 1>(a, &map, &stmap, &padmap, L, ring, bars, cx, r_begin, r_end, swaps);
  else
    run_segment<NW, FORCE, RULE, 0>(a, &map, &stmap, &padmap, L, ring, bars, cx, r_begin, r_end, swaps);
  if (FORCE) {
    unsigned long long s = swaps;
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(kFull, s, o);
    if (L.lane == 0 && s) atomicAdd(a.swaps, s);
  }
}

// ---------------------------------------------------------------------------
// CTA-shared row ring (default). One CTA = one band x a segment of rows; a
// producer warp streams the segment's source rows into a ring of kRing
// slots with TMA (full barriers), kCons consumer warps take destination rows
// round-robin (warp k: rows R0 + k, R0 + k + kCons, ...), read their three
// source rows from the shared ring and release them (empty barriers, 3
// consumers per source row). Sharing the ring lets 20 warps per SM stream
// with a deep prefetch in the shared-memory budget that per-warp rings
// spend on 16.
// ---------------------------------------------------------------------------
// Consumer warps per CTA and ring slots (A/B on cfg4: 16/36 1570, 20/44
// 1695, 24/52 1766, 30/64 1876, 31/48 1889 GSUPS).
// Back-off of a consumer polling a slot's tag (ns): spinning warps take
// issue slots from the working ones.
#ifndef FHPG_TAG_SLEEP
#define FHPG_TAG_SLEEP 64
#endif
// Source rows per TMA box: the producer warp's issue rate (one elected
// thread: empty-barrier wait, tag, expect_tx, TMA per box) bounds the ring's
// throughput, so each box carries several rows.
#ifndef FHPG_BOX_ROWS
#define FHPG_BOX_ROWS 4  // (2: 1972, 4: 1987-1995 GSUPS on cfg4)
#endif
#ifndef FHPG_EXTRA_CTAS
#define FHPG_EXTRA_CTAS 1
#endif
#ifndef FHPG_EXTRA_BUBBLE_ROWS
#define FHPG_EXTRA_BUBBLE_ROWS 20
#endif
#ifndef FHPG_RING_CONS
#define FHPG_RING_CONS 31
#endif
// Consumers take destination rows from a shared counter (1) instead of the
// static round-robin (0) (measured: 2097 vs 2111 GSUPS on cfg4, kept off).
#ifndef FHPG_DYN_ROWS
#define FHPG_DYN_ROWS 0
#endif
// Back-off (ns) of the producer between polls of a ring slot's empty barrier
// (measured: no effect at 200 or 1000 ns).
#ifndef FHPG_PROD_SLEEP
#define FHPG_PROD_SLEEP 0
#endif
template <int NW, bool FORCE>
struct RingGeo {
  using G = Geo<NW, FORCE>;
  static constexpr int kCons = FHPG_RING_CONS;
#ifdef FHPG_RING_SLOTS
  static constexpr int kRing = FORCE ? FHPG_RING_SLOTS_F : FHPG_RING_SLOTS;
#else
  // Powers of two: the consumer loop divides by the ring and group counts
  // (the forcing variant's two key tables leave room for 56 slots, but 32
  // measured 1-3% faster on the forced BASELINE shapes than 56 or 48).
  static constexpr int kRing = FORCE ? 32 : 64;
#endif
  static constexpr int kThreads = (kCons + 1) * 32;
  static constexpr int kKeys = (FORCE ? 2 : 1) * G::kBandCols * 8;
  static constexpr int kRingOff = (kKeys + 127) / 128 * 128;
  static constexpr int kStageOff = kRingOff + kRing * G::kSlot;
  static constexpr int kBarOff = kStageOff + kCons * G::kStageAll;
  static constexpr int kTagOff = kBarOff + 2 * 8 * kRing;
  static constexpr int kCtrOff = kTagOff + 4 * kRing;  // dynamic row counters (2 parts)
  static constexpr int kSmem = kCtrOff + 8;
  static_assert(kSmem <= 232448, "shared memory per CTA");
  static constexpr int kBox = FHPG_BOX_ROWS;     // source rows per TMA box (a "group")
  static constexpr int kGroups = kRing / kBox;   // ring slots of whole groups
  static_assert(kRing % kBox == 0, "row groups");
};

__device__ __forceinline__ void mbar_arrive(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}

template <int NW, bool FORCE, int RULE>
__global__ void __launch_bounds__(RingGeo<NW, FORCE>::kThreads, 1)
    step_ring_kernel(StepArgs a, const __grid_constant__ CUtensorMap map,
                     const __grid_constant__ CUtensorMap stmap,
                     const __grid_constant__ CUtensorMap padmap,
                     const __grid_constant__ CUtensorMap map2) {
  using G = Geo<NW, FORCE>;
  using RG = RingGeo<NW, FORCE>;
  extern __shared__ __align__(128) uint8_t smem[];
  const uint32_t sbase = smem_u32(smem);
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  // Work of this CTA: part A = band bA, rows [RA0, RA0 + nA), and for the
  // extra CTAs (the SMs left over by nbands x segment groups) part B = band
  // bA + 1 over the same rows. Main CTAs: a band x a segment of one of the
  // row ranges (the second range: a strip's boundary rows); with extra CTAs
  // the first range's last extra_rows rows of every band go to them, the
  // bands still walking the same rows at the same time (adjacent bands share
  // the sectors at their edges in L2).
  const int nmain = a.nbands * (a.segs1 + a.segs2);
  int bA, RA0, nA, nB = 0;
  int row_lo;
  if (static_cast<int>(blockIdx.x) < nmain) {
    bA = blockIdx.x % a.nbands;
    const bool second = static_cast<int>(blockIdx.x / a.nbands) >= a.segs1;
    const int seg_group = blockIdx.x / a.nbands - (second ? a.segs1 : 0);
    row_lo = second ? a.row_lo2 : a.row_lo;
    const int row_hi = second ? a.row_hi2 : a.row_hi - a.extra_rows;
    RA0 = row_lo + seg_group * a.seg_rows;
    nA = max(0, min(row_hi, RA0 + a.seg_rows) - RA0);
  } else {
    bA = 2 * (blockIdx.x - nmain);
    row_lo = a.row_hi - a.extra_rows;
    RA0 = row_lo;
    nA = a.extra_rows;
    nB = bA + 1 < a.nbands ? a.extra_rows : 0;
  }
  constexpr uint32_t B = RG::kBox;
  // Ring index layout: part A's source rows RA0-1 .. RA0+nA, then part B's
  // (row_lo-1 .. row_lo+nB) from the next whole group on.
  const uint32_t offB = (static_cast<uint32_t>(nA) + 2 + B - 1) / B * B;
  const uint32_t kc_base = sbase;
  const uint32_t kf_base = sbase + G::kBandCols * 8;
  const uint32_t ring = sbase + RG::kRingOff;
  const uint32_t full = sbase + RG::kBarOff;
  const uint32_t empty = full + 8 * RG::kRing;
  // tag[k] = ring index of the row the producer last issued into slot k. A
  // consumer visits only every kCons-th row, so a bare parity wait could
  // mistake a slot two phases old for the one it needs; it first waits for
  // the tag, after which the full barrier's parity is unambiguous.
  const uint32_t tags = sbase + RG::kTagOff;
  if (threadIdx.x == 0) {
    for (int k = 0; k < RG::kRing; ++k) {
      // Source rows come in groups of kBox (one TMA box): group P = index /
      // kBox uses barriers / tag P mod kGroups (3 consumers per row).
      mbar_init(full + k * 8, 1);
      mbar_init(empty + k * 8, 3 * RG::kBox);
      sts32(tags + k * 4, 0xFFFFFFFFu);
    }
    sts32(sbase + RG::kCtrOff, 0u);
    sts32(sbase + RG::kCtrOff + 4, 0u);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // The band's column keys, made here from the step keys (they depend on
  // nothing the previous step wrote, so this overlaps its tail under PDL).
  auto make_keys = [&](int b, int t0, int nt) {
    for (int c = t0; c < G::kBandCols; c += nt) {
      const uint64_t x = static_cast<uint64_t>(b * G::kBandCols + c) + 1;
      sts64(kc_base + c * 8, column_key(a.kc_cur, x));
      if (FORCE) sts64(kf_base + c * 8, column_key(a.kf_cur, x));
    }
  };
  make_keys(bA, threadIdx.x, blockDim.x);
#if FHPG_PDL
  // Let the next step's grid launch now; wait for the previous step's grid
  // (the lattice rows it wrote, the key buffers it read) before going on.
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
#endif
  if (a.zc_next) {  // next step's column keys (read by the next launch only)
    const int n = gridDim.x * blockDim.x;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < a.W; i += n) {
      a.zc_next[i] = column_key(a.kc_next, static_cast<uint64_t>(i) + 1);
      if (a.zf_next) a.zf_next[i] = column_key(a.kf_next, static_cast<uint64_t>(i) + 1);
    }
  }
  __syncthreads();
  if (nA + nB <= 0) return;

  if (warp == RG::kCons) {  // producer (tensor row = local row + 1)
    if (lane == 0) {
      constexpr uint32_t kG = RG::kGroups;
      const uint32_t gA = offB / B;
      const uint32_t ngroups = gA + (nB > 0 ? (static_cast<uint32_t>(nB) + 2 + B - 1) / B : 0u);
      for (uint32_t P = 0; P < ngroups; ++P) {
        const uint32_t k = P % kG;
        if (P >= kG) {
#if FHPG_PROD_SLEEP
          uint32_t done;
          for (;;) {
            asm volatile(
                "{ .reg .pred p; mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                : "=r"(done) : "r"(empty + k * 8), "r"((P / kG - 1) & 1u) : "memory");
            if (done) break;
            __nanosleep(FHPG_PROD_SLEEP);
          }
#else
          mbar_wait(empty + k * 8, (P / kG - 1) & 1u);
#endif
        }
        {  // tag: an atomic store (consumers poll it; not a data race)
          uint32_t prev;
          asm volatile("atom.shared.exch.b32 %0, [%1], %2;" : "=r"(prev) : "r"(tags + k * 4), "r"(P) : "memory");
        }
        const bool inA = P < gA;
        const int word = (inA ? bA : bA + 1) * G::kBandWords;
        const int trow = inA ? RA0 + static_cast<int>(B * P) : row_lo + static_cast<int>(B * P - offB);
#if FHPG_STREAM_ONLY == 3 || FHPG_STREAM_ONLY >= 5  // timing experiments: no loads
        if (FHPG_STREAM_ONLY >= 5 && P < kG) {  // 5, 6: compute on the first ring fill
          mbar_expect_tx(full + k * 8, B * G::kRowBytes);
          tma_row(ring + B * k * G::kSlot, &map2, word, trow, full + k * 8);
        } else {
          mbar_arrive(full + k * 8, 1);
        }
#else
        mbar_expect_tx(full + k * 8, B * G::kRowBytes);
        tma_row(ring + B * k * G::kSlot, &map2, word, trow, full + k * 8);  // tensor rows
#endif
        // Ring indices no destination row reads (the tail of part A's last
        // group when part B follows) still count 3 arrivals each, or the
        // slot is never freed.
        if (nB > 0 && P + 1 == gA && offB > static_cast<uint32_t>(nA) + 2)
          mbar_arrive(empty + k * 8, 3 * (offB - static_cast<uint32_t>(nA) - 2));
      }
    }
    return;
  }

  Lanes L;
  L.lane = lane;
  L.WW = a.W >> 5;
  L.PW = L.WW + 8;
  auto set_band = [&](int b) {
    L.w0 = b * G::kBandWords;
    const int wl = L.w0 + L.lane * NW;
    L.pad = wl < 4 ? G::kPadR + wl * 4 : (wl >= L.WW - 4 ? G::kPadL + (wl - (L.WW - 4)) * 4 : -1);
    L.padx = (L.w0 + G::kBandWords == L.WW ? 1 : 0) | (L.w0 == 0 ? 2 : 0) | (L.WW << 2);
    L.pad_band = L.w0 == 0 || L.w0 + G::kBandWords == L.WW;
  };
  set_band(bA);
  const uint32_t stage = sbase + RG::kStageOff + warp * G::kStageAll;
  Ctx<NW, FORCE> cx;
  cx.kc = kc_base;
  cx.kf = kf_base;
  cx.lsm = stage;
  cx.osm = stage + G::kList;
  cx.stage = stage;
  cx.thr = a.thr;
  cx.four = a.k4;
  unsigned swaps = 0;
  const uint32_t lane_off = 16u + lane * NW * 4u;
  const uint32_t y0 = static_cast<uint32_t>(a.row0);  // global rows < 2^31
  // Destination rows [Rb, Re) of the current band, warp-interleaved; source
  // row r - 1 sits at ring index ibase + r - Rb. Inlined once per part (one
  // copy inside a loop over the parts measured 8% slower: spills).
  auto rows = [&](const int Rb, const int Re, const uint32_t ibase, const uint32_t ctr) {
#if FHPG_DYN_ROWS
    for (;;) {
      int r = 0;
      if (lane == 0) asm volatile("atom.shared.add.u32 %0, [%1], 1;" : "=r"(r) : "r"(ctr) : "memory");
      r = Rb + __shfl_sync(kFull, r, 0);
      if (r >= Re) break;
#else
    (void)ctr;
    for (int r = Rb + warp; r < Re; r += RG::kCons) {
#endif
      const uint32_t i = ibase + static_cast<uint32_t>(r - Rb);  // ring index of source row r - 1
      const bool first_row = r == Rb, last_row = r == Re - 1;
      constexpr uint32_t kG = RG::kGroups;
      uint32_t sl[3];
#pragma unroll
      for (uint32_t d = 0; d < 3; ++d) {
        const uint32_t P = (i + d) / B;
        if (d == 0 || ((i + d) % B) == 0) {  // a new group
          const uint32_t kp = P % kG;
          for (;;) {
            uint32_t tag;
            asm volatile("ld.relaxed.cta.shared.u32 %0, [%1];"
                         : "=r"(tag) : "r"(tags + kp * 4) : "memory");
            if (tag == P) break;
            __nanosleep(FHPG_TAG_SLEEP);
          }
          mbar_wait(full + kp * 8, (P / kG) & 1u);
        }
        sl[d] = ring + ((i + d) % RG::kRing) * G::kSlot + lane_off;
      }
      // Release the three source rows as soon as they are in registers (3
      // consumers per row; segment edges make up for the destination rows
      // outside [Rb, Re)); one arrive per group the rows fall in.
      auto release = [&] {
        __syncwarp();
        if (lane == 0) {
          const uint32_t first = first_row ? 1u : 0u, lastr = last_row ? 1u : 0u;
          const uint32_t c0 = 1 + 2 * first, c1 = 1 + first + lastr, c2 = 1 + 2 * lastr;
          const uint32_t g0 = i / B, g1 = (i + 1) / B, g2 = (i + 2) / B;
          if (g0 == g2) {
            mbar_arrive(empty + (g0 % kG) * 8, c0 + c1 + c2);
          } else {
            mbar_arrive(empty + (g0 % kG) * 8, c0 + (g1 == g0 ? c1 : 0u));
            mbar_arrive(empty + (g2 % kG) * 8, c2 + (g1 == g2 ? c1 : 0u));
          }
        }
      };
      if ((a.row0 + r) & 1)
        dest_row<NW, FORCE, RULE, 1>(sl[0], sl[1], sl[2], cx, lane, y0 + r, &stmap, &padmap, L.w0, r + 1,
                               L.pad, L.padx, L.pad_band, swaps, release);
      else
        dest_row<NW, FORCE, RULE, 0>(sl[0], sl[1], sl[2], cx, lane, y0 + r, &stmap, &padmap, L.w0, r + 1,
                               L.pad, L.padx, L.pad_band, swaps, release);
      }
  };
  rows(RA0, RA0 + nA, 0u, sbase + RG::kCtrOff);
  if (nB > 0) {
    // Extra CTA: on to band bA + 1 once every consumer is done with band bA
    // (the key table is rewritten); the producer streams on meanwhile.
    asm volatile("bar.sync 1, %0;" ::"r"(RG::kCons * 32) : "memory");
    make_keys(bA + 1, threadIdx.x, RG::kCons * 32);
    asm volatile("bar.sync 1, %0;" ::"r"(RG::kCons * 32) : "memory");
    set_band(bA + 1);
    rows(row_lo, row_lo + nB, offB, sbase + RG::kCtrOff + 4);
  }
  if (lane == 0) bulk_wait_all();  // the stores have landed before the kernel ends
  if (FORCE) {
    unsigned long long sw = swaps;
    for (int o = 16; o; o >>= 1) sw += __shfl_xor_sync(kFull, sw, o);
    if (lane == 0 && sw) atomicAdd(a.swaps, sw);
  }
}

// ---------------------------------------------------------------------------
// Row-pair ring kernel (default for the 2048-column bands). The same shared
// row ring as step_ring_kernel, but a consumer warp takes two destination
// rows at a time (rows r, r+1 from source rows r-1 .. r+2): the per-row
// costs of the ring protocol (slot waits and releases), of the chirality
// walk's setup (one balanced walk over both rows' sites) and of the output
// (one TMA store of a 2-row box) are paid once per pair. Registers: up to
// 128 per thread, 16 consumer warps (+ the producer).
// ---------------------------------------------------------------------------
#ifndef FHPG_PAIR_CONS
#define FHPG_PAIR_CONS 15
#endif
#ifndef FHPG_PAIR_RING
#define FHPG_PAIR_RING 64
#endif
#ifndef FHPG_PAIR_RING_F
#define FHPG_PAIR_RING_F 32
#endif
#ifndef FHPG_PAIR
#define FHPG_PAIR 0
#endif
template <int NW, bool FORCE>
struct PairGeo {
  using G = Geo<NW, FORCE>;
  static constexpr int kCons = FHPG_PAIR_CONS;
  static constexpr int kRing = FORCE ? FHPG_PAIR_RING_F : FHPG_PAIR_RING;
  static constexpr int kThreads = (kCons + 1) * 32;
  static constexpr int kKeys = (FORCE ? 2 : 1) * G::kBandCols * 8;
  static constexpr int kRingOff = (kKeys + 127) / 128 * 128;
  // Per consumer: the outputs of two rows [row][plane][band words] (the
  // 2-row TMA store box), then the two 2-row pad boxes [row][plane][4 words].
  // The walk's list (up to 2 x 32 NW entries) and result words (2 rows) live
  // in the output area while it is dead.
  static constexpr int kRowOut = G::kStage;  // 7 planes x band words x 4 B
  static constexpr int kPadL = 2 * kRowOut, kPadR = 2 * kRowOut + 256;
  static constexpr int kList = 0;
  static constexpr int kOut = 16 * 2 * 32 * NW;
  static constexpr int kStage = 2 * kRowOut + 512;
  static_assert(kOut + 2 * 4 * 32 * NW <= 2 * kRowOut, "walk scratch must fit the output area");
  static constexpr int kStageOff = kRingOff + kRing * G::kSlot;
  static constexpr int kBarOff = kStageOff + kCons * kStage;
  static constexpr int kTagOff = kBarOff + 2 * 8 * kRing;
  static constexpr int kCtrOff = kTagOff + 4 * kRing;  // dynamic pair counters (2 parts)
  static constexpr int kSmem = kCtrOff + 8;
  static_assert(kSmem <= 232448, "shared memory per CTA");
  static constexpr int kBox = FHPG_BOX_ROWS;
  static constexpr int kGroups = kRing / kBox;
  static_assert(kRing % kBox == 0, "row groups");
};

// The planes of destination row r (parity Q) pulled from the ring slots of
// rows r-1 (sm), r (sc), r+1 (sn) (backends.cpp:64-73, as in dest_row).
template <int NW, int Q>
__device__ __forceinline__ void pull_row(uint32_t sm, uint32_t sc, uint32_t sn,
                                         uint32_t (&a)[6][NW], uint32_t (&rr)[NW],
                                         uint32_t (&so)[NW]) {
  constexpr int P = Geo<NW, false>::kPlane;
  if (Q) rd_shr<NW>(sn + 0 * P, a[0]); else rd_al<NW>(sn + 0 * P, a[0]);
  if (Q) rd_al<NW>(sn + 1 * P, a[1]); else rd_shl<NW>(sn + 1 * P, a[1]);
  rd_shl<NW>(sc + 2 * P, a[2]);
  if (Q) rd_al<NW>(sm + 3 * P, a[3]); else rd_shl<NW>(sm + 3 * P, a[3]);
  if (Q) rd_shr<NW>(sm + 4 * P, a[4]); else rd_al<NW>(sm + 4 * P, a[4]);
  rd_shr<NW>(sc + 5 * P, a[5]);
  rd_al<NW>(sc + 6 * P, rr);
  rd_al<NW>(sc + 7 * P, so);
}

// The balanced walk of `walk` over the set bits of two rows' masks (m[0]:
// row r, m[1]: row r + 1). List entries carry the row in bit 31 of the
// sites-before field; fn(key address, row) returns the site's bit, ORed into
// the result words [row][band word] at osm.
template <int NW, int NR, typename Fn>
__device__ __forceinline__ int walk_rows(const uint32_t (&m)[2][NW], uint32_t lsm, uint32_t osm,
                                         uint32_t keys, int lane, const Fn& fn) {
  int cnt = 0, nz = 0;
#pragma unroll
  for (int q = 0; q < NR; ++q)
#pragma unroll
    for (int w = 0; w < NW; ++w) {
      cnt += __popc(m[q][w]);
      nz += m[q][w] != 0u;
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
    int q0 = excl >> 16, c = excl & 0xFFFF;
#pragma unroll
    for (int q = 0; q < NR; ++q)
#pragma unroll
      for (int w = 0; w < NW; ++w) {
        const uint32_t wi = static_cast<uint32_t>(lane * NW + w);
        const uint32_t ow = osm + (static_cast<uint32_t>(q) * 32u * NW + wi) * 4u;
        if (m[q][w]) {
          sts128(lsm + q0 * 16, m[q][w], keys + wi * 256u,
                 static_cast<uint32_t>(c) | (static_cast<uint32_t>(q) << 31), ow);
          ++q0;
          c += __popc(m[q][w]);
        }
        sts32(ow, 0u);
      }
  }
  __syncwarp();
  const int s = (lane * T) >> 5;
  const int e = ((lane + 1) * T) >> 5;
  const int icnt = incl & 0xFFFF;
  int o = 0;
#pragma unroll
  for (int step = 16; step; step >>= 1) {
    const int v = __shfl_sync(kFull, icnt, o + step - 1);
    if (v <= s) o += step;
  }
  const int o_excl = __shfl_sync(kFull, excl, o);
  if (s < e) {
    uint32_t qa = lsm + (o_excl >> 16) * 16u;
    uint4 en = lds128(qa);
#pragma unroll
    for (int w = 1; w < NR * NW; ++w) {
      if (s >= static_cast<int>(en.z & 0x7FFFFFFFu) + __popc(en.x)) {
        qa += 16u;
        en = lds128(qa);
      }
    }
    uint32_t mask = en.x, kw = en.y, ow = en.w, dy = en.z >> 31;
    for (int k = s - static_cast<int>(en.z & 0x7FFFFFFFu); k > 0; --k) mask &= mask - 1u;
    auto next = [&](uint32_t& ka, uint32_t& wa, uint32_t& v, uint32_t& row) {
      if (mask == 0u) {
        qa += 16u;
        const uint4 n = lds128(qa);
        mask = n.x;
        kw = n.y;
        ow = n.w;
        dy = n.z >> 31;
      }
      v = mask & (0u - mask);
      mask ^= v;
      ka = kw + top_bit(v) * 8u;
      wa = ow;
      row = dy;
    };
    int it = s;
    for (; it + 1 < e; it += 2) {
      uint32_t k0, w0, v0, r0, k1, w1, v1, r1;
      next(k0, w0, v0, r0);
      next(k1, w1, v1, r1);
      const uint32_t b0 = fn(k0, r0), b1 = fn(k1, r1);
      red_or(w0, b0 * v0);
      red_or(w1, b1 * v1);
    }
    if (it < e) {
      uint32_t k0, w0, v0, r0;
      next(k0, w0, v0, r0);
      red_or(w0, fn(k0, r0) * v0);
    }
  }
  __syncwarp();
  return T;
}

// Per-site result bits of the walks (functors with forced inlining: lambdas
// passed down here were kept out of line, their closures in local memory).
struct ChirBit {
  uint32_t y, four;
  __device__ __forceinline__ uint32_t operator()(uint32_t ka, uint32_t row) const {
    return chir_bit(lds64(ka) + (y + row), four);
  }
};
struct ForceBit {
  uint32_t y;
  uint64_t thr;
  __device__ __forceinline__ uint32_t operator()(uint32_t ka, uint32_t row) const {
    return (fin64(lds64(ka) + (y + row)) >> 32) < thr ? 1u : 0u;
  }
};

// Empty-barrier arrivals of a pair's source rows r-1 .. r+2 (ring index i
// of row r-1): one per (destination row, source row) use, plus the missing
// destination rows outside [Rb, Re) at the part's edges, 3 per source row.
struct PairRelease {
  uint32_t empty, i;
  int lane;
  bool two, first, last;
  template <uint32_t B, uint32_t kG>
  __device__ __forceinline__ void arrive() const {
    __syncwarp();
    if (lane == 0) {
      uint32_t c0 = 1u, c1 = two ? 2u : 1u, c2 = two ? 2u : 1u, c3 = two ? 1u : 0u;
      if (first) {
        c0 += 2u;
        c1 += 1u;
      }
      if (last) {  // source rows Re (2 missing users) and Re - 1 (1)
        if (two) {
          c3 += 2u;
          c2 += 1u;
        } else {
          c2 += 2u;
          c1 += 1u;
        }
      }
      const uint32_t g0 = i / B;
      uint32_t s0 = c0, s1 = 0;
      ((i + 1) / B == g0 ? s0 : s1) += c1;
      ((i + 2) / B == g0 ? s0 : s1) += c2;
      ((i + 3) / B == g0 ? s0 : s1) += c3;
      mbar_arrive(empty + (g0 % kG) * 8, s0);
      if (s1) mbar_arrive(empty + ((g0 + 1) % kG) * 8, s1);
    }
  }
};

// Destination rows r (parity Q) and, when NR == 2, r + 1, from the slots of
// source rows r-1 .. r+NR (sl[0..NR+1], this lane's word address in plane
// 0). `released()` is called once the source rows are in registers.
template <int NW, bool FORCE, int RULE, int Q, int NR>
__device__ __forceinline__ void dest_rows(const uint32_t (&sl)[4], uint32_t stage,
                                          const Ctx<NW, FORCE>& cx, int lane, uint32_t y,
                                          const CUtensorMap* stmap, const CUtensorMap* padmap,
                                          int w0, int trow, int pad, int padx, bool pad_band,
                                          unsigned& swaps, const PairRelease& rel) {
  using PG = PairGeo<NW, FORCE>;
  uint32_t a[2][6][NW], rr[2][NW], so[2][NW];
  pull_row<NW, Q>(sl[0], sl[1], sl[2], a[0], rr[0], so[0]);
  if constexpr (NR == 2) pull_row<NW, Q ^ 1>(sl[1], sl[2], sl[3], a[1], rr[1], so[1]);
  rel.arrive<PG::kBox, PG::kGroups>();
  typename PlaneRule<RULE>::Class K[2][NW];
  uint32_t dep[2][NW];
#pragma unroll
  for (int q = 0; q < NR; ++q)
#pragma unroll
    for (int w = 0; w < NW; ++w) {
      const uint32_t aw[6] = {a[q][0][w], a[q][1][w], a[q][2][w], a[q][3][w], a[q][4][w], a[q][5][w]};
      K[q][w] = PlaneRule<RULE>::classify(aw, rr[q][w], so[q][w]);
      dep[q][w] = K[q][w].dep;
    }
  // The previous pair's TMA stores must have read the output area (which
  // also holds the walk scratch) before it is rewritten.
  if (lane == 0) bulk_wait_read();
  __syncwarp();
  const uint32_t lsm = stage + PG::kList, osm = stage + PG::kOut;
  // Chirality: bit 0 of node_random(seed, Chirality, step, x + 1, y)
  // = fin64(key[x] + y) (rng.hpp:25-33, step.cpp:73-76).
  const int T = walk_rows<NW, NR>(dep, lsm, osm, cx.kc, lane, ChirBit{y, cx.four});
  uint32_t o[2][NW][7];
#pragma unroll
  for (int q = 0; q < NR; ++q) {
    const uint32_t mine = osm + (static_cast<uint32_t>(q) * 32u * NW + lane * NW) * 4u;
#pragma unroll
    for (int w = 0; w < NW; ++w) {
      const uint32_t c = T ? lds32(mine + w * 4) : 0u;
      uint32_t oo[6], orr;
      const uint32_t aw[6] = {a[q][0][w], a[q][1][w], a[q][2][w], a[q][3][w], a[q][4][w], a[q][5][w]};
      PlaneRule<RULE>::apply(K[q][w], c, rr[q][w], aw, oo, orr, so[q][w]);
#pragma unroll
      for (int p = 0; p < 6; ++p) o[q][w][p] = oo[p];
      o[q][w][6] = orr;
    }
  }
  if constexpr (FORCE) {
    // step.cpp:79-88: fluid, W (bit 5) set, E (bit 2) clear after collision.
    uint32_t f[2][NW];
#pragma unroll
    for (int q = 0; q < NR; ++q)
#pragma unroll
      for (int w = 0; w < NW; ++w) f[q][w] = ~so[q][w] & o[q][w][5] & ~o[q][w][2];
    const int TF = walk_rows<NW, NR>(f, lsm, osm, cx.kf, lane, ForceBit{y, cx.thr});
    if (TF) {
#pragma unroll
      for (int q = 0; q < NR; ++q) {
        const uint32_t mine = osm + (static_cast<uint32_t>(q) * 32u * NW + lane * NW) * 4u;
#pragma unroll
        for (int w = 0; w < NW; ++w) {
          const uint32_t acc = lds32(mine + w * 4);
          o[q][w][5] ^= acc;
          o[q][w][2] ^= acc;
          swaps += __popc(acc);
        }
      }
    }
  }
#pragma unroll
  for (int q = 0; q < NR; ++q)
#pragma unroll
    for (int p = 0; p < 7; ++p) {
      uint32_t v[NW];
#pragma unroll
      for (int w = 0; w < NW; ++w) v[w] = o[q][w][p];
      stsv<NW>(stage + q * PG::kRowOut + p * (4 * 32 * NW) + lane * NW * 4, v);
      // periodic wrap copies: lanes holding words 0..3 / WW-4..WW-1
      if (pad_band && pad >= 0) stsv<NW>(stage + pad + q * 112 + p * 16, v);
    }
  fence_async_smem();
  __syncwarp();
  if (lane == 0) {
    tma_store(stmap, w0 + 4, trow, stage);
    if (pad_band) {
      if (padx & 1) tma_store(padmap, 0, trow, stage + PG::kPadL);
      if (padx & 2) tma_store(padmap, (padx >> 2) + 4, trow, stage + PG::kPadR);
    }
    bulk_commit();
  }
}

template <int NW, bool FORCE, int RULE>
__global__ void __launch_bounds__(PairGeo<NW, FORCE>::kThreads, 1)
    step_pair_kernel(StepArgs a, const __grid_constant__ CUtensorMap ldmap,
                     const __grid_constant__ CUtensorMap stmap1,
                     const __grid_constant__ CUtensorMap padmap1,
                     const __grid_constant__ CUtensorMap stmap2,
                     const __grid_constant__ CUtensorMap padmap2) {
  using G = Geo<NW, FORCE>;
  using PG = PairGeo<NW, FORCE>;
  extern __shared__ __align__(128) uint8_t smem[];
  const uint32_t sbase = smem_u32(smem);
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  // Work split as in step_ring_kernel: part A = band bA, rows [RA0, RA0+nA);
  // extra CTAs also do part B = band bA + 1 over the same rows.
  const int nmain = a.nbands * (a.segs1 + a.segs2);
  int bA, RA0, nA, nB = 0;
  int row_lo;
  if (static_cast<int>(blockIdx.x) < nmain) {
    bA = blockIdx.x % a.nbands;
    const bool second = static_cast<int>(blockIdx.x / a.nbands) >= a.segs1;
    const int seg_group = blockIdx.x / a.nbands - (second ? a.segs1 : 0);
    row_lo = second ? a.row_lo2 : a.row_lo;
    const int row_hi = second ? a.row_hi2 : a.row_hi - a.extra_rows;
    RA0 = row_lo + seg_group * a.seg_rows;
    nA = max(0, min(row_hi, RA0 + a.seg_rows) - RA0);
  } else {
    bA = 2 * (blockIdx.x - nmain);
    row_lo = a.row_hi - a.extra_rows;
    RA0 = row_lo;
    nA = a.extra_rows;
    nB = bA + 1 < a.nbands ? a.extra_rows : 0;
  }
  constexpr uint32_t B = PG::kBox;
  const uint32_t offB = (static_cast<uint32_t>(nA) + 2 + B - 1) / B * B;
  const uint32_t kc_base = sbase;
  const uint32_t kf_base = sbase + G::kBandCols * 8;
  const uint32_t ring = sbase + PG::kRingOff;
  const uint32_t full = sbase + PG::kBarOff;
  const uint32_t empty = full + 8 * PG::kRing;
  const uint32_t tags = sbase + PG::kTagOff;
  if (threadIdx.x == 0) {
    for (int k = 0; k < PG::kRing; ++k) {
      mbar_init(full + k * 8, 1);
      mbar_init(empty + k * 8, 3 * PG::kBox);
      sts32(tags + k * 4, 0xFFFFFFFFu);
    }
    sts32(sbase + PG::kCtrOff, 0u);
    sts32(sbase + PG::kCtrOff + 4, 0u);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // (The lambdas below capture plain locals, not the kernel parameter `a`:
  // capturing it by reference puts the whole StepArgs in local memory.)
  const uint64_t kc_cur = a.kc_cur, kf_cur = a.kf_cur;
  const int row0 = static_cast<int>(a.row0);  // global rows < 2^31
  auto make_keys = [&](int b, int t0, int nt) {
    for (int c = t0; c < G::kBandCols; c += nt) {
      const uint64_t x = static_cast<uint64_t>(b * G::kBandCols + c) + 1;
      sts64(kc_base + c * 8, column_key(kc_cur, x));
      if (FORCE) sts64(kf_base + c * 8, column_key(kf_cur, x));
    }
  };
  make_keys(bA, threadIdx.x, blockDim.x);
#if FHPG_PDL
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
#endif
  if (a.zc_next) {
    const int n = gridDim.x * blockDim.x;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < a.W; i += n) {
      a.zc_next[i] = column_key(a.kc_next, static_cast<uint64_t>(i) + 1);
      if (a.zf_next) a.zf_next[i] = column_key(a.kf_next, static_cast<uint64_t>(i) + 1);
    }
  }
  __syncthreads();
  if (nA + nB <= 0) return;

  if (warp == PG::kCons) {  // producer (tensor row = local row + 1)
    if (lane == 0) {
      constexpr uint32_t kG = PG::kGroups;
      const uint32_t gA = offB / B;
      const uint32_t ngroups = gA + (nB > 0 ? (static_cast<uint32_t>(nB) + 2 + B - 1) / B : 0u);
      for (uint32_t P = 0; P < ngroups; ++P) {
        const uint32_t k = P % kG;
        if (P >= kG) mbar_wait(empty + k * 8, (P / kG - 1) & 1u);
        {
          uint32_t prev;
          asm volatile("atom.shared.exch.b32 %0, [%1], %2;" : "=r"(prev) : "r"(tags + k * 4), "r"(P) : "memory");
        }
        const bool inA = P < gA;
        const int word = (inA ? bA : bA + 1) * G::kBandWords;
        const int trow = inA ? RA0 + static_cast<int>(B * P) : row_lo + static_cast<int>(B * P - offB);
        mbar_expect_tx(full + k * 8, B * G::kRowBytes);
        tma_row(ring + B * k * G::kSlot, &ldmap, word, trow, full + k * 8);
        if (nB > 0 && P + 1 == gA && offB > static_cast<uint32_t>(nA) + 2)
          mbar_arrive(empty + k * 8, 3 * (offB - static_cast<uint32_t>(nA) - 2));
      }
    }
    return;
  }

  Lanes L;
  L.lane = lane;
  L.WW = a.W >> 5;
  L.PW = L.WW + 8;
  auto set_band = [&](int b) {
    L.w0 = b * G::kBandWords;
    const int wl = L.w0 + L.lane * NW;
    L.pad = wl < 4 ? PG::kPadR + wl * 4 : (wl >= L.WW - 4 ? PG::kPadL + (wl - (L.WW - 4)) * 4 : -1);
    L.padx = (L.w0 + G::kBandWords == L.WW ? 1 : 0) | (L.w0 == 0 ? 2 : 0) | (L.WW << 2);
    L.pad_band = L.w0 == 0 || L.w0 + G::kBandWords == L.WW;
  };
  set_band(bA);
  const uint32_t stage = sbase + PG::kStageOff + warp * PG::kStage;
  Ctx<NW, FORCE> cx;
  cx.kc = kc_base;
  cx.kf = kf_base;
  cx.lsm = stage + PG::kList;
  cx.osm = stage + PG::kOut;
  cx.stage = stage;
  cx.thr = a.thr;
  cx.four = a.k4;
  unsigned swaps = 0;
  const uint32_t lane_off = 16u + lane * NW * 4u;
  const uint32_t y0 = static_cast<uint32_t>(a.row0);
  // Destination rows [Rb, Re) in pairs, pair j to consumer j mod kCons;
  // source row r - 1 of the pair at r sits at ring index ibase + r - Rb.
  auto rows = [&](const int Rb, const int Re, const uint32_t ibase, const uint32_t ctr)
                  __attribute__((always_inline)) {
#if FHPG_DYN_ROWS
    for (;;) {
      int r = 0;
      if (lane == 0) asm volatile("atom.shared.add.u32 %0, [%1], 2;" : "=r"(r) : "r"(ctr) : "memory");
      r = Rb + __shfl_sync(kFull, r, 0);
      if (r >= Re) break;
#else
    (void)ctr;
    for (int r = Rb + 2 * warp; r < Re; r += 2 * PG::kCons) {
#endif
      const bool two = r + 1 < Re;
      const uint32_t i = ibase + static_cast<uint32_t>(r - Rb);
      constexpr uint32_t kG = PG::kGroups;
      const uint32_t nsrc = two ? 4u : 3u;
      uint32_t sl[4];
#pragma unroll
      for (uint32_t d = 0; d < 4; ++d) {
        if (d < nsrc) {
          const uint32_t P = (i + d) / B;
          if (d == 0 || ((i + d) % B) == 0) {
            const uint32_t kp = P % kG;
            for (;;) {
              uint32_t tag;
              asm volatile("ld.relaxed.cta.shared.u32 %0, [%1];" : "=r"(tag) : "r"(tags + kp * 4) : "memory");
              if (tag == P) break;
              __nanosleep(FHPG_TAG_SLEEP);
            }
            mbar_wait(full + kp * 8, (P / kG) & 1u);
          }
          sl[d] = ring + ((i + d) % PG::kRing) * G::kSlot + lane_off;
        } else {
          sl[d] = sl[d - 1];
        }
      }
      const PairRelease rel{empty, i, lane, two, r == Rb, r + (two ? 1 : 0) == Re - 1};
      const bool q = (row0 + r) & 1;
      if (two) {
        if (q)
          dest_rows<NW, FORCE, RULE, 1, 2>(sl, stage, cx, lane, y0 + r, &stmap2, &padmap2, L.w0, r + 1,
                                           L.pad, L.padx, L.pad_band, swaps, rel);
        else
          dest_rows<NW, FORCE, RULE, 0, 2>(sl, stage, cx, lane, y0 + r, &stmap2, &padmap2, L.w0, r + 1,
                                           L.pad, L.padx, L.pad_band, swaps, rel);
      } else {
        if (q)
          dest_rows<NW, FORCE, RULE, 1, 1>(sl, stage, cx, lane, y0 + r, &stmap1, &padmap1, L.w0, r + 1,
                                           L.pad, L.padx, L.pad_band, swaps, rel);
        else
          dest_rows<NW, FORCE, RULE, 0, 1>(sl, stage, cx, lane, y0 + r, &stmap1, &padmap1, L.w0, r + 1,
                                           L.pad, L.padx, L.pad_band, swaps, rel);
      }
    }
  };
  rows(RA0, RA0 + nA, 0u, sbase + PG::kCtrOff);
  if (nB > 0) {
    asm volatile("bar.sync 1, %0;" ::"r"(PG::kCons * 32) : "memory");
    make_keys(bA + 1, threadIdx.x, PG::kCons * 32);
    asm volatile("bar.sync 1, %0;" ::"r"(PG::kCons * 32) : "memory");
    set_band(bA + 1);
    rows(row_lo, row_lo + nB, offB, sbase + PG::kCtrOff + 4);
  }
  if (lane == 0) bulk_wait_all();
  if (FORCE) {
    unsigned long long sw = swaps;
    for (int o = 16; o; o >>= 1) sw += __shfl_xor_sync(kFull, sw, o);
    if (lane == 0 && sw) atomicAdd(a.swaps, sw);
  }
}

// Grid of the ring / pair kernels: nbands x segment groups of the row range
// (plus the second range's segments), with the SMs left over by nbands x
// segment groups (148 - 8 x 18 = 4 at W = 16384) taking the last rows of two
// bands each, so that every SM has the same work: x rows per band go to them,
// x(2S + 1) = rows - S b with b rows of equivalent cost for their mid-kernel
// band switch.
template <int NW>
int ring_grid(StepArgs& a, int num_sms) {
  using G = Geo<NW, false>;
  const int rows = a.row_hi - a.row_lo;
  a.k4 = 4u;
  a.nbands = a.W / G::kBandCols;
  int seg_groups = num_sms / a.nbands;
  if (seg_groups < 1) seg_groups = 1;
  int seg = (rows + seg_groups - 1) / seg_groups;
  if (seg < 1) seg = 1;
  a.seg_rows = seg;
  seg_groups = (rows + seg - 1) / seg;
  a.segs1 = seg_groups;
  const int rows2 = a.row_hi2 > a.row_lo2 ? a.row_hi2 - a.row_lo2 : 0;
  a.segs2 = (rows2 + seg - 1) / seg;
  a.extra_rows = 0;
  int grid = a.nbands * (seg_groups + a.segs2);
  const int spare = num_sms - a.nbands * (num_sms / a.nbands);
  if (FHPG_EXTRA_CTAS && rows2 == 0 && a.nbands % 2 == 0 && 2 * spare >= a.nbands &&
      num_sms / a.nbands >= 2) {
    const int S = num_sms / a.nbands;
    const int x = (rows - FHPG_EXTRA_BUBBLE_ROWS * S) / (2 * S + 1);
    if (x >= 16) {
      a.extra_rows = x;
      a.seg_rows = (rows - x + S - 1) / S;
      a.segs1 = (rows - x + a.seg_rows - 1) / a.seg_rows;
      a.segs2 = 0;
      grid = a.nbands * a.segs1 + a.nbands / 2;
    }
  }
  return grid;
}

// Launch with programmatic dependent launch: the next step's grid is
// launched while this one runs and its CTAs take SMs as they free up
// (griddepcontrol.wait in the kernel orders every read of the previous
// step's output).
template <typename K, typename... Args>
void launch_pdl(K kernel, int grid, int threads, int smem, cudaStream_t st, Args... args) {
#if FHPG_PDL
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kernel, args...);
#else
  kernel<<<grid, threads, smem, st>>>(args...);
#endif
}

// maps: [0] row loads, [1] band stores, [2] pad stores, [3] 4-row loads,
// [4] 2-row band stores, [5] 2-row pad stores (make_planes_map kinds).
template <int NW, bool FORCE, int RULE>
void launch_ring(StepArgs a, const CUtensorMap* src, const CUtensorMap* dst, int num_sms,
                 cudaStream_t st) {
  using RG = RingGeo<NW, FORCE>;
  const int grid = ring_grid<NW>(a, num_sms);
  ensure_smem_optin(reinterpret_cast<const void*>(step_ring_kernel<NW, FORCE, RULE>), RG::kSmem);
  launch_pdl(step_ring_kernel<NW, FORCE, RULE>, grid, RG::kThreads, RG::kSmem, st, a, src[0],
             dst[1], dst[2], src[3]);
}

template <int NW, bool FORCE, int RULE>
void launch_pair(StepArgs a, const CUtensorMap* src, const CUtensorMap* dst, int num_sms,
                 cudaStream_t st) {
  using PG = PairGeo<NW, FORCE>;
  const int grid = ring_grid<NW>(a, num_sms);
  ensure_smem_optin(reinterpret_cast<const void*>(step_pair_kernel<NW, FORCE, RULE>), PG::kSmem);
  launch_pdl(step_pair_kernel<NW, FORCE, RULE>, grid, PG::kThreads, PG::kSmem, st, a, src[3],
             dst[1], dst[2], dst[4], dst[5]);
}

template <int NW, bool FORCE>
int smem_bytes(int bpc) {
  using G = Geo<NW, FORCE>;
  return (FORCE ? 2 : 1) * bpc * G::kBandCols * 8 + kPWarps<NW> * G::kWarp;
}

template <int NW, bool FORCE, int RULE>
void launch_nw(StepArgs a, const CUtensorMap* src, const CUtensorMap* dst, int num_sms,
               cudaStream_t st) {
  using G = Geo<NW, FORCE>;
  const int rows = a.row_hi - a.row_lo;
  a.k4 = 4u;
  a.nbands = a.W / G::kBandCols;
  // Bands per CTA: as many as the shared-memory budget allows (the column
  // keys of every band a CTA covers are staged).
  constexpr int kWarps = kPWarps<NW>;
  int bpc = a.nbands < kWarps ? a.nbands : kWarps;
  while (bpc > 1 && smem_bytes<NW, FORCE>(bpc) > 226 * 1024) bpc >>= 1;
  while (kWarps % bpc) --bpc;
  a.bpc = bpc;
  a.spc = kWarps / bpc;
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
  // (The kernel also holds 1 KB of static shared memory for the bulk-copy
  // machinery, so the dynamic opt-in is set to exactly what is used.)
  ensure_smem_optin(reinterpret_cast<const void*>(step_planes_kernel<NW, FORCE, RULE>), smem);
#if FHPG_PDL
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kWarps * 32);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, step_planes_kernel<NW, FORCE, RULE>, a, src[0], dst[1], dst[2]);
#else
  step_planes_kernel<NW, FORCE, RULE><<<grid, kWarps * 32, smem, st>>>(a, src[0], dst[1], dst[2]);
#endif
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
    const int PW = WW + 8;  // padded plane row
    const int pad = i < 4 ? WW : (i >= WW - 4 ? -WW : 0);
    uint32_t* d = reinterpret_cast<uint32_t*>(dst + r * static_cast<long long>(pitch)) + 4 + i;
    uint32_t* o = reinterpret_cast<uint32_t*>(dst_obst + r * static_cast<long long>(pitch)) + 4 + i;
#pragma unroll
    for (int p = 0; p < 8; ++p) {
      uint32_t w = 0;
#pragma unroll
      for (int k = 0; k < 8; ++k)  // bytes 4k..4k+3: bit p of each -> 4 bits
        w |= ((((v[k] >> p) & 0x01010101u) * 0x01020408u) >> 24 & 0xFu) << (4 * k);
      d[p * PW] = w;
      if (pad) d[p * PW + pad] = w;
      if (p == 7) {
        o[7 * PW] = w;
        if (pad) o[7 * PW + pad] = w;
      }
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
    const uint32_t* s =
        reinterpret_cast<const uint32_t*>(src + r * static_cast<long long>(pitch)) + 4 + i;
    uint32_t p[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) p[q] = s[q * (WW + 8)];
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
  if (bands1 % 4 == 0) return FHPG_PLANES_NW4;
  if (bands1 % 2 == 0) return 2;
  return 1;
}

bool planes_ok(int W) { return planes_words_per_lane(W) != 0; }

size_t planes_row_bytes(int W) { return static_cast<size_t>(W) + 256; }

bool make_planes_map(void* tmap, uint8_t* buffer, int W, size_t pitch, int rows, int kind) {
  static PFN_cuTensorMapEncodeTiled encode = nullptr;
  if (!encode) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) !=
            cudaSuccess || q != cudaDriverEntryPointSuccess || !fn)
      return false;
    encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled>(fn);
  }
  // Tensor {padded words, planes, rows}. Boxes: kind 0 (load) one band of
  // 32 NW words + 4 on each side, all 8 planes; kind 1 (store) the band's
  // words, planes 0-6; kind 2 (pad store) 4 words, planes 0-6; kind 3 (load)
  // as kind 0 for FHPG_BOX_ROWS consecutive rows; kinds 4 / 5 as 1 / 2 for
  // two consecutive rows.
  const int nw = planes_words_per_lane(W);
  const cuuint64_t dims[3] = {static_cast<cuuint64_t>(W / 32 + 8), 8,
                              static_cast<cuuint64_t>(rows)};
  const cuuint64_t strides[2] = {static_cast<cuuint64_t>((W / 32 + 8) * 4),
                                 static_cast<cuuint64_t>(pitch)};
  const bool load = kind == 0 || kind == 3;
  const bool band = kind == 1 || kind == 4;
  const cuuint32_t box[3] = {
      static_cast<cuuint32_t>(load ? 32 * nw + 8 : band ? 32 * nw : 4), load ? 8u : 7u,
      kind == 3 ? static_cast<cuuint32_t>(FHPG_BOX_ROWS) : (kind >= 4 ? 2u : 1u)};
  const cuuint32_t estr[3] = {1, 1, 1};
  const CUresult r = encode(static_cast<CUtensorMap*>(tmap), CU_TENSOR_MAP_DATA_TYPE_UINT32, 3,
                            buffer, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

int launch_step_planes(const StepArgs& a, const void* src_maps, const void* dst_maps,
                       int num_sms, cudaStream_t st) {
  const int nw = planes_words_per_lane(a.W);
  const bool force = a.thr != 0;
  const CUtensorMap* src = static_cast<const CUtensorMap*>(src_maps);
  const CUtensorMap* dst = static_cast<const CUtensorMap*>(dst_maps);
  // a.rule: 2 = FHP-III, 1 = FHP-I, 0 = DEFAULT (the circuit the kernels instantiate)
  auto ring = [&](auto rule) {
    constexpr int R = decltype(rule)::value;
#if FHPG_PAIR
    if (force) launch_pair<2, true, R>(a, src, dst, num_sms, st);
    else launch_pair<2, false, R>(a, src, dst, num_sms, st);
#else
    if (force) launch_ring<2, true, R>(a, src, dst, num_sms, st);
    else launch_ring<2, false, R>(a, src, dst, num_sms, st);
#endif
  };
  auto nwk = [&](auto rule) {
    constexpr int R = decltype(rule)::value;
    if (nw == 4) {
      if (force) launch_nw<4, true, R>(a, src, dst, num_sms, st);
      else launch_nw<4, false, R>(a, src, dst, num_sms, st);
    } else if (nw == 2) {
      if (force) launch_nw<2, true, R>(a, src, dst, num_sms, st);
      else launch_nw<2, false, R>(a, src, dst, num_sms, st);
    } else {
      if (force) launch_nw<1, true, R>(a, src, dst, num_sms, st);
      else launch_nw<1, false, R>(a, src, dst, num_sms, st);
    }
  };
#if FHPG_PLANES_RING
  if (nw == 2) {
    if (a.rule == 0) ring(std::integral_constant<int, 0>{});
    else if (a.rule == 1) ring(std::integral_constant<int, 1>{});
    else ring(std::integral_constant<int, 2>{});
    return 1;
  }
#endif
  if (a.row_hi2 > a.row_lo2) {  // per-warp-ring kernels take one range per launch
    StepArgs a1 = a, a2 = a;
    a1.row_lo2 = a1.row_hi2 = a2.row_lo2 = a2.row_hi2 = 0;
    a2.row_lo = a.row_lo2;
    a2.row_hi = a.row_hi2;
    return launch_step_planes(a1, src_maps, dst_maps, num_sms, st) +
           launch_step_planes(a2, src_maps, dst_maps, num_sms, st);
  }
  if (a.rule == 0) nwk(std::integral_constant<int, 0>{});
  else if (a.rule == 1) nwk(std::integral_constant<int, 1>{});
  else nwk(std::integral_constant<int, 2>{});
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
