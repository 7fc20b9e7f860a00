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
// Layout (fhpg_kernels.cuh). A lattice row holds 8 bit planes (0-5 movers
// NW..W, 6 rest, 7 obstacle); bit j of word i of a plane = column 32 i + j.
// A plane row is 32 lead words, the W/32 data words and 32 trail words (the
// data starts on a 128-byte line). The obstacle plane is static: the pack
// kernel writes it into both ping-pong buffers and the step never does, so a
// step moves the algorithmic 15 bits per site (8 planes read, 7 written).
//
// Kernels. step_ring_kernel (W % 2048 == 0): one CTA per SM = a band of 2048
// columns x a segment of rows; a producer warp streams the segment's source
// rows into a shared ring with 4-row TMA boxes, 31 consumer warps take
// destination rows round-robin (lane l: words 2l, 2l+1 of every plane),
// evaluate the circuit, draw the chirality / forcing bits of the sites that
// need them (walk_own over folded column keys) and store the 7 output planes
// with one TMA store per row. step_planes_kernel (W = 1024 x odd): per-warp
// rings, the same row code. See DESIGN.md for the measured design choices.

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
#if FHPG_TIMELINE
constexpr unsigned long long kTimelineMax = 1 << 16;
__device__ unsigned long long g_timeline[kTimelineMax * 4];
__device__ unsigned long long g_timeline_n;
#endif
namespace {

#include "fhpg_planes_dev.cuh"  // shared device helpers (in this anonymous namespace)
// padx (PADS: the per-warp kernel, which keeps the periodic wrap in the
// plane rows' lead / trail sectors): bit 0 = the band is the last one (its
// last kPlaneWrap words are the left wrap sector), bit 1 = the first one (its
// first words are the right wrap sector), padx >> 2 = W / 32.
// E (the ring kernel, which writes no wrap sectors): the edge reads of
// rd_shl_e / rd_shr_e; wm, wc, wn: side-buffer rows of source rows r-1, r,
// r+1 ([8 planes][4 words], E = 1: data words W/32-4 .., E = 2: words 0 ..).
// FOLD: every row of the call lies inside the column keys' span (the ring
// kernel re-keys at span boundaries); otherwise rows past it hash from the
// step keys.
template <int NW, bool FORCE, int RULE, int Q, int E, bool PADS, bool FOLD, typename Rel>
__device__ __forceinline__ void dest_row(uint32_t sm, uint32_t sc, uint32_t sn, uint32_t wm,
                                         uint32_t wc, uint32_t wn, const Ctx<NW, FORCE>& cx,
                                         int lane, uint32_t y, const CUtensorMap* stmap,
                                         const CUtensorMap* padmap, int w0, int trow, int padx,
                                         unsigned& swaps, Rel&& released) {
  using G = Geo<NW, FORCE>;
  constexpr int P = G::kPlane;
  constexpr uint32_t kWo = E == 1 ? 12u : 0u;  // the wrap word inside a side-buffer plane
  uint32_t a0[NW], a1[NW], a2[NW], a3[NW], a4[NW], a5[NW], rr[NW], so[NW];
  // Pull sources (backends.cpp:64-73): k0 (x+q, r+1), k1 (x+q-1, r+1),
  // k2 (x-1, r), k3 (x+q-1, r-1), k4 (x+q, r-1), k5 (x+1, r).
  if (Q) rd_shr_e<NW, E>(sn + 0 * P, wn + 0 * 16 + kWo, lane, a0); else rd_al<NW>(sn + 0 * P, a0);
  if (Q) rd_al<NW>(sn + 1 * P, a1); else rd_shl_e<NW, E>(sn + 1 * P, wn + 1 * 16 + kWo, lane, a1);
  rd_shl_e<NW, E>(sc + 2 * P, wc + 2 * 16 + kWo, lane, a2);
  if (Q) rd_al<NW>(sm + 3 * P, a3); else rd_shl_e<NW, E>(sm + 3 * P, wm + 3 * 16 + kWo, lane, a3);
  if (Q) rd_shr_e<NW, E>(sm + 4 * P, wm + 4 * 16 + kWo, lane, a4); else rd_al<NW>(sm + 4 * P, a4);
  rd_shr_e<NW, E>(sc + 5 * P, wc + 5 * 16 + kWo, lane, a5);
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
  (void)swaps; (void)y; (void)padx; (void)padmap; (void)stmap;
  return;
#endif
  fence_async_smem();
  __syncwarp();
  if (lane == 0 && FHPG_STREAM_ONLY != 2) {  // 2: loads only
    tma_store(stmap, w0 + kPlaneLead, trow, cx.stage);
    bulk_commit();
  }
  (void)swaps; (void)y; (void)padx; (void)padmap;
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
  // Chirality: bit 0 of node_random(seed, Chirality, step, x + 1, y)
  // = fin64(key[x] + y) (rng.hpp:25-33, step.cpp:73-76), drawn only for the
  // dep sites, each lane walking its own (walk_own).
  uint32_t o[NW][7];
  // Column keys folded at the band's key base row (fhpg_common.cuh ColKey);
  // rows past their span (a key's low word would cross a 2^30 block) hash
  // from the step keys (rare: warp-uniform branch).
  const uint32_t dy = y - cx.ybase;
  const bool folded = FOLD || dy < cx.span;
  auto chir_fast = [&](uint32_t col) -> uint32_t {
    const uint4 k = lds128(cx.kc + col * 16u);
    return chir_mask_pre(k.x + dy, k.y, k.z);
  };
  auto chir_slow = [&](uint32_t col) -> uint32_t {
    return chir_mask(column_key(cx.kcur, cx.x1 + col) + y, cx.four);
  };
  uint32_t cw[NW];
  if (folded) walk_own<NW>(dep, lane, cw, chir_fast);
  else walk_own<NW>(dep, lane, cw, chir_slow);
#pragma unroll
  for (int w = 0; w < NW; ++w) {
    uint32_t oo[6], orr;
    const uint32_t a[6] = {a0[w], a1[w], a2[w], a3[w], a4[w], a5[w]};
    PlaneRule<RULE>::apply(K[w], cw[w], rr[w], a, oo, orr, so[w]);
#pragma unroll
    for (int p = 0; p < 6; ++p) o[w][p] = oo[p];
    o[w][6] = orr;
  }
  if constexpr (FORCE) {
    // step.cpp:79-88: fluid, W (bit 5) set, E (bit 2) clear after collision.
    uint32_t f[NW];
#pragma unroll
    for (int w = 0; w < NW; ++w) f[w] = ~so[w] & o[w][5] & ~o[w][2];
    auto force_fast = [&](uint32_t col) -> uint32_t {
      const uint4 k = lds128(cx.kf + col * 16u);
      const uint32_t h = fin64_hi_pre(k.x + dy, k.y, k.z);
      return static_cast<uint64_t>(h) < cx.thr ? ~0u : 0u;
    };
    auto force_slow = [&](uint32_t col) -> uint32_t {
      const uint32_t h = static_cast<uint32_t>(fin64(column_key(cx.kfcur, cx.x1 + col) + y) >> 32);
      return static_cast<uint64_t>(h) < cx.thr ? ~0u : 0u;
    };
    uint32_t fw[NW];
    if (!folded) {
      walk_own<NW>(f, lane, fw, force_slow);
    } else if (cx.thr <= (1ull << 31)) {  // p <= 1/2: compare z2's high word
      const uint32_t thr = static_cast<uint32_t>(cx.thr);
      walk_own_lt<NW>(f, lane, fw, thr, [&](uint32_t col) -> uint32_t {
        const uint4 k = lds128(cx.kf + col * 16u);
        return fin64_z2hi_pre(k.x + dy, k.y, k.z);
      });
    } else {
      walk_own<NW>(f, lane, fw, force_fast);
    }
#pragma unroll
    for (int w = 0; w < NW; ++w) {
      o[w][5] ^= fw[w];
      o[w][2] ^= fw[w];
      swaps += __popc(fw[w]);
    }
  }
  // The previous row's TMA store must have read the staging area before it
  // is rewritten.
  if (lane == 0) bulk_wait_read();
  __syncwarp();
#pragma unroll
  for (int p = 0; p < 7; ++p) {
    uint32_t v[NW];
#pragma unroll
    for (int w = 0; w < NW; ++w) v[w] = o[w][p];
    stsv<NW>(cx.stage + p * (4 * 32 * NW) + lane * NW * 4, v);
    // The edge bands' periodic-wrap sectors (one staging box of kPlaneWrap
    // words per plane): the first band's first words (right wrap), else the
    // last band's last words (left wrap).
    if (PADS && (padx & 3)) {
      const int wl = lane * NW;
      if ((padx & 2) ? wl < kPlaneWrap : wl >= 32 * NW - kPlaneWrap)
        stsv<NW>(cx.stage + G::kPad + p * (4 * kPlaneWrap) + (wl & (kPlaneWrap - 1)) * 4, v);
    }
  }
  fence_async_smem();
  __syncwarp();
  if (lane == 0) {
#if FHPG_STREAM_ONLY != 6  // 6: no stores (timing experiment)
    tma_store(stmap, w0 + kPlaneLead, trow, cx.stage);
    if (PADS && (padx & 3))
      tma_store(padmap, (padx & 2) ? kPlaneLead + (padx >> 2) : kPlaneLead - kPlaneWrap, trow,
                cx.stage + G::kPad);
#endif
    bulk_commit();
  }
  if (PADS && (padx & 3) == 3) {  // a single band (W = 32 * 32 NW): its left wrap goes second
    if (lane == 0) bulk_wait_read();
    __syncwarp();
    const int wl = lane * NW;
    if (wl >= 32 * NW - kPlaneWrap) {
#pragma unroll
      for (int p = 0; p < 7; ++p) {
        uint32_t v[NW];
#pragma unroll
        for (int w = 0; w < NW; ++w) v[w] = o[w][p];
        stsv<NW>(cx.stage + G::kPad + p * (4 * kPlaneWrap) + (wl & (kPlaneWrap - 1)) * 4, v);
      }
    }
    fence_async_smem();
    __syncwarp();
    if (lane == 0) {
      tma_store(padmap, kPlaneLead - kPlaneWrap, trow, cx.stage + G::kPad);
      bulk_commit();
    }
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
  const uint32_t lane_off = 4u * kSlotPad + L.lane * NW * 4u;
  // Ring position of the next row to issue / of rows r-1, r, r+1, and the
  // mbarrier phase of each slot, tracked incrementally.
  uint32_t phase = 0;  // bit k: phase of slot k's next completion
  int issue_row = first, issue_slot = 0;
  auto issue = [&]() {
    if (L.lane == 0) {
      const uint32_t bar = bars + issue_slot * 8u;
      mbar_expect_tx(bar, G::kRowBytes);
      tma_row(ring + issue_slot * G::kSlot, map, L.w0 + kPlaneLead - kSlotPad, issue_row + 1, bar);
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
    dest_row<NW, FORCE, RULE, Q, 0, true, false>(ring + sm * G::kSlot + lane_off,
                                          ring + sc * G::kSlot + lane_off,
                                          ring + sn * G::kSlot + lane_off, 0u, 0u, 0u, cx, L.lane,
                                          y0 + r, stmap, padmap, L.w0, r + 1, L.padx, swaps, [] {});
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
    step_planes_kernel(const __grid_constant__ StepArgs a, const __grid_constant__ CUtensorMap map,
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
  // smem: chirality column keys ({lo, t2} [cta_cols], g [cta_cols]), the
  // forcing ones, 32 span slots, then per warp the row ring, the walk list
  // and results, the ring's mbarriers.
  const uint32_t kc_base = sbase;
  const uint32_t kf_base = kc_base + cta_cols * 16;
  const uint32_t slots = sbase + (FORCE ? 2 : 1) * cta_cols * 16;
  const uint32_t wbase = slots + 128 + warp * G::kWarp;
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
  // this overlaps its tail under PDL), then wait for the previous grid. Key
  // base row: the CTA's first row.
  const uint32_t ybase =
      static_cast<uint32_t>(a.row0 + a.row_lo + seg_group * a.spc * a.seg_rows);
  span_put(slots, make_col_keys<FORCE>(kc_base, kf_base, a.kc_cur, a.kf_cur,
                                       static_cast<uint32_t>(cta_x0) + 1u, ybase, threadIdx.x,
                                       blockDim.x, cta_cols));
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
  L.PW = plane_stride_words(a.W);
  L.w0 = band * G::kBandWords;
  // Lanes holding words 0..3 / WW-4..WW-1 also stage the right / left pad
  // box (periodic wrap copies): words 0..3 go to padded words WW+4..WW+7,
  // words WW-4..WW-1 to padded words 0..3.
  L.padx = (L.w0 + G::kBandWords == L.WW ? 1 : 0) | (L.w0 == 0 ? 2 : 0) | (L.WW << 2);
  Ctx<NW, FORCE> cx;
  cx.kc = kc_base + bic * G::kBandCols * 16;
  cx.kf = kf_base + bic * G::kBandCols * 16;
  cx.ybase = ybase;
  cx.span = min(span_get(slots), a.span_cap);
  cx.x1 = static_cast<uint32_t>(cta_x0 + bic * G::kBandCols) + 1u;
  cx.kcur = a.kc_cur;
  cx.kfcur = a.kf_cur;
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
// Ring slots (any multiple of the box rows: the consumers track slot indices
// incrementally). A shallow ring keeps the bands' CTAs on the same rows (a
// row's 8 band segments leave DRAM together): the memory-bound rules (the
// reference's DEFAULT, FHP-I: few collisions) run 32 slots (DEFAULT table at
// cfg4: 2348 GSUPS with 56 slots, 2900 with 32); the compute-bound FHP-III is
// insensitive (2544 / 2535) and keeps 56; forcing runs 32.
#ifndef FHPG_RING_SLOTS
#define FHPG_RING_SLOTS 56
#endif
#ifndef FHPG_RING_SLOTS_F
#define FHPG_RING_SLOTS_F 32
#endif
#ifndef FHPG_RING_SLOTS_L
#define FHPG_RING_SLOTS_L 32
#endif
#ifndef FHPG_RING_CONS_L
#define FHPG_RING_CONS_L FHPG_RING_CONS  // consumer warps of the memory-bound rules
#endif
template <int NW, bool FORCE, int RULE = 2>
struct RingGeo {
  using G = Geo<NW, FORCE>;
  static constexpr int kCons = (FORCE || RULE == 2) ? FHPG_RING_CONS : FHPG_RING_CONS_L;
  static constexpr int kRing = FORCE ? FHPG_RING_SLOTS_F
                               : RULE == 2 ? FHPG_RING_SLOTS : FHPG_RING_SLOTS_L;
  // (the consumers' slot step wraps once: s + kCons < 2 kRing)
  static_assert(kRing > kCons, "ring slots > consumer warps");
  static constexpr int kThreads = (kCons + 1) * 32;
  // Column keys: {lo, t2, g, 0} per column (chirality, then forcing), then
  // 32 span slots.
  static constexpr int kKeyTab = G::kBandCols * 16;
  static constexpr int kSpanOff = (FORCE ? 2 : 1) * kKeyTab;
  static constexpr int kKeys = kSpanOff + 128;
  static constexpr int kRingOff = (kKeys + 127) / 128 * 128;
  static constexpr int kStageOff = kRingOff + kRing * G::kSlot;
  static constexpr int kBarOff = kStageOff + kCons * G::kStage;  // (no wrap-sector box)
  static constexpr int kBox = FHPG_BOX_ROWS;     // source rows per TMA box (a "group")
  static constexpr int kGroups = kRing / kBox;   // ring slots of whole groups
  static_assert(kRing % kBox == 0, "row groups");
  static_assert((kBox & (kBox - 1)) == 0, "box rows: a power of two");
  // Full barriers, one per group modulo kFullBars (a power of two >= 4
  // kGroups). A consumer waiting on group P has finished its previous row
  // (31 rows = at most 9 groups back), so the producer has issued group
  // P - 9 and with it every group up to P - 9 - kGroups has been consumed:
  // the barrier's use for group P - kFullBars is complete and the parity
  // wait for group P is unambiguous (static round-robin rows, no slot tags).
  static constexpr int kFullBars = kGroups <= 8 ? 32 : kGroups <= 16 ? 64 : 128;
  static_assert(kFullBars > kGroups + (kCons + kBox) / kBox + 1, "tag-free ring bound");
  static_assert(kCons <= 31, "consumer warps");
  // mbarriers: kFullBars full (per group) and the empty barriers: per slot
  // (3 readers: a consumer releases its three source rows with three plain
  // arrives, the producer checks the 4 slots of a group; the compute-bound
  // FHP-III, +1.1%) or per group (12 arrivals, a consumer merges its rows'
  // arrivals per group; the memory-bound rules, whose producer thread's
  // per-group cost shows: DEFAULT table 2862 vs 2894).
  static constexpr bool kSlotEmpty = RULE == 2;
  static constexpr int kEmpties = kSlotEmpty ? kRing : kGroups;
  static constexpr int kCtrOff = kBarOff + 8 * (kFullBars + kEmpties);
  // Side buffer of the edge bands: per group, the 4 data words across the
  // periodic wrap of every plane and row ([kBox rows][8 planes][4 words]).
  static constexpr int kSideGroup = kBox * 8 * 16;
  static constexpr int kSideOff = (kCtrOff + 8 + 127) / 128 * 128;
  static constexpr int kSmem = kSideOff + kGroups * kSideGroup;
  static_assert(kSmem <= 232448, "shared memory per CTA");
};

// Re-keying by the consumer warps of a ring CTA (barrier 2): once every
// consumer is past the rows of the current keys, the band's column keys are
// rebuilt for key base row ybase (a band switch, or rows reaching the
// keys' span); returns the new span. Not inlined: it runs a few times per
// thousand CTA steps.
template <bool FORCE, int NCONS, int NCOLS>
__device__ __noinline__ uint32_t rekey_consumers(uint32_t kc, uint32_t kf,
                                                 uint32_t slots, uint64_t kcur, uint64_t kfcur,
                                                 uint32_t x1, uint32_t ybase) {
  asm volatile("bar.sync 2, %0;" ::"n"(NCONS) : "memory");
  span_put(slots, make_col_keys<FORCE>(kc, kf, kcur, kfcur, x1, ybase, threadIdx.x, NCONS,
                                       NCOLS));
  if (threadIdx.x == 0) sts32(slots + (NCONS / 32) * 4, 0xFFFFFFFFu);  // the producer's slot
  asm volatile("bar.sync 2, %0;" ::"n"(NCONS) : "memory");
  return span_get(slots);
}

__device__ __forceinline__ void mbar_arrive(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}

template <int NW, bool FORCE, int RULE>
__global__ void __launch_bounds__(RingGeo<NW, FORCE, RULE>::kThreads, 1)
    step_ring_kernel(const __grid_constant__ StepArgs a, const __grid_constant__ CUtensorMap stmap,
                     const __grid_constant__ CUtensorMap sidemap,
                     const __grid_constant__ CUtensorMap map2) {
  using G = Geo<NW, FORCE>;
  using RG = RingGeo<NW, FORCE, RULE>;
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
  const uint32_t kf_base = kc_base + RG::kKeyTab;
  const uint32_t slots = sbase + RG::kSpanOff;
  const uint32_t ring = sbase + RG::kRingOff;
  const uint32_t full = sbase + RG::kBarOff;
  const uint32_t empty = full + 8 * RG::kFullBars;
  const uint32_t side = sbase + RG::kSideOff;
  // Which wrap a band's rows need from the side buffer (1: band 0 of several,
  // 2: the last band of several; a single band finds both in its own box).
  auto edge_of = [&](int b) { return a.nbands == 1 ? 3 : b == 0 ? 1 : b == a.nbands - 1 ? 2 : 0; };
  if (threadIdx.x == 0) {
    // Source rows come in groups of kBox (one TMA box): group P = index /
    // kBox fills ring group P mod kGroups and completes full barrier P mod
    // kFullBars; each slot is released on its own empty barrier (3
    // consumers per row).
    for (int k = 0; k < RG::kFullBars; ++k) mbar_init(full + k * 8, 1);
    for (int k = 0; k < RG::kEmpties; ++k) mbar_init(empty + k * 8, RG::kSlotEmpty ? 3 : 3 * RG::kBox);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // The band's column keys, made here from the step keys (they depend on
  // nothing the previous step wrote, so this overlaps its tail under PDL).
  // Key base row: the part's first destination row.
  auto make_keys = [&](int b, uint32_t ybase, int t0, int nt) {
    span_put(slots, make_col_keys<FORCE>(kc_base, kf_base, a.kc_cur, a.kf_cur,
                                         static_cast<uint32_t>(b * G::kBandCols) + 1u, ybase, t0,
                                         nt, G::kBandCols));
  };
  make_keys(bA, static_cast<uint32_t>(a.row0 + RA0), threadIdx.x, blockDim.x);
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
#if FHPG_TIMELINE  // timing instrument: CTA start (after the PDL wait) and end, per launch
  unsigned long long t_start = 0;
  if (threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));
#endif

  if (warp == RG::kCons) {  // producer (tensor row = local row + 1)
    if (lane == 0) {
      constexpr uint32_t kG = RG::kGroups;
      const uint32_t gA = offB / B;
      const uint32_t ngroups = gA + (nB > 0 ? (static_cast<uint32_t>(nB) + 2 + B - 1) / B : 0u);
      // k = P mod kG (ring group), lap = P / kG, tracked incrementally
      uint32_t k = 0, lap = 0;
      for (uint32_t P = 0; P < ngroups; ++P) {
        if (lap > 0) {
          if constexpr (RG::kSlotEmpty) {
#pragma unroll
            for (uint32_t q = 0; q < B; ++q) mbar_wait(empty + (B * k + q) * 8, (lap - 1) & 1u);
          } else {
            mbar_wait(empty + k * 8, (lap - 1) & 1u);
          }
        }
        const uint32_t fb = full + (P % RG::kFullBars) * 8;
        const bool inA = P < gA;
        const int word = (inA ? bA : bA + 1) * G::kBandWords + kPlaneLead - kSlotPad;
        const int trow = inA ? RA0 + static_cast<int>(B * P) : row_lo + static_cast<int>(B * P - offB);
#if FHPG_STREAM_ONLY == 3 || FHPG_STREAM_ONLY >= 5  // timing experiments: no loads
        if (FHPG_STREAM_ONLY >= 5 && P < kG) {  // 5, 6: compute on the first ring fill
          mbar_expect_tx(fb, B * G::kRowBytes);
          tma_row(ring + B * k * G::kSlot, &map2, word, trow, fb);
        } else {
          mbar_arrive(fb, 1);
        }
#else
        const int e = edge_of(inA ? bA : bA + 1);
        const bool sided = e == 1 || e == 2;
        mbar_expect_tx(fb, B * G::kRowBytes + (sided ? RG::kSideGroup : 0));
        tma_row(ring + B * k * G::kSlot, &map2, word, trow, fb);  // tensor rows
        if (sided)  // data words W/32-4 .. W/32-1 (left wrap) or 0 .. 3 (right wrap)
          tma_row(side + k * RG::kSideGroup, &sidemap,
                  e == 1 ? kPlaneLead + (a.W >> 5) - 4 : kPlaneLead, trow, fb);
#endif
        // Ring indices no destination row reads (the tail of part A's last
        // group when part B follows) still count 3 arrivals each, or the
        // slot is never freed.
        if (nB > 0 && P + 1 == gA && offB > static_cast<uint32_t>(nA) + 2) {
          if constexpr (RG::kSlotEmpty) {
            for (uint32_t q = static_cast<uint32_t>(nA) + 2; q < offB; ++q)
              mbar_arrive(empty + (B * k + (q - B * P)) * 8, 3);
          } else {
            mbar_arrive(empty + k * 8, 3 * (offB - static_cast<uint32_t>(nA) - 2));
          }
        }
        if (++k == kG) {
          k = 0;
          ++lap;
        }
      }
    }
    return;
  }

  Lanes L;
  L.lane = lane;
  L.WW = a.W >> 5;
  L.PW = plane_stride_words(a.W);
  auto set_band = [&](int b) {
    L.w0 = b * G::kBandWords;
    L.padx = (L.w0 + G::kBandWords == L.WW ? 1 : 0) | (L.w0 == 0 ? 2 : 0) | (L.WW << 2);
  };
  set_band(bA);
  const uint32_t stage = sbase + RG::kStageOff + warp * G::kStage;
  Ctx<NW, FORCE> cx;
  cx.kc = kc_base;
  cx.kf = kf_base;
  cx.ybase = static_cast<uint32_t>(a.row0 + RA0);
  cx.span = max(1u, min(span_get(slots), a.span_cap));
  cx.x1 = static_cast<uint32_t>(bA * G::kBandCols) + 1u;
  cx.kcur = a.kc_cur;
  cx.kfcur = a.kf_cur;
  cx.lsm = stage;
  cx.osm = stage + G::kList;
  cx.stage = stage;
  cx.thr = a.thr;
  cx.four = a.k4;
  unsigned swaps = 0;
  const uint32_t lane_off = 4u * kSlotPad + lane * NW * 4u;
  const uint32_t y0 = static_cast<uint32_t>(a.row0);  // global rows < 2^31
  // Destination rows [Rb, Re) of the current band, warp-interleaved; source
  // row r - 1 sits at ring index ibase + r - Rb. Inlined once per part (one
  // copy inside a loop over the parts measured 8% slower: spills).
  // Column keys are valid for rows [key_row, key_row + span) of the band;
  // reaching the end re-keys (all consumers, rekey_consumers).
  int key_row = RA0;
  auto key_end = [&](int Re) { return key_row + static_cast<int>(min(cx.span, static_cast<uint32_t>(Re - key_row))); };
  auto rekey = [&](int b, int row) {
    cx.span = max(1u, min(rekey_consumers<FORCE, RG::kCons * 32, G::kBandCols>(
                              kc_base, kf_base, slots, a.kc_cur, a.kf_cur,
                              static_cast<uint32_t>(b * G::kBandCols) + 1u,
                              y0 + static_cast<uint32_t>(row)),
                          a.span_cap));
    cx.ybase = y0 + static_cast<uint32_t>(row);
    key_row = row;
  };
  auto rows = [&](auto ec, const int b, const int Rb, const int Re, const uint32_t ibase,
                  const uint32_t ctr) __attribute__((always_inline)) {
    constexpr int E = decltype(ec)::value;
    int kend = key_end(Re);
    (void)ctr;
    // Ring index i of source row r - 1 and its slot s0 = i mod kRing, both
    // advanced by kCons per row of this warp.
    uint32_t i = ibase + static_cast<uint32_t>(warp);
    uint32_t s0 = i % RG::kRing;
    auto wrap = [](uint32_t x) { return x >= static_cast<uint32_t>(RG::kRing) ? x - RG::kRing : x; };
    for (int r = Rb + warp; r < Re;
         r += RG::kCons, i += RG::kCons, s0 = wrap(s0 + RG::kCons)) {
      while (r >= kend) {  // rows past the keys' span: re-key at kend
        rekey(b, kend);
        kend = key_end(Re);
      }
      const bool first_row = r == Rb, last_row = r == Re - 1;
      const uint32_t sd[3] = {s0, wrap(s0 + 1), wrap(s0 + 2)};
      uint32_t sl[3];
#pragma unroll
      for (uint32_t d = 0; d < 3; ++d) {
        if (d == 0 || (sd[d] % B) == 0) {  // a new group
          const uint32_t P = (i + d) / B;
          mbar_wait(full + (P % RG::kFullBars) * 8, (P / RG::kFullBars) & 1u);
        }
        sl[d] = ring + sd[d] * G::kSlot + lane_off;
      }
      uint32_t sw[3] = {0u, 0u, 0u};  // side-buffer rows of the source rows
      if constexpr (E == 1 || E == 2) {
        static_assert(RG::kSideGroup == B * 8 * 16, "side rows");
#pragma unroll
        for (uint32_t d = 0; d < 3; ++d) sw[d] = side + sd[d] * (8u * 16u);
      }
      // Release the three source rows as soon as they are in registers (3
      // consumers per row; segment edges make up for the destination rows
      // outside [Rb, Re)): one arrive per slot, or per group the rows fall
      // in (ring group of slot s = s / B).
      auto release = [&] {
        __syncwarp();
        if (lane == 0 && !RG::kSlotEmpty) {
          const uint32_t first = first_row ? 1u : 0u, lastr = last_row ? 1u : 0u;
          const uint32_t c0 = 1 + 2 * first, c1 = 1 + first + lastr, c2 = 1 + 2 * lastr;
          const uint32_t g0 = i / B, g1 = (i + 1) / B, g2 = (i + 2) / B;
          if (g0 == g2) {
            mbar_arrive(empty + (sd[0] / B) * 8, c0 + c1 + c2);
          } else {
            mbar_arrive(empty + (sd[0] / B) * 8, c0 + (g1 == g0 ? c1 : 0u));
            mbar_arrive(empty + (sd[2] / B) * 8, c2 + (g1 == g2 ? c1 : 0u));
          }
        } else if (lane == 0) {
          if (!first_row && !last_row) {
            mbar_arrive(empty + sd[0] * 8, 1);
            mbar_arrive(empty + sd[1] * 8, 1);
            mbar_arrive(empty + sd[2] * 8, 1);
          } else {
            const uint32_t first = first_row ? 1u : 0u, lastr = last_row ? 1u : 0u;
            mbar_arrive(empty + sd[0] * 8, 1 + 2 * first);
            mbar_arrive(empty + sd[1] * 8, 1 + first + lastr);
            mbar_arrive(empty + sd[2] * 8, 1 + 2 * lastr);
          }
        }
      };
      if ((a.row0 + r) & 1)
        dest_row<NW, FORCE, RULE, 1, E, false, true>(sl[0], sl[1], sl[2], sw[0], sw[1], sw[2], cx, lane,
                                               y0 + r, &stmap, nullptr, L.w0, r + 1, 0, swaps,
                                               release);
      else
        dest_row<NW, FORCE, RULE, 0, E, false, true>(sl[0], sl[1], sl[2], sw[0], sw[1], sw[2], cx, lane,
                                               y0 + r, &stmap, nullptr, L.w0, r + 1, 0, swaps,
                                               release);
      }
    while (kend < Re) {  // re-keyings the other consumers still take part in
      rekey(b, kend);
      kend = key_end(Re);
    }
  };
  // One inlined copy of the row loop per edge kind (interior bands pay
  // nothing for the wrap).
  auto rows_e = [&](int b, const int Rb, const int Re, const uint32_t ibase,
                    const uint32_t ctr) __attribute__((always_inline)) {
    switch (edge_of(b)) {
      case 0: rows(std::integral_constant<int, 0>{}, b, Rb, Re, ibase, ctr); break;
      case 1: rows(std::integral_constant<int, 1>{}, b, Rb, Re, ibase, ctr); break;
      case 2: rows(std::integral_constant<int, 2>{}, b, Rb, Re, ibase, ctr); break;
      default: rows(std::integral_constant<int, 3>{}, b, Rb, Re, ibase, ctr); break;
    }
  };
  rows_e(bA, RA0, RA0 + nA, 0u, sbase + RG::kCtrOff);
  if (nB > 0) {
    // Extra CTA: on to band bA + 1 once every consumer is done with band bA
    // (the key table is rewritten); the producer streams on meanwhile.
    rekey(bA + 1, row_lo);
    cx.x1 = static_cast<uint32_t>((bA + 1) * G::kBandCols) + 1u;
    set_band(bA + 1);
    rows_e(bA + 1, row_lo, row_lo + nB, offB, sbase + RG::kCtrOff + 4);
  }
  if (lane == 0) bulk_wait_all();  // the stores have landed before the kernel ends
#if FHPG_TIMELINE
  asm volatile("bar.sync 3, %0;" ::"r"(RG::kCons * 32) : "memory");
  if (threadIdx.x == 0) {
    unsigned long long t_end;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_end));
    const unsigned long long slot = atomicAdd(&g_timeline_n, 1ull);
    if (slot < kTimelineMax) {
      g_timeline[slot * 4 + 0] = blockIdx.x;
      g_timeline[slot * 4 + 1] = t_start;
      g_timeline[slot * 4 + 2] = t_end;
      g_timeline[slot * 4 + 3] = static_cast<unsigned long long>(nA + nB);
    }
  }
#endif
  if (FORCE) {
    unsigned long long sw = swaps;
    for (int o = 16; o; o >>= 1) sw += __shfl_xor_sync(kFull, sw, o);
    if (lane == 0 && sw) atomicAdd(a.swaps, sw);
  }
}

// Grid of the ring kernel: nbands x segment groups of the row range
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

// maps: make_planes_map kinds (kMapLoad, kMapStore, kMapLoadRows, kMapPad, kMapSide).
template <int NW, bool FORCE, int RULE>
void launch_ring(StepArgs a, const CUtensorMap* src, const CUtensorMap* dst, int num_sms,
                 cudaStream_t st) {
  using RG = RingGeo<NW, FORCE, RULE>;
  const int grid = ring_grid<NW>(a, num_sms);
  ensure_smem_optin(reinterpret_cast<const void*>(step_ring_kernel<NW, FORCE, RULE>), RG::kSmem);
  launch_pdl(step_ring_kernel<NW, FORCE, RULE>, grid, RG::kThreads, RG::kSmem, st, a,
             dst[kMapStore], src[kMapSide], src[kMapLoadRows]);
}

template <int NW, bool FORCE>
int smem_bytes(int bpc) {
  using G = Geo<NW, FORCE>;
  return (FORCE ? 2 : 1) * bpc * G::kBandCols * 16 + 128 + kPWarps<NW> * G::kWarp;
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
  cudaLaunchKernelEx(&cfg, step_planes_kernel<NW, FORCE, RULE>, a, src[kMapLoad], dst[kMapStore],
                     dst[kMapPad]);
#else
  step_planes_kernel<NW, FORCE, RULE><<<grid, kWarps * 32, smem, st>>>(a, src[kMapLoad], dst[kMapStore],
                                                                      dst[kMapPad]);
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
    const int PW = plane_stride_words(W);
    // periodic-wrap copies: data words 0..7 after the data, W/32-8.. before it
    const int pad = i < kPlaneWrap ? WW : (i >= WW - kPlaneWrap ? -WW : 0);
    uint32_t* d = reinterpret_cast<uint32_t*>(dst + r * static_cast<long long>(pitch)) + kPlaneLead + i;
    uint32_t* o = reinterpret_cast<uint32_t*>(dst_obst + r * static_cast<long long>(pitch)) + kPlaneLead + i;
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
        reinterpret_cast<const uint32_t*>(src + r * static_cast<long long>(pitch)) + kPlaneLead + i;
    const int PW = plane_stride_words(W);
    uint32_t p[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) p[q] = s[q * PW];
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

size_t planes_row_bytes(int W) { return static_cast<size_t>(plane_stride_words(W)) * 32; }

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
  // Tensor {plane-row words, planes, rows}. Boxes: kMapLoad one band of 32
  // NW words + 4 on either side, all 8 planes; kMapStore the band's words,
  // planes 0-6; kMapLoadRows as kMapLoad for FHPG_BOX_ROWS consecutive rows.
  const int nw = planes_words_per_lane(W);
  const int xw = plane_stride_words(W);
  const cuuint64_t dims[3] = {static_cast<cuuint64_t>(xw), 8, static_cast<cuuint64_t>(rows)};
  const cuuint64_t strides[2] = {static_cast<cuuint64_t>(xw * 4), static_cast<cuuint64_t>(pitch)};
  const bool load = kind == kMapLoad || kind == kMapLoadRows || kind == kMapSide;
  const cuuint32_t box[3] = {
      static_cast<cuuint32_t>(kind == kMapSide ? 4 : load ? 32 * nw + 2 * kSlotPad
                              : kind == kMapPad ? kPlaneWrap : 32 * nw),
      load ? 8u : 7u,
      kind == kMapLoadRows || kind == kMapSide ? static_cast<cuuint32_t>(FHPG_BOX_ROWS) : 1u};
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
    if (force) launch_ring<2, true, R>(a, src, dst, num_sms, st);
    else launch_ring<2, false, R>(a, src, dst, num_sms, st);
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

#if FHPG_TIMELINE
// Timing instrument (FHPG_TIMELINE builds only; not in include/): copies the
// recorded (block, start ns, end ns, rows) records out and resets the log.
extern "C" int fhpg_debug_timeline(unsigned long long* out, int max_records) {
  unsigned long long n = 0;
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(&n, g_timeline_n, sizeof(n));
  if (n > kTimelineMax) n = kTimelineMax;
  if (static_cast<long long>(n) > max_records) n = max_records;
  cudaMemcpyFromSymbol(out, g_timeline, n * 4 * sizeof(unsigned long long));
  const unsigned long long zero = 0;
  cudaMemcpyToSymbol(g_timeline_n, &zero, sizeof(zero));
  return static_cast<int>(n);
}
#endif
}  // namespace fhpg
