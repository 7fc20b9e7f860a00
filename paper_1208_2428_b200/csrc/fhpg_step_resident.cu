// fhpg_step_resident.cu — small bit-plane lattices (cfg1: 1024 x 1024): a
// whole advance call in ONE cooperative launch, the lattice held in shared
// memory, time-blocked with deep halos.
//
// At 1M sites a step is ~0.5 us of work but a launch of the streaming ring
// kernel costs ~5 us (grid start, ring fill, drain; profiles/height_r01h.json)
// — the small BASELINE shape is launch-bound. Here each CTA owns a band of
// rows [r0, r1) of the whole lattice and works in blocks of k steps: it loads
// rows [r0 - k, r1 + k) (all 8 planes, with the periodic-wrap pad words) into
// shared memory, computes k steps there on a shrinking row range (row r of
// step j needs rows r-1..r+1 of step j-1, so after k steps exactly [r0, r1) is
// valid; rows outside the lattice stay zero, the reference's out-of-grid
// rows, step.cpp:47), writes [r0, r1) back to the other global buffer and
// meets the other CTAs at a grid barrier — one barrier and one L2 round trip
// per k steps instead of a launch per step. The halo rows are recomputed by
// the neighbouring CTAs; every random decision is keyed by global (x, y,
// step), so the redundant copies are bit-identical and the result is the
// streaming kernels' (and the reference's) exactly.
//
// Per destination row and 1024-column band, one warp evaluates the same
// pull / circuit / lazy-chirality walk as the ring kernel (fhpg_planes_dev.cuh,
// fhpg_planes_rules.cuh), reading and writing shared memory only.
#include <cstdint>
#include <type_traits>

#include <cuda.h>
#include <cudaTypedefs.h>

#include "fhpg_common.cuh"
#include "fhpg_kernels.cuh"
#include "fhpg_planes_rules.cuh"

namespace fhpg {
namespace {

#include "fhpg_planes_dev.cuh"

// Warps per CTA and halo depth per kind of run (tools/ab_small.py, cfg1 =
// FHP-I 1024^2 p = 0; FHP-III p = 0.01 at 1024^2 / 2048^2): a k-step block
// computes rows_per_cta + 2 (k - 1 - j) rows at its step j, so with 7 rows
// per CTA 24 warps take every step of a depth-9 block in one row round
// (16 warps: 3 of 8 steps in two): cfg1 539 -> 569 GSUPS. The forced runs
// (two walks per row, twice the key table) keep 16 warps and depth 8
// (1024^2: 313 vs 306 with 24 warps).
#ifndef FHPG_RES_WARPS
#define FHPG_RES_WARPS 24
#endif
#ifndef FHPG_RES_WARPS_F
#define FHPG_RES_WARPS_F 16
#endif
template <bool FORCE>
constexpr int res_warps() { return FORCE ? FHPG_RES_WARPS_F : FHPG_RES_WARPS; }

struct ResArgs {
  uint8_t* g0;             // the engine's two plane buffers, local row 0
  uint8_t* g1;
  int cur;                 // buffer holding the state at `first`
  size_t pitch;
  int W, H;
  int rows_per_cta;
  int depth;               // k: steps per block (halo depth)
  long long first, count;  // global step indices first .. first + count - 1
  uint64_t seed, thr;
  uint32_t k4;             // 4, at run time (chir_bit)
  unsigned long long* swaps;
  unsigned* bar;           // grid barrier: [0] arrivals, [1] generation
};

// u / n for the small run-time divisors of the index loops (bands, 16-byte
// chunks per row / plane) without the ~20-instruction integer division:
// with m = ceil(2^32 / n), umulhi(u, m) is exact for u < 2^32 / n.
struct FastDiv {
  uint32_t n, m;
  __device__ explicit FastDiv(uint32_t d)
      : n(d), m(d > 1 ? static_cast<uint32_t>(((1ull << 32) + d - 1) / d) : 0u) {}
  __device__ __forceinline__ uint32_t div(uint32_t u) const { return n == 1 ? u : __umulhi(u, m); }
};
// x mod n for x in [-n, 2n).
__device__ __forceinline__ int wrap_mod(int x, int n) { return x < 0 ? x + n : x >= n ? x - n : x; }

__device__ __forceinline__ uint4 ldcg128(const void* p) {
  return __ldcg(reinterpret_cast<const uint4*>(p));  // L2 only: other SMs wrote it
}

// All CTAs of the (cooperative) grid: every global store issued before the
// barrier is visible to every load issued after it.
__device__ __forceinline__ void grid_barrier(unsigned* bar) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    unsigned gen;
    asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(gen) : "l"(bar + 1) : "memory");
    if (atomicAdd(bar, 1u) == gridDim.x - 1) {
      atomicExch(bar, 0u);
      __threadfence();
      atomicAdd(bar + 1, 1u);
    } else {
      for (;;) {
        unsigned now;
        asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(now) : "l"(bar + 1) : "memory");
        if (now != gen) break;
        __nanosleep(32);
      }
    }
    __threadfence();
  }
  __syncthreads();
}

// One destination row (parity Q) of one band: sm, sc, sn = this lane's word
// in plane 0 of rows r-1, r, r+1 of the source buffer; dst = the same word of
// row r in the destination buffer; P = plane stride (bytes); pad = byte
// offset of this word's periodic-wrap copy (0: none).
template <int RULE, bool FORCE, int Q>
__device__ __forceinline__ void resident_row(uint32_t sm, uint32_t sc, uint32_t sn, uint32_t dst,
                                             uint32_t P, int pad, uint32_t kc, uint32_t kf, int lane, uint32_t y,
                                             uint32_t four, uint64_t thr, bool own, unsigned& swaps) {
  uint32_t a0[1], a1[1], a2[1], a3[1], a4[1], a5[1], rr[1], so[1];
  // Pull sources (backends.cpp:64-73): k0 (x+q, r+1), k1 (x+q-1, r+1),
  // k2 (x-1, r), k3 (x+q-1, r-1), k4 (x+q, r-1), k5 (x+1, r).
  if (Q) rd_shr<1>(sn + 0 * P, a0); else rd_al<1>(sn + 0 * P, a0);
  if (Q) rd_al<1>(sn + 1 * P, a1); else rd_shl<1>(sn + 1 * P, a1);
  rd_shl<1>(sc + 2 * P, a2);
  if (Q) rd_al<1>(sm + 3 * P, a3); else rd_shl<1>(sm + 3 * P, a3);
  if (Q) rd_shr<1>(sm + 4 * P, a4); else rd_al<1>(sm + 4 * P, a4);
  rd_shr<1>(sc + 5 * P, a5);
  rd_al<1>(sc + 6 * P, rr);
  rd_al<1>(sc + 7 * P, so);
  const uint32_t a[6] = {a0[0], a1[0], a2[0], a3[0], a4[0], a5[0]};
  const auto K = PlaneRule<RULE>::classify(a, rr[0], so[0]);
  const uint32_t dep[1] = {K.dep};
  // chirality: bit 0 of node_random(seed, Chirality, step, x + 1, y) (step.cpp:73-76)
  // (each lane walks its own dep bits, walk_own: no per-row setup — the
  // rules this kernel runs at small shapes have few dep sites)
  uint32_t c[1];
  walk_own<1>(dep, lane, c, [&](uint32_t col) { return chir_mask(lds64(kc + col * 8u) + y, four); });
  uint32_t o[7];
  PlaneRule<RULE>::apply(K, c[0], rr[0], a, o, o[6], so[0]);
  if constexpr (FORCE) {
    // step.cpp:79-88: fluid, W (bit 5) set, E (bit 2) clear after collision
    const uint32_t f[1] = {~so[0] & o[5] & ~o[2]};
    uint32_t acc[1];
    walk_own<1>(f, lane, acc, [&](uint32_t col) -> uint32_t {
      return (fin64(lds64(kf + col * 8u) + y) >> 32) < thr ? ~0u : 0u;
    });
    o[5] ^= acc[0];
    o[2] ^= acc[0];
    if (own) swaps += __popc(acc[0]);  // halo rows are counted by their owner CTA
  }
#pragma unroll
  for (int p = 0; p < 7; ++p) sts32(dst + p * P, o[p]);
  sts32(dst + 7 * P, so[0]);  // the obstacle plane travels with the row
  if (pad) {
#pragma unroll
    for (int p = 0; p < 7; ++p) sts32(dst + p * P + pad, o[p]);
    sts32(dst + 7 * P + pad, so[0]);
  }
}

template <int RULE, bool FORCE>
__global__ void __launch_bounds__(res_warps<FORCE>() * 32, 1) step_resident_kernel(ResArgs a) {
  constexpr int kResWarps = res_warps<FORCE>();
  extern __shared__ __align__(128) uint8_t smem[];
  const uint32_t sbase = smem_u32(smem);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int WW = a.W >> 5;
  const uint32_t P = static_cast<uint32_t>(WW + 8) * 4u;  // shared plane row (4 wrap words each side)
  const uint32_t GP = static_cast<uint32_t>(plane_stride_words(a.W)) * 4u;  // global plane row
  const uint32_t RB = 8u * P;                              // row of 8 planes
  const int nb = a.W >> 10;                                // 1024-column bands
  const FastDiv dnb(nb), dn16(RB / 16u), dp16(P / 16u);
  const FastDiv dsn16(7u * ((WW + 2 * kPlaneWrap) / 4u)), dsp16((WW + 2 * kPlaneWrap) / 4u);
  const int k = a.depth;
  const int r0 = blockIdx.x * a.rows_per_cta, r1 = min(a.H, r0 + a.rows_per_cta);
  const int base = r0 - k - 1;  // global row of local row 0
  const int nloc = (r1 - r0) + 2 * k + 2;
  const uint32_t kc = sbase, kf = sbase + a.W * 8;
  const uint32_t bufs = sbase + (FORCE ? 2u : 1u) * static_cast<uint32_t>(a.W) * 8u;
  const uint32_t bufsz = static_cast<uint32_t>(nloc) * RB;
  // Zero rows stand for the rows outside the lattice.
  for (uint32_t o = threadIdx.x * 16u; o < 2u * bufsz; o += blockDim.x * 16u) sts128(bufs + o, 0, 0, 0, 0);
  unsigned swaps = 0;
  int g = a.cur;
  for (long long done = 0; done < a.count;) {
    const int kb = static_cast<int>(min(static_cast<long long>(k), a.count - done));
    __syncthreads();
    // Rows [r0 - kb, r1 + kb) of the current state into buffer 0.
    // (Shared memory keeps 4 wrap words on either side of each plane's data,
    // made here from the data words: the streaming ring kernel does not
    // maintain the global rows' wrap sectors.)
    {
      const int lo = max(0, r0 - kb), hi = min(a.H, r1 + kb);
      const uint32_t n16 = RB / 16u, p16 = P / 16u;
      const uint32_t total = static_cast<uint32_t>(hi - lo) * n16;
      for (uint32_t t = threadIdx.x; t < total; t += blockDim.x) {
        const uint32_t rr = dn16.div(t), c = t - rr * n16, pl = dp16.div(c), j = c - pl * p16;
        const int d = static_cast<int>(4 * j) - 4;  // data word of the chunk
        const uint32_t gw = kPlaneLead + static_cast<uint32_t>(wrap_mod(d, WW));
        const uint4 v = ldcg128((g ? a.g1 : a.g0) + static_cast<size_t>(lo + rr) * a.pitch +
                                pl * GP + gw * 4u);
        sts128(bufs + static_cast<uint32_t>(lo + rr - base) * RB + c * 16u, v.x, v.y, v.z, v.w);
      }
    }
    int sb = 0;
    for (int j = 0; j < kb; ++j) {
      const uint64_t s = static_cast<uint64_t>(a.first + done + j);
      const uint64_t kcs = step_key(a.seed, kChirality, s), kfs = step_key(a.seed, kForcing, s);
      for (int c = threadIdx.x; c < a.W; c += blockDim.x) {
        sts64(kc + c * 8, column_key(kcs, static_cast<uint64_t>(c) + 1));
        if (FORCE) sts64(kf + c * 8, column_key(kfs, static_cast<uint64_t>(c) + 1));
      }
      __syncthreads();
      const int clo = max(0, r0 - kb + 1 + j), chi = min(a.H, r1 + kb - 1 - j);
      const uint32_t src = bufs + static_cast<uint32_t>(sb) * bufsz;
      const uint32_t dst = bufs + static_cast<uint32_t>(sb ^ 1) * bufsz;
      const int units = (chi - clo) * nb;
      for (int u = warp; u < units; u += kResWarps) {
        const int q = static_cast<int>(dnb.div(static_cast<uint32_t>(u)));
        const int r = clo + q, b = u - q * nb;
        const uint32_t off = static_cast<uint32_t>(r - base) * RB + static_cast<uint32_t>(4 + b * 32 + lane) * 4u;
        const int pad = (b == 0 && lane < 4) ? WW * 4 : (b == nb - 1 && lane >= 28) ? -WW * 4 : 0;
        const uint32_t y = static_cast<uint32_t>(r);
        const bool own = r >= r0 && r < r1;
        if (r & 1)
          resident_row<RULE, FORCE, 1>(src + off - RB, src + off, src + off + RB, dst + off, P, pad,
                                       kc + b * 8192, kf + b * 8192, lane, y, a.k4, a.thr,
                                       own, swaps);
        else
          resident_row<RULE, FORCE, 0>(src + off - RB, src + off, src + off + RB, dst + off, P, pad,
                                       kc + b * 8192, kf + b * 8192, lane, y, a.k4, a.thr,
                                       own, swaps);
      }
      __syncthreads();
      sb ^= 1;
    }
    // Rows [r0, r1), planes 0-6 with their wrap sectors (global words
    // kPlaneLead - 8 .. kPlaneLead + WW + 8), into the other buffer (plane
    // 7, the obstacles, is static in both).
    {
      const uint32_t p16 = static_cast<uint32_t>(WW + 2 * kPlaneWrap) / 4u, n16 = 7u * p16;
      const uint32_t total = static_cast<uint32_t>(r1 - r0) * n16;
      const uint32_t src = bufs + static_cast<uint32_t>(sb) * bufsz;
      for (uint32_t t = threadIdx.x; t < total; t += blockDim.x) {
        const uint32_t rr = dsn16.div(t), c = t - rr * n16, pl = dsp16.div(c), j = c - pl * p16;
        const int d = static_cast<int>(4 * j) - kPlaneWrap;  // data word of the chunk
        const uint32_t sw = 4u + static_cast<uint32_t>(wrap_mod(d, WW));
        const uint4 v = lds128(src + static_cast<uint32_t>(r0 + rr - base) * RB + pl * P + sw * 4u);
        __stcg(reinterpret_cast<uint4*>((g ? a.g0 : a.g1) + static_cast<size_t>(r0 + rr) * a.pitch +
                                        pl * GP + (kPlaneLead - kPlaneWrap + 4 * j) * 4u),
               v);
      }
    }
    g ^= 1;
    done += kb;
    grid_barrier(a.bar);
  }
  if (FORCE) {
    unsigned long long sw = swaps;
    for (int o = 16; o; o >>= 1) sw += __shfl_xor_sync(0xFFFFFFFFu, sw, o);
    if (lane == 0 && sw) atomicAdd(a.swaps, sw);
  }
}

int resident_smem(int W, int rows_per_cta, int depth, bool force) {
  const int RB = 8 * (W / 32 + 8) * 4;
  const int nloc = rows_per_cta + 2 * depth + 2;
  return (force ? 2 : 1) * W * 8 + 2 * nloc * RB;
}

}  // namespace

// Halo depth (steps per block), unforced / forced. Unforced: cfg1 with 16
// warps 2 -> 320, 4 -> 416, 8 -> 422, 12 -> 397 GSUPS (round 2 start); with
// 24 warps depth 9 fills every row round (569 vs 564 at depth 8).
#ifndef FHPG_RESIDENT_DEPTH
#define FHPG_RESIDENT_DEPTH 9
#endif
#ifndef FHPG_RESIDENT_DEPTH_F
#define FHPG_RESIDENT_DEPTH_F 8
#endif
// Largest lattice (sites) the resident kernel takes: above it the streaming
// kernels' per-launch cost is a small fraction of a step. Measured crossover
// (tools/ab_small.py AB_WIDE=1, GSUPS resident / streaming): unforced 2048^2
// FHP-I 1205 / 1045, FHP-III 866 / 860; forced FHP-III 2048 x 1024 395 / 376,
// 2048^2 597 / 671 — the forced runs switch at 2M sites.
#ifndef FHPG_RESIDENT_MAX_SITES
#define FHPG_RESIDENT_MAX_SITES (4LL << 20)
#endif
#ifndef FHPG_RESIDENT_MAX_SITES_F
#define FHPG_RESIDENT_MAX_SITES_F (2LL << 20)
#endif

int resident_plan(int W, int H, uint64_t thr, int num_sms, int* rows_per_cta, int* grid) {
  const bool force = thr != 0;
  const long long max_sites = force ? FHPG_RESIDENT_MAX_SITES_F : FHPG_RESIDENT_MAX_SITES;
  if (W % 1024 || H < 3 || static_cast<long long>(W) * H > max_sites) return 0;
  const int rpc = (H + num_sms - 1) / num_sms;
  const int depth = force ? FHPG_RESIDENT_DEPTH_F : FHPG_RESIDENT_DEPTH;
  if (resident_smem(W, rpc, depth, force) > 227 * 1024) return 0;
  *rows_per_cta = rpc;
  *grid = (H + rpc - 1) / rpc;
  return depth;
}

// Returns the number of global-buffer flips (blocks of depth steps).
int launch_step_resident(uint8_t* const g[2], int cur, size_t pitch, int W, int H, int rule,
                         uint64_t seed, uint64_t thr, long long first, long long count,
                         unsigned long long* swaps, unsigned* bar, int num_sms, cudaStream_t st,
                         cudaError_t* err) {
  int rpc = 0, grid = 0;
  const int depth = resident_plan(W, H, thr, num_sms, &rpc, &grid);
  ResArgs a{};
  a.g0 = g[0];
  a.g1 = g[1];
  a.cur = cur;
  a.pitch = pitch;
  a.W = W;
  a.H = H;
  a.rows_per_cta = rpc;
  a.depth = depth;
  a.first = first;
  a.count = count;
  a.seed = seed;
  a.thr = thr;
  a.k4 = 4u;
  a.swaps = swaps;
  a.bar = bar;
  const bool f = thr != 0;
  const int smem = resident_smem(W, rpc, depth, f);
  void* args[] = {&a};
  auto go = [&](auto kernel) {
    ensure_smem_optin(reinterpret_cast<const void*>(kernel), smem);
    *err = cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(kernel), dim3(grid),
                                       dim3((f ? res_warps<true>() : res_warps<false>()) * 32),
                                       args, smem, st);
  };
  if (rule == 0) f ? go(step_resident_kernel<0, true>) : go(step_resident_kernel<0, false>);
  else if (rule == 1) f ? go(step_resident_kernel<1, true>) : go(step_resident_kernel<1, false>);
  else f ? go(step_resident_kernel<2, true>) : go(step_resident_kernel<2, false>);
  return static_cast<int>((count + depth - 1) / depth);
}

}  // namespace fhpg
