// fhpg_kernels.cu — sm_100a kernels of the B200 FHP engine.
//
// Hot path: one fused kernel per time step doing, for every site, the
// reference's pull motion (step.cpp:40-61, pull offsets backends.cpp:64-73),
// the 512-entry LUT collision with counter-RNG chirality and the stochastic
// W->E forcing (step.cpp:63-93). Ghost-column sync (lattice.cpp:32-39) is
// replaced by in-kernel periodic wrap; the buffer swap by ping-pong pointers.
//
// Fast path (W % 16 == 0): byte-per-site rows streamed top to bottom by warps.
// A warp owns a 512-column band (16 sites per lane, one 128-bit load and one
// 128-bit store per lane per row) and walks a segment of rows keeping rows
// r-1, r, r+1 in registers, so each source row is read from HBM once. The +-1
// column shifts are byte permutes (PRMT) with the neighbour lane's edge word
// fetched by warp shuffle. The collision LUT is replicated per shared-memory
// bank (lane-private copy: conflict-free LDS), each entry holding the outcome
// for both chiralities; the RNG is evaluated lazily, only for sites whose two
// outcomes differ, from per-column keys precomputed once per step.
#include <cstdio>
#include <type_traits>

#include "fhpg_common.cuh"
#include "fhpg_kernels.cuh"

namespace fhpg {

namespace {

constexpr unsigned kFull = 0xFFFFFFFFu;
constexpr int kFastThreads = 512;   // 16 warps per CTA
constexpr int kWarps = kFastThreads / 32;

__device__ __forceinline__ uint4 ldg128(const uint8_t* p) {
  return __ldg(reinterpret_cast<const uint4*>(p));
}
__device__ __forceinline__ uint32_t ldg32(const uint8_t* p) {
  return __ldg(reinterpret_cast<const uint32_t*>(p));
}
__device__ __forceinline__ void stg128_cs(uint8_t* p, uint4 v) {
  __stcs(reinterpret_cast<uint4*>(p), v);
}

// 0x80 in every byte of t that is nonzero.
__device__ __forceinline__ uint32_t nonzero_bytes(uint32_t t) {
  return (((t & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) | t) & 0x80808080u;
}

// Next-step column keys, spread over every thread of the launch.
__device__ __forceinline__ void column_keys_next(const StepArgs& a) {
  if (!a.zc_next) return;
  const int n = gridDim.x * blockDim.x;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < a.W; i += n) {
    a.zc_next[i] = column_key(a.kc_next, static_cast<uint64_t>(i) + 1);
    if (a.zf_next) a.zf_next[i] = column_key(a.kf_next, static_cast<uint64_t>(i) + 1);
  }
}

// ---------------------------------------------------------------------------
// Generic path: one thread per site, any W >= 1. Used for W % 16 != 0 and as
// an independent cross-check of the fast path.
// ---------------------------------------------------------------------------
template <bool FORCE>
__global__ void __launch_bounds__(256) step_generic_kernel(StepArgs a) {
  __shared__ uint8_t lut[512];
  for (int i = threadIdx.x; i < 512; i += blockDim.x) lut[i] = a.table[i];
  __syncthreads();
  column_keys_next(a);

  const long long nsites = static_cast<long long>(a.row_hi - a.row_lo) * a.W;
  unsigned long long swaps = 0;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < nsites;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int r = a.row_lo + static_cast<int>(i / a.W);
    const int x = static_cast<int>(i % a.W);
    const int q = static_cast<int>((a.row0 + r) & 1);
    const uint8_t* s = a.src + static_cast<long long>(r) * static_cast<long long>(a.pitch);
    const long long p = static_cast<long long>(a.pitch);
    const int xm = x == 0 ? a.W - 1 : x - 1;
    const int xp = x == a.W - 1 ? 0 : x + 1;
    const int xq0 = q ? xp : x;   // x + q
    const int xq1 = q ? x : xm;   // x + q - 1
    uint32_t v = s[x] & (kRestBit | kObstacleBit);  // rest stays; bit 7 = own mask
    v |= s[p + xq0] & 0x01u;   // NW from (x+q, r+1)
    v |= s[p + xq1] & 0x02u;   // NE from (x+q-1, r+1)
    v |= s[xm] & 0x04u;        // E  from (x-1, r)
    v |= s[-p + xq1] & 0x08u;  // SE from (x+q-1, r-1)
    v |= s[-p + xq0] & 0x10u;  // SW from (x+q, r-1)
    v |= s[xp] & 0x20u;        // W  from (x+1, r)
    const uint64_t y = static_cast<uint64_t>(a.row0 + r);
    uint32_t out = lut[v];
    if (out != lut[256 + v] && fin64_bit0(a.zc[x] + y)) out = lut[256 + v];
    if (FORCE && !(out & 0x80u) && (out & 0x20u) && !(out & 0x04u)) {
      if ((fin64(a.zf[x] + y) >> 32) < a.thr) {
        out ^= 0x24u;
        ++swaps;
      }
    }
    a.dst[static_cast<long long>(r) * p + x] = static_cast<uint8_t>(out);
  }
  if (FORCE) {
    for (int o = 16; o; o >>= 1) swaps += __shfl_xor_sync(kFull, swaps, o);
    if ((threadIdx.x & 31) == 0 && swaps) atomicAdd(a.swaps, swaps);
  }
}

// ---------------------------------------------------------------------------
// Fast path.
// ---------------------------------------------------------------------------
struct RawRow {
  uint4 v;     // 16 sites of this lane
  uint32_t e;  // lane 0: word left of the band; last lane: word right of it
};

struct Row {
  uint32_t w[4];
  uint32_t L;  // word whose top byte is column x0-1
  uint32_t R;  // word whose low byte is column x0+16
};

struct Lane {
  int lane, last, x0;
  bool active;
  int W;
  int eoff;  // byte offset of the edge word this lane loads (lane 0 / last)
};

__device__ __forceinline__ RawRow load_raw(const uint8_t* rowp, const Lane& ln) {
  RawRow r;
  r.v = ln.active ? ldg128(rowp + ln.x0) : make_uint4(0, 0, 0, 0);
  r.e = (ln.lane == 0 || ln.lane == ln.last) ? ldg32(rowp + ln.eoff) : 0u;
  return r;
}

__device__ __forceinline__ Row finish_row(const RawRow& r, const Lane& ln) {
  Row o;
  o.w[0] = r.v.x;
  o.w[1] = r.v.y;
  o.w[2] = r.v.z;
  o.w[3] = r.v.w;
  const uint32_t up = __shfl_up_sync(kFull, r.v.w, 1);
  const uint32_t dn = __shfl_down_sync(kFull, r.v.x, 1);
  o.L = ln.lane == 0 ? r.e : up;
  o.R = ln.lane == ln.last ? r.e : dn;
  return o;
}

// Value of column x-1 at every byte of word j.
__device__ __forceinline__ uint32_t shl1(const Row& r, int j) {
  return __byte_perm(j == 0 ? r.L : r.w[j - 1], r.w[j], 0x6543);
}
// Value of column x+1 at every byte of word j.
__device__ __forceinline__ uint32_t shr1(const Row& r, int j) {
  return __byte_perm(r.w[j], j == 3 ? r.R : r.w[j + 1], 0x4321);
}

// One destination row: motion (pull) + collision + forcing. Q = row parity.
template <int Q, bool FORCE>
__device__ __forceinline__ uint4 site_update(const Row& P, const Row& C, const Row& N,
                                             const uint32_t* __restrict__ lut_lane,
                                             const Lane& ln, uint64_t y,
                                             const uint64_t* __restrict__ zc,
                                             const uint64_t* __restrict__ zf, uint64_t thr,
                                             unsigned& swaps) {
  uint32_t out0[4], dep[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    // Pull sources (backends.cpp:64-73): k0 (x+q, r+1), k1 (x+q-1, r+1),
    // k2 (x-1, r), k3 (x+q-1, r-1), k4 (x+q, r-1), k5 (x+1, r).
    const uint32_t n0 = Q ? shr1(N, j) : N.w[j];
    const uint32_t n1 = Q ? N.w[j] : shl1(N, j);
    const uint32_t p3 = Q ? P.w[j] : shl1(P, j);
    const uint32_t p4 = Q ? shr1(P, j) : P.w[j];
    uint32_t m = C.w[j] & 0xC0C0C0C0u;  // rest bit stays, bit 7 = own obstacle
    m |= n0 & 0x01010101u;
    m |= n1 & 0x02020202u;
    m |= shl1(C, j) & 0x04040404u;
    m |= p3 & 0x08080808u;
    m |= p4 & 0x10101010u;
    m |= shr1(C, j) & 0x20202020u;
    // LUT: entry (state << 5) of the lane's private copy = out(ch0) | out(ch1) << 8.
    const uint32_t v0 = lut_lane[(m & 0xFFu) << 5];
    const uint32_t v1 = lut_lane[((m >> 8) & 0xFFu) << 5];
    const uint32_t v2 = lut_lane[((m >> 16) & 0xFFu) << 5];
    const uint32_t v3 = lut_lane[(m >> 24) << 5];
    const uint32_t A = __byte_perm(v0, v1, 0x5140);
    const uint32_t B = __byte_perm(v2, v3, 0x5140);
    out0[j] = __byte_perm(A, B, 0x5410);
    dep[j] = out0[j] ^ __byte_perm(A, B, 0x7632);
  }
  // Chirality: only where the two outcomes differ (rng.hpp:25-33 keyed by the
  // 1-based storage column and the global row, step.cpp:73-76).
  if ((dep[0] | dep[1] | dep[2] | dep[3]) != 0u) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      uint32_t nz = nonzero_bytes(dep[j]);
      while (nz) {
        const int b = (__ffs(nz) - 1) >> 3;
        nz &= nz - 1;
        if (fin64_bit0(__ldg(zc + ln.x0 + 4 * j + b) + y))
          out0[j] ^= dep[j] & (0xFFu << (8 * b));
      }
    }
  }
  // Forcing on the post-collision state (step.cpp:79-88): fluid, W set, E clear.
  if (FORCE) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint32_t f = out0[j];
      uint32_t el = (f >> 5) & ~(f >> 2) & ~(f >> 7) & 0x01010101u;
      while (el) {
        const int b = (__ffs(el) - 1) >> 3;
        el &= el - 1;
        if ((fin64(__ldg(zf + ln.x0 + 4 * j + b) + y) >> 32) < thr) {
          out0[j] ^= 0x24u << (8 * b);
          ++swaps;
        }
      }
    }
  }
  return make_uint4(out0[0], out0[1], out0[2], out0[3]);
}

template <bool FORCE>
__global__ void __launch_bounds__(kFastThreads, 2) step_fast_kernel(StepArgs a) {
  __shared__ uint32_t lut[256 * 32];
  // Lane-replicated LUT: word (e*32 + lane) holds both chirality outcomes of
  // state e, so lane l always hits bank l.
  for (int i = threadIdx.x; i < 256 * 32; i += blockDim.x) {
    const int e = i >> 5;
    lut[i] = static_cast<uint32_t>(a.table[e]) | (static_cast<uint32_t>(a.table[256 + e]) << 8);
  }
  __syncthreads();
  column_keys_next(a);

  const int warp = threadIdx.x >> 5;
  const long long task = static_cast<long long>(blockIdx.x) * kWarps + warp;
  const int band = static_cast<int>(task % a.nbands);
  const int seg = static_cast<int>(task / a.nbands);
  const int r_begin = a.row_lo + seg * a.seg_rows;
  if (r_begin >= a.row_hi) return;  // whole warp
  const int r_end = min(a.row_hi, r_begin + a.seg_rows);

  Lane ln;
  ln.lane = threadIdx.x & 31;
  ln.W = a.W;
  const int band_x = band * 512;
  ln.x0 = band_x + ln.lane * 16;
  ln.active = ln.x0 < a.W;
  ln.last = min(31, (a.W - band_x) / 16 - 1);
  ln.eoff = ln.lane == 0 ? (ln.x0 == 0 ? a.W - 4 : ln.x0 - 4)
                         : (ln.x0 + 16 == a.W ? 0 : ln.x0 + 16);
  const uint32_t* lut_lane = lut + ln.lane;
  const long long pitch = static_cast<long long>(a.pitch);
  const uint8_t* src = a.src;

  unsigned swaps = 0;
  // Window: P = row r-1, C = row r; prefetch ring q1 = r+1, q2 = r+2.
  Row P = finish_row(load_raw(src + (r_begin - 1) * pitch, ln), ln);
  Row C = finish_row(load_raw(src + r_begin * pitch, ln), ln);
  RawRow q1 = load_raw(src + (r_begin + 1) * pitch, ln);
  RawRow q2 = (r_begin + 2 <= r_end) ? load_raw(src + (r_begin + 2) * pitch, ln) : RawRow{};

  auto advance_row = [&](int r, auto parity) {
    constexpr int Q = decltype(parity)::value;
    const Row N = finish_row(q1, ln);
    q1 = q2;
    if (r + 3 <= r_end) q2 = load_raw(src + (r + 3) * pitch, ln);
    const uint4 o = site_update<Q, FORCE>(P, C, N, lut_lane, ln,
                                          static_cast<uint64_t>(a.row0 + r), a.zc, a.zf,
                                          a.thr, swaps);
    if (ln.active) stg128_cs(a.dst + r * pitch + ln.x0, o);
    P = C;
    C = N;
  };
  using Even = std::integral_constant<int, 0>;
  using Odd = std::integral_constant<int, 1>;

  int r = r_begin;
  if (((a.row0 + r) & 1) && r < r_end) advance_row(r++, Odd{});
  for (; r + 1 < r_end; r += 2) {
    advance_row(r, Even{});
    advance_row(r + 1, Odd{});
  }
  if (r < r_end) advance_row(r, Even{});

  if (FORCE) {
    unsigned long long s = swaps;
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(kFull, s, o);
    if (ln.lane == 0 && s) atomicAdd(a.swaps, s);
  }
}

__global__ void column_keys_kernel(uint64_t* zc, uint64_t* zf, uint64_t kc, uint64_t kf, int W) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= W) return;
  zc[i] = column_key(kc, static_cast<uint64_t>(i) + 1);
  if (zf) zf[i] = column_key(kf, static_cast<uint64_t>(i) + 1);
}

__global__ void apply_mask_kernel(uint8_t* base, const uint8_t* mask, size_t pitch, int W,
                                  int nrows) {
  const long long n = static_cast<long long>(nrows) * W;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long r = i / W, x = i % W;
    uint8_t* p = base + r * static_cast<long long>(pitch) + x;
    *p = static_cast<uint8_t>((*p & 0x7Fu) | (mask[r * static_cast<long long>(pitch) + x] ? 0x80u : 0u));
  }
}

// lattice.cpp:57-93: walls on global rows 0 and H-1, geometry obstacles, then
// random_fill (lattice.cpp:44-55) of the remaining nodes.
__global__ void init_kernel(uint8_t* base, const uint8_t* mask, size_t pitch, int W, int nrows,
                            long long row0, long long H, uint64_t seed, uint64_t thr,
                            uint64_t kinit) {
  const long long n = static_cast<long long>(nrows) * W;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long r = i / W, x = i % W;
    const long long gr = row0 + r;
    const long long off = r * static_cast<long long>(pitch) + x;
    if (gr == 0 || gr == H - 1 || mask[off]) {
      base[off] = 0x80;
      continue;
    }
    const uint64_t w = fin64(column_key(kinit, static_cast<uint64_t>(x) + 1) +
                             static_cast<uint64_t>(gr));
    uint32_t s = 0;
#pragma unroll
    for (int b = 0; b < 7; ++b)
      if ((mix64(w + static_cast<uint64_t>(b)) >> 32) < thr) s |= 1u << b;
    base[off] = static_cast<uint8_t>(s);
  }
}

// Integer momentum of the moving bits of the four bytes of w, fluid bytes
// only (node_state.hpp:54-74): px = NE+SE-NW-SW + 2(E-W), py = NW+NE-SE-SW.
__device__ __forceinline__ void word_momentum(uint32_t w, int& px, int& py) {
  const uint32_t fluid = ((~w >> 7) & 0x01010101u) * 0xFFu;
  const uint32_t f = w & fluid;
  auto cnt = [&](int bit) { return __popc(f & (0x01010101u << bit)); };
  px = cnt(1) + cnt(3) - cnt(0) - cnt(4) + 2 * (cnt(2) - cnt(5));
  py = cnt(0) + cnt(1) - cnt(3) - cnt(4);
}

__device__ __forceinline__ int byte_popc7(uint32_t b) { return __popc(b & 0x7Fu); }

__device__ __forceinline__ void byte_momentum(uint32_t s, int& px, int& py) {
  if (s & 0x80u) { px = py = 0; return; }
  px = ((s >> 1) & 1) + ((s >> 3) & 1) - (s & 1) - ((s >> 4) & 1) +
       2 * (static_cast<int>((s >> 2) & 1) - static_cast<int>((s >> 5) & 1));
  py = (s & 1) + ((s >> 1) & 1) - ((s >> 3) & 1) - ((s >> 4) & 1);
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}

__global__ void reduce_global_kernel(const uint8_t* base, size_t pitch, int W, int nrows,
                                     long long* acc) {
  long long mass = 0, px = 0, py = 0;
  const long long n = static_cast<long long>(nrows) * W;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long r = i / W, x = i % W;
    const uint32_t s = base[r * static_cast<long long>(pitch) + x];
    mass += byte_popc7(s);
    int a, b;
    byte_momentum(s, a, b);
    px += a;
    py += b;
  }
  mass = warp_sum(mass);
  px = warp_sum(px);
  py = warp_sum(py);
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(reinterpret_cast<unsigned long long*>(acc + 0), static_cast<unsigned long long>(mass));
    atomicAdd(reinterpret_cast<unsigned long long*>(acc + 1), static_cast<unsigned long long>(px));
    atomicAdd(reinterpret_cast<unsigned long long*>(acc + 2), static_cast<unsigned long long>(py));
  }
}

// One thread per (cell, local row inside the cell grid row): sums the B
// columns of one row of one cell, then atomically adds into the cell.
__global__ void reduce_cells_kernel(const uint8_t* base, size_t pitch, int W, int nrows,
                                    long long row0, long long H, int B, int cells_x, int* nodes,
                                    int* particles, long long* pxo, long long* pyo) {
  const long long n = static_cast<long long>(nrows) * cells_x;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long r = i / cells_x;
    const int cx = static_cast<int>(i % cells_x);
    const long long gr = row0 + r;
    if (gr < 1 || gr > H - 2) continue;
    const long long cy = (gr - 1) / B;
    const uint8_t* p = base + r * static_cast<long long>(pitch);
    const int x1 = min(W, (cx + 1) * B);
    int parts = 0, px = 0, py = 0;
    for (int x = cx * B; x < x1; ++x) {
      const uint32_t s = p[x];
      parts += byte_popc7(s);
      int a, b;
      byte_momentum(s, a, b);
      px += a;
      py += b;
    }
    const long long c = cy * cells_x + cx;
    atomicAdd(nodes + c, x1 - cx * B);
    atomicAdd(particles + c, parts);
    atomicAdd(reinterpret_cast<unsigned long long*>(pxo + c), static_cast<unsigned long long>(static_cast<long long>(px)));
    atomicAdd(reinterpret_cast<unsigned long long*>(pyo + c), static_cast<unsigned long long>(static_cast<long long>(py)));
  }
}

// One CTA per owned row.
__global__ void reduce_rows_kernel(const uint8_t* base, size_t pitch, int W, int nrows,
                                   long long row0, long long H, long long* pxo, int* fluido) {
  const int r = blockIdx.x;
  const long long gr = row0 + r;
  if (gr < 1 || gr > H - 2) return;
  const uint8_t* p = base + static_cast<long long>(r) * static_cast<long long>(pitch);
  long long px = 0;
  int fluid = 0;
  for (int x = threadIdx.x; x < W; x += blockDim.x) {
    const uint32_t s = p[x];
    if (s & 0x80u) continue;
    ++fluid;
    int a, b;
    byte_momentum(s, a, b);
    px += a;
  }
  __shared__ long long spx[32];
  __shared__ int sfl[32];
  px = warp_sum(px);
  fluid = warp_sum(fluid);
  if ((threadIdx.x & 31) == 0) {
    spx[threadIdx.x >> 5] = px;
    sfl[threadIdx.x >> 5] = fluid;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (blockDim.x + 31) / 32; ++w) {
      px += spx[w];
      fluid += sfl[w];
    }
    pxo[gr - 1] = px;
    fluido[gr - 1] = fluid;
  }
}

int grid_for(long long n, int threads, int num_sms) {
  long long g = (n + threads - 1) / threads;
  const long long cap = static_cast<long long>(num_sms) * 32;
  if (g > cap) g = cap;
  return static_cast<int>(g < 1 ? 1 : g);
}

}  // namespace

bool fast_path_ok(int W) { return W >= 32 && W % 16 == 0 && W % 512 != 16; }

int launch_step(const StepArgs& a0, int num_sms, cudaStream_t st, bool force_generic) {
  StepArgs a = a0;
  const int rows = a.row_hi - a.row_lo;
  if (rows <= 0) return 0;
  const bool force = a.thr != 0;
  if (force_generic || !fast_path_ok(a.W)) {
    const int g = grid_for(static_cast<long long>(rows) * a.W, 256, num_sms);
    if (force) step_generic_kernel<true><<<g, 256, 0, st>>>(a);
    else step_generic_kernel<false><<<g, 256, 0, st>>>(a);
    return 1;
  }
  // Fast path: warp tasks = (band, row segment). Size the segments so that
  // one wave of resident warps covers the strip (2 CTAs x 16 warps per SM).
  a.nbands = (a.W + 511) / 512;
  const long long slots = static_cast<long long>(num_sms) * 2 * kWarps;
  long long nseg = (slots + a.nbands - 1) / a.nbands;
  int seg = static_cast<int>((rows + nseg - 1) / nseg);
  if (seg < 16) seg = 16;
  a.seg_rows = seg;
  nseg = (rows + seg - 1) / seg;
  const long long tasks = nseg * a.nbands;
  const int grid = static_cast<int>((tasks + kWarps - 1) / kWarps);
  if (force) step_fast_kernel<true><<<grid, kFastThreads, 0, st>>>(a);
  else step_fast_kernel<false><<<grid, kFastThreads, 0, st>>>(a);
  return 1;
}

void launch_column_keys(uint64_t* zc, uint64_t* zf, uint64_t kc, uint64_t kf, int W,
                        cudaStream_t st) {
  column_keys_kernel<<<(W + 255) / 256, 256, 0, st>>>(zc, zf, kc, kf, W);
}

void launch_apply_mask(uint8_t* base, const uint8_t* mask, size_t pitch, int W, int nrows,
                       cudaStream_t st) {
  apply_mask_kernel<<<grid_for(static_cast<long long>(nrows) * W, 256, 148), 256, 0, st>>>(
      base, mask, pitch, W, nrows);
}

void launch_init(uint8_t* base, const uint8_t* mask, size_t pitch, int W, int nrows,
                 long long row0, long long H, uint64_t seed, uint64_t thr, cudaStream_t st) {
  const uint64_t kinit = step_key(seed, kInit, 0);
  init_kernel<<<grid_for(static_cast<long long>(nrows) * W, 256, 148), 256, 0, st>>>(
      base, mask, pitch, W, nrows, row0, H, seed, thr, kinit);
}

void launch_reduce_global(const uint8_t* base, size_t pitch, int W, int nrows, long long* acc,
                          cudaStream_t st) {
  reduce_global_kernel<<<grid_for(static_cast<long long>(nrows) * W, 256, 148), 256, 0, st>>>(
      base, pitch, W, nrows, acc);
}

void launch_reduce_cells(const uint8_t* base, size_t pitch, int W, int nrows, long long row0,
                         long long H, int B, int* nodes, int* particles, long long* px,
                         long long* py, cudaStream_t st) {
  const int cells_x = (W + B - 1) / B;
  reduce_cells_kernel<<<grid_for(static_cast<long long>(nrows) * cells_x, 256, 148), 256, 0,
                        st>>>(base, pitch, W, nrows, row0, H, B, cells_x, nodes, particles, px,
                              py);
}

void launch_reduce_rows(const uint8_t* base, size_t pitch, int W, int nrows, long long row0,
                        long long H, long long* px, int* fluid, cudaStream_t st) {
  if (nrows <= 0) return;
  reduce_rows_kernel<<<nrows, 256, 0, st>>>(base, pitch, W, nrows, row0, H, px, fluid);
}

}  // namespace fhpg
