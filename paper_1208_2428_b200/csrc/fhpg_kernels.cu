// fhpg_kernels.cu — sm_100a kernels of the B200 FHP engine.
//
// Hot path: one fused kernel per time step doing, for every site, the
// reference's pull motion (step.cpp:40-61, pull offsets backends.cpp:64-73),
// the 512-entry LUT collision with counter-RNG chirality and the stochastic
// W->E forcing (step.cpp:63-93). Ghost-column sync (lattice.cpp:32-39) is
// replaced by in-kernel periodic wrap; the buffer swap by ping-pong pointers.
//
// The fast path (W % 16 == 0) lives in fhpg_step_fast.cu; this file holds
// the generic one-thread-per-site step, init, mask and reduction kernels.
#include <cstdio>
#include <map>
#include <mutex>
#include <tuple>
#include <type_traits>

#include "fhpg_common.cuh"
#include "fhpg_kernels.cuh"

namespace fhpg {

namespace {

constexpr unsigned kFull = 0xFFFFFFFFu;



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

// SM count of the current device (grid-stride helpers size their grids by
// it), cached per device.
int current_sms() {
  static int cache[64] = {0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 148;
  if (dev >= 0 && dev < 64 && cache[dev]) return cache[dev];
  int n = 0;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n < 1) n = 148;
  if (dev >= 0 && dev < 64) cache[dev] = n;
  return n;
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
  return launch_step_fast(a, num_sms, st);
}

cudaError_t ensure_smem_optin(const void* kernel, int bytes) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, int> done;  // (kernel, device) -> bytes
  int dev = 0;
  cudaError_t err = cudaGetDevice(&dev);
  if (err != cudaSuccess) return err;
  std::lock_guard<std::mutex> lock(mu);
  auto it = done.find({kernel, dev});
  if (it != done.end() && it->second == bytes) return cudaSuccess;
  err = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (err == cudaSuccess) done[{kernel, dev}] = bytes;
  return err;
}

void launch_column_keys(uint64_t* zc, uint64_t* zf, uint64_t kc, uint64_t kf, int W,
                        cudaStream_t st) {
  column_keys_kernel<<<(W + 255) / 256, 256, 0, st>>>(zc, zf, kc, kf, W);
}

void launch_apply_mask(uint8_t* base, const uint8_t* mask, size_t pitch, int W, int nrows,
                       cudaStream_t st) {
  apply_mask_kernel<<<grid_for(static_cast<long long>(nrows) * W, 256, current_sms()), 256, 0, st>>>(
      base, mask, pitch, W, nrows);
}

void launch_init(uint8_t* base, const uint8_t* mask, size_t pitch, int W, int nrows,
                 long long row0, long long H, uint64_t seed, uint64_t thr, cudaStream_t st) {
  const uint64_t kinit = step_key(seed, kInit, 0);
  init_kernel<<<grid_for(static_cast<long long>(nrows) * W, 256, current_sms()), 256, 0, st>>>(
      base, mask, pitch, W, nrows, row0, H, seed, thr, kinit);
}

void launch_reduce_global(const uint8_t* base, size_t pitch, int W, int nrows, long long* acc,
                          cudaStream_t st) {
  reduce_global_kernel<<<grid_for(static_cast<long long>(nrows) * W, 256, current_sms()), 256, 0, st>>>(
      base, pitch, W, nrows, acc);
}

void launch_reduce_cells(const uint8_t* base, size_t pitch, int W, int nrows, long long row0,
                         long long H, int B, int* nodes, int* particles, long long* px,
                         long long* py, cudaStream_t st) {
  const int cells_x = (W + B - 1) / B;
  reduce_cells_kernel<<<grid_for(static_cast<long long>(nrows) * cells_x, 256, current_sms()), 256, 0,
                        st>>>(base, pitch, W, nrows, row0, H, B, cells_x, nodes, particles, px,
                              py);
}

void launch_reduce_rows(const uint8_t* base, size_t pitch, int W, int nrows, long long row0,
                        long long H, long long* px, int* fluid, cudaStream_t st) {
  if (nrows <= 0) return;
  reduce_rows_kernel<<<nrows, 256, 0, st>>>(base, pitch, W, nrows, row0, H, px, fluid);
}

}  // namespace fhpg
