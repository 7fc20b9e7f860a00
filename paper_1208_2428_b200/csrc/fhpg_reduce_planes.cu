// fhpg_reduce_planes.cu — the integer observables straight from the bit-plane
// lattice (no unpack): total_mass / total_momentum (observables.cpp:27-47),
// coarse_grain's per-cell integer sums (observables.cpp:49-82) and
// velocity_profile's per-row sums (observables.cpp:84-102).
//
// Plane layout (fhpg_step_planes.cu): row r of a buffer starts at
// base + r * pitch; plane p of it holds W/32 words after 4 pad words, plane
// stride PW = W/32 + 8 words; bit j of word i = column 32 i + j. Per word of
// 32 sites: mass = sum of popc over planes 0-6 (every node, obstacles
// included), momentum over the fluid sites (plane 7 clear) with
// kDirectionMomentum (node_state.hpp:54-61): NW (-1,1), NE (1,1), E (2,0),
// SE (1,-1), SW (-1,-1), W (-2,0). Each kernel reads the 8 plane words of a
// site word once: 1 byte per site, the HBM roofline of an observable.
#include <cstdint>

#include "fhpg_kernels.cuh"

namespace fhpg {
namespace {

constexpr unsigned kFull = 0xFFFFFFFFu;

struct WordSums {
  int mass, px, py, fluid;
};

// Sums of 32 sites (the bits of `sel`) of one row: w[p] = plane p's word.
__device__ __forceinline__ WordSums word_sums(const uint32_t (&w)[8], uint32_t sel) {
  const uint32_t fl = ~w[7] & sel;
  WordSums s;
  s.mass = 0;
#pragma unroll
  for (int p = 0; p < 7; ++p) s.mass += __popc(w[p] & sel);
  const int nw = __popc(w[0] & fl), ne = __popc(w[1] & fl), e = __popc(w[2] & fl);
  const int se = __popc(w[3] & fl), sw = __popc(w[4] & fl), ww = __popc(w[5] & fl);
  s.px = ne + se - nw - sw + 2 * (e - ww);
  s.py = nw + ne - se - sw;
  s.fluid = __popc(fl);
  return s;
}

__device__ __forceinline__ void load_word(const uint8_t* base, size_t pitch, int PW, long long r,
                                          int i, uint32_t (&w)[8]) {
  const uint32_t* row = reinterpret_cast<const uint32_t*>(base + r * static_cast<long long>(pitch));
#pragma unroll
  for (int p = 0; p < 8; ++p) w[p] = __ldcs(row + p * PW + kPlaneLead + i);
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}

__global__ void reduce_global_planes_kernel(const uint8_t* base, size_t pitch, int W, int nrows,
                                            long long* acc) {
  const int WW = W >> 5, PW = plane_stride_words(W);
  const long long n = static_cast<long long>(nrows) * WW;
  long long mass = 0, px = 0, py = 0;
  for (long long t = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; t < n;
       t += static_cast<long long>(gridDim.x) * blockDim.x) {
    uint32_t w[8];
    load_word(base, pitch, PW, t / WW, static_cast<int>(t % WW), w);
    const WordSums s = word_sums(w, kFull);
    mass += s.mass;
    px += s.px;
    py += s.py;
  }
  __shared__ long long red[3][32];
  mass = warp_sum(mass);
  px = warp_sum(px);
  py = warp_sum(py);
  const int wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    red[0][wid] = mass;
    red[1][wid] = px;
    red[2][wid] = py;
  }
  __syncthreads();
  if (threadIdx.x < 3) {
    long long v = 0;
    for (int k = 0; k < nw; ++k) v += red[threadIdx.x][k];
    atomicAdd(reinterpret_cast<unsigned long long*>(acc + threadIdx.x),
              static_cast<unsigned long long>(v));
  }
}

// One CTA per owned interior row: (sum px over fluid sites, fluid count).
__global__ void reduce_rows_planes_kernel(const uint8_t* base, size_t pitch, int W, int nrows,
                                          long long row0, long long H, long long* pxo,
                                          int* fluido) {
  const int r = blockIdx.x;
  const long long gr = row0 + r;
  if (gr < 1 || gr > H - 2) return;
  const int WW = W >> 5, PW = plane_stride_words(W);
  long long px = 0;
  int fluid = 0;
  for (int i = threadIdx.x; i < WW; i += blockDim.x) {
    uint32_t w[8];
    load_word(base, pitch, PW, r, i, w);
    const WordSums s = word_sums(w, kFull);
    px += s.px;
    fluid += s.fluid;
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
    for (int k = 1; k < static_cast<int>(blockDim.x >> 5); ++k) {
      px += spx[k];
      fluid += sfl[k];
    }
    pxo[gr - 1] = px;
    fluido[gr - 1] = fluid;
  }
}

// One thread per (cell row, word column): the B (or fewer, at the strip and
// lattice edges) rows of the cell row that this strip owns, every cell the
// word's 32 columns touch. A cell lies inside one word and one strip when B
// divides 32 and the strip holds the whole cell row: the thread is its only
// contributor and stores; otherwise it adds atomically (the arrays start at 0).
__global__ void reduce_cells_planes_kernel(const uint8_t* base, size_t pitch, int W, int nrows,
                                           long long row0, long long H, int B, int cells_x,
                                           int cy0, int ncy, int* nodes, int* particles,
                                           long long* pxo, long long* pyo) {
  const int WW = W >> 5, PW = plane_stride_words(W);
  const long long n = static_cast<long long>(ncy) * WW;
  for (long long t = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; t < n;
       t += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int cy = cy0 + static_cast<int>(t / WW);
    const int i = static_cast<int>(t % WW);
    // global rows of the cell row, clipped to the interior and to this strip
    const long long g0 = 1 + static_cast<long long>(cy) * B;
    const long long g1 = min(g0 + B, H - 1);
    const long long a = max(g0, row0), b = min(g1, row0 + nrows);
    if (a >= b) continue;
    const bool whole_rows = a == g0 && b == g1;
    const int x0 = 32 * i, x1 = min(W, x0 + 32);
    for (int cx = x0 / B; cx * B < x1; ++cx) {
      const int c0 = max(cx * B, x0), c1 = min(min((cx + 1) * B, W), x1);
      const uint32_t sel = (c1 - c0 == 32 ? kFull : ((1u << (c1 - c0)) - 1u)) << (c0 - x0);
      int parts = 0, px = 0, py = 0;
      for (long long g = a; g < b; ++g) {
        uint32_t w[8];
        load_word(base, pitch, PW, g - row0, i, w);
        const WordSums s = word_sums(w, sel);
        parts += s.mass;
        px += s.px;
        py += s.py;
      }
      const long long c = static_cast<long long>(cy) * cells_x + cx;
      const int cnt = static_cast<int>(b - a) * (c1 - c0);
      const bool own = whole_rows && cx * B >= x0 && min((cx + 1) * B, W) <= x1;
      if (own) {
        nodes[c] = cnt;
        particles[c] = parts;
        pxo[c] = px;
        pyo[c] = py;
      } else {
        atomicAdd(nodes + c, cnt);
        atomicAdd(particles + c, parts);
        atomicAdd(reinterpret_cast<unsigned long long*>(pxo + c),
                  static_cast<unsigned long long>(static_cast<long long>(px)));
        atomicAdd(reinterpret_cast<unsigned long long*>(pyo + c),
                  static_cast<unsigned long long>(static_cast<long long>(py)));
      }
    }
  }
}

int grid_cap(long long n, int threads, int num_sms, int per_sm) {
  long long g = (n + threads - 1) / threads;
  const long long cap = static_cast<long long>(num_sms) * per_sm;
  if (g > cap) g = cap;
  return static_cast<int>(g < 1 ? 1 : g);
}

}  // namespace

void launch_reduce_global_planes(const uint8_t* base, size_t pitch, int W, int nrows,
                                 long long* acc, int num_sms, cudaStream_t st) {
  const long long n = static_cast<long long>(nrows) * (W >> 5);
  reduce_global_planes_kernel<<<grid_cap(n, 256, num_sms, 8), 256, 0, st>>>(base, pitch, W, nrows,
                                                                            acc);
}

void launch_reduce_rows_planes(const uint8_t* base, size_t pitch, int W, int nrows, long long row0,
                               long long H, long long* px, int* fluid, cudaStream_t st) {
  if (nrows <= 0) return;
  reduce_rows_planes_kernel<<<nrows, 128, 0, st>>>(base, pitch, W, nrows, row0, H, px, fluid);
}

void launch_reduce_cells_planes(const uint8_t* base, size_t pitch, int W, int nrows,
                                long long row0, long long H, int B, int* nodes, int* particles,
                                long long* px, long long* py, int num_sms, cudaStream_t st) {
  const int cells_x = (W + B - 1) / B;
  // cell rows this strip touches (interior rows 1..H-2 only)
  const long long lo = row0 < 1 ? 1 : row0;
  const long long hi = (row0 + nrows < H - 1 ? row0 + nrows : H - 1);
  if (hi <= lo) return;
  const int cy0 = static_cast<int>((lo - 1) / B), cy1 = static_cast<int>((hi - 2) / B);
  const int ncy = cy1 - cy0 + 1;
  const long long n = static_cast<long long>(ncy) * (W >> 5);
  reduce_cells_planes_kernel<<<grid_cap(n, 128, num_sms, 16), 128, 0, st>>>(
      base, pitch, W, nrows, row0, H, B, cells_x, cy0, ncy, nodes, particles, px, py);
}

}  // namespace fhpg
