// Memory-pipeline calibration for the step kernel (timing tool, not product):
// what the B200 sustains for the bit-plane lattice's traffic pattern with
// plain vectorized loads / stores and no compute.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/membw tools/membw.cu
//   ./tools/membw [W] [H]
// Kernels (all over the engine's plane layout: H+2 rows x 8 planes x
// (W/32 + 8) words, two buffers):
//   copy    : every byte of buffer A -> buffer B (torch copy_-like)
//   planes  : read the 8 planes of each row, write 7 (the step's traffic)
//   readonly: read the 8 planes (sum into a register)
//   writeonly: write 7 planes
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  printf("%s: %s\n", #x, cudaGetErrorString(e_)); exit(1); } } while (0)

__global__ void copy_k(const uint4* __restrict__ a, uint4* __restrict__ b, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    b[i] = a[i];
}

// row = 8 planes x pw words; write planes 0..6 (each plane pw words = pw/4 uint4).
__global__ void planes_k(const uint4* __restrict__ a, uint4* __restrict__ b, int rows, int pw4) {
  const size_t row_v = 8 * (size_t)pw4;
  const size_t n = (size_t)rows * row_v;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const size_t in_row = i % row_v;
    const uint4 v = a[i];
    if (in_row < 7 * (size_t)pw4) b[i] = make_uint4(v.x ^ 1, v.y, v.z, v.w);
  }
}

__global__ void read_k(const uint4* __restrict__ a, unsigned* out, size_t n) {
  unsigned acc = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const uint4 v = a[i];
    acc ^= v.x ^ v.y ^ v.z ^ v.w;
  }
  if (acc == 0x12345678u) *out = acc;
}

__global__ void write_k(uint4* __restrict__ b, int rows, int pw4) {
  const size_t row_v = 8 * (size_t)pw4;
  const size_t n = (size_t)rows * row_v;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    if (i % row_v < 7 * (size_t)pw4) b[i] = make_uint4((unsigned)i, 0, 0, 0);
}

template <typename F>
float best_ms(F f, int reps = 20) {
  cudaEvent_t s, e;
  CK(cudaEventCreate(&s));
  CK(cudaEventCreate(&e));
  float best = 1e30f;
  for (int r = 0; r < reps + 3; ++r) {
    CK(cudaEventRecord(s));
    f();
    CK(cudaEventRecord(e));
    CK(cudaEventSynchronize(e));
    float ms;
    CK(cudaEventElapsedTime(&ms, s, e));
    if (r >= 3 && ms < best) best = ms;
  }
  return best;
}

int main(int argc, char** argv) {
  const int W = argc > 1 ? atoi(argv[1]) : 16384;
  const int H = argc > 2 ? atoi(argv[2]) : 16384;
  const int pw = W / 32 + 8, pw4 = pw / 4;
  const int rows = H + 2;
  const size_t bytes = (size_t)rows * 8 * pw * 4;
  const double sites = (double)W * H;
  uint4 *a, *b;
  unsigned* out;
  CK(cudaMalloc(&a, bytes));
  CK(cudaMalloc(&b, bytes));
  CK(cudaMalloc(&out, 4));
  CK(cudaMemset(a, 1, bytes));
  CK(cudaMemset(b, 2, bytes));
  int sms;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const size_t n = bytes / 16;
  printf("{\"W\": %d, \"H\": %d, \"buffer_bytes\": %zu, \"sms\": %d", W, H, bytes, sms);
  for (int bpsm : {4, 8, 16}) {
    const int grid = sms * bpsm, block = 256;
    float ms = best_ms([&] { copy_k<<<grid, block>>>(a, b, n); });
    printf(", \"copy_b%d_gbs\": %.1f", bpsm, 2.0 * bytes / ms / 1e6);
    ms = best_ms([&] { planes_k<<<grid, block>>>(a, b, rows, pw4); });
    printf(", \"planes_b%d_gbs\": %.1f, \"planes_b%d_gsups_eq\": %.1f", bpsm, 15.0 / 16 * 2.0 * bytes / ms / 1e6,
           bpsm, sites / ms / 1e6);
    ms = best_ms([&] { read_k<<<grid, block>>>(a, out, n); });
    printf(", \"read_b%d_gbs\": %.1f", bpsm, 1.0 * bytes / ms / 1e6);
    ms = best_ms([&] { write_k<<<grid, block>>>(b, rows, pw4); });
    printf(", \"write7_b%d_gbs\": %.1f", bpsm, 7.0 / 8 * bytes / ms / 1e6);
  }
  CK(cudaGetLastError());
  printf("}\n");
  return 0;
}
