// Integer-pipe throughput microbenchmark ("measure the INT
// peak with a LOP3/IMAD microbenchmark on the box"). Each kernel runs 8
// independent dependency chains per thread of one instruction kind, on every
// SM, and reports warp instructions per clock per SM and lane-ops/s.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o int_peak tools/int_peak.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

#define CHAINS 8
#define ITERS 4096

#define OP_LOOP(BODY)                                        \
  uint32_t v[CHAINS];                                        \
  _Pragma("unroll") for (int c = 0; c < CHAINS; ++c) v[c] = seed + threadIdx.x * 7 + c; \
  const uint32_t b = seed ^ 0x9E3779B9u, d = seed * 3u + 1u; \
  for (int it = 0; it < ITERS; ++it) {                       \
    _Pragma("unroll") for (int c = 0; c < CHAINS; ++c) { BODY; } \
  }                                                          \
  uint32_t acc = 0;                                          \
  _Pragma("unroll") for (int c = 0; c < CHAINS; ++c) acc ^= v[c]; \
  if (acc == 0x12345678u) out[threadIdx.x] = acc;

__global__ void k_lop3(uint32_t seed, uint32_t* out) {
  OP_LOOP(asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(v[c]) : "r"(b), "r"(d)))
}
__global__ void k_iadd3(uint32_t seed, uint32_t* out) {
  OP_LOOP(asm volatile("add.u32 %0, %0, %1;" : "+r"(v[c]) : "r"(b)))
}
__global__ void k_shf(uint32_t seed, uint32_t* out) {
  OP_LOOP(asm volatile("shf.l.wrap.b32 %0, %0, %1, 3;" : "+r"(v[c]) : "r"(b)))
}
__global__ void k_prmt(uint32_t seed, uint32_t* out) {
  OP_LOOP(asm volatile("prmt.b32 %0, %0, %1, 0x3210;" : "+r"(v[c]) : "r"(b)))
}
__global__ void k_imad(uint32_t seed, uint32_t* out) {
  OP_LOOP(asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(v[c]) : "r"(b), "r"(d)))
}
__global__ void k_lop3_imad(uint32_t seed, uint32_t* out) {
  // alternating ALU and FMA-pipe work: do the two pipes issue in parallel?
  OP_LOOP(if (c & 1) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(v[c]) : "r"(b), "r"(d));
          else asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(v[c]) : "r"(b), "r"(d)))
}

typedef void (*Kern)(uint32_t, uint32_t*);

int main() {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  int clk_khz = 0;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  uint32_t* out;
  cudaMalloc(&out, 4096);
  const int threads = 1024, blocks = p.multiProcessorCount * 2;
  struct { const char* name; Kern k; } ks[] = {{"lop3", k_lop3}, {"iadd", k_iadd3}, {"shf", k_shf},
                                              {"prmt", k_prmt}, {"imad", k_imad},
                                              {"lop3+imad", k_lop3_imad}};
  cudaEvent_t a, z;
  cudaEventCreate(&a);
  cudaEventCreate(&z);
  printf("{\"sms\": %d, \"clock_khz_attr\": %d, \"kernels\": {", p.multiProcessorCount, clk_khz);
  for (int i = 0; i < 6; ++i) {
    ks[i].k<<<blocks, threads>>>(1, out);  // warm-up
    cudaEventRecord(a);
    for (int r = 0; r < 5; ++r) ks[i].k<<<blocks, threads>>>(r + 2, out);
    cudaEventRecord(z);
    cudaEventSynchronize(z);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, z);
    const double ops = 5.0 * blocks * threads * (double)ITERS * CHAINS;
    const double lane_ops_s = ops / (ms * 1e-3);
    printf("%s\"%s\": {\"lane_ops_per_s\": %.4e, \"ms\": %.3f}", i ? ", " : "", ks[i].name,
           lane_ops_s, ms);
  }
  printf("}, \"error\": \"%s\"}\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
