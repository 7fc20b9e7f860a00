// Store-path calibration for the step kernel's output (timing tool, not
// product): one step's worth of output rows of the bit-plane layout (16384
// rows x 8 bands x 7 planes x 256 B, plane rows at 2304-byte stride, row
// pitch 18432 B) written by 148 CTAs x 31 warps, each warp staging in shared
// memory and storing row after row (waiting for the previous store's smem
// read before re-staging, as the ring kernel does). Variants:
//   0: one 3D TMA tensor store per row, box {64 words, 7 planes, 1 row} (the kernel)
//   1: seven 2D TMA stores per row, box {64 words, 1 plane}
//   2: seven 1D bulk copies (cp.async.bulk.global.shared::cta) of 256 B
//   3: one 1D bulk copy of 1792 contiguous bytes (a band-major layout)
//   4: one 3D TMA store per two rows, box {64, 7, 2}
//   5: direct st.global.v2 from registers (no staging)
//   6: one 3D TMA store per row, no wait before re-staging (upper bound)
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tma_store_bench tools/tma_store_bench.cu -lcuda
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  printf("%s: %s\n", #x, cudaGetErrorString(e_)); exit(1); } } while (0)

constexpr int kRows = 16384, kBands = 8, kBandWords = 64, kPW = 576, kCons = 31;
constexpr size_t kPitch = 8ull * kPW * 4;  // 18432

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

template <int V>
__global__ void __launch_bounds__(kCons * 32, 1)
    store_k(const __grid_constant__ CUtensorMap m7, const __grid_constant__ CUtensorMap m1,
            const __grid_constant__ CUtensorMap m72, uint8_t* out, int rows_per_cta, int drift) {
  extern __shared__ __align__(128) uint8_t smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t stage = smem_u32(smem) + warp * 3584;
  const int band = blockIdx.x % kBands;
  const int seg = blockIdx.x / kBands;
  const int r0 = seg * rows_per_cta, r1 = min(kRows, r0 + rows_per_cta);
  const int step = V == 4 ? 2 : 1;
  // drift: band b starts b * drift rows later in its segment (wrapping), so
  // the 8 bands of a row are written at different times.
  const int span = r1 - r0;
  for (int t = warp * step; t < span; t += kCons * step) {
    const int r = r0 + (t + band * drift) % span;
    const uint32_t v0 = r * 7 + lane, v1 = r ^ lane;
    if (V == 5) {
      uint8_t* row = out + static_cast<size_t>(r) * kPitch + (32 + band * kBandWords + lane * 2) * 4;
      for (int p = 0; p < 7; ++p)
        asm volatile("st.global.v2.u32 [%0], {%1,%2};" ::"l"(row + p * kPW * 4), "r"(v0 + p), "r"(v1)
                     : "memory");
      continue;
    }
    if (V != 6 && lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    __syncwarp();
    for (int q = 0; q < (V == 4 ? 2 : 1); ++q)
      for (int p = 0; p < 7; ++p)
        asm volatile("st.shared.v2.u32 [%0], {%1,%2};" ::"r"(stage + q * 1792 + p * 256 + lane * 8),
                     "r"(v0 + p), "r"(v1));
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    if (lane == 0) {
      const int word = 32 + band * kBandWords;
      if (V == 0 || V == 6) {
        asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.tile.bulk_group [%0, {%1, %2, %3}], [%4];"
                     ::"l"(&m7), "r"(word), "r"(0), "r"(r), "r"(stage) : "memory");
      } else if (V == 1) {
        for (int p = 0; p < 7; ++p)
          asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.tile.bulk_group [%0, {%1, %2, %3}], [%4];"
                       ::"l"(&m1), "r"(word), "r"(p), "r"(r), "r"(stage + p * 256) : "memory");
      } else if (V == 2) {
        for (int p = 0; p < 7; ++p) {
          uint8_t* g = out + static_cast<size_t>(r) * kPitch + (static_cast<size_t>(p) * kPW + word) * 4;
          asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], 256;"
                       ::"l"(g), "r"(stage + p * 256) : "memory");
        }
      } else if (V == 3) {
        uint8_t* g = out + static_cast<size_t>(r) * kPitch + static_cast<size_t>(band) * 2048;
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], 1792;"
                     ::"l"(g), "r"(stage) : "memory");
      } else if (V == 4) {
        asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.tile.bulk_group [%0, {%1, %2, %3}], [%4];"
                     ::"l"(&m72), "r"(word), "r"(0), "r"(r), "r"(stage) : "memory");
      }
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
  }
  if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

static PFN_cuTensorMapEncodeTiled encode_fn() {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
  return reinterpret_cast<PFN_cuTensorMapEncodeTiled>(fn);
}

static CUtensorMap make_map(void* base, unsigned planes, unsigned rows_box) {
  CUtensorMap m;
  const cuuint64_t dims[3] = {kPW, 8, kRows};
  const cuuint64_t strides[2] = {kPW * 4, kPitch};
  const cuuint32_t box[3] = {kBandWords, planes, rows_box};
  const cuuint32_t es[3] = {1, 1, 1};
  if (encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_UINT32, 3, base, dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
    printf("encode failed\n");
    exit(1);
  }
  return m;
}

template <int V>
static void run(const CUtensorMap& m7, const CUtensorMap& m1, const CUtensorMap& m72, uint8_t* out,
                int sms, const char* name, int drift = 0) {
  const int segs = sms / kBands;
  const int rows_per_cta = (kRows + segs - 1) / segs;
  const int grid = kBands * segs;
  const int smem = kCons * 3584;
  CK(cudaFuncSetAttribute(store_k<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  for (int i = 0; i < 3; ++i) store_k<V><<<grid, kCons * 32, smem>>>(m7, m1, m72, out, rows_per_cta, drift);
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  const int reps = 20;
  CK(cudaEventRecord(a));
  for (int i = 0; i < reps; ++i) store_k<V><<<grid, kCons * 32, smem>>>(m7, m1, m72, out, rows_per_cta, drift);
  CK(cudaEventRecord(b));
  CK(cudaEventSynchronize(b));
  float ms = 0;
  CK(cudaEventElapsedTime(&ms, a, b));
  const double bytes = static_cast<double>(kRows) * kBands * 1792;
  printf("%s drift %3d: %.1f us per step-store, %.0f GB/s, %.0f GSUPS-equivalent store ceiling\n", name,
         drift, 1e3 * ms / reps, bytes / (ms / reps * 1e-3) / 1e9,
         static_cast<double>(kRows) * 16384 / (ms / reps * 1e-3) / 1e9);
}

int main() {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  uint8_t* out = nullptr;
  CK(cudaMalloc(&out, kPitch * (kRows + 2)));
  const CUtensorMap m7 = make_map(out, 7, 1), m1 = make_map(out, 1, 1), m72 = make_map(out, 7, 2);
  run<0>(m7, m1, m72, out, sms, "tma3d box{64,7,1}        ");
  run<1>(m7, m1, m72, out, sms, "tma3d 7 x box{64,1,1}    ");
  run<2>(m7, m1, m72, out, sms, "bulk1d 7 x 256 B         ");
  run<3>(m7, m1, m72, out, sms, "bulk1d 1792 B contiguous ");
  run<4>(m7, m1, m72, out, sms, "tma3d box{64,7,2}        ");
  run<5>(m7, m1, m72, out, sms, "st.global.v2 direct      ");
  run<6>(m7, m1, m72, out, sms, "tma3d box{64,7,1} no wait");
  for (int d : {8, 32, 128, 400}) run<0>(m7, m1, m72, out, sms, "tma3d box{64,7,1}        ", d);
  return 0;
}
