// fhpg_kernels.cuh — device kernels of the FHP engine and their host launchers.
#pragma once
#include <cstddef>
#include <cstdint>

#include <cuda_runtime.h>

namespace fhpg {

// Device lattice view of one strip of rows. The buffer holds nrows+4 rows of
// `pitch` bytes: local row -1 (top halo), rows 0..nrows-1 (owned), row nrows
// (bottom halo). Halo rows are zero where the strip touches the global grid
// edge (the reference's "out-of-grid rows contribute nothing", step.cpp:47)
// and hold the neighbour strip's boundary row otherwise; two spare zero rows
// follow the bottom halo so the fast path may prefetch past it. `base` points at
// local row 0, column 0 (reference storage column 1).
struct StepArgs {
  const uint8_t* src;
  uint8_t* dst;
  size_t pitch;
  int W;
  int nrows;
  long long row0;            // global index of local row 0 (row parity, RNG y)
  const uint8_t* table;      // 512-entry collision table (device)
  const uint64_t* zc;        // chirality column keys for this step, index x-1
  const uint64_t* zf;        // forcing column keys for this step (thr > 0)
  uint64_t thr;              // bernoulli threshold, 0 = no forcing
  unsigned long long* swaps; // accumulated accepted forcing swaps
  uint64_t* zc_next;         // column keys of the next step (may be null)
  uint64_t* zf_next;
  uint64_t kc_next, kf_next; // step keys of the next step
  uint64_t kc_cur, kf_cur;   // step keys of this step (ring kernel: column keys made in-kernel)
  // Powers of two passed at run time so that ptxas keeps the byte moves that
  // use them as IMAD / IMAD.HI (FMA pipe) instead of folding them into
  // shifts on the ALU pipe, which the fast path saturates (fast path only).
  uint32_t k1, k2, k4, k16, k32, k256, k2p24;
  int seg_rows;              // rows per warp task (fast path)
  int nbands;                // 512-column bands (fast path)
  int nbands_groups;         // CTA column groups (fast path)
  int bpc, spc;              // bands x segments per CTA (fast path)
  int row_lo, row_hi;        // local row range to update, [row_lo, row_hi)
  int row_lo2 = 0, row_hi2 = 0;  // optional second range (bit-plane path: boundary rows)
  int segs1 = 0;             // row segments of the first range (bit-plane ring kernel)
  int segs2 = 0;             //   ... of the second range
  int extra_rows = 0;        // ring kernel: last rows of every band done by the extra CTAs
  uint32_t span_cap = 0xFFFFFFFFu;  // bit-plane kernels: rows per column-key base (testing aid)
  int rule = 2;              // bit-plane kernels: collision circuit, 2 = FHP-III, 1 = FHP-I,
                             // 0 = DEFAULT (FHPG_RULES_*)
};

// Dynamic shared-memory opt-in of `kernel` on the CURRENT device (the
// attribute is per device: an engine on a second GPU of the same process
// needs its own). Remembered per (kernel, device, bytes); thread-safe.
cudaError_t ensure_smem_optin(const void* kernel, int bytes);

// Fast path launcher (fhpg_step_fast.cu).
int launch_step_fast(const StepArgs& a, int num_sms, cudaStream_t st);

// Kernel selection for a lattice width.
bool fast_path_ok(int W);

// Bit-plane path (fhpg_step_planes.cu): rows hold 8 planes (plane p: bit p
// of every node; bit j of word i = column 32 i + j). A plane row is
// plane_stride_words(W) = W/32 + 64 words: 32 lead words, the W/32 data
// words, 32 trail words. The data starts on a 128-byte line (W % 1024 == 0,
// row pitch planes_row_bytes(W) = W + 2048), so the step kernel's band
// stores are whole lines and never share a sector with another band's. The
// lead words [24, 32) hold the periodic wrap of data words W/32-8 .. W/32-1
// and the trail words [W/32+32, W/32+40) that of data words 0..7 — one
// 32-byte sector each (readers use the inner 4 words).
constexpr int kPlaneLead = 32;
constexpr int kPlaneWrap = 8;
#ifndef FHPG_PLANE_TRAIL
#define FHPG_PLANE_TRAIL 32
#endif
constexpr int kPlaneTrail = FHPG_PLANE_TRAIL;
#if defined(__CUDACC__)
__host__ __device__
#endif
constexpr int plane_stride_words(int W) { return W / 32 + kPlaneLead + kPlaneTrail; }
bool planes_ok(int W);  // W % 1024 == 0
int planes_words_per_lane(int W);
size_t planes_row_bytes(int W);
// TMA descriptors (CUtensorMap, 64-byte aligned, 128 bytes each) of a plane
// buffer whose row 0 is at `buffer` (the top halo row), `rows` rows:
// kMapLoad = row loads (band + 4 edge words on either side, 8 planes),
// kMapStore = band stores (7 planes), kMapLoadRows = FHPG_BOX_ROWS-row loads,
// kMapPad = periodic-wrap sector stores (kPlaneWrap words, 7 planes; the
// per-warp kernel), kMapSide = 4 words x 8 planes x FHPG_BOX_ROWS rows (the
// ring kernel's edge bands load the wrap words instead of storing sectors).
constexpr int kMapLoad = 0, kMapStore = 1, kMapLoadRows = 2, kMapPad = 3, kMapSide = 4;
constexpr int kPlaneMaps = 5;
bool make_planes_map(void* tmap, uint8_t* buffer, int W, size_t pitch, int rows, int kind);
// One time step with a collision circuit (a.rule) over rows [row_lo, row_hi)
// (and the optional second range): loads through the source buffer's maps,
// stores through the destination buffer's (src_maps / dst_maps: the
// kPlaneMaps descriptors of each buffer, in kind order).
int launch_step_planes(const StepArgs& a, const void* src_maps, const void* dst_maps,
                       int num_sms, cudaStream_t st);
// Small whole lattices (fhpg_step_resident.cu): the depth (steps per grid
// barrier) the shared-memory-resident kernel would use for W x H, or 0 when
// the lattice is not eligible (W % 1024, too large, shared memory).
int resident_plan(int W, int H, uint64_t thr, int num_sms, int* rows_per_cta, int* grid);
// `count` steps from global step `first` of a whole plane lattice held in
// g[cur] in ONE cooperative launch; returns the number of buffer flips (the
// state ends in g[cur ^ (flips & 1)]). `bar`: 2 zeroed words of device memory.
int launch_step_resident(uint8_t* const g[2], int cur, size_t pitch, int W, int H, int rule,
                         uint64_t seed, uint64_t thr, long long first, long long count,
                         unsigned long long* swaps, unsigned* bar, int num_sms, cudaStream_t st,
                         cudaError_t* err);

// Bytes (rows 0..nrows-1 of src) -> planes in dst; plane 7 from the mask,
// also written into dst_obst (the other ping-pong buffer).
void launch_pack_planes(const uint8_t* src, const uint8_t* mask, uint8_t* dst, uint8_t* dst_obst,
                        size_t pitch, int W, int nrows, int num_sms, cudaStream_t st);
// Planes -> bytes (bit 7 from plane 7).
void launch_unpack_planes(const uint8_t* src, uint8_t* dst, size_t pitch, int W, int nrows,
                          int num_sms, cudaStream_t st);

// One time step (motion -> collision -> forcing) over rows [row_lo,row_hi).
// Returns the number of kernel launches enqueued.
int launch_step(const StepArgs& a, int num_sms, cudaStream_t st, bool force_generic);

// Column keys for one step: zc[i] = column_key(kc, i+1), same for zf.
void launch_column_keys(uint64_t* zc, uint64_t* zf, uint64_t kc, uint64_t kf, int W,
                        cudaStream_t st);

// src bit 7 := obstacle mask (bytes 0/1), bits 0-6 untouched, on owned rows.
void launch_apply_mask(uint8_t* base, const uint8_t* mask, size_t pitch, int W, int nrows,
                       cudaStream_t st);

// init_lattice on device (lattice.cpp:44-93) for owned rows of a strip.
void launch_init(uint8_t* base, const uint8_t* mask, size_t pitch, int W, int nrows,
                 long long row0, long long H, uint64_t seed, uint64_t thr, cudaStream_t st);

// Reductions. acc: 3 x int64 (mass, px, py) over owned rows (observables.cpp:27-47).
void launch_reduce_global(const uint8_t* base, size_t pitch, int W, int nrows,
                          long long* acc, cudaStream_t st);
// Per cell (nodes, particles, px, py) over global interior rows 1..H-2
// (observables.cpp:49-82); output arrays are the full global cell grid.
void launch_reduce_cells(const uint8_t* base, size_t pitch, int W, int nrows, long long row0,
                         long long H, int B, int* nodes, int* particles, long long* px,
                         long long* py, cudaStream_t st);
// Per owned interior row (px sum, fluid count) (observables.cpp:84-102);
// index = global row - 1.
void launch_reduce_rows(const uint8_t* base, size_t pitch, int W, int nrows, long long row0,
                        long long H, long long* px, int* fluid, cudaStream_t st);

// The same observables on a bit-plane lattice (fhpg_reduce_planes.cu), read
// straight from the planes of the current buffer (`base` = local row 0).
void launch_reduce_global_planes(const uint8_t* base, size_t pitch, int W, int nrows,
                                 long long* acc, int num_sms, cudaStream_t st);
void launch_reduce_cells_planes(const uint8_t* base, size_t pitch, int W, int nrows,
                                long long row0, long long H, int B, int* nodes, int* particles,
                                long long* px, long long* py, int num_sms, cudaStream_t st);
void launch_reduce_rows_planes(const uint8_t* base, size_t pitch, int W, int nrows, long long row0,
                               long long H, long long* px, int* fluid, cudaStream_t st);

}  // namespace fhpg
