/*
 * fhpg.h — C ABI of the B200 FHP lattice-gas engine (libfhpg.so).
 *
 * This is the drop-in boundary for the reference's evolution path:
 *
 *   std::uint64_t fhp::advance(Lattice& lat, const CollisionTable& table,
 *                              const SimConfig& cfg, int first_step,
 *                              int step_count);
 *     (/root/reference/proj/core/include/fhp/step.hpp:46-47,
 *      proj/core/src/step.cpp:103-133)
 *
 * A `case Backend::Cuda:` in that switch uploads
 * lat.src() and the obstacle mask, sets the table, calls fhpg_advance and
 * downloads the result into lat.src(). The framework's own C++ host layer
 * (paper_1208_2428_b200/host, namespace fhp_b200) keeps the state resident on
 * the device between calls instead.
 *
 * Plain C types only. Every function returns 0 on success, FHPG_EINVAL (2)
 * for the conditions the reference reports with std::invalid_argument and
 * FHPG_ERUNTIME (3) for the ones it reports with std::runtime_error (CUDA
 * failures included) — the same split the reference CLI maps to exit codes 2
 * and 3 (proj/tools/fhp_main.cpp:171-182). fhpg_last_error() gives the
 * message of the last failure on the calling thread.
 *
 * Byte layout of every host buffer: row-major rows of W node bytes (the
 * reference's storage columns 1..W), consecutive rows `stride` bytes apart;
 * pass lat.src() + 1 with stride W + 2 for a reference Lattice. Node byte:
 * bits 0-5 movers NW,NE,E,SE,SW,W, bit 6 rest, bit 7 obstacle
 * (node_state.hpp:9-20). Obstacle masks: one byte per node, nonzero = solid
 * (the Lattice's obstacle_ vector, lattice.hpp:67).
 */
#ifndef FHPG_H
#define FHPG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FHPG_OK 0
#define FHPG_EINVAL 2
#define FHPG_ERUNTIME 3

typedef struct fhpg_engine fhpg_engine;

/* Engine for a whole W x H lattice on the current CUDA device.
 * Replaces Lattice::Lattice (lattice.cpp:10-17): W >= 1, H >= 3. */
int fhpg_create(int width, int height, fhpg_engine** out);

/* Engine for the row strip [row_begin, row_end) of a W x H lattice on CUDA
 * device `device` (multi-GPU row strips, the device analog of the strips
 * backend's worker rows, backends.cpp:140-145). Halo rows row_begin-1 and
 * row_end are filled by the caller through fhpg_halo() before every step. */
int fhpg_create_strip(int width, int height, int row_begin, int row_end, int device,
                      fhpg_engine** out);

/* Engine for a whole W x H lattice split into n_strips row strips, strip i on
 * CUDA device devices[i] (devices == NULL: device i; several strips may share
 * a device). Rows follow make_strip_plan + worker_rows (backends.cpp:20-36,
 * 140-145): balanced interior strips, strip 0 also owns wall row 0 and the
 * last strip row H-1; n_strips > H-2 is FHPG_EINVAL with the reference's
 * message. The engine owns every strip's buffers and streams and runs the
 * halo exchange itself (peer copies over NVLink between neighbouring strips,
 * overlapped with the interior rows of each step): every call below works on
 * it as on a single-device engine over the whole lattice (uploads, masks and
 * downloads cover all H rows; observables and swaps are summed over the
 * strips), except fhpg_set_stream, fhpg_advance_part and fhpg_halo
 * (FHPG_EINVAL: the engine orders its strips' streams itself). This is the
 * `gpus` of fhp_b200::SimConfig. */
int fhpg_create_multi(int width, int height, int n_strips, const int* devices,
                      fhpg_engine** out);

/* Number of CUDA devices visible to the library (for strip placement). */
int fhpg_device_count(int* n);

/* Strip layout of an engine: *n_strips (1 for a single-strip engine) and,
 * for each strip i (arrays of n_strips entries, each may be NULL), its rows
 * [row_begin[i], row_end[i]) and CUDA device. */
int fhpg_strips(fhpg_engine* e, int* n_strips, int* row_begin, int* row_end, int* device);

void fhpg_destroy(fhpg_engine* e);

/* Thread-local message of the last failure ("" if none). */
const char* fhpg_last_error(void);

/* Stream all engine work is enqueued on (a cudaStream_t; NULL = the legacy
 * default stream). Until this is called the engine uses its own stream. */
int fhpg_set_stream(fhpg_engine* e, void* cuda_stream);

/* 512-entry collision table, index (chirality << 8) | state
 * (CollisionTable, collision.hpp:17-23). Rejected (FHPG_EINVAL) if any entry
 * changes bit 7: the engine keeps the obstacle flag in bit 7 of the state
 * (the reference re-derives it from the mask during motion, step.cpp:50). */
int fhpg_set_table(fhpg_engine* e, const uint8_t table[512]);

/* Obstacle mask for the engine's rows (Lattice::set_obstacle, lattice.cpp:19-30). */
int fhpg_set_obstacles(fhpg_engine* e, const uint8_t* mask, size_t stride);

/* Copy the engine's rows from / to host memory (bit 7 included). An upload
 * is kept byte-exact until the first step; stepping derives bit 7 from the
 * obstacle mask exactly like the reference's motion pass. */
int fhpg_upload(fhpg_engine* e, const uint8_t* state, size_t stride);
int fhpg_download(fhpg_engine* e, uint8_t* state, size_t stride);

/* init_lattice(cfg) on the device, bit-exact with lattice.cpp:44-93: walls on
 * global rows 0 and H-1, the obstacle mask set by fhpg_set_obstacles (the
 * geometry), counter-RNG fill of every other node. Also sets bit 7. */
int fhpg_init(fhpg_engine* e, uint64_t seed, double fill_density);

/* The hot path: step_count full steps with global step indices
 * first_step .. first_step+step_count-1 (step.cpp:95-133). force_thr is the
 * bernoulli threshold of rng.hpp:37-42 (fhpg_bernoulli_threshold(force_p)),
 * 0 = no forcing. step_count <= 0 is a no-op. Blocks until done and returns
 * the accepted forcing swaps in *swaps (may be NULL). */
int fhpg_advance(fhpg_engine* e, uint64_t seed, uint64_t force_thr, int64_t first_step,
                 int64_t step_count, uint64_t* swaps);

/* Same, enqueue only: swaps accumulate on the device, read with fhpg_swaps. */
int fhpg_advance_async(fhpg_engine* e, uint64_t seed, uint64_t force_thr, int64_t first_step,
                       int64_t step_count);

/* One step split in two launches so a strip can overlap its halo exchange
 * with the interior (the device analog of run_strips' per-step phases,
 * backends.cpp:196-209): part 0 updates rows 1..nrows-2 (needs no halo),
 * part 1 updates rows 0 and nrows-1 (needs the halos of this step) and
 * swaps the buffers. Enqueue only; swaps accumulate on the device. */
int fhpg_advance_part(fhpg_engine* e, uint64_t seed, uint64_t force_thr, int64_t step, int part);

/* Synchronise and read (optionally reset) the device swap counter. */
int fhpg_swaps(fhpg_engine* e, uint64_t* swaps, int reset);

/* Block until all enqueued engine work is done. */
int fhpg_synchronize(fhpg_engine* e);

/* rng.hpp:37-42 threshold: p >= 1 ? 2^32 : (uint64_t)(p * 2^32). */
uint64_t fhpg_bernoulli_threshold(double p);

/* FNV-1a-64 over n host bytes: the reference's state_digest
 * (lattice.cpp:122-132) of a downloaded lattice (rows x W bytes, bit 7
 * included); also the checkpoint integrity digest. Host-side, no engine. */
uint64_t fhpg_digest(const uint8_t* bytes, size_t n);

/* Integer observables of the engine's rows (observables.cpp:27-47):
 * mass = sum popcount(s & 0x7F) over all nodes, momentum over fluid nodes. */
int fhpg_reduce_global(fhpg_engine* e, int64_t* mass, int64_t* px, int64_t* py);

/* coarse_grain integer sums (observables.cpp:49-82) on the GLOBAL cell grid
 * cells_x = ceil(W/B), cells_y = ceil((H-2)/B), row-major; a strip adds only
 * its own rows (sum the arrays over strips). */
int fhpg_reduce_cells(fhpg_engine* e, int block, int32_t* nodes, int32_t* particles,
                      int64_t* px, int64_t* py);

/* The same sums without blocking (the dump pipeline, step.cpp:150-166 /
 * fhp_main.cpp:52-59, at a dump_every cadence): the reduction and the copy
 * of its result into engine-owned pinned host memory are enqueued on the
 * engine's stream(s) behind the steps already enqueued, and the call returns
 * at once, so the next steps can be enqueued while the sums travel.
 * fhpg_cells_wait() blocks until they have landed and copies them out
 * (summed over the strips of a multi-strip engine). One request is
 * outstanding per engine; a new request first waits for the previous one. */
int fhpg_reduce_cells_async(fhpg_engine* e, int block);
int fhpg_cells_wait(fhpg_engine* e, int32_t* nodes, int32_t* particles, int64_t* px,
                    int64_t* py);

/* velocity_profile integer sums (observables.cpp:84-102): for global interior
 * row r (1..H-2) entry r-1 = (sum px over fluid nodes, fluid node count);
 * only the engine's own rows are written. */
int fhpg_reduce_rows(fhpg_engine* e, int64_t* px, int32_t* fluid_count);

/* Device pointers of the current state's boundary rows and halo rows for
 * the halo exchange of a strip (each row_bytes long, valid until the next
 * step): send_top = first owned row, send_bottom = last owned row,
 * recv_top = halo row above, recv_bottom = halo row below. */
int fhpg_halo(fhpg_engine* e, void** send_top, void** send_bottom, void** recv_top,
              void** recv_bottom, size_t* row_bytes);

/* Introspection: W, H, row_begin, row_end, which step kernel runs
 * (2 = bit-plane path, 1 = byte streaming path, 0 = generic), and the number
 * of kernels the stepping has enqueued so far (step kernels, the per-call
 * column keys, bit-7 normalisation). */
int fhpg_info(fhpg_engine* e, int* width, int* height, int* row_begin, int* row_end,
              int* fast_path, uint64_t* step_launches);

/* Testing aid: force the generic (one-thread-per-site) step kernel. */
int fhpg_force_generic(fhpg_engine* e, int on);

/* Testing aid: rows per column-key base of the bit-plane kernels (the
 * kernels fold each band's column keys at a base row and re-key — or, in
 * the per-warp kernel, hash from the step keys — where a key's low word
 * would leave its 2^30 block; this caps that span, 0xFFFFFFFF = automatic).
 * Results are identical for every value. */
int fhpg_debug_key_span(fhpg_engine* e, uint32_t rows);

/* Step-kernel selection: 0 = automatic (bit-plane path when the table has a
 * bit-sliced circuit — FHP-III, FHP-I, DEFAULT — and W % 1024 == 0, with the
 * shared-memory-resident kernel for multi-step calls on small lattices; else
 * the byte streaming path when W allows it, else generic), 1 = byte paths
 * only, 2 = generic, 3 = bit-plane streaming kernels only (no resident kernel).
 * The resident state is converted between layouts on the device; results
 * are identical on every path. */
int fhpg_select_path(fhpg_engine* e, int path);

/* Introspection: the halo depth (steps per block, > 0) the shared-memory-
 * resident kernel would run a multi-step fhpg_advance call with at this
 * forcing threshold, or 0 when the call goes to the streaming kernels (the
 * lattice or its shared-memory footprint is too large, a strip engine, or a
 * path other than automatic selected). */
int fhpg_resident_depth(fhpg_engine* e, uint64_t force_thr, int* depth);

#ifdef __cplusplus
}
#endif
#endif /* FHPG_H */
