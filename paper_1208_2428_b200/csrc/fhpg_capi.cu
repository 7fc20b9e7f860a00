// fhpg_capi.cu — the C ABI (include/fhpg.h): engine object, device memory,
// error mapping, and the step loop that drives the kernels.
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include "../../include/fhpg.h"
#include "../../include/fhpg_tables.h"
#include "fhpg_common.cuh"
#include "fhpg_kernels.cuh"

struct fhpg_engine {
  int W = 0, H = 0, row_begin = 0, row_end = 0, nrows = 0, device = 0;
  size_t pitch = 0;
  uint8_t* buf[2] = {nullptr, nullptr};  // (nrows + 4) * pitch each: halo, rows, halo, 2 spare
  int cur = 0;
  uint8_t* mask = nullptr;               // nrows * pitch, 0/1
  // Bit-plane layout (fhpg_step_planes.cu): used while the table has a
  // bit-sliced circuit and W allows it. `scratch` then holds a byte image of
  // the state when `scratch_valid` (exact uploaded bytes until the first
  // step, an unpacked copy afterwards).
  bool planes = false;
  bool table_planes = false;
  int planes_rule = 2;                   // circuit of the table: FHPG_RULES_* (fhpg_tables.h)
  int path_pref = 0;                     // 0 auto, 1 byte fast path, 2 generic, 3 streaming planes
  uint32_t span_cap = 0xFFFFFFFFu;       // fhpg_debug_key_span (testing aid)
  uint8_t* scratch = nullptr;            // nrows * pitch
  alignas(64) unsigned char tmap[2][fhpg::kPlaneMaps][128];  // TMA descriptors of buf[0], buf[1] (planes)
  bool scratch_valid = false;
  uint8_t* table = nullptr;              // 512 bytes
  uint64_t* zkeys = nullptr;             // [parity][purpose][W]
  unsigned long long* swaps = nullptr;
  long long* acc = nullptr;              // reduction scratch (3)
  unsigned* bar = nullptr;               // grid barrier of the resident kernel (2 words)
  cudaStream_t stream = nullptr;
  cudaStream_t own_stream = nullptr;
  cudaEvent_t tail = nullptr;            // recorded after the last enqueued work (any stream)
  // Coarse-grain request (fhpg_reduce_cells_async): device sums copied into
  // pinned host memory on the stream, `cells_ev` marks their arrival.
  void* cells_dev = nullptr;
  void* cells_host = nullptr;
  size_t cells_cap = 0;                  // bytes of each buffer
  size_t cells_n = 0;                    // cells of the pending request
  bool cells_pending = false;
  cudaEvent_t cells_ev = nullptr;
  bool table_set = false;
  bool normalized = true;                // state bit 7 == mask
  int num_sms = 148;
  uint64_t launches = 0;                 // kernels enqueued by stepping (step, keys, mask)
  int64_t keys_step = -1;                // step whose column keys are in keys(step & 1)
  uint64_t keys_seed = 0;
  bool keys_force = false;

  // Multi-strip engine (fhpg_create_multi): the strips, one engine each (on
  // its own device and stream), and the halo-exchange machinery. Empty for
  // a single-strip engine.
  std::vector<fhpg_engine*> parts;
  std::vector<cudaStream_t> halo_stream;   // per strip: the halo copies into it
  std::vector<cudaEvent_t> ev_done;        // per strip: its last step's boundary rows are done
  std::vector<cudaEvent_t> ev_halo;        // per strip: its halos for this step have landed

  bool multi() const { return !parts.empty(); }
  uint8_t* base(int which) const { return buf[which] + pitch; }  // local row 0
  uint64_t* keys(int parity, int purpose) const {
    return zkeys + (static_cast<size_t>(parity) * 2 + purpose) * static_cast<size_t>(W);
  }
};

namespace {

thread_local std::string g_last_error;

struct Failure {
  int code;
  std::string msg;
};

[[noreturn]] void invalid(const std::string& m) { throw Failure{FHPG_EINVAL, m}; }

void ck(cudaError_t err, const char* what) {
  if (err != cudaSuccess)
    throw Failure{FHPG_ERUNTIME, std::string(what) + ": " + cudaGetErrorString(err)};
}

class DeviceGuard {
 public:
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev_);
    if (prev_ != dev) ck(cudaSetDevice(dev), "cudaSetDevice");
  }
  ~DeviceGuard() {
    int now = -1;
    cudaGetDevice(&now);
    if (now != prev_) cudaSetDevice(prev_);
  }

 private:
  int prev_ = 0;
};

template <typename F>
int guarded(F&& f) {
  try {
    f();
    g_last_error.clear();
    return FHPG_OK;
  } catch (const Failure& e) {
    g_last_error = e.msg;
    return e.code;
  } catch (const std::bad_alloc&) {
    g_last_error = "out of host memory";
    return FHPG_ERUNTIME;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return FHPG_ERUNTIME;
  }
}

void need(const fhpg_engine* e) {
  if (!e) invalid("null engine");
}

void release(fhpg_engine* e) {
  if (!e) return;
  for (size_t i = 0; i < e->parts.size(); ++i) {
    cudaSetDevice(e->parts[i]->device);
    if (i < e->halo_stream.size() && e->halo_stream[i]) cudaStreamDestroy(e->halo_stream[i]);
    if (i < e->ev_done.size() && e->ev_done[i]) cudaEventDestroy(e->ev_done[i]);
    if (i < e->ev_halo.size() && e->ev_halo[i]) cudaEventDestroy(e->ev_halo[i]);
    release(e->parts[i]);
  }
  if (e->multi()) {
    delete e;
    return;
  }
  cudaFree(e->buf[0]);
  cudaFree(e->buf[1]);
  cudaFree(e->mask);
  cudaFree(e->scratch);
  cudaFree(e->table);
  cudaFree(e->zkeys);
  cudaFree(e->swaps);
  cudaFree(e->acc);
  cudaFree(e->bar);
  cudaFree(e->cells_dev);
  cudaFreeHost(e->cells_host);
  if (e->cells_ev) cudaEventDestroy(e->cells_ev);
  if (e->own_stream) cudaStreamDestroy(e->own_stream);
  if (e->tail) cudaEventDestroy(e->tail);
  delete e;
}

void create(int W, int H, int rb, int re, int device, fhpg_engine** out) {
  if (!out) invalid("null output pointer");
  *out = nullptr;
  // Same messages as Lattice::Lattice (lattice.cpp:11-12) and make_strip_plan.
  if (W < 1) invalid("lattice width must be >= 1");
  if (H < 3) invalid("lattice height must be >= 3");
  if (rb < 0 || re > H || re <= rb) invalid("strip rows must satisfy 0 <= row_begin < row_end <= height");
  int ndev = 0;
  ck(cudaGetDeviceCount(&ndev), "cudaGetDeviceCount");
  if (device < 0 || device >= ndev) invalid("CUDA device index out of range");
  DeviceGuard g(device);
  auto* e = new fhpg_engine;
  try {
    e->W = W;
    e->H = H;
    e->row_begin = rb;
    e->row_end = re;
    e->nrows = re - rb;
    e->device = device;
    // Room for the bit-plane rows (W + 2048 bytes, line-aligned) when the
    // width allows them.
    e->pitch = fhpg::planes_ok(W) ? fhpg::planes_row_bytes(W)
                                  : (static_cast<size_t>(W) + 15) / 16 * 16;
    // halo above, rows, halo below, 3 spare zero rows the streaming kernels may prefetch
    const size_t bytes = (static_cast<size_t>(e->nrows) + 5) * e->pitch;
    for (int i = 0; i < 2; ++i) {
      ck(cudaMalloc(&e->buf[i], bytes), "cudaMalloc(state)");
      ck(cudaMemset(e->buf[i], 0, bytes), "cudaMemset(state)");
      for (int kind = 0; kind < fhpg::kPlaneMaps && fhpg::planes_ok(W); ++kind)
        if (!fhpg::make_planes_map(e->tmap[i][kind], e->buf[i], W, e->pitch, e->nrows + 5, kind))
          throw Failure{FHPG_ERUNTIME, "cuTensorMapEncodeTiled failed"};
    }
    ck(cudaMalloc(&e->mask, static_cast<size_t>(e->nrows) * e->pitch), "cudaMalloc(mask)");
    ck(cudaMemset(e->mask, 0, static_cast<size_t>(e->nrows) * e->pitch), "cudaMemset(mask)");
    ck(cudaMalloc(&e->table, 512), "cudaMalloc(table)");
    ck(cudaMalloc(&e->zkeys, sizeof(uint64_t) * 4 * static_cast<size_t>(W)), "cudaMalloc(keys)");
    ck(cudaMalloc(&e->swaps, sizeof(unsigned long long)), "cudaMalloc(swaps)");
    ck(cudaMemset(e->swaps, 0, sizeof(unsigned long long)), "cudaMemset(swaps)");
    ck(cudaMalloc(&e->acc, sizeof(long long) * 4), "cudaMalloc(acc)");
    ck(cudaMalloc(&e->bar, sizeof(unsigned) * 2), "cudaMalloc(bar)");
    ck(cudaMemset(e->bar, 0, sizeof(unsigned) * 2), "cudaMemset(bar)");
    ck(cudaStreamCreateWithFlags(&e->own_stream, cudaStreamNonBlocking), "cudaStreamCreate");
    e->stream = e->own_stream;
    ck(cudaEventCreateWithFlags(&e->tail, cudaEventDisableTiming), "cudaEventCreate");
    ck(cudaEventCreateWithFlags(&e->cells_ev, cudaEventDisableTiming), "cudaEventCreate");
    ck(cudaDeviceGetAttribute(&e->num_sms, cudaDevAttrMultiProcessorCount, device),
       "cudaDeviceGetAttribute");
    ck(cudaDeviceSynchronize(), "cudaDeviceSynchronize");
  } catch (...) {
    release(e);
    throw;
  }
  *out = e;
}

bool want_planes(const fhpg_engine* e) {
  return e->table_set && e->table_planes && (e->path_pref == 0 || e->path_pref == 3) &&
         fhpg::planes_ok(e->W);
}

void need_scratch(fhpg_engine* e) {
  if (e->scratch) return;
  ck(cudaMalloc(&e->scratch, static_cast<size_t>(e->nrows) * e->pitch), "cudaMalloc(scratch)");
}

// Byte image of the current state (device, local row 0, pitch e->pitch).
uint8_t* bytes_view(fhpg_engine* e) {
  if (!e->planes) return e->base(e->cur);
  if (!e->scratch_valid) {
    need_scratch(e);
    fhpg::launch_unpack_planes(e->base(e->cur), e->scratch, e->pitch, e->W, e->nrows,
                               e->num_sms, e->stream);
    ck(cudaGetLastError(), "unpack launch");
    e->scratch_valid = true;
  }
  return e->scratch;
}

// scratch (bytes) -> current plane buffer; plane 7 (obstacles, from the mask)
// into both buffers. The step never writes plane 7.
void pack_from_scratch(fhpg_engine* e) {
  fhpg::launch_pack_planes(e->scratch, e->mask, e->base(e->cur), e->base(e->cur ^ 1), e->pitch,
                           e->W, e->nrows, e->num_sms, e->stream);
  ck(cudaGetLastError(), "pack launch");
}

// Put the resident state in the layout the table / path selection wants.
void sync_layout(fhpg_engine* e) {
  const bool want = want_planes(e);
  if (want == e->planes) return;
  if (want) {
    need_scratch(e);
    ck(cudaMemcpy2DAsync(e->scratch, e->pitch, e->base(e->cur), e->pitch, e->W, e->nrows,
                         cudaMemcpyDeviceToDevice, e->stream), "layout copy");
    e->scratch_valid = true;
    pack_from_scratch(e);
    e->planes = true;
  } else {
    const uint8_t* v = bytes_view(e);
    ck(cudaMemcpy2DAsync(e->base(e->cur), e->pitch, v, e->pitch, e->W, e->nrows,
                         cudaMemcpyDeviceToDevice, e->stream), "layout copy");
    e->planes = false;
    e->scratch_valid = false;
    e->normalized = false;  // re-derived from the mask at the next step
  }
  ck(cudaStreamSynchronize(e->stream), "layout sync");
}

// Enqueue one step launch over rows [a.row_lo, a.row_hi) with the kernel the
// layout selects.
void launch_any(fhpg_engine* e, const fhpg::StepArgs& a) {
  if (e->planes) {
    const int which = a.src == e->base(0) ? 0 : 1;
#if FHPG_FIXED_SRC  // timing experiment (wrong results): every step reads buffer 0, writes buffer 1
    e->launches += fhpg::launch_step_planes(a, e->tmap[0], e->tmap[1], e->num_sms,
#else
    e->launches += fhpg::launch_step_planes(a, e->tmap[which], e->tmap[which ^ 1], e->num_sms,
#endif
                                            e->stream);
    e->scratch_valid = false;
  } else {
    e->launches += fhpg::launch_step(a, e->num_sms, e->stream, e->path_pref == 2);
  }
  ck(cudaGetLastError(), "step launch");
}

void step_loop(fhpg_engine* e, uint64_t seed, uint64_t thr, int64_t first, int64_t count) {
  using namespace fhpg;
  if (!e->table_set) invalid("collision table not set (fhpg_set_table)");
  if (thr > (1ull << 32)) invalid("force threshold must be <= 2^32");
  cudaStream_t st = e->stream;
  if (!e->planes && !e->normalized) {
    launch_apply_mask(e->base(e->cur), e->mask, e->pitch, e->W, e->nrows, st);
    ck(cudaGetLastError(), "apply_mask launch");
    ++e->launches;
    e->normalized = true;
  }
  const bool force = thr != 0;
  // Small whole lattices: the shared-memory-resident kernel, one cooperative
  // launch for the whole call (fhpg_step_resident.cu).
  int rpc = 0, grid = 0;
  if (e->planes && e->path_pref == 0 && count >= 2 && e->row_begin == 0 && e->row_end == e->H &&
      resident_plan(e->W, e->H, thr, e->num_sms, &rpc, &grid) > 0) {
    uint8_t* const g[2] = {e->base(0), e->base(1)};
    cudaError_t err = cudaSuccess;
    const int flips = launch_step_resident(g, e->cur, e->pitch, e->W, e->H, e->planes_rule, seed, thr,
                                           first, count, e->swaps, e->bar, e->num_sms, st, &err);
    ck(err, "resident step launch");
    ck(cudaGetLastError(), "resident step launch");
    e->cur ^= flips & 1;
    e->scratch_valid = false;
    ++e->launches;
    e->keys_step = -1;
    ck(cudaEventRecord(e->tail, st), "cudaEventRecord");
    return;
  }
  const uint64_t s0 = static_cast<uint64_t>(first);
  launch_column_keys(e->keys(s0 & 1, 0), force ? e->keys(s0 & 1, 1) : nullptr,
                     step_key(seed, kChirality, s0), step_key(seed, kForcing, s0), e->W, st);
  ck(cudaGetLastError(), "column_keys launch");
  ++e->launches;
  for (int64_t i = 0; i < count; ++i) {
    const uint64_t s = static_cast<uint64_t>(first + i);
    StepArgs a{};
    a.src = e->base(e->cur);
    a.dst = e->base(e->cur ^ 1);
    a.pitch = e->pitch;
    a.W = e->W;
    a.nrows = e->nrows;
    a.row0 = e->row_begin;
    a.table = e->table;
    a.zc = e->keys(s & 1, 0);
    a.zf = force ? e->keys(s & 1, 1) : nullptr;
    a.kc_cur = step_key(seed, kChirality, s);
    a.kf_cur = step_key(seed, kForcing, s);
    a.thr = thr;
    a.swaps = e->swaps;
    a.rule = e->planes_rule;
  a.span_cap = e->span_cap;
    if (i + 1 < count) {
      a.zc_next = e->keys((s + 1) & 1, 0);
      a.zf_next = force ? e->keys((s + 1) & 1, 1) : nullptr;
      a.kc_next = step_key(seed, kChirality, s + 1);
      a.kf_next = step_key(seed, kForcing, s + 1);
    }
    a.row_lo = 0;
    a.row_hi = e->nrows;
    launch_any(e, a);
    e->cur ^= 1;
  }
  e->keys_step = -1;
  ck(cudaEventRecord(e->tail, st), "cudaEventRecord");
}

// One step in two parts for strips that overlap the halo exchange with the
// interior: part 0 = rows [1, nrows-1) (needs no halo row), part 1 = the
// boundary rows 0 and nrows-1, then the buffer swap.
void step_part(fhpg_engine* e, uint64_t seed, uint64_t thr, int64_t step, int part) {
  using namespace fhpg;
  if (!e->table_set) invalid("collision table not set (fhpg_set_table)");
  if (thr > (1ull << 32)) invalid("force threshold must be <= 2^32");
  if (part != 0 && part != 1) invalid("part must be 0 (interior) or 1 (boundary rows)");
  cudaStream_t st = e->stream;
  if (!e->planes && !e->normalized) {
    launch_apply_mask(e->base(e->cur), e->mask, e->pitch, e->W, e->nrows, st);
    ck(cudaGetLastError(), "apply_mask launch");
    ++e->launches;
    e->normalized = true;
  }
  const bool force = thr != 0;
  const uint64_t s = static_cast<uint64_t>(step);
  if (e->keys_step != step || e->keys_seed != seed || (force && !e->keys_force)) {
    launch_column_keys(e->keys(s & 1, 0), force ? e->keys(s & 1, 1) : nullptr,
                       step_key(seed, kChirality, s), step_key(seed, kForcing, s), e->W, st);
    ck(cudaGetLastError(), "column_keys launch");
    ++e->launches;
    e->keys_step = step;
    e->keys_seed = seed;
    e->keys_force = force;
  }
  StepArgs a{};
  a.src = e->base(e->cur);
  a.dst = e->base(e->cur ^ 1);
  a.pitch = e->pitch;
  a.W = e->W;
  a.nrows = e->nrows;
  a.row0 = e->row_begin;
  a.table = e->table;
  a.zc = e->keys(s & 1, 0);
  a.zf = force ? e->keys(s & 1, 1) : nullptr;
  a.kc_cur = step_key(seed, kChirality, s);
  a.kf_cur = step_key(seed, kForcing, s);
  a.thr = thr;
  a.swaps = e->swaps;
  a.rule = e->planes_rule;
  a.span_cap = e->span_cap;
  const bool interior = e->nrows >= 3;
  auto run = [&](int lo, int hi, bool with_next_keys) {
    StepArgs b = a;
    b.row_lo = lo;
    b.row_hi = hi;
    if (with_next_keys) {
      b.zc_next = e->keys((s + 1) & 1, 0);
      b.zf_next = force ? e->keys((s + 1) & 1, 1) : nullptr;
      b.kc_next = step_key(seed, kChirality, s + 1);
      b.kf_next = step_key(seed, kForcing, s + 1);
    }
    launch_any(e, b);
  };
  if (part == 0) {
    if (interior) run(1, e->nrows - 1, true);
    ck(cudaEventRecord(e->tail, st), "cudaEventRecord");
    return;
  }
  if (interior && e->planes) {
    // both boundary rows in one launch of the ring kernel
    StepArgs b = a;
    b.row_lo = 0;
    b.row_hi = 1;
    b.row_lo2 = e->nrows - 1;
    b.row_hi2 = e->nrows;
    launch_any(e, b);
  } else if (interior) {
    run(0, 1, false);
    run(e->nrows - 1, e->nrows, false);
  } else {
    run(0, e->nrows, true);
  }
  e->cur ^= 1;
  e->keys_step = step + 1;  // computed by part 0 (or by the single launch above)
  ck(cudaEventRecord(e->tail, st), "cudaEventRecord");
}

void copy_rows_h2d(uint8_t* dev, size_t pitch, const uint8_t* host, size_t stride, int W,
                   int rows, cudaStream_t st) {
  ck(cudaMemcpy2DAsync(dev, pitch, host, stride, W, rows, cudaMemcpyHostToDevice, st),
     "cudaMemcpy2D H2D");
}

// ---------------------------------------------------------------------------
// Multi-strip engine: the device analog of the strips backend (make_strip_plan
// backends.cpp:20-36, worker_rows :140-145, run_strips :149-219) with one
// strip per GPU. Per step and strip j (stream S_j, halo stream T_j):
//   T_j: wait done(j-1), done(j), done(j+1) of the previous step, copy the
//        neighbours' boundary rows into j's halo rows (peer copies over
//        NVLink when the strips sit on different GPUs), record halo(j);
//   S_j: interior rows (no halo needed; overlaps the copies), wait halo(j),
//        boundary rows + buffer swap, record done(j).
// The waits order every read of a boundary row after the step that wrote
// it, and every overwrite of a halo row or boundary row after the last read
// of its previous contents (the neighbour's boundary launch of the step
// before). Every random decision is keyed by global (x, y, step), so the
// strips reproduce the single-engine bits exactly.
// ---------------------------------------------------------------------------
std::vector<std::pair<int, int>> strip_plan(int H, int n) {
  // make_strip_plan (same messages) + worker_rows: strip 0 also owns wall
  // row 0, the last strip wall row H-1.
  const int interior = H - 2;
  if (n < 1) invalid("strip count must be >= 1");
  if (n > interior) invalid("strip count exceeds interior row count");
  std::vector<std::pair<int, int>> rows;
  const int base = interior / n, extra = interior % n;
  int r = 1;
  for (int i = 0; i < n; ++i) {
    const int k = base + (i < extra ? 1 : 0);
    rows.emplace_back(r, r + k);
    r += k;
  }
  rows.front().first = 0;
  rows.back().second = H;
  return rows;
}

void create_multi(int W, int H, int n, const int* devices, fhpg_engine** out) {
  if (!out) invalid("null output pointer");
  *out = nullptr;
  if (W < 1) invalid("lattice width must be >= 1");
  if (H < 3) invalid("lattice height must be >= 3");
  const auto plan = strip_plan(H, n);
  int ndev = 0;
  ck(cudaGetDeviceCount(&ndev), "cudaGetDeviceCount");
  std::vector<int> dev(n);
  for (int i = 0; i < n; ++i) {
    dev[i] = devices ? devices[i] : i;
    if (dev[i] < 0 || dev[i] >= ndev) invalid("CUDA device index out of range");
  }
  auto* m = new fhpg_engine;
  m->W = W;
  m->H = H;
  m->row_begin = 0;
  m->row_end = H;
  m->nrows = H;
  m->device = dev[0];
  try {
    for (int i = 0; i < n; ++i) {
      fhpg_engine* p = nullptr;
      create(W, H, plan[i].first, plan[i].second, dev[i], &p);
      m->parts.push_back(p);
      DeviceGuard g(dev[i]);
      cudaStream_t hs = nullptr;
      cudaEvent_t d = nullptr, h = nullptr;
      ck(cudaStreamCreateWithFlags(&hs, cudaStreamNonBlocking), "cudaStreamCreate(halo)");
      m->halo_stream.push_back(hs);
      ck(cudaEventCreateWithFlags(&d, cudaEventDisableTiming), "cudaEventCreate");
      m->ev_done.push_back(d);
      ck(cudaEventCreateWithFlags(&h, cudaEventDisableTiming), "cudaEventCreate");
      m->ev_halo.push_back(h);
    }
    // Peer access between neighbouring strips on different GPUs (NVLink).
    for (int i = 0; i + 1 < n; ++i) {
      if (dev[i] == dev[i + 1]) continue;
      for (const auto& pr : {std::make_pair(dev[i], dev[i + 1]), std::make_pair(dev[i + 1], dev[i])}) {
        int can = 0;
        ck(cudaDeviceCanAccessPeer(&can, pr.first, pr.second), "cudaDeviceCanAccessPeer");
        if (!can) continue;  // cudaMemcpyPeerAsync still works, staged by the driver
        DeviceGuard g(pr.first);
        const cudaError_t err = cudaDeviceEnablePeerAccess(pr.second, 0);
        if (err == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
        else ck(err, "cudaDeviceEnablePeerAccess");
      }
    }
  } catch (...) {
    release(m);
    throw;
  }
  *out = m;
}

struct Halo {
  uint8_t *send_top, *send_bottom, *recv_top, *recv_bottom;
  size_t row_bytes;
};
Halo halo_of(fhpg_engine* e) {
  uint8_t* b = e->base(e->cur);
  return {b, b + static_cast<size_t>(e->nrows - 1) * e->pitch, b - e->pitch,
          b + static_cast<size_t>(e->nrows) * e->pitch,
          e->planes ? fhpg::planes_row_bytes(e->W) : static_cast<size_t>(e->W)};
}

void multi_step_loop(fhpg_engine* m, uint64_t seed, uint64_t thr, int64_t first, int64_t count) {
  const int n = static_cast<int>(m->parts.size());
  auto& P = m->parts;
  if (n == 1) {
    DeviceGuard g(P[0]->device);
    step_loop(P[0], seed, thr, first, count);
    return;
  }
  nvtxRangePushA("fhpg.advance(multi)");
  for (int j = 0; j < n; ++j) {  // the work already enqueued on every strip
    DeviceGuard g(P[j]->device);
    ck(cudaEventRecord(m->ev_done[j], P[j]->stream), "cudaEventRecord");
  }
  for (int64_t i = 0; i < count; ++i) {
    const int64_t s = first + i;
    nvtxRangePushA("fhpg.step");
    nvtxRangePushA("fhpg.halo");
    for (int j = 0; j < n; ++j) {
      DeviceGuard g(P[j]->device);
      const cudaStream_t hs = m->halo_stream[j];
      for (int k = std::max(0, j - 1); k <= std::min(n - 1, j + 1); ++k)
        ck(cudaStreamWaitEvent(hs, m->ev_done[k], 0), "cudaStreamWaitEvent");
      const Halo me = halo_of(P[j]);
      if (j > 0) {
        const Halo up = halo_of(P[j - 1]);
        ck(cudaMemcpyPeerAsync(me.recv_top, P[j]->device, up.send_bottom, P[j - 1]->device,
                               me.row_bytes, hs), "halo copy (top)");
      }
      if (j + 1 < n) {
        const Halo dn = halo_of(P[j + 1]);
        ck(cudaMemcpyPeerAsync(me.recv_bottom, P[j]->device, dn.send_top, P[j + 1]->device,
                               me.row_bytes, hs), "halo copy (bottom)");
      }
      ck(cudaEventRecord(m->ev_halo[j], hs), "cudaEventRecord");
    }
    nvtxRangePop();
    nvtxRangePushA("fhpg.interior");
    for (int j = 0; j < n; ++j) {
      DeviceGuard g(P[j]->device);
      step_part(P[j], seed, thr, s, 0);
    }
    nvtxRangePop();
    nvtxRangePushA("fhpg.boundary");
    for (int j = 0; j < n; ++j) {
      DeviceGuard g(P[j]->device);
      ck(cudaStreamWaitEvent(P[j]->stream, m->ev_halo[j], 0), "cudaStreamWaitEvent");
      step_part(P[j], seed, thr, s, 1);
      ck(cudaEventRecord(m->ev_done[j], P[j]->stream), "cudaEventRecord");
    }
    nvtxRangePop();
    nvtxRangePop();
  }
  nvtxRangePop();
}

// Apply fn to every strip of a multi engine (on its device), or to e itself.
template <typename F>
void each(fhpg_engine* e, F&& fn) {
  if (!e->multi()) {
    DeviceGuard g(e->device);
    fn(e);
    return;
  }
  for (fhpg_engine* p : e->parts) {
    DeviceGuard g(p->device);
    fn(p);
  }
}

void single_only(const fhpg_engine* e, const char* what) {
  if (e->multi()) invalid(std::string(what) + " is not available on a multi-strip engine");
}

}  // namespace

extern "C" {

const char* fhpg_last_error(void) { return g_last_error.c_str(); }

uint64_t fhpg_bernoulli_threshold(double p) { return fhpg::bernoulli_threshold(p); }

uint64_t fhpg_digest(const uint8_t* bytes, size_t n) {
  uint64_t h = 0xCBF29CE484222325ull;
  for (size_t i = 0; i < n; ++i) h = (h ^ bytes[i]) * 0x100000001B3ull;
  return h;
}

int fhpg_device_count(int* n) {
  return guarded([&] {
    if (!n) invalid("null output pointer");
    *n = 0;
    ck(cudaGetDeviceCount(n), "cudaGetDeviceCount");
  });
}

int fhpg_create(int width, int height, fhpg_engine** out) {
  return guarded([&] {
    int dev = 0;
    ck(cudaGetDevice(&dev), "cudaGetDevice");
    create(width, height, 0, height, dev, out);
  });
}

int fhpg_create_strip(int width, int height, int row_begin, int row_end, int device,
                      fhpg_engine** out) {
  return guarded([&] { create(width, height, row_begin, row_end, device, out); });
}

int fhpg_create_multi(int width, int height, int n_strips, const int* devices,
                      fhpg_engine** out) {
  return guarded([&] { create_multi(width, height, n_strips, devices, out); });
}

void fhpg_destroy(fhpg_engine* e) {
  if (!e) return;
  int prev = 0;
  cudaGetDevice(&prev);
  each(e, [](fhpg_engine* p) {
    // The tail event, not the stream: a caller stream set with
    // fhpg_set_stream may already be gone.
    cudaEventSynchronize(p->tail);
  });
  for (size_t i = 0; i < e->halo_stream.size(); ++i) {
    cudaSetDevice(e->parts[i]->device);
    cudaStreamSynchronize(e->halo_stream[i]);
  }
  release(e);
  cudaSetDevice(prev);
}

int fhpg_set_stream(fhpg_engine* e, void* s) {
  return guarded([&] {
    need(e);
    single_only(e, "fhpg_set_stream");
    DeviceGuard g(e->device);
    // Work already enqueued on the old stream (PDL step kernels run
    // asynchronously) is ordered before anything enqueued on the new one.
    ck(cudaEventRecord(e->tail, e->stream), "cudaEventRecord");
    const cudaStream_t ns = static_cast<cudaStream_t>(s);  // NULL = the legacy default stream
    ck(cudaStreamWaitEvent(ns, e->tail, 0), "cudaStreamWaitEvent");
    e->stream = ns;
  });
}

int fhpg_set_table(fhpg_engine* e, const uint8_t* t) {
  return guarded([&] {
    need(e);
    if (!t) invalid("null table");
    for (int i = 0; i < 512; ++i)
      if ((t[i] & 0x80u) != (i & 0x80))
        invalid("collision table: entry " + std::to_string(i) + " changes the obstacle bit");
    // The bit-plane kernels evaluate FHP-III, FHP-I and the reference's
    // DEFAULT rule as circuits (fhpg_planes_rules.cuh); any other table runs
    // the byte LUT path.
    bool planes = false;
    int rule = 2;
    for (const int v : {FHPG_RULES_FHP_III, FHPG_RULES_FHP_I, FHPG_RULES_DEFAULT}) {
      uint8_t ref[512];
      fhpg_build_table(v, ref);
      if (std::memcmp(t, ref, 512) == 0) {
        planes = true;
        rule = v;
        break;
      }
    }
    each(e, [&](fhpg_engine* p) {
      ck(cudaMemcpyAsync(p->table, t, 512, cudaMemcpyHostToDevice, p->stream), "table upload");
      ck(cudaStreamSynchronize(p->stream), "table upload sync");
      p->table_set = true;
      p->table_planes = planes;
      p->planes_rule = rule;
      sync_layout(p);
    });
    e->table_set = true;
  });
}

int fhpg_set_obstacles(fhpg_engine* e, const uint8_t* mask, size_t stride) {
  return guarded([&] {
    need(e);
    if (!mask) invalid("null mask");
    if (stride < static_cast<size_t>(e->W)) invalid("stride < width");
    each(e, [&](fhpg_engine* p) {
      // Raw bytes (nonzero = solid) go straight to the device mask.
      copy_rows_h2d(p->mask, p->pitch, mask + static_cast<size_t>(p->row_begin - e->row_begin) * stride, stride,
                    p->W, p->nrows, p->stream);
      // Lattice::set_obstacle also sets / clears bit 7 of the node (lattice.cpp:25-29).
      uint8_t* v = bytes_view(p);
      fhpg::launch_apply_mask(v, p->mask, p->pitch, p->W, p->nrows, p->stream);
      ck(cudaGetLastError(), "apply_mask launch");
      if (p->planes) pack_from_scratch(p);
      ck(cudaStreamSynchronize(p->stream), "mask sync");
    });
  });
}

int fhpg_upload(fhpg_engine* e, const uint8_t* state, size_t stride) {
  return guarded([&] {
    need(e);
    if (!state) invalid("null state");
    if (stride < static_cast<size_t>(e->W)) invalid("stride < width");
    each(e, [&](fhpg_engine* p) {
      const uint8_t* src = state + static_cast<size_t>(p->row_begin - e->row_begin) * stride;
      if (p->planes) {
        // The byte image stays exact until the first step; the planes take
        // bit 7 from the mask like the reference's motion pass.
        need_scratch(p);
        copy_rows_h2d(p->scratch, p->pitch, src, stride, p->W, p->nrows, p->stream);
        p->scratch_valid = true;
        pack_from_scratch(p);
      } else {
        copy_rows_h2d(p->base(p->cur), p->pitch, src, stride, p->W, p->nrows, p->stream);
        p->normalized = false;
      }
    });
    each(e, [&](fhpg_engine* p) { ck(cudaStreamSynchronize(p->stream), "upload sync"); });
  });
}

int fhpg_download(fhpg_engine* e, uint8_t* state, size_t stride) {
  return guarded([&] {
    need(e);
    if (!state) invalid("null state");
    if (stride < static_cast<size_t>(e->W)) invalid("stride < width");
    each(e, [&](fhpg_engine* p) {
      ck(cudaMemcpy2DAsync(state + static_cast<size_t>(p->row_begin - e->row_begin) * stride,
                           stride, bytes_view(p), p->pitch, p->W, p->nrows,
                           cudaMemcpyDeviceToHost, p->stream),
         "cudaMemcpy2D D2H");
    });
    each(e, [&](fhpg_engine* p) { ck(cudaStreamSynchronize(p->stream), "download sync"); });
  });
}

int fhpg_init(fhpg_engine* e, uint64_t seed, double fill_density) {
  return guarded([&] {
    need(e);
    // lattice.cpp:58-60
    if (!(fill_density >= 0.0 && fill_density <= 1.0)) invalid("fill_density must be in [0,1]");
    each(e, [&](fhpg_engine* p) {
      if (p->planes) need_scratch(p);
      uint8_t* target = p->planes ? p->scratch : p->base(p->cur);
      fhpg::launch_init(target, p->mask, p->pitch, p->W, p->nrows, p->row_begin, p->H, seed,
                        fhpg::bernoulli_threshold(fill_density), p->stream);
      ck(cudaGetLastError(), "init launch");
      // Walls join the obstacle mask (init_impl calls set_obstacle on them).
      for (int r = 0; r < p->nrows; ++r) {
        const long long gr = p->row_begin + r;
        if (gr == 0 || gr == p->H - 1)
          ck(cudaMemsetAsync(p->mask + static_cast<size_t>(r) * p->pitch, 1, p->W, p->stream),
             "wall mask");
      }
      if (p->planes) {
        p->scratch_valid = true;
        pack_from_scratch(p);
      }
      p->normalized = true;
    });
    each(e, [&](fhpg_engine* p) { ck(cudaStreamSynchronize(p->stream), "init sync"); });
  });
}

int fhpg_advance_async(fhpg_engine* e, uint64_t seed, uint64_t thr, int64_t first, int64_t count) {
  return guarded([&] {
    need(e);
    if (count <= 0) return;  // backends.cpp:157 — no-op, state untouched
    if (e->multi()) {
      multi_step_loop(e, seed, thr, first, count);
      return;
    }
    DeviceGuard g(e->device);
    step_loop(e, seed, thr, first, count);
  });
}

int fhpg_advance(fhpg_engine* e, uint64_t seed, uint64_t thr, int64_t first, int64_t count,
                 uint64_t* swaps) {
  return guarded([&] {
    need(e);
    if (swaps) *swaps = 0;
    if (count <= 0) return;
    each(e, [&](fhpg_engine* p) {
      ck(cudaMemsetAsync(p->swaps, 0, sizeof(unsigned long long), p->stream), "swap reset");
    });
    if (e->multi()) {
      multi_step_loop(e, seed, thr, first, count);
    } else {
      DeviceGuard g(e->device);
      step_loop(e, seed, thr, first, count);
    }
    unsigned long long total = 0;
    each(e, [&](fhpg_engine* p) {
      unsigned long long s = 0;
      ck(cudaMemcpyAsync(&s, p->swaps, sizeof s, cudaMemcpyDeviceToHost, p->stream), "swap read");
      ck(cudaStreamSynchronize(p->stream), "advance sync");
      total += s;
    });
    if (swaps) *swaps = total;
  });
}

int fhpg_advance_part(fhpg_engine* e, uint64_t seed, uint64_t thr, int64_t step, int part) {
  return guarded([&] {
    need(e);
    single_only(e, "fhpg_advance_part");
    DeviceGuard g(e->device);
    step_part(e, seed, thr, step, part);
  });
}

int fhpg_swaps(fhpg_engine* e, uint64_t* swaps, int reset) {
  return guarded([&] {
    need(e);
    unsigned long long total = 0;
    each(e, [&](fhpg_engine* p) {
      unsigned long long s = 0;
      ck(cudaMemcpyAsync(&s, p->swaps, sizeof s, cudaMemcpyDeviceToHost, p->stream), "swap read");
      if (reset) ck(cudaMemsetAsync(p->swaps, 0, sizeof s, p->stream), "swap reset");
      ck(cudaStreamSynchronize(p->stream), "swap sync");
      total += s;
    });
    if (swaps) *swaps = total;
  });
}

int fhpg_synchronize(fhpg_engine* e) {
  return guarded([&] {
    need(e);
    each(e, [&](fhpg_engine* p) { ck(cudaStreamSynchronize(p->stream), "synchronize"); });
  });
}

int fhpg_reduce_global(fhpg_engine* e, int64_t* mass, int64_t* px, int64_t* py) {
  return guarded([&] {
    need(e);
    long long tot[3] = {0, 0, 0};
    each(e, [&](fhpg_engine* p) {
      ck(cudaMemsetAsync(p->acc, 0, sizeof(long long) * 3, p->stream), "acc reset");
      if (p->planes && !p->scratch_valid)  // else: the exact uploaded bytes
        fhpg::launch_reduce_global_planes(p->base(p->cur), p->pitch, p->W, p->nrows, p->acc,
                                          p->num_sms, p->stream);
      else
        fhpg::launch_reduce_global(bytes_view(p), p->pitch, p->W, p->nrows, p->acc, p->stream);
      ck(cudaGetLastError(), "reduce launch");
      long long h[3];
      ck(cudaMemcpyAsync(h, p->acc, sizeof h, cudaMemcpyDeviceToHost, p->stream), "acc read");
      ck(cudaStreamSynchronize(p->stream), "reduce sync");
      for (int k = 0; k < 3; ++k) tot[k] += h[k];
    });
    if (mass) *mass = tot[0];
    if (px) *px = tot[1];
    if (py) *py = tot[2];
  });
}

int fhpg_reduce_cells_async(fhpg_engine* e, int B) {
  return guarded([&] {
    need(e);
    if (B < 1) invalid("block size must be >= 1");  // observables.cpp:50
    const size_t cx = (static_cast<size_t>(e->W) + B - 1) / B;
    const size_t cy = (static_cast<size_t>(e->H) - 2 + B - 1) / B;
    const size_t n = cx * cy;
    each(e, [&](fhpg_engine* p) {
      // The previous request's host buffer may still be in use.
      if (p->cells_pending) ck(cudaEventSynchronize(p->cells_ev), "cells wait");
      p->cells_pending = false;
      p->cells_n = n;
      if (n == 0) return;
      if (p->cells_cap < n * 24) {
        cudaFree(p->cells_dev);
        cudaFreeHost(p->cells_host);
        p->cells_dev = p->cells_host = nullptr;
        p->cells_cap = 0;
        ck(cudaMalloc(&p->cells_dev, n * 24), "cudaMalloc(cells)");
        ck(cudaMallocHost(&p->cells_host, n * 24), "cudaMallocHost(cells)");
        p->cells_cap = n * 24;
      }
      // [nodes i32 | particles i32 | px i64 | py i64]
      int* dn = static_cast<int*>(p->cells_dev);
      int* dp = dn + n;
      long long* dx = reinterpret_cast<long long*>(static_cast<char*>(p->cells_dev) + n * 8);
      long long* dy = dx + n;
      ck(cudaMemsetAsync(p->cells_dev, 0, n * 24, p->stream), "cells reset");
      if (p->planes && !p->scratch_valid)  // else: the exact uploaded bytes
        fhpg::launch_reduce_cells_planes(p->base(p->cur), p->pitch, p->W, p->nrows, p->row_begin,
                                         p->H, B, dn, dp, dx, dy, p->num_sms, p->stream);
      else
        fhpg::launch_reduce_cells(bytes_view(p), p->pitch, p->W, p->nrows, p->row_begin, p->H, B,
                                  dn, dp, dx, dy, p->stream);
      ck(cudaGetLastError(), "cells launch");
      ck(cudaMemcpyAsync(p->cells_host, p->cells_dev, n * 24, cudaMemcpyDeviceToHost, p->stream),
         "cells read");
      ck(cudaEventRecord(p->cells_ev, p->stream), "cudaEventRecord");
      p->cells_pending = true;
    });
    e->cells_n = n;
    e->cells_pending = true;
  });
}

int fhpg_cells_wait(fhpg_engine* e, int32_t* nodes, int32_t* particles, int64_t* px,
                    int64_t* py) {
  return guarded([&] {
    need(e);
    if (!e->cells_pending) invalid("no coarse-grain request pending (fhpg_reduce_cells_async)");
    if (!nodes || !particles || !px || !py) invalid("null output array");
    const size_t n = e->cells_n;
    bool first = true;
    each(e, [&](fhpg_engine* p) {
      if (!p->cells_pending || n == 0) return;
      ck(cudaEventSynchronize(p->cells_ev), "cells wait");
      p->cells_pending = false;
      const int32_t* hn = static_cast<const int32_t*>(p->cells_host);
      const int32_t* hp = hn + n;
      const int64_t* hx = reinterpret_cast<const int64_t*>(static_cast<char*>(p->cells_host) + n * 8);
      const int64_t* hy = hx + n;
      if (first) {
        std::memcpy(nodes, hn, n * 4);
        std::memcpy(particles, hp, n * 4);
        std::memcpy(px, hx, n * 8);
        std::memcpy(py, hy, n * 8);
      } else {
        for (size_t i = 0; i < n; ++i) {
          nodes[i] += hn[i];
          particles[i] += hp[i];
          px[i] += hx[i];
          py[i] += hy[i];
        }
      }
      first = false;
    });
    e->cells_pending = false;
  });
}

int fhpg_reduce_cells(fhpg_engine* e, int B, int32_t* nodes, int32_t* particles, int64_t* px,
                      int64_t* py) {
  if (e && (!nodes || !particles || !px || !py)) {
    g_last_error = "null output array";
    return FHPG_EINVAL;
  }
  const int rc = fhpg_reduce_cells_async(e, B);
  if (rc != FHPG_OK) return rc;
  if (e->cells_n == 0) {
    e->cells_pending = false;
    return FHPG_OK;
  }
  return fhpg_cells_wait(e, nodes, particles, px, py);
}

int fhpg_reduce_rows(fhpg_engine* e, int64_t* px, int32_t* fluid) {
  return guarded([&] {
    need(e);
    if (!px || !fluid) invalid("null output array");
    each(e, [&](fhpg_engine* p) {
      const int lo = std::max(1, p->row_begin), hi = std::min(p->H - 1, p->row_end);
      if (hi <= lo) return;
      const size_t n = static_cast<size_t>(p->H - 2);
      void* d = nullptr;
      ck(cudaMallocAsync(&d, n * 12, p->stream), "cudaMallocAsync(rows)");
      long long* dx = static_cast<long long*>(d);
      int* df = reinterpret_cast<int*>(dx + n);
      if (p->planes && !p->scratch_valid)  // else: the exact uploaded bytes
        fhpg::launch_reduce_rows_planes(p->base(p->cur), p->pitch, p->W, p->nrows, p->row_begin,
                                        p->H, dx, df, p->stream);
      else
        fhpg::launch_reduce_rows(bytes_view(p), p->pitch, p->W, p->nrows, p->row_begin, p->H, dx,
                                 df, p->stream);
      ck(cudaGetLastError(), "rows launch");
      ck(cudaMemcpyAsync(px + (lo - 1), dx + (lo - 1), (hi - lo) * 8, cudaMemcpyDeviceToHost,
                         p->stream), "rows read");
      ck(cudaMemcpyAsync(fluid + (lo - 1), df + (lo - 1), (hi - lo) * 4, cudaMemcpyDeviceToHost,
                         p->stream), "rows read");
      ck(cudaFreeAsync(d, p->stream), "cudaFreeAsync(rows)");
      ck(cudaStreamSynchronize(p->stream), "rows sync");
    });
  });
}

int fhpg_halo(fhpg_engine* e, void** send_top, void** send_bottom, void** recv_top,
              void** recv_bottom, size_t* row_bytes) {
  return guarded([&] {
    need(e);
    single_only(e, "fhpg_halo");
    const Halo h = halo_of(e);
    if (send_top) *send_top = h.send_top;
    if (send_bottom) *send_bottom = h.send_bottom;
    if (recv_top) *recv_top = h.recv_top;
    if (recv_bottom) *recv_bottom = h.recv_bottom;
    if (row_bytes) *row_bytes = h.row_bytes;
  });
}

int fhpg_info(fhpg_engine* e, int* width, int* height, int* row_begin, int* row_end,
              int* fast_path, uint64_t* step_launches) {
  return guarded([&] {
    need(e);
    if (width) *width = e->W;
    if (height) *height = e->H;
    if (row_begin) *row_begin = e->row_begin;
    if (row_end) *row_end = e->row_end;
    const fhpg_engine* p0 = e->multi() ? e->parts[0] : e;
    if (fast_path)
      *fast_path = p0->planes ? 2 : (p0->path_pref != 2 && fhpg::fast_path_ok(p0->W)) ? 1 : 0;
    uint64_t n = 0;
    if (e->multi())
      for (const fhpg_engine* p : e->parts) n += p->launches;
    else
      n = e->launches;
    if (step_launches) *step_launches = n;
  });
}

int fhpg_strips(fhpg_engine* e, int* n_strips, int* row_begin, int* row_end, int* device) {
  return guarded([&] {
    need(e);
    const int n = e->multi() ? static_cast<int>(e->parts.size()) : 1;
    if (n_strips) *n_strips = n;
    for (int i = 0; i < n; ++i) {
      const fhpg_engine* p = e->multi() ? e->parts[i] : e;
      if (row_begin) row_begin[i] = p->row_begin;
      if (row_end) row_end[i] = p->row_end;
      if (device) device[i] = p->device;
    }
  });
}

int fhpg_force_generic(fhpg_engine* e, int on) {
  return guarded([&] {
    need(e);
    each(e, [&](fhpg_engine* p) {
      p->path_pref = on ? 2 : 0;
      sync_layout(p);
    });
  });
}

int fhpg_debug_key_span(fhpg_engine* e, uint32_t rows) {
  return guarded([&] {
    need(e);
    each(e, [&](fhpg_engine* p) { p->span_cap = rows; });
  });
}

int fhpg_select_path(fhpg_engine* e, int path) {
  return guarded([&] {
    need(e);
    if (path < 0 || path > 3)
      invalid("path must be 0 (auto), 1 (byte fast path), 2 (generic) or 3 (streaming kernels only)");
    each(e, [&](fhpg_engine* p) {
      p->path_pref = path;
      sync_layout(p);
    });
  });
}

int fhpg_resident_depth(fhpg_engine* e, uint64_t thr, int* depth) {
  return guarded([&] {
    need(e);
    if (!depth) invalid("depth is null");
    int rpc = 0, grid = 0;
    *depth = (!e->multi() && e->planes && e->path_pref == 0 && e->row_begin == 0 &&
              e->row_end == e->H)
                 ? fhpg::resident_plan(e->W, e->H, thr, e->num_sms, &rpc, &grid)
                 : 0;
  });
}

}  // extern "C"
