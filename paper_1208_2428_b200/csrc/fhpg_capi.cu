// fhpg_capi.cu — the C ABI (include/fhpg.h): engine object, device memory,
// error mapping, and the step loop that drives the kernels.
#include <cstdio>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include <cuda_runtime.h>

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
  int path_pref = 0;                     // 0 auto, 1 byte fast path, 2 generic
  uint8_t* scratch = nullptr;            // nrows * pitch
  alignas(64) unsigned char tmap[2][4][128];  // TMA descriptors of buf[0], buf[1] (planes)
  bool scratch_valid = false;
  uint8_t* table = nullptr;              // 512 bytes
  uint64_t* zkeys = nullptr;             // [parity][purpose][W]
  unsigned long long* swaps = nullptr;
  long long* acc = nullptr;              // reduction scratch (3)
  cudaStream_t stream = nullptr;
  cudaStream_t own_stream = nullptr;
  bool table_set = false;
  bool normalized = true;                // state bit 7 == mask
  int num_sms = 148;
  uint64_t launches = 0;
  int64_t keys_step = -1;                // step whose column keys are in keys(step & 1)
  uint64_t keys_seed = 0;
  bool keys_force = false;

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
  cudaFree(e->buf[0]);
  cudaFree(e->buf[1]);
  cudaFree(e->mask);
  cudaFree(e->scratch);
  cudaFree(e->table);
  cudaFree(e->zkeys);
  cudaFree(e->swaps);
  cudaFree(e->acc);
  if (e->own_stream) cudaStreamDestroy(e->own_stream);
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
    // Room for the bit-plane rows (W + 256 bytes) when the width allows them.
    e->pitch = (static_cast<size_t>(W) + 15) / 16 * 16 + (fhpg::planes_ok(W) ? 256 : 0);
    // halo above, rows, halo below, 3 spare zero rows the streaming kernels may prefetch
    const size_t bytes = (static_cast<size_t>(e->nrows) + 5) * e->pitch;
    for (int i = 0; i < 2; ++i) {
      ck(cudaMalloc(&e->buf[i], bytes), "cudaMalloc(state)");
      ck(cudaMemset(e->buf[i], 0, bytes), "cudaMemset(state)");
      for (int kind = 0; kind < 4 && fhpg::planes_ok(W); ++kind)
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
    ck(cudaStreamCreateWithFlags(&e->own_stream, cudaStreamNonBlocking), "cudaStreamCreate");
    e->stream = e->own_stream;
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
  return e->table_set && e->table_planes && e->path_pref == 0 && fhpg::planes_ok(e->W);
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
    e->launches += fhpg::launch_step_planes(a, e->tmap[which][0], e->tmap[which ^ 1][1],
                                            e->tmap[which ^ 1][2], e->tmap[which][3],
                                            e->num_sms, e->stream);
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
    e->normalized = true;
  }
  const bool force = thr != 0;
  const uint64_t s0 = static_cast<uint64_t>(first);
  launch_column_keys(e->keys(s0 & 1, 0), force ? e->keys(s0 & 1, 1) : nullptr,
                     step_key(seed, kChirality, s0), step_key(seed, kForcing, s0), e->W, st);
  ck(cudaGetLastError(), "column_keys launch");
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
    e->normalized = true;
  }
  const bool force = thr != 0;
  const uint64_t s = static_cast<uint64_t>(step);
  if (e->keys_step != step || e->keys_seed != seed || (force && !e->keys_force)) {
    launch_column_keys(e->keys(s & 1, 0), force ? e->keys(s & 1, 1) : nullptr,
                       step_key(seed, kChirality, s), step_key(seed, kForcing, s), e->W, st);
    ck(cudaGetLastError(), "column_keys launch");
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
}

void copy_rows_h2d(uint8_t* dev, size_t pitch, const uint8_t* host, size_t stride, int W,
                   int rows, cudaStream_t st) {
  ck(cudaMemcpy2DAsync(dev, pitch, host, stride, W, rows, cudaMemcpyHostToDevice, st),
     "cudaMemcpy2D H2D");
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

void fhpg_destroy(fhpg_engine* e) {
  if (!e) return;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(e->device);
  cudaStreamSynchronize(e->stream);
  release(e);
  cudaSetDevice(prev);
}

int fhpg_set_stream(fhpg_engine* e, void* s) {
  return guarded([&] {
    need(e);
    e->stream = static_cast<cudaStream_t>(s);  // NULL = the legacy default stream
  });
}

int fhpg_set_table(fhpg_engine* e, const uint8_t* t) {
  return guarded([&] {
    need(e);
    if (!t) invalid("null table");
    for (int i = 0; i < 512; ++i)
      if ((t[i] & 0x80u) != (i & 0x80)) invalid("collision table: entry " + std::to_string(i) + " changes the obstacle bit");
    DeviceGuard g(e->device);
    ck(cudaMemcpyAsync(e->table, t, 512, cudaMemcpyHostToDevice, e->stream), "table upload");
    ck(cudaStreamSynchronize(e->stream), "table upload sync");
    e->table_set = true;
    // The bit-plane kernels evaluate FHP-III, FHP-I and the reference's
    // DEFAULT rule as circuits (fhpg_planes_rules.cuh); any other table runs
    // the byte LUT path.
    e->table_planes = false;
    for (const int v : {FHPG_RULES_FHP_III, FHPG_RULES_FHP_I, FHPG_RULES_DEFAULT}) {
      uint8_t ref[512];
      fhpg_build_table(v, ref);
      if (std::memcmp(t, ref, 512) == 0) {
        e->table_planes = true;
        e->planes_rule = v;
        break;
      }
    }
    sync_layout(e);
  });
}

int fhpg_set_obstacles(fhpg_engine* e, const uint8_t* mask, size_t stride) {
  return guarded([&] {
    need(e);
    if (!mask) invalid("null mask");
    if (stride < static_cast<size_t>(e->W)) invalid("stride < width");
    DeviceGuard g(e->device);
    // Raw bytes (nonzero = solid) go straight to the device mask.
    copy_rows_h2d(e->mask, e->pitch, mask, stride, e->W, e->nrows, e->stream);
    // Lattice::set_obstacle also sets / clears bit 7 of the node (lattice.cpp:25-29).
    uint8_t* v = bytes_view(e);
    fhpg::launch_apply_mask(v, e->mask, e->pitch, e->W, e->nrows, e->stream);
    ck(cudaGetLastError(), "apply_mask launch");
    if (e->planes) pack_from_scratch(e);
    ck(cudaStreamSynchronize(e->stream), "mask sync");
  });
}

int fhpg_upload(fhpg_engine* e, const uint8_t* state, size_t stride) {
  return guarded([&] {
    need(e);
    if (!state) invalid("null state");
    if (stride < static_cast<size_t>(e->W)) invalid("stride < width");
    DeviceGuard g(e->device);
    if (e->planes) {
      // The byte image stays exact until the first step; the planes take
      // bit 7 from the mask like the reference's motion pass.
      need_scratch(e);
      copy_rows_h2d(e->scratch, e->pitch, state, stride, e->W, e->nrows, e->stream);
      e->scratch_valid = true;
      pack_from_scratch(e);
    } else {
      copy_rows_h2d(e->base(e->cur), e->pitch, state, stride, e->W, e->nrows, e->stream);
      e->normalized = false;
    }
    ck(cudaStreamSynchronize(e->stream), "upload sync");
  });
}

int fhpg_download(fhpg_engine* e, uint8_t* state, size_t stride) {
  return guarded([&] {
    need(e);
    if (!state) invalid("null state");
    if (stride < static_cast<size_t>(e->W)) invalid("stride < width");
    DeviceGuard g(e->device);
    ck(cudaMemcpy2DAsync(state, stride, bytes_view(e), e->pitch, e->W, e->nrows,
                         cudaMemcpyDeviceToHost, e->stream),
       "cudaMemcpy2D D2H");
    ck(cudaStreamSynchronize(e->stream), "download sync");
  });
}

int fhpg_init(fhpg_engine* e, uint64_t seed, double fill_density) {
  return guarded([&] {
    need(e);
    // lattice.cpp:58-60
    if (!(fill_density >= 0.0 && fill_density <= 1.0)) invalid("fill_density must be in [0,1]");
    DeviceGuard g(e->device);
    if (e->planes) need_scratch(e);
    uint8_t* target = e->planes ? e->scratch : e->base(e->cur);
    fhpg::launch_init(target, e->mask, e->pitch, e->W, e->nrows, e->row_begin, e->H,
                      seed, fhpg::bernoulli_threshold(fill_density), e->stream);
    ck(cudaGetLastError(), "init launch");
    // Walls join the obstacle mask (init_impl calls set_obstacle on them).
    for (int r = 0; r < e->nrows; ++r) {
      const long long gr = e->row_begin + r;
      if (gr == 0 || gr == e->H - 1)
        ck(cudaMemsetAsync(e->mask + static_cast<size_t>(r) * e->pitch, 1, e->W, e->stream),
           "wall mask");
    }
    if (e->planes) {
      e->scratch_valid = true;
      pack_from_scratch(e);
    }
    ck(cudaStreamSynchronize(e->stream), "init sync");
    e->normalized = true;
  });
}

int fhpg_advance_async(fhpg_engine* e, uint64_t seed, uint64_t thr, int64_t first, int64_t count) {
  return guarded([&] {
    need(e);
    if (count <= 0) return;  // backends.cpp:157 — no-op, state untouched
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
    DeviceGuard g(e->device);
    ck(cudaMemsetAsync(e->swaps, 0, sizeof(unsigned long long), e->stream), "swap reset");
    step_loop(e, seed, thr, first, count);
    unsigned long long s = 0;
    ck(cudaMemcpyAsync(&s, e->swaps, sizeof s, cudaMemcpyDeviceToHost, e->stream), "swap read");
    ck(cudaStreamSynchronize(e->stream), "advance sync");
    if (swaps) *swaps = s;
  });
}

int fhpg_advance_part(fhpg_engine* e, uint64_t seed, uint64_t thr, int64_t step, int part) {
  return guarded([&] {
    need(e);
    DeviceGuard g(e->device);
    step_part(e, seed, thr, step, part);
  });
}

int fhpg_swaps(fhpg_engine* e, uint64_t* swaps, int reset) {
  return guarded([&] {
    need(e);
    DeviceGuard g(e->device);
    unsigned long long s = 0;
    ck(cudaMemcpyAsync(&s, e->swaps, sizeof s, cudaMemcpyDeviceToHost, e->stream), "swap read");
    if (reset) ck(cudaMemsetAsync(e->swaps, 0, sizeof s, e->stream), "swap reset");
    ck(cudaStreamSynchronize(e->stream), "swap sync");
    if (swaps) *swaps = s;
  });
}

int fhpg_synchronize(fhpg_engine* e) {
  return guarded([&] {
    need(e);
    DeviceGuard g(e->device);
    ck(cudaStreamSynchronize(e->stream), "synchronize");
  });
}

int fhpg_reduce_global(fhpg_engine* e, int64_t* mass, int64_t* px, int64_t* py) {
  return guarded([&] {
    need(e);
    DeviceGuard g(e->device);
    ck(cudaMemsetAsync(e->acc, 0, sizeof(long long) * 3, e->stream), "acc reset");
    fhpg::launch_reduce_global(bytes_view(e), e->pitch, e->W, e->nrows, e->acc, e->stream);
    ck(cudaGetLastError(), "reduce launch");
    long long h[3];
    ck(cudaMemcpyAsync(h, e->acc, sizeof h, cudaMemcpyDeviceToHost, e->stream), "acc read");
    ck(cudaStreamSynchronize(e->stream), "reduce sync");
    if (mass) *mass = h[0];
    if (px) *px = h[1];
    if (py) *py = h[2];
  });
}

int fhpg_reduce_cells(fhpg_engine* e, int B, int32_t* nodes, int32_t* particles, int64_t* px,
                      int64_t* py) {
  return guarded([&] {
    need(e);
    if (B < 1) invalid("block size must be >= 1");  // observables.cpp:50
    if (!nodes || !particles || !px || !py) invalid("null output array");
    DeviceGuard g(e->device);
    const size_t cx = (static_cast<size_t>(e->W) + B - 1) / B;
    const size_t cy = (static_cast<size_t>(e->H) - 2 + B - 1) / B;
    const size_t n = cx * cy;
    if (n == 0) return;
    void* d = nullptr;
    ck(cudaMallocAsync(&d, n * 24, e->stream), "cudaMallocAsync(cells)");
    int* dn = static_cast<int*>(d);
    int* dp = dn + n;
    long long* dx = reinterpret_cast<long long*>(static_cast<char*>(d) + n * 8);
    long long* dy = dx + n;
    ck(cudaMemsetAsync(d, 0, n * 24, e->stream), "cells reset");
    fhpg::launch_reduce_cells(bytes_view(e), e->pitch, e->W, e->nrows, e->row_begin, e->H, B,
                              dn, dp, dx, dy, e->stream);
    ck(cudaGetLastError(), "cells launch");
    ck(cudaMemcpyAsync(nodes, dn, n * 4, cudaMemcpyDeviceToHost, e->stream), "cells read");
    ck(cudaMemcpyAsync(particles, dp, n * 4, cudaMemcpyDeviceToHost, e->stream), "cells read");
    ck(cudaMemcpyAsync(px, dx, n * 8, cudaMemcpyDeviceToHost, e->stream), "cells read");
    ck(cudaMemcpyAsync(py, dy, n * 8, cudaMemcpyDeviceToHost, e->stream), "cells read");
    ck(cudaFreeAsync(d, e->stream), "cudaFreeAsync(cells)");
    ck(cudaStreamSynchronize(e->stream), "cells sync");
  });
}

int fhpg_reduce_rows(fhpg_engine* e, int64_t* px, int32_t* fluid) {
  return guarded([&] {
    need(e);
    if (!px || !fluid) invalid("null output array");
    DeviceGuard g(e->device);
    const int lo = std::max(1, e->row_begin), hi = std::min(e->H - 1, e->row_end);
    if (hi <= lo) return;
    const size_t n = static_cast<size_t>(e->H - 2);
    void* d = nullptr;
    ck(cudaMallocAsync(&d, n * 12, e->stream), "cudaMallocAsync(rows)");
    long long* dx = static_cast<long long*>(d);
    int* df = reinterpret_cast<int*>(dx + n);
    fhpg::launch_reduce_rows(bytes_view(e), e->pitch, e->W, e->nrows, e->row_begin, e->H, dx,
                             df, e->stream);
    ck(cudaGetLastError(), "rows launch");
    ck(cudaMemcpyAsync(px + (lo - 1), dx + (lo - 1), (hi - lo) * 8, cudaMemcpyDeviceToHost, e->stream), "rows read");
    ck(cudaMemcpyAsync(fluid + (lo - 1), df + (lo - 1), (hi - lo) * 4, cudaMemcpyDeviceToHost, e->stream), "rows read");
    ck(cudaFreeAsync(d, e->stream), "cudaFreeAsync(rows)");
    ck(cudaStreamSynchronize(e->stream), "rows sync");
  });
}

int fhpg_halo(fhpg_engine* e, void** send_top, void** send_bottom, void** recv_top,
              void** recv_bottom, size_t* row_bytes) {
  return guarded([&] {
    need(e);
    uint8_t* b = e->base(e->cur);
    if (send_top) *send_top = b;
    if (send_bottom) *send_bottom = b + static_cast<size_t>(e->nrows - 1) * e->pitch;
    if (recv_top) *recv_top = b - e->pitch;
    if (recv_bottom) *recv_bottom = b + static_cast<size_t>(e->nrows) * e->pitch;
    if (row_bytes) *row_bytes = e->planes ? fhpg::planes_row_bytes(e->W) : static_cast<size_t>(e->W);
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
    if (fast_path)
      *fast_path = e->planes ? 2 : (e->path_pref != 2 && fhpg::fast_path_ok(e->W)) ? 1 : 0;
    if (step_launches) *step_launches = e->launches;
  });
}

int fhpg_force_generic(fhpg_engine* e, int on) {
  return guarded([&] {
    need(e);
    DeviceGuard g(e->device);
    e->path_pref = on ? 2 : 0;
    sync_layout(e);
  });
}

int fhpg_select_path(fhpg_engine* e, int path) {
  return guarded([&] {
    need(e);
    if (path < 0 || path > 2) invalid("path must be 0 (auto), 1 (byte fast path) or 2 (generic)");
    DeviceGuard g(e->device);
    e->path_pref = path;
    sync_layout(e);
  });
}

}  // extern "C"
