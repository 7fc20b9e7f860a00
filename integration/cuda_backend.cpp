// The Backend::Cuda shim of fhp::advance (installed into the reference's
// src/ by integration/Makefile). It is the whole integration: a cached
// engine of the C ABI (include/fhpg.h) per calling thread.
#include "fhp/cuda_backend.hpp"

#include <array>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <vector>

#include "fhpg.h"

namespace fhp {

namespace {

void fhpg_check(int rc) {
  if (rc == FHPG_OK) return;
  if (rc == FHPG_EINVAL) throw std::invalid_argument(fhpg_last_error());
  throw std::runtime_error(fhpg_last_error());
}

struct EngineCache {
  int width = 0, height = 0, gpus = 0;
  std::array<std::uint8_t, 512> table{};
  bool table_set = false;
  std::unique_ptr<fhpg_engine, void (*)(fhpg_engine*)> engine{nullptr, fhpg_destroy};

  fhpg_engine* get(int w, int h, int n, const CollisionTable& t) {
    if (!engine || w != width || h != height || n != gpus) {
      engine.reset();
      fhpg_engine* e = nullptr;
      if (n > 1) {
        // strip i on GPU i, wrapping around when there are fewer GPUs
        int ndev = 0;
        fhpg_check(fhpg_device_count(&ndev));
        std::vector<int> dev(static_cast<std::size_t>(n));
        for (int i = 0; i < n; ++i) dev[i] = ndev > 0 ? i % ndev : 0;
        fhpg_check(fhpg_create_multi(w, h, n, dev.data(), &e));
      } else {
        fhpg_check(fhpg_create(w, h, &e));
      }
      engine.reset(e);
      width = w;
      height = h;
      gpus = n;
      table_set = false;
    }
    if (!table_set || std::memcmp(table.data(), t.entries.data(), 512) != 0) {
      fhpg_check(fhpg_set_table(engine.get(), t.entries.data()));
      std::memcpy(table.data(), t.entries.data(), 512);
      table_set = true;
    }
    return engine.get();
  }
};

}  // namespace

std::uint64_t cuda_advance(Lattice& lat, const CollisionTable& table, const SimConfig& cfg,
                           int first_step, int step_count) {
  if (step_count <= 0) return 0;  // the lattice is not touched (backends.cpp:157)
  thread_local EngineCache cache;
  fhpg_engine* e = cache.get(lat.width(), lat.height(), cfg.gpus, table);
  const std::size_t stride = static_cast<std::size_t>(lat.stride());  // W + 2
  fhpg_check(fhpg_set_obstacles(e, lat.obstacle_mask() + 1, stride));
  fhpg_check(fhpg_upload(e, lat.src() + 1, stride));  // interior columns 1..W, bit 7 included
  std::uint64_t swaps = 0;
  fhpg_check(fhpg_advance(e, cfg.seed, fhpg_bernoulli_threshold(cfg.force_p), first_step,
                          step_count, &swaps));
  fhpg_check(fhpg_download(e, lat.src() + 1, stride));
  return swaps;  // ghost columns and dst() are unspecified on exit, as for every backend
}

}  // namespace fhp
