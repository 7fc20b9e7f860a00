// fhp_b200/step.hpp — the evolution entry points (mirrors
// proj/core/include/fhp/step.hpp:46-68).
#pragma once

#include <cstdint>
#include <functional>
#include <vector>

#include "fhp_b200/collision.hpp"
#include "fhp_b200/config.hpp"
#include "fhp_b200/engine.hpp"
#include "fhp_b200/lattice.hpp"
#include "fhp_b200/observables.hpp"

namespace fhp_b200 {

// Drop-in for fhp::advance (step.cpp:103-133) with cfg.backend == Cuda:
// uploads lat.src() and the mask, runs step_count steps with global indices
// first_step.. on the device, downloads into lat.src(). step_count <= 0 is a
// no-op. Returns the accepted forcing swaps. Other backends throw
// std::invalid_argument (they live in the reference).
std::uint64_t advance(Lattice& lat, const CollisionTable& table, const SimConfig& cfg,
                      int first_step, int step_count);

struct ObservableSample {
  int step = 0;
  std::int64_t mass = 0;
  MomentumVec momentum{};
};

struct RunResult {
  Lattice lattice;
  std::vector<ObservableSample> series;
  std::uint64_t forcing_swaps = 0;
};

// Host-lattice dump callback (the reference's DumpFn, step.hpp:62): gets a
// downloaded Lattice at every dump point.
using DumpFn = std::function<void(int step, const Lattice&)>;
// Device dump callback: gets the resident engine (reduce on the GPU, no
// lattice download).
using DeviceDumpFn = std::function<void(int step, const Engine&)>;

// fhp::run (step.cpp:135-175) on a device-resident lattice: init on the
// device, sample(0), advance in dump_every chunks, sample + dump, final
// sample / dump. The state never leaves HBM except for DumpFn and the final
// RunResult::lattice.
RunResult run(const SimConfig& cfg, const CollisionTable& table, const DumpFn& dump = {},
              const DeviceDumpFn& device_dump = {});
RunResult run(const SimConfig& cfg);

// run() with asynchronous coarse-grain dumps: every dump_every steps (and at
// the end) fn gets the coarse_grain(block) field of that step; the sums are
// reduced on the device and copied back while the next chunk of steps runs.
using CellDumpFn = std::function<void(int step, const FlowField& field)>;
RunResult run_cell_dumps(const SimConfig& cfg, const CollisionTable& table, int block,
                         const CellDumpFn& fn);

}  // namespace fhp_b200
