// Drop-in proof: the reference library (proj/core, built from its own
// sources with integration/backend_cuda.patch applied) running
// Backend::Cuda through its own fhp::run / fhp::advance, against its own CPU
// backends. Built by integration/Makefile into oracle/_ref/dropin/.
//
//  1. acceptance criterion 3's 24 deterministic configs (acceptance.cpp:58-97:
//     same generator) — Scalar vs Cuda digests and forcing swaps;
//  2. "all four backends agree on one config" (test_backends.cpp:161-171)
//     with Cuda as a fifth;
//  3. the bit-plane path through the drop-in: FHP-III (data/fhp3.fhptab,
//     read by the reference's own read_table_file) at 2048 x 258, forcing,
//     Strips x N threads vs Cuda, and Cuda with gpus = 2 (two strips);
//  4. optional (argv[1] == "e2e"): fhp::advance(Backend::Cuda) at the cfg4
//     shape (16384^2, FHP-III), host Lattice in, host Lattice out, timed.
// Prints one JSON line per part and exits 1 on any mismatch.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <string>
#include <thread>

#include "fhp/bench.hpp"
#include "fhp/collision.hpp"
#include "fhp/lattice.hpp"
#include "fhp/rng.hpp"
#include "fhp/step.hpp"

using namespace fhp;

namespace {

int failures = 0;

std::uint64_t digest_of(SimConfig cfg, Backend b, std::uint64_t* swaps) {
  cfg.backend = b;
  const RunResult r = run(cfg);
  if (swaps) *swaps = r.forcing_swaps;
  return state_digest(r.lattice);
}

void criterion3() {
  const double force_ps[] = {0.0, 0.01, 0.2};
  const int thread_choices[] = {1, 2, 4, 7};
  const int lane_choices[] = {16, 32, 64};
  int mismatches = 0;
  for (int i = 0; i < 24; ++i) {
    const auto pick = [&](int salt, int mod) {
      return static_cast<int>(rng::mix64(1000 + i * 16 + salt) % mod);
    };
    SimConfig cfg;
    cfg.width = 8 + pick(0, 121);
    cfg.height = 8 + pick(1, 89);
    cfg.steps = 10 + pick(2, 191);
    cfg.fill_density = 0.35;
    cfg.force_p = force_ps[pick(3, 3)];
    cfg.seed = rng::mix64(i);
    cfg.threads = std::min(thread_choices[pick(4, 4)], cfg.height - 2);
    cfg.lanes = lane_choices[pick(5, 3)];
    cfg.tile_x = 1 + pick(6, 24);
    cfg.tile_y = 1 + pick(7, 12);
    std::uint64_t s0 = 0, s1 = 0;
    const std::uint64_t d0 = digest_of(cfg, Backend::Scalar, &s0);
    const std::uint64_t d1 = digest_of(cfg, Backend::Cuda, &s1);
    if (d0 != d1 || s0 != s1) ++mismatches;
  }
  std::printf("{\"part\": \"acceptance criterion 3 (24 configs), Scalar vs Cuda\", \"mismatches\": %d}\n",
              mismatches);
  failures += mismatches;
}

void all_backends() {
  SimConfig cfg;
  cfg.width = 48;
  cfg.height = 33;
  cfg.fill_density = 0.35;
  cfg.seed = 5;
  cfg.force_p = 0.01;
  cfg.threads = 4;
  cfg.tile_x = 7;
  cfg.tile_y = 5;
  cfg.steps = 60;
  const Backend all[] = {Backend::Scalar, Backend::Lanes, Backend::Strips, Backend::Tiles, Backend::Cuda};
  std::uint64_t d[5];
  for (int b = 0; b < 5; ++b) d[b] = digest_of(cfg, all[b], nullptr);
  const bool ok = std::all_of(d, d + 5, [&](std::uint64_t v) { return v == d[0]; });
  std::printf("{\"part\": \"all backends on one config (test_backends.cpp:161-171) + Cuda\", "
              "\"digest\": \"%#018llx\", \"agree\": %s}\n",
              static_cast<unsigned long long>(d[0]), ok ? "true" : "false");
  failures += ok ? 0 : 1;
}

void planes_path(const std::string& table_file) {
  SimConfig cfg;
  cfg.width = 2048;
  cfg.height = 258;
  cfg.fill_density = 0.2;
  cfg.seed = 3;
  cfg.force_p = 0.01;
  cfg.steps = 40;
  cfg.table_file = table_file;
  cfg.threads = static_cast<int>(std::max(1u, std::thread::hardware_concurrency()));
  std::uint64_t s0 = 0, s1 = 0, s2 = 0;
  const std::uint64_t d0 = digest_of(cfg, Backend::Strips, &s0);
  const std::uint64_t d1 = digest_of(cfg, Backend::Cuda, &s1);
  cfg.gpus = 2;  // two row strips (on GPUs 0 and 1 when present)
  const std::uint64_t d2 = digest_of(cfg, Backend::Cuda, &s2);
  const bool ok = d0 == d1 && d0 == d2 && s0 == s1 && s0 == s2;
  std::printf("{\"part\": \"FHP-III 2048x258 p=0.01 40 steps: Strips vs Cuda vs Cuda(gpus=2)\", "
              "\"digest\": \"%#018llx\", \"swaps\": %llu, \"agree\": %s}\n",
              static_cast<unsigned long long>(d0), static_cast<unsigned long long>(s0),
              ok ? "true" : "false");
  failures += ok ? 0 : 1;
}

void e2e(const std::string& table_file, int steps) {
  SimConfig cfg;
  cfg.width = 16384;
  cfg.height = 16384;
  cfg.fill_density = 0.2;
  cfg.seed = 4;
  cfg.table_file = table_file;
  cfg.backend = Backend::Cuda;
  const CollisionTable table = load_table(read_table_file(table_file));
  Lattice lat = init_lattice(cfg);
  advance(lat, table, cfg, 0, 5);  // warm-up: engine created and cached
  const auto t0 = std::chrono::steady_clock::now();
  advance(lat, table, cfg, 5, steps);
  const double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  std::printf("{\"part\": \"e2e: fhp::advance(Backend::Cuda) on a host Lattice, cfg4 16384^2 FHP-III\", "
              "\"steps\": %d, \"seconds\": %.6f, \"gsups\": %.3f, \"digest\": \"%#018llx\"}\n",
              steps, secs, 16384.0 * 16384.0 * steps / secs / 1e9,
              static_cast<unsigned long long>(state_digest(lat)));
}

}  // namespace

int main(int argc, char** argv) {
  const std::string mode = argc > 1 ? argv[1] : "check";
  const std::string table_file = argc > 2 ? argv[2] : "data/fhp3.fhptab";
  try {
    if (mode == "check" || mode == "all") {
      criterion3();
      all_backends();
      planes_path(table_file);
    }
    if (mode == "e2e" || mode == "all") e2e(table_file, argc > 3 ? std::atoi(argv[3]) : 20);
  } catch (const std::exception& e) {
    std::printf("{\"error\": \"%s\"}\n", e.what());
    return 1;
  }
  std::printf("{\"failures\": %d}\n", failures);
  return failures ? 1 : 0;
}
