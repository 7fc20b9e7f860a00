// advance (the Backend::Cuda shim of fhp::advance, step.cpp:103-133) and
// run (step.cpp:135-175) on a device-resident lattice.
#include "fhp_b200/step.hpp"

#include <algorithm>
#include <stdexcept>

#include "fhp_b200/checkpoint.hpp"
#include "fhp_b200/observables.hpp"

namespace fhp_b200 {

std::uint64_t advance(Lattice& lat, const CollisionTable& table, const SimConfig& cfg,
                      int first_step, int step_count) {
  if (cfg.backend != Backend::Cuda)
    throw std::invalid_argument(std::string("backend '") + backend_name(cfg.backend) +
                                "' is not provided by fhp_b200 (use Backend::Cuda)");
  if (step_count <= 0) return 0;  // backends.cpp:157: the lattice is not touched
  Engine e(lat.width(), lat.height());
  e.set_table(table);
  e.upload(lat);
  const std::uint64_t swaps = e.advance(cfg.seed, cfg.force_p, first_step, step_count);
  e.download(lat);
  return swaps;
}

RunResult run(const SimConfig& cfg, const CollisionTable& table, const DumpFn& dump,
              const DeviceDumpFn& device_dump) {
  cfg.validate();
  if (cfg.backend != Backend::Cuda)
    throw std::invalid_argument(std::string("backend '") + backend_name(cfg.backend) +
                                "' is not provided by fhp_b200 (use Backend::Cuda)");
  Engine e(cfg.width, cfg.height);
  e.set_table(table);
  Lattice host(cfg.width, cfg.height);
  int step = 0;
  std::uint64_t swaps0 = 0;
  if (!cfg.resume_file.empty()) {
    // Resume: the checkpoint replaces init (and geometry: its bit 7 is the mask).
    const Checkpoint ck = read_checkpoint_file(cfg.resume_file);
    if (ck.width != cfg.width || ck.height != cfg.height)
      throw std::invalid_argument("resume: checkpoint is " + std::to_string(ck.width) + "x" +
                                  std::to_string(ck.height) + ", config is " +
                                  std::to_string(cfg.width) + "x" + std::to_string(cfg.height));
    if (ck.seed != cfg.seed || ck.force_p != cfg.force_p)
      throw std::invalid_argument("resume: seed / force-p differ from the checkpoint's");
    if (ck.table.entries != table.entries)
      throw std::invalid_argument("resume: collision table differs from the checkpoint's");
    if (ck.next_step < 0 || ck.next_step > cfg.steps)
      throw std::invalid_argument("resume: checkpoint step " + std::to_string(ck.next_step) +
                                  " is outside [0, steps]");
    restore_checkpoint(e, ck);
    for (int r = 0; r < cfg.height; ++r)
      for (int x = 1; x <= cfg.width; ++x)
        if (ck.state[static_cast<std::size_t>(r) * cfg.width + (x - 1)] & kObstacleBit)
          host.set_obstacle(r, x, true);
    step = static_cast<int>(ck.next_step);
    swaps0 = ck.swaps;
  } else {
    if (!cfg.geometry_file.empty()) {
      const auto g = read_geometry_file(cfg.geometry_file);
      if (static_cast<int>(g.size()) != cfg.height) throw std::runtime_error("geometry height mismatch");
      for (int r = 0; r < cfg.height; ++r) {
        if (static_cast<int>(g[r].size()) != cfg.width)
          throw std::runtime_error("geometry width mismatch on row " + std::to_string(r));
        for (int x = 1; x <= cfg.width; ++x)
          if (g[r][x - 1] == '#') host.set_obstacle(r, x, true);
      }
      e.set_obstacles(host.obstacle_mask() + 1, static_cast<std::size_t>(host.stride()));
    }
    if (cfg.fill_density < 0.0 || cfg.fill_density > 1.0)
      throw std::invalid_argument("fill_density must be in [0,1]");
    e.init(cfg.seed, cfg.fill_density);
    if (cfg.clear_rest) {
      e.download(host);
      for (int r = 0; r < cfg.height; ++r)
        for (int x = 1; x <= cfg.width; ++x) host.set_node(r, x, host.node(r, x) & ~kRestBit);
      e.upload(host.src() + 1, static_cast<std::size_t>(host.stride()));
    }
  }

  RunResult result{Lattice(cfg.width, cfg.height), {}, swaps0};
  auto sample = [&](int s) {
    result.series.push_back({s, e.total_mass(), e.total_momentum()});
  };
  auto do_dump = [&](int s) {
    if (device_dump) device_dump(s, e);
    if (dump) {
      e.download(host);
      dump(s, host);
    }
  };
  auto checkpoint = [&](int s) {
    write_checkpoint_file(cfg.checkpoint_file,
                          capture_checkpoint(e, s, cfg.seed, cfg.force_p, result.forcing_swaps, table));
  };
  // Chunks end at every dump and checkpoint boundary.
  auto next_stop = [&](int s) {
    int t = cfg.steps;
    if (cfg.dump_every > 0) t = std::min(t, (s / cfg.dump_every + 1) * cfg.dump_every);
    if (cfg.checkpoint_every > 0 && !cfg.checkpoint_file.empty())
      t = std::min(t, (s / cfg.checkpoint_every + 1) * cfg.checkpoint_every);
    return t;
  };
  const int first = step;
  sample(step);
  int last_dumped = -1;
  while (step < cfg.steps) {
    const int stop = next_stop(step);
    result.forcing_swaps += e.advance(cfg.seed, cfg.force_p, step, stop - step);
    step = stop;
    if (cfg.dump_every > 0 && step % cfg.dump_every == 0) {
      sample(step);
      do_dump(step);
      last_dumped = step;
    }
    if (!cfg.checkpoint_file.empty() && cfg.checkpoint_every > 0 && step % cfg.checkpoint_every == 0)
      checkpoint(step);
  }
  if (last_dumped != cfg.steps) {
    if (cfg.steps > first) sample(cfg.steps);
    do_dump(cfg.steps);
  }
  if (!cfg.checkpoint_file.empty()) checkpoint(cfg.steps);
  // Obstacle mask of the result lattice = the geometry + walls.
  for (int r = 0; r < cfg.height; ++r)
    for (int x = 1; x <= cfg.width; ++x)
      if (host.obstacle(r, x) || r == 0 || r == cfg.height - 1) result.lattice.set_obstacle(r, x, true);
  e.download(result.lattice);
  return result;
}

RunResult run(const SimConfig& cfg) { return run(cfg, table_for(cfg)); }

}  // namespace fhp_b200
