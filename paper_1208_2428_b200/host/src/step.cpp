// advance (the Backend::Cuda shim of fhp::advance, step.cpp:103-133) and
// run (step.cpp:135-175) on a device-resident lattice.
#include "fhp_b200/step.hpp"

#include <algorithm>
#include <stdexcept>

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

  RunResult result{Lattice(cfg.width, cfg.height), {}, 0};
  auto sample = [&](int step) {
    result.series.push_back({step, e.total_mass(), e.total_momentum()});
  };
  auto do_dump = [&](int step) {
    if (device_dump) device_dump(step, e);
    if (dump) {
      e.download(host);
      dump(step, host);
    }
  };
  sample(0);
  const int chunk = cfg.dump_every > 0 ? cfg.dump_every : cfg.steps;
  int step = 0, last_dumped = -1;
  while (step < cfg.steps) {
    const int count = std::min(chunk, cfg.steps - step);
    result.forcing_swaps += e.advance(cfg.seed, cfg.force_p, step, count);
    step += count;
    if (cfg.dump_every > 0 && step % cfg.dump_every == 0) {
      sample(step);
      do_dump(step);
      last_dumped = step;
    }
  }
  if (last_dumped != cfg.steps) {
    if (cfg.steps > 0) sample(cfg.steps);
    do_dump(cfg.steps);
  }
  // Obstacle mask of the result lattice = the geometry + walls.
  for (int r = 0; r < cfg.height; ++r)
    for (int x = 1; x <= cfg.width; ++x)
      if (host.obstacle(r, x) || r == 0 || r == cfg.height - 1) result.lattice.set_obstacle(r, x, true);
  e.download(result.lattice);
  return result;
}

RunResult run(const SimConfig& cfg) { return run(cfg, table_for(cfg)); }

}  // namespace fhp_b200
