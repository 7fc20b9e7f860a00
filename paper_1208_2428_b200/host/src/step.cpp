// advance (the Backend::Cuda shim of fhp::advance, step.cpp:103-133) and
// run (step.cpp:135-175) on a device-resident lattice.
#include "fhp_b200/step.hpp"

#include <algorithm>
#include <array>
#include <memory>
#include <stdexcept>

#include "fhp_b200/checkpoint.hpp"
#include "fhp_b200/observables.hpp"

namespace fhp_b200 {

namespace {

void need_cuda(const SimConfig& cfg) {
  if (cfg.backend != Backend::Cuda)
    throw std::invalid_argument(std::string("backend '") + backend_name(cfg.backend) +
                                "' is not provided by fhp_b200 (use Backend::Cuda)");
}

// One GPU (cfg.device) or cfg.gpus row strips (fhpg_create_multi).
Engine make_engine(const SimConfig& cfg) {
  if (cfg.gpus > 1) return Engine(cfg.width, cfg.height, cfg.gpus, cfg.devices);
  return Engine(cfg.width, cfg.height, 0, cfg.height, cfg.device);
}

// The drop-in's engine, kept between calls (the reference's Lattice is
// uploaded and downloaded every call, the device buffers, streams and TMA
// descriptors are not rebuilt): keyed by lattice shape and device layout,
// the table re-sent only when it changes.
struct CachedEngine {
  int width = 0, height = 0, device = -1, gpus = 0;
  std::vector<int> devices;
  std::array<NodeState, 512> table{};
  bool table_set = false;
  std::unique_ptr<Engine> engine;
};

Engine& cached_engine(const SimConfig& cfg, int width, int height, const CollisionTable& table) {
  thread_local CachedEngine c;
  if (!c.engine || c.width != width || c.height != height || c.device != cfg.device ||
      c.gpus != cfg.gpus || c.devices != cfg.devices) {
    c.engine.reset();
    SimConfig shape = cfg;
    shape.width = width;
    shape.height = height;
    c.engine = std::make_unique<Engine>(make_engine(shape));
    c.width = width;
    c.height = height;
    c.device = cfg.device;
    c.gpus = cfg.gpus;
    c.devices = cfg.devices;
    c.table_set = false;
  }
  if (!c.table_set || c.table != table.entries) {
    c.engine->set_table(table);
    c.table = table.entries;
    c.table_set = true;
  }
  return *c.engine;
}

}  // namespace

std::uint64_t advance(Lattice& lat, const CollisionTable& table, const SimConfig& cfg,
                      int first_step, int step_count) {
  need_cuda(cfg);
  if (step_count <= 0) return 0;  // backends.cpp:157: the lattice is not touched
  Engine& e = cached_engine(cfg, lat.width(), lat.height(), table);
  e.upload(lat);
  const std::uint64_t swaps = e.advance(cfg.seed, cfg.force_p, first_step, step_count);
  e.download(lat);
  return swaps;
}

RunResult run(const SimConfig& cfg, const CollisionTable& table, const DumpFn& dump,
              const DeviceDumpFn& device_dump) {
  cfg.validate();
  need_cuda(cfg);
  Engine e = make_engine(cfg);
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

// run() with asynchronous coarse-grain dumps (the dump pipeline of
// step.cpp:150-166 / fhp_main.cpp:52-59): at every dump point the cell sums
// are requested on the device behind the chunk of steps that ends there, the
// next chunk is enqueued at once, and the previous dump is finalised and
// handed to the callback on the host while the GPU runs that chunk.
RunResult run_cell_dumps(const SimConfig& cfg, const CollisionTable& table, int block,
                         const CellDumpFn& fn) {
  cfg.validate();
  need_cuda(cfg);
  if (block < 1) throw std::invalid_argument("block size must be >= 1");
  Engine e = make_engine(cfg);
  e.set_table(table);
  if (!cfg.geometry_file.empty()) {
    const auto g = read_geometry_file(cfg.geometry_file);
    if (static_cast<int>(g.size()) != cfg.height) throw std::runtime_error("geometry height mismatch");
    std::vector<std::uint8_t> mask(static_cast<std::size_t>(cfg.width) * cfg.height, 0);
    for (int r = 0; r < cfg.height; ++r) {
      if (static_cast<int>(g[r].size()) != cfg.width)
        throw std::runtime_error("geometry width mismatch on row " + std::to_string(r));
      for (int x = 0; x < cfg.width; ++x) mask[static_cast<std::size_t>(r) * cfg.width + x] = g[r][x] == '#';
    }
    e.set_obstacles(mask.data(), static_cast<std::size_t>(cfg.width));
  }
  e.init(cfg.seed, cfg.fill_density);
  RunResult result{Lattice(cfg.width, cfg.height), {}, 0};
  auto sample = [&](int s) { result.series.push_back({s, e.total_mass(), e.total_momentum()}); };
  sample(0);
  e.swaps(true);
  int pending = -1;  // step of the requested, not yet delivered dump
  auto deliver = [&] {
    if (pending < 0) return;
    const FlowField f = finalize_cells(e.collect_cells(), block);
    if (fn) fn(pending, f);
    pending = -1;
  };
  int step = 0;
  while (step < cfg.steps) {
    const int stop = cfg.dump_every > 0
                         ? std::min(cfg.steps, (step / cfg.dump_every + 1) * cfg.dump_every)
                         : cfg.steps;
    e.advance_async(cfg.seed, cfg.force_p, step, stop - step);
    deliver();  // host work while the chunk runs
    step = stop;
    e.request_cells(block);
    pending = step;
    sample(step);
  }
  if (cfg.steps == 0) {
    e.request_cells(block);
    pending = 0;
  }
  deliver();
  result.forcing_swaps = e.swaps(false);
  Lattice host(cfg.width, cfg.height);
  e.download(host.src() + 1, static_cast<std::size_t>(host.stride()));
  for (int r = 0; r < cfg.height; ++r)
    for (int x = 1; x <= cfg.width; ++x) {
      const NodeState v = host.node(r, x);
      if (v & kObstacleBit) result.lattice.set_obstacle(r, x, true);
      result.lattice.set_node(r, x, v);
    }
  sync_ghost_columns(result.lattice);
  return result;
}

}  // namespace fhp_b200
