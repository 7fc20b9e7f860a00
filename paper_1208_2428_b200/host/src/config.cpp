// SimConfig checks (the messages of SimConfig::validate, step.cpp:22-38,
// plus the Cuda backend's own fields) and backend names (step.cpp:12-20).
#include "fhp_b200/config.hpp"

#include <stdexcept>

namespace fhp_b200 {

const char* backend_name(Backend b) noexcept {
  static constexpr const char* kNames[] = {"scalar", "lanes", "strips", "tiles", "cuda"};
  const auto i = static_cast<unsigned>(b);
  return i < sizeof kNames / sizeof kNames[0] ? kNames[i] : "?";
}

void SimConfig::validate() const {
  struct Rule {
    bool broken;
    const char* message;
  };
  const bool lanes_ok = lanes == 16 || lanes == 32 || lanes == 64;
  bool devices_ok = devices.empty() || static_cast<int>(devices.size()) == gpus;
  for (int d : devices) devices_ok = devices_ok && d >= 0;
  const Rule rules[] = {
      {width < 1, "width must be >= 1"},
      {height < 3, "height must be >= 3"},
      {steps < 0, "steps must be >= 0"},
      {!(fill_density >= 0.0 && fill_density <= 1.0), "density must be in [0,1]"},
      {!(force_p >= 0.0 && force_p <= 1.0), "force-p must be in [0,1]"},
      {threads < 1, "threads must be >= 1"},
      {!lanes_ok, "lanes must be 16, 32 or 64"},
      {tile_x < 1 || tile_y < 1, "tile dimensions must be >= 1"},
      {dump_every < 0, "dump-every must be >= 0"},
      {repeats < 1, "repeats must be >= 1"},
      {warmup_steps < 0, "warmup must be >= 0"},
      // Cuda backend
      {device < 0, "device must be >= 0"},
      {gpus < 1, "gpus must be >= 1"},
      {gpus > 1 && gpus > height - 2, "strip count exceeds interior row count"},
      {!devices_ok, "devices must list one non-negative GPU index per strip"},
      {checkpoint_every < 0, "checkpoint-every must be >= 0"},
  };
  for (const Rule& r : rules)
    if (r.broken) throw std::invalid_argument(r.message);
}

}  // namespace fhp_b200
