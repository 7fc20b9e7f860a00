// RAII wrapper over the C ABI (include/fhpg.h).
#include "fhp_b200/engine.hpp"

#include <utility>

#include "fhpg.h"

namespace fhp_b200 {

void check_status(int rc) {
  if (rc == FHPG_OK) return;
  const std::string msg = fhpg_last_error();
  if (rc == FHPG_EINVAL) throw std::invalid_argument(msg);
  throw std::runtime_error(msg);
}

Engine::Engine(int width, int height) : width_(width), height_(height), row_end_(height) {
  check_status(fhpg_create(width, height, &h_));
}

Engine::Engine(int width, int height, int row_begin, int row_end, int device)
    : width_(width), height_(height), row_begin_(row_begin), row_end_(row_end) {
  check_status(fhpg_create_strip(width, height, row_begin, row_end, device, &h_));
}

Engine::Engine(int width, int height, int strips, const std::vector<int>& devices)
    : width_(width), height_(height), row_end_(height) {
  if (!devices.empty() && static_cast<int>(devices.size()) != strips)
    throw std::invalid_argument("devices must list one GPU index per strip");
  check_status(fhpg_create_multi(width, height, strips, devices.empty() ? nullptr : devices.data(), &h_));
}

Engine::~Engine() { fhpg_destroy(h_); }

Engine::Engine(Engine&& o) noexcept { *this = std::move(o); }

Engine& Engine::operator=(Engine&& o) noexcept {
  if (this != &o) {
    fhpg_destroy(h_);
    h_ = std::exchange(o.h_, nullptr);
    width_ = o.width_;
    height_ = o.height_;
    row_begin_ = o.row_begin_;
    row_end_ = o.row_end_;
    cells_block_ = o.cells_block_;
  }
  return *this;
}

bool Engine::fast_path() const {
  int fast = 0;
  check_status(fhpg_info(h_, nullptr, nullptr, nullptr, nullptr, &fast, nullptr));
  return fast != 0;
}

std::uint64_t Engine::step_launches() const {
  std::uint64_t n = 0;
  check_status(fhpg_info(h_, nullptr, nullptr, nullptr, nullptr, nullptr, &n));
  return n;
}

void Engine::set_stream(void* s) { check_status(fhpg_set_stream(h_, s)); }
void Engine::set_table(const CollisionTable& t) { check_status(fhpg_set_table(h_, t.entries.data())); }
void Engine::set_obstacles(const std::uint8_t* m, std::size_t stride) {
  check_status(fhpg_set_obstacles(h_, m, stride));
}
void Engine::upload(const std::uint8_t* rows, std::size_t stride) {
  check_status(fhpg_upload(h_, rows, stride));
}
void Engine::download(std::uint8_t* rows, std::size_t stride) const {
  check_status(fhpg_download(h_, rows, stride));
}

void Engine::upload(const Lattice& lat) {
  if (lat.width() != width_ || lat.height() != row_end_ - row_begin_)
    throw std::invalid_argument("lattice shape does not match the engine");
  set_obstacles(lat.obstacle_mask() + 1, static_cast<std::size_t>(lat.stride()));
  upload(lat.src() + 1, static_cast<std::size_t>(lat.stride()));
}

void Engine::download(Lattice& lat) const {
  if (lat.width() != width_ || lat.height() != row_end_ - row_begin_)
    throw std::invalid_argument("lattice shape does not match the engine");
  download(lat.src() + 1, static_cast<std::size_t>(lat.stride()));
  sync_ghost_columns(lat);
}

void Engine::init(std::uint64_t seed, double density) { check_status(fhpg_init(h_, seed, density)); }

std::uint64_t Engine::advance(std::uint64_t seed, double force_p, std::int64_t first,
                              std::int64_t count) {
  std::uint64_t sw = 0;
  check_status(fhpg_advance(h_, seed, fhpg_bernoulli_threshold(force_p), first, count, &sw));
  return sw;
}

void Engine::advance_async(std::uint64_t seed, double force_p, std::int64_t first,
                           std::int64_t count) {
  check_status(fhpg_advance_async(h_, seed, fhpg_bernoulli_threshold(force_p), first, count));
}

std::uint64_t Engine::swaps(bool reset) {
  std::uint64_t s = 0;
  check_status(fhpg_swaps(h_, &s, reset ? 1 : 0));
  return s;
}

void Engine::synchronize() { check_status(fhpg_synchronize(h_)); }

std::int64_t Engine::total_mass() const {
  int64_t m = 0;
  check_status(fhpg_reduce_global(h_, &m, nullptr, nullptr));
  return m;
}

MomentumVec Engine::total_momentum() const {
  int64_t px = 0, py = 0;
  check_status(fhpg_reduce_global(h_, nullptr, &px, &py));
  return {static_cast<int>(px), static_cast<int>(py)};
}

CellSums Engine::cell_sums(int block) const {
  if (block < 1) throw std::invalid_argument("block size must be >= 1");
  CellSums s;
  s.cells_x = (width_ + block - 1) / block;
  s.cells_y = (height_ - 2 + block - 1) / block;
  const std::size_t n = static_cast<std::size_t>(s.cells_x) * s.cells_y;
  s.nodes.assign(n, 0);
  s.particles.assign(n, 0);
  s.px.assign(n, 0);
  s.py.assign(n, 0);
  check_status(fhpg_reduce_cells(h_, block, s.nodes.data(), s.particles.data(), s.px.data(),
                                 s.py.data()));
  return s;
}

void Engine::request_cells(int block) {
  check_status(fhpg_reduce_cells_async(h_, block));
  cells_block_ = block;
}

CellSums Engine::collect_cells() {
  if (cells_block_ < 1) throw std::invalid_argument("no coarse-grain request pending");
  CellSums s;
  s.cells_x = (width_ + cells_block_ - 1) / cells_block_;
  s.cells_y = (height_ - 2 + cells_block_ - 1) / cells_block_;
  const std::size_t n = static_cast<std::size_t>(s.cells_x) * s.cells_y;
  s.nodes.assign(n, 0);
  s.particles.assign(n, 0);
  s.px.assign(n, 0);
  s.py.assign(n, 0);
  if (n) check_status(fhpg_cells_wait(h_, s.nodes.data(), s.particles.data(), s.px.data(), s.py.data()));
  cells_block_ = 0;
  return s;
}

int Engine::strips() const {
  int n = 1;
  check_status(fhpg_strips(h_, &n, nullptr, nullptr, nullptr));
  return n;
}

void Engine::row_sums(std::vector<std::int64_t>& px, std::vector<std::int32_t>& fluid) const {
  px.assign(static_cast<std::size_t>(height_ - 2), 0);
  fluid.assign(static_cast<std::size_t>(height_ - 2), 0);
  check_status(fhpg_reduce_rows(h_, px.data(), fluid.data()));
}

}  // namespace fhp_b200
