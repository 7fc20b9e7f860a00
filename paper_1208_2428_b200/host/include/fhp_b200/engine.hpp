// fhp_b200/engine.hpp — RAII wrapper of the device-resident engine
// (include/fhpg.h). State stays in HBM between calls; host Lattices are only
// touched on upload / download.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "fhp_b200/collision.hpp"
#include "fhp_b200/lattice.hpp"

struct fhpg_engine;

namespace fhp_b200 {

// Maps an fhpg status to the reference's exception types (invalid_argument
// for status 2, runtime_error for 3).
void check_status(int rc);

struct CellSums {
  int cells_x = 0, cells_y = 0;
  std::vector<std::int32_t> nodes, particles;
  std::vector<std::int64_t> px, py;
};

class Engine {
 public:
  Engine(int width, int height);                                     // whole lattice
  Engine(int width, int height, int row_begin, int row_end, int device);  // row strip
  // Whole lattice in `strips` row strips, strip i on devices[i] (empty: GPU
  // i); the library exchanges the halo rows (fhpg_create_multi).
  Engine(int width, int height, int strips, const std::vector<int>& devices);
  ~Engine();
  Engine(const Engine&) = delete;
  Engine& operator=(const Engine&) = delete;
  Engine(Engine&& o) noexcept;
  Engine& operator=(Engine&& o) noexcept;

  int width() const noexcept { return width_; }
  int height() const noexcept { return height_; }
  int row_begin() const noexcept { return row_begin_; }
  int row_end() const noexcept { return row_end_; }
  bool fast_path() const;
  std::uint64_t step_launches() const;
  fhpg_engine* handle() noexcept { return h_; }

  void set_stream(void* cuda_stream);
  void set_table(const CollisionTable& t);
  void set_obstacles(const std::uint8_t* mask, std::size_t stride);
  void upload(const std::uint8_t* rows, std::size_t stride);
  void download(std::uint8_t* rows, std::size_t stride) const;
  // Whole-lattice Lattice <-> device (src() interior and obstacle mask).
  void upload(const Lattice& lat);
  void download(Lattice& lat) const;
  void init(std::uint64_t seed, double density);

  std::uint64_t advance(std::uint64_t seed, double force_p, std::int64_t first_step,
                        std::int64_t step_count);
  void advance_async(std::uint64_t seed, double force_p, std::int64_t first_step,
                     std::int64_t step_count);
  std::uint64_t swaps(bool reset);
  void synchronize();

  std::int64_t total_mass() const;
  MomentumVec total_momentum() const;
  CellSums cell_sums(int block) const;
  // The same sums without blocking: request_cells enqueues the reduction
  // behind the steps already enqueued; collect_cells waits for it.
  void request_cells(int block);
  CellSums collect_cells();
  int strips() const;
  // Per interior row r (index r-1): px sum over fluid nodes, fluid count.
  void row_sums(std::vector<std::int64_t>& px, std::vector<std::int32_t>& fluid) const;

 private:
  fhpg_engine* h_ = nullptr;
  int width_ = 0, height_ = 0, row_begin_ = 0, row_end_ = 0;
  int cells_block_ = 0;
};

}  // namespace fhp_b200
