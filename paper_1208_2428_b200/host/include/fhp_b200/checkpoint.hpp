// fhp_b200/checkpoint.hpp — checkpoint / resume of a device-resident run
// (not in the reference). Exact by
// construction: every random draw is keyed by (seed, purpose, step, x, y), so
// the state bytes plus the next global step index, seed, forcing probability
// and table are the whole simulation state.
//
// File "FHPCKPT1" (little-endian):
//   0  magic "FHPCKPT1"         8 B
//   8  u32 width, u32 height    8 B
//  16  i64 next_step            the first step index still to run
//  24  u64 seed
//  32  f64 force_p
//  40  u64 forcing swaps accumulated so far
//  48  u64 FNV-1a-64 of the state bytes (== state_digest of the lattice)
//  56  512 B collision table
// 568  height x width state bytes, row-major, bit 7 = obstacle
#pragma once

#include <array>
#include <cstdint>
#include <string>
#include <vector>

#include "fhp_b200/collision.hpp"
#include "fhp_b200/engine.hpp"

namespace fhp_b200 {

inline constexpr char kCheckpointMagic[9] = "FHPCKPT1";
inline constexpr std::size_t kCheckpointHeader = 56 + 512;

struct Checkpoint {
  int width = 0, height = 0;
  std::int64_t next_step = 0;
  std::uint64_t seed = 0;
  double force_p = 0.0;
  std::uint64_t swaps = 0;
  CollisionTable table{};
  std::vector<std::uint8_t> state;  // height * width bytes, bit 7 = obstacle
};

// FNV-1a-64 over a byte range (the reference's state_digest, lattice.cpp:122-132).
std::uint64_t fnv1a64(const std::uint8_t* p, std::size_t n) noexcept;

// Downloads the engine's whole lattice into a checkpoint record.
Checkpoint capture_checkpoint(const Engine& e, std::int64_t next_step, std::uint64_t seed,
                              double force_p, std::uint64_t swaps, const CollisionTable& table);
// Table, obstacles (from bit 7) and state back into an engine of the same size.
void restore_checkpoint(Engine& e, const Checkpoint& c);

std::vector<std::uint8_t> serialize_checkpoint(const Checkpoint& c);
// Throws std::runtime_error on a bad magic, size or digest.
Checkpoint parse_checkpoint(const std::vector<std::uint8_t>& bytes);
void write_checkpoint_file(const std::string& path, const Checkpoint& c);
Checkpoint read_checkpoint_file(const std::string& path);

}  // namespace fhp_b200
