// fhp/cuda_backend.hpp — Backend::Cuda of fhp::advance (installed into the
// reference's include/fhp/ by integration/Makefile).
#pragma once

#include <cstdint>

#include "fhp/collision.hpp"
#include "fhp/config.hpp"
#include "fhp/lattice.hpp"

namespace fhp {

// fhp::advance on the B200 engine (libfhpg.so, include/fhpg.h): uploads
// lat.src() and the obstacle mask, runs step_count steps with global indices
// first_step.., downloads into lat.src(). step_count <= 0 is a no-op
// (backends.cpp:157). cfg.gpus > 1 splits the lattice into row strips, strip
// i on GPU i (modulo the GPUs present). The engine (device buffers, streams, TMA descriptors) is
// kept between calls for the same lattice shape; library errors are thrown
// as std::invalid_argument / std::runtime_error like the other backends.
std::uint64_t cuda_advance(Lattice& lat, const CollisionTable& table, const SimConfig& cfg,
                           int first_step, int step_count);

}  // namespace fhp
