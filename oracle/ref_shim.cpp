// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// extern "C" shim over the UNMODIFIED reference library (proj/core), compiled
// straight from /root/reference/proj/core/src/*.cpp by oracle/Makefile into
// oracle/_ref/libfhpref.so. Lets the Python tests, the golden-vector
// generator and bench.py's reference arm drive the reference's own public
// API (fhp::run, fhp::advance, fhp::run_bench, observables) on plain byte
// buffers.
//
// Buffer convention used by every function here ("interior layout"):
// H rows x W bytes, row-major, columns 1..W of the reference Lattice, bit 7
// included. Obstacle masks use the same layout with bytes 0/1.

#include <cstdint>
#include <cstdio>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <string>
#include <vector>
#include <unistd.h>

#include "fhp/backends.hpp"
#include "fhp/bench.hpp"
#include "fhp/collision.hpp"
#include "fhp/lattice.hpp"
#include "fhp/observables.hpp"
#include "fhp/rng.hpp"
#include "fhp/step.hpp"

namespace {

thread_local std::string g_err;

int fail(const std::exception& e, int code) {
  g_err = e.what();
  return code;
}

fhp::Backend backend_of(int b) {
  switch (b) {
    case 0: return fhp::Backend::Scalar;
    case 1: return fhp::Backend::Lanes;
    case 2: return fhp::Backend::Strips;
    default: return fhp::Backend::Tiles;
  }
}

fhp::CollisionTable table_of(const uint8_t* t) {
  if (!t) return fhp::build_table();
  fhp::CollisionTable tab;
  std::memcpy(tab.entries.data(), t, 512);
  return tab;
}

void copy_out(const fhp::Lattice& lat, uint8_t* out) {
  const int W = lat.width();
  for (int r = 0; r < lat.height(); ++r)
    for (int x = 1; x <= W; ++x) out[(size_t)r * W + (x - 1)] = lat.node(r, x);
}

std::vector<std::string> geometry_of(const uint8_t* mask, int W, int H) {
  std::vector<std::string> g(H, std::string(W, '.'));
  for (int r = 0; r < H; ++r)
    for (int x = 0; x < W; ++x)
      if (mask[(size_t)r * W + x]) g[r][x] = '#';
  return g;
}

// Lattice with obstacle mask + arbitrary node bytes (what an upload does).
fhp::Lattice lattice_of(int W, int H, const uint8_t* state, const uint8_t* mask) {
  fhp::Lattice lat(W, H);
  if (mask) {
    for (int r = 0; r < H; ++r)
      for (int x = 1; x <= W; ++x)
        if (mask[(size_t)r * W + x - 1]) lat.set_obstacle(r, x, true);
  }
  for (int r = 0; r < H; ++r)
    for (int x = 1; x <= W; ++x) lat.set_node(r, x, state[(size_t)r * W + x - 1]);
  fhp::sync_ghost_columns(lat);
  return lat;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

uint64_t ref_mix64(uint64_t z) { return fhp::rng::mix64(z); }

uint64_t ref_node_random(uint64_t seed, int purpose, uint64_t step, uint64_t x,
                         uint64_t y) {
  return fhp::rng::node_random(seed, static_cast<fhp::rng::Purpose>(purpose), step, x, y);
}

int ref_bernoulli(uint64_t word, double p) { return fhp::rng::bernoulli(word, p) ? 1 : 0; }

void ref_build_table(uint8_t* out512) {
  const auto t = fhp::build_table();
  std::memcpy(out512, t.entries.data(), 512);
}

// Number of validation issues (0 = valid).
int ref_validate_table(const uint8_t* t512) {
  return static_cast<int>(fhp::validate_table(table_of(t512)).issues.size());
}

// init_lattice(cfg[, geometry]); out = interior layout.
int ref_init(int W, int H, uint64_t seed, double density, const uint8_t* mask,
             uint8_t* out) {
  try {
    fhp::SimConfig cfg;
    cfg.width = W;
    cfg.height = H;
    cfg.seed = seed;
    cfg.fill_density = density;
    fhp::Lattice lat = mask ? fhp::init_lattice(cfg, geometry_of(mask, W, H))
                            : fhp::init_lattice(cfg);
    copy_out(lat, out);
    return 0;
  } catch (const std::invalid_argument& e) {
    return fail(e, 2);
  } catch (const std::exception& e) {
    return fail(e, 3);
  }
}

// fhp::run(cfg, table): init (+geometry) then `steps` steps on `backend`.
// Final state into out (may be null); swaps/mass/momentum/digest returned.
int ref_run(int W, int H, int steps, double density, double force_p, uint64_t seed,
            int backend, int threads, const uint8_t* table512, const uint8_t* mask,
            uint8_t* out, uint64_t* swaps, int64_t* mass, int64_t* px, int64_t* py,
            uint64_t* digest) {
  try {
    fhp::SimConfig cfg;
    cfg.width = W;
    cfg.height = H;
    cfg.steps = steps;
    cfg.fill_density = density;
    cfg.force_p = force_p;
    cfg.seed = seed;
    cfg.backend = backend_of(backend);
    cfg.threads = threads;
    cfg.lanes = 64;
    std::string geom_path;
    if (mask) {
      char tmpl[] = "/tmp/fhpref_geomXXXXXX";
      int fd = mkstemp(tmpl);
      if (fd < 0) throw std::runtime_error("mkstemp failed");
      std::string text;
      for (const auto& row : geometry_of(mask, W, H)) text += row + "\n";
      if (write(fd, text.data(), text.size()) != (ssize_t)text.size())
        throw std::runtime_error("geometry write failed");
      close(fd);
      geom_path = tmpl;
      cfg.geometry_file = geom_path;
    }
    auto res = fhp::run(cfg, table_of(table512));
    if (!geom_path.empty()) unlink(geom_path.c_str());
    if (out) copy_out(res.lattice, out);
    if (swaps) *swaps = res.forcing_swaps;
    if (mass) *mass = fhp::total_mass(res.lattice);
    const auto p = fhp::total_momentum(res.lattice);
    if (px) *px = p.px;
    if (py) *py = p.py;
    if (digest) *digest = fhp::state_digest(res.lattice);
    return 0;
  } catch (const std::invalid_argument& e) {
    return fail(e, 2);
  } catch (const std::exception& e) {
    return fail(e, 3);
  }
}

// fhp::advance on an uploaded state: the drop-in boundary's contract.
int ref_advance(int W, int H, uint8_t* state, const uint8_t* mask,
                const uint8_t* table512, uint64_t seed, double force_p,
                int first_step, int step_count, int backend, int threads,
                uint64_t* swaps) {
  try {
    fhp::Lattice lat = lattice_of(W, H, state, mask);
    fhp::SimConfig cfg;
    cfg.width = W;
    cfg.height = H;
    cfg.seed = seed;
    cfg.force_p = force_p;
    cfg.backend = backend_of(backend);
    cfg.threads = threads;
    cfg.lanes = 64;
    const uint64_t s = fhp::advance(lat, table_of(table512), cfg, first_step, step_count);
    copy_out(lat, state);
    if (swaps) *swaps = s;
    return 0;
  } catch (const std::invalid_argument& e) {
    return fail(e, 2);
  } catch (const std::exception& e) {
    return fail(e, 3);
  }
}

// Observables on an interior-layout state (mask only matters through bit 7).
void ref_observables(int W, int H, const uint8_t* state, int64_t* mass, int64_t* px,
                     int64_t* py, uint64_t* digest) {
  fhp::Lattice lat = lattice_of(W, H, state, nullptr);
  *mass = fhp::total_mass(lat);
  const auto p = fhp::total_momentum(lat);
  *px = p.px;
  *py = p.py;
  *digest = fhp::state_digest(lat);
}

// coarse_grain(lat, block): per-cell nodes/particles + doubles rho/ux/uy.
int ref_coarse_grain(int W, int H, const uint8_t* state, int block, int* cells_x,
                     int* cells_y, int32_t* nodes, int32_t* particles, double* rho,
                     double* ux, double* uy) {
  try {
    fhp::Lattice lat = lattice_of(W, H, state, nullptr);
    const auto f = fhp::coarse_grain(lat, block);
    *cells_x = f.cells_x;
    *cells_y = f.cells_y;
    if (nodes) {
      for (size_t i = 0; i < f.cells.size(); ++i) {
        nodes[i] = f.cells[i].nodes;
        particles[i] = f.cells[i].particles;
        rho[i] = f.cells[i].rho;
        ux[i] = f.cells[i].ux;
        uy[i] = f.cells[i].uy;
      }
    }
    return 0;
  } catch (const std::exception& e) {
    return fail(e, 2);
  }
}

// velocity_profile(lat): H-2 rows of (mean_ux, sample_count).
void ref_velocity_profile(int W, int H, const uint8_t* state, double* mean_ux,
                          int32_t* count) {
  fhp::Lattice lat = lattice_of(W, H, state, nullptr);
  const auto prof = fhp::velocity_profile(lat);
  for (size_t i = 0; i < prof.size(); ++i) {
    mean_ux[i] = prof[i].mean_ux;
    count[i] = prof[i].sample_count;
  }
}

// fhp::run_bench(cfg, repeats): median Mups and digest. table512 null = DEFAULT,
// else written to a temporary FHPTAB01 file and passed via cfg.table_file.
int ref_bench(int W, int H, int steps, int warmup, double density, double force_p,
              uint64_t seed, int backend, int threads, const uint8_t* table512,
              int repeats, double* mups, double* wall_seconds, uint64_t* digest) {
  try {
    fhp::SimConfig cfg;
    cfg.width = W;
    cfg.height = H;
    cfg.steps = steps;
    cfg.warmup_steps = warmup;
    cfg.fill_density = density;
    cfg.force_p = force_p;
    cfg.seed = seed;
    cfg.backend = backend_of(backend);
    cfg.threads = threads;
    cfg.lanes = 64;
    std::string path;
    if (table512) {
      char tmpl[] = "/tmp/fhpref_tabXXXXXX";
      int fd = mkstemp(tmpl);
      if (fd < 0) throw std::runtime_error("mkstemp failed");
      close(fd);
      path = tmpl;
      fhp::write_table_file(path, table_of(table512));
      cfg.table_file = path;
    }
    const auto res = fhp::run_bench(cfg, repeats);
    if (!path.empty()) unlink(path.c_str());
    *mups = res.median.mups;
    *wall_seconds = res.median.wall_seconds;
    *digest = res.median.state_digest;
    return 0;
  } catch (const std::invalid_argument& e) {
    return fail(e, 2);
  } catch (const std::exception& e) {
    return fail(e, 3);
  }
}

// fhp::run_bench(cfg, repeats) with cfg.table_file = an FHPTAB01 file (the
// reference's own read_table_file / load_table, collision.cpp:137-170, reads
// it; nullptr = the DEFAULT table).
int ref_bench_file(int W, int H, int steps, int warmup, double density, double force_p,
                   uint64_t seed, int backend, int threads, const char* table_file,
                   int repeats, double* mups, double* wall_seconds, uint64_t* digest) {
  try {
    fhp::SimConfig cfg;
    cfg.width = W;
    cfg.height = H;
    cfg.steps = steps;
    cfg.warmup_steps = warmup;
    cfg.fill_density = density;
    cfg.force_p = force_p;
    cfg.seed = seed;
    cfg.backend = backend_of(backend);
    cfg.threads = threads;
    cfg.lanes = 64;
    if (table_file) cfg.table_file = table_file;
    const auto res = fhp::run_bench(cfg, repeats);
    *mups = res.median.mups;
    *wall_seconds = res.median.wall_seconds;
    *digest = res.median.state_digest;
    return 0;
  } catch (const std::invalid_argument& e) {
    return fail(e, 2);
  } catch (const std::exception& e) {
    return fail(e, 3);
  }
}

}  // extern "C"
