/*
 * fhp_oracle.c — TEST INFRASTRUCTURE ONLY (the parity checker, never the
 * product). Plain-C restatement of the reference FHP evolution path
 * (/root/reference/proj/core), used by tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline leg. The CUDA engine must never call into this.
 *
 * Parity pinned: tests/test_oracle.py checks every function here against the
 * reference's own golden values (test_rng.cpp:15-26, test_collision.cpp,
 * test_step.cpp, test_observables.cpp) and against digests produced by the
 * reference library itself (oracle/_ref/libfhpref.so, fixtures in
 * tests/golden/ made by tests/golden/make_golden.py).
 *
 * Layout ("interior layout"): H rows x W bytes, row-major, the reference's
 * storage columns 1..W (lattice.hpp:36-68 without the ghost columns);
 * periodic wrap in x is done with modular arithmetic instead of ghost
 * columns (lattice.cpp:32-39).
 */
#include "fhp_oracle.h"

#include <stdlib.h>
#include <string.h>

#define GOLDEN_GAMMA 0x9E3779B97F4A7C15ull

/* rng.hpp:15-23 */
uint64_t fo_mix64(uint64_t z) {
  z += GOLDEN_GAMMA;
  z ^= z >> 30;
  z *= 0xBF58476D1CE4E5B9ull;
  z ^= z >> 27;
  z *= 0x94D049BB133111EBull;
  z ^= z >> 31;
  return z;
}

/* rng.hpp:25-33 */
uint64_t fo_node_random(uint64_t seed, uint64_t purpose, uint64_t step, uint64_t x,
                        uint64_t y) {
  uint64_t z = seed + GOLDEN_GAMMA * purpose;
  z = fo_mix64(z);
  z = fo_mix64(z + step);
  z = fo_mix64(z + x);
  return fo_mix64(z + y);
}

/* rng.hpp:37-42, threshold part (the only floating-point step). */
uint64_t fo_bernoulli_threshold(double p) {
  return p >= 1.0 ? (1ull << 32) : (uint64_t)(p * 4294967296.0);
}

/* rng.hpp:37-42 */
int fo_bernoulli(uint64_t word, uint64_t threshold) { return (word >> 32) < threshold; }

static int popc7(unsigned s) { return __builtin_popcount(s & 0x7Fu); }

/* node_state.hpp:82-85 */
static unsigned reverse6(unsigned m) { m &= 0x3Fu; return ((m << 3) | (m >> 3)) & 0x3Fu; }

/* collision.cpp:12-18 */
static unsigned rotate6(unsigned moving, int by) {
  unsigned out = 0;
  for (int i = 0; i < 6; ++i)
    if (moving & (1u << i)) out |= 1u << ((i + by) % 6);
  return out;
}

/* collision.cpp:22-51 (DEFAULT rule set, fluid states) */
static unsigned fluid_outcome(unsigned s, int chirality) {
  const unsigned moving = s & 0x3Fu;
  const int rest = (s & 0x40u) != 0;
  const int n = __builtin_popcount(moving);
  if (n == 2 && !rest && reverse6(moving) == moving) return rotate6(moving, chirality ? 1 : 2);
  if (n == 3 && !rest && (moving == 0x15 || moving == 0x2A)) return moving ^ 0x3Fu;
  if (n == 1 && rest) {
    const int i = __builtin_ctz(moving);
    return (1u << ((i + 5) % 6)) | (1u << ((i + 1) % 6));
  }
  if (n == 2 && !rest) {
    for (int i = 0; i < 6; ++i) {
      const unsigned pair = (1u << i) | (1u << ((i + 2) % 6));
      if (moving == pair) return (1u << ((i + 1) % 6)) | 0x40u;
    }
  }
  return s;
}

/* collision.cpp:55-72 */
void fo_build_default_table(uint8_t* t) {
  for (int ch = 0; ch < 2; ++ch)
    for (unsigned s = 0; s < 256; ++s) {
      unsigned out;
      if (s & 0x80u) out = (s & 0xC0u) | reverse6(s & 0x3Fu);
      else out = fluid_outcome(s, ch);
      t[(ch << 8) | s] = (uint8_t)out;
    }
}

/* node_state.hpp:54-74: integer momentum of the moving bits. */
static const int kPx[6] = {-1, 1, 2, 1, -1, -2};
static const int kPy[6] = {1, 1, 0, -1, -1, 0};
static void momentum(unsigned s, int* px, int* py) {
  int a = 0, b = 0;
  for (int k = 0; k < 6; ++k)
    if (s & (1u << k)) { a += kPx[k]; b += kPy[k]; }
  *px = a;
  *py = b;
}

/* collision.cpp:74-101: number of violations (0 = valid). */
int fo_validate_table(const uint8_t* t) {
  int issues = 0;
  for (int idx = 0; idx < 512; ++idx) {
    const unsigned s = (unsigned)idx & 0xFFu, out = t[idx];
    if ((out & 0x80u) != (s & 0x80u)) { ++issues; continue; }
    if (s & 0x80u) {
      if (out != ((s & 0xC0u) | reverse6(s & 0x3Fu))) ++issues;
      continue;
    }
    if (popc7(out) != popc7(s)) ++issues;
    int a, b, c, d;
    momentum(out, &a, &b);
    momentum(s, &c, &d);
    if (a != c || b != d) ++issues;
  }
  return issues;
}

/* lattice.cpp:44-55 (random_fill) + lattice.cpp:57-93 (init_impl).
 * mask: interior-layout obstacle bytes (0/1) from the geometry, or NULL. */
void fo_init(int W, int H, uint64_t seed, double density, const uint8_t* mask,
             uint8_t* out) {
  const uint64_t thr = fo_bernoulli_threshold(density);
  for (int r = 0; r < H; ++r)
    for (int x = 1; x <= W; ++x) {
      const size_t i = (size_t)r * W + (x - 1);
      const int obst = (r == 0 || r == H - 1) || (mask && mask[i]);
      if (obst) { out[i] = 0x80; continue; }
      const uint64_t w = fo_node_random(seed, 0, 0, (uint64_t)x, (uint64_t)r);
      unsigned s = 0;
      for (int b = 0; b < 7; ++b)
        if (fo_bernoulli(fo_mix64(w + (uint64_t)b), thr)) s |= 1u << b;
      out[i] = (uint8_t)s;
    }
}

/* backends.cpp:64-73 (pull offsets) with step.cpp:40-52 (motion_gather).
 * Bit 7 of the destination comes from the obstacle mask (step.cpp:50); src
 * bit 7 is never read. */
static const int kPullDr[6] = {1, 1, 0, -1, -1, 0};
static void pull_dx(int q, int* dx) {
  dx[0] = q; dx[1] = q - 1; dx[2] = -1; dx[3] = q - 1; dx[4] = q; dx[5] = 1;
}

static void motion(int W, int H, const uint8_t* src, const uint8_t* mask, uint8_t* dst) {
  for (int r = 0; r < H; ++r) {
    int dx[6];
    pull_dx(r & 1, dx);
    for (int x = 0; x < W; ++x) {
      unsigned v = src[(size_t)r * W + x] & 0x40u;
      for (int k = 0; k < 6; ++k) {
        const int sr = r + kPullDr[k];
        if (sr < 0 || sr >= H) continue;
        const int sx = ((x + dx[k]) % W + W) % W;
        v |= src[(size_t)sr * W + sx] & (1u << k);
      }
      if (mask[(size_t)r * W + x]) v |= 0x80u;
      dst[(size_t)r * W + x] = (uint8_t)v;
    }
  }
}

/* step.cpp:63-93 (collide_rows over all rows). Returns accepted swaps. */
static uint64_t collide(int W, int H, uint8_t* buf, const uint8_t* table, uint64_t seed,
                        uint64_t step, uint64_t thr) {
  uint64_t swaps = 0;
  for (int r = 0; r < H; ++r)
    for (int x = 1; x <= W; ++x) {
      const size_t i = (size_t)r * W + (x - 1);
      const unsigned s = buf[i];
      const unsigned ch = (unsigned)(fo_node_random(seed, 2, step, (uint64_t)x, (uint64_t)r) & 1u);
      unsigned out = table[(ch << 8) | s];
      if (!(out & 0x80u) && (out & 0x20u) && !(out & 0x04u)) {
        const uint64_t w = fo_node_random(seed, 1, step, (uint64_t)x, (uint64_t)r);
        if (fo_bernoulli(w, thr)) {
          out = (out & ~0x20u) | 0x04u;
          ++swaps;
        }
      }
      buf[i] = (uint8_t)out;
    }
  return swaps;
}

/* step.cpp:95-133: advance = step_count x (motion -> swap -> collision),
 * global step index first_step + i. step_count <= 0 is a no-op
 * (backends.cpp:157). `state` is updated in place. mask: interior-layout
 * obstacle bytes (the Lattice's obstacle_ vector, lattice.hpp:67); NULL means
 * "bit 7 of the input state", which is what init_lattice produces. */
uint64_t fo_advance(int W, int H, uint8_t* state, const uint8_t* mask, const uint8_t* table,
                    uint64_t seed, uint64_t force_thr, int64_t first_step, int64_t step_count) {
  if (step_count <= 0) return 0;
  const size_t n = (size_t)W * H;
  uint8_t* tmp = (uint8_t*)malloc(n);
  uint8_t* own_mask = NULL;
  if (!mask) { /* no separate mask: the obstacle set is bit 7 of the input */
    own_mask = (uint8_t*)malloc(n);
    for (size_t i = 0; i < n; ++i) own_mask[i] = (uint8_t)(state[i] >> 7);
    mask = own_mask;
  }
  uint64_t swaps = 0;
  for (int64_t s = first_step; s < first_step + step_count; ++s) {
    motion(W, H, state, mask, tmp);
    swaps += collide(W, H, tmp, table, seed, (uint64_t)s, force_thr);
    memcpy(state, tmp, n);
  }
  free(tmp);
  free(own_mask);
  return swaps;
}

/* lattice.cpp:122-132 */
uint64_t fo_digest(int W, int H, const uint8_t* state) {
  uint64_t h = 0xCBF29CE484222325ull;
  const size_t n = (size_t)W * H;
  for (size_t i = 0; i < n; ++i) {
    h ^= state[i];
    h *= 0x100000001B3ull;
  }
  return h;
}

/* observables.cpp:27-47 */
void fo_global(int W, int H, const uint8_t* state, int64_t* mass, int64_t* px, int64_t* py) {
  int64_t m = 0, a = 0, b = 0;
  const size_t n = (size_t)W * H;
  for (size_t i = 0; i < n; ++i) {
    const unsigned s = state[i];
    m += popc7(s);
    if (s & 0x80u) continue;
    int c, d;
    momentum(s, &c, &d);
    a += c;
    b += d;
  }
  *mass = m;
  *px = a;
  *py = b;
}

/* observables.cpp:49-82, integer part: per cell (nodes, particles, px, py)
 * over rows 1..H-2, cells ((r-1)/B, (x-1)/B); momentum over fluid nodes. */
void fo_cells(int W, int H, const uint8_t* state, int B, int32_t* nodes, int32_t* particles,
              int64_t* px, int64_t* py) {
  const int cx = (W + B - 1) / B, cy = (H - 2 + B - 1) / B;
  const size_t nc = (size_t)cx * cy;
  memset(nodes, 0, nc * sizeof(int32_t));
  memset(particles, 0, nc * sizeof(int32_t));
  memset(px, 0, nc * sizeof(int64_t));
  memset(py, 0, nc * sizeof(int64_t));
  for (int r = 1; r <= H - 2; ++r)
    for (int x = 1; x <= W; ++x) {
      const size_t c = (size_t)((r - 1) / B) * cx + (size_t)((x - 1) / B);
      const unsigned s = state[(size_t)r * W + (x - 1)];
      nodes[c] += 1;
      particles[c] += popc7(s);
      if (!(s & 0x80u)) {
        int a, b;
        momentum(s, &a, &b);
        px[c] += a;
        py[c] += b;
      }
    }
}

/* observables.cpp:84-102, integer part: per interior row (px sum, fluid count). */
void fo_rows(int W, int H, const uint8_t* state, int64_t* px, int32_t* fluid) {
  for (int r = 1; r <= H - 2; ++r) {
    int64_t a = 0;
    int32_t c = 0;
    for (int x = 0; x < W; ++x) {
      const unsigned s = state[(size_t)r * W + x];
      if (s & 0x80u) continue;
      ++c;
      int p, q;
      momentum(s, &p, &q);
      a += p;
    }
    px[r - 1] = a;
    fluid[r - 1] = c;
  }
}

/* Adversarial input used by the parity tests (after test_backends.cpp:25-39,
 * scramble()): obstacle mask = walls + sites with node_random(seed,Init,2,x,r)
 * % 13 == 0; node bytes = node_random(seed,Init,1,x,r) & 0x7F, plus bit 7 on
 * obstacles. Rest, wall-row and obstacle nodes all carry particles. */
void fo_scramble(int W, int H, uint64_t seed, uint8_t* state, uint8_t* mask) {
  for (int r = 0; r < H; ++r)
    for (int x = 1; x <= W; ++x) {
      const size_t i = (size_t)r * W + (x - 1);
      const int obst = r == 0 || r == H - 1 ||
                       fo_node_random(seed, 0, 2, (uint64_t)x, (uint64_t)r) % 13 == 0;
      mask[i] = (uint8_t)obst;
      state[i] = (uint8_t)((fo_node_random(seed, 0, 1, (uint64_t)x, (uint64_t)r) & 0x7Fu) |
                           (obst ? 0x80u : 0u));
    }
}

/* Cylinder geometry of BASELINE config 3: '#' disc of radius R centred at
 * (cx, cy) in storage coordinates (1-based column, row), odd rows shifted by
 * one half column. mask = interior layout bytes 0/1. */
void fo_cylinder(int W, int H, double cx, double cy, double R, uint8_t* mask) {
  for (int r = 0; r < H; ++r)
    for (int x = 1; x <= W; ++x) {
      const double px = x + 0.5 * (r & 1) - cx;
      const double py = (r - cy) * 0.8660254037844386;
      mask[(size_t)r * W + (x - 1)] = (uint8_t)(px * px + py * py <= R * R);
    }
}

/* One step of a row strip, for the multi-process decomposition tests: the
 * strip owns global rows [row0, row0+nrows) of a W x H lattice; `src` holds
 * nrows+2 rows (halo row above, owned rows, halo row below; halos are zero
 * where the strip touches the grid edge), `mask` the owned rows' obstacle
 * bytes. Writes the owned rows after motion + collision + forcing of global
 * step `step` into `dst` (nrows rows). Same rules as fo_advance with the RNG
 * keyed by the global row. Returns the accepted swaps. */
uint64_t fo_step_strip(int W, int H, int row0, int nrows, const uint8_t* src, const uint8_t* mask,
                       const uint8_t* table, uint64_t seed, uint64_t thr, uint64_t step,
                       uint8_t* dst) {
  (void)H;
  uint64_t swaps = 0;
  for (int lr = 0; lr < nrows; ++lr) {
    const int r = row0 + lr;
    int dx[6];
    pull_dx(r & 1, dx);
    for (int x = 0; x < W; ++x) {
      const uint8_t* c = src + (size_t)(lr + 1) * W; /* row r in the halo-extended buffer */
      unsigned v = c[x] & 0x40u;
      for (int k = 0; k < 6; ++k) {
        const uint8_t* s = src + (size_t)(lr + 1 + kPullDr[k]) * W;
        const int sx = ((x + dx[k]) % W + W) % W;
        v |= s[sx] & (1u << k);
      }
      if (mask[(size_t)lr * W + x]) v |= 0x80u;
      const unsigned ch =
          (unsigned)(fo_node_random(seed, 2, step, (uint64_t)x + 1, (uint64_t)r) & 1u);
      unsigned out = table[(ch << 8) | v];
      if (!(out & 0x80u) && (out & 0x20u) && !(out & 0x04u) &&
          fo_bernoulli(fo_node_random(seed, 1, step, (uint64_t)x + 1, (uint64_t)r), thr)) {
        out = (out & ~0x20u) | 0x04u;
        ++swaps;
      }
      dst[(size_t)lr * W + x] = (uint8_t)out;
    }
  }
  return swaps;
}
