// fhpg_step_fast.cu — the hot path: one fused FHP time step for W % 16 == 0.
//
// Replaces, per step, sync_ghost_columns (lattice.cpp:32-39), motion_step
// (step.cpp:40-61, pull offsets backends.cpp:64-73), swap_buffers and
// collide_rows with its counter-RNG chirality and forcing (step.cpp:63-93).
//
// Layout: byte-per-site rows (bit 7 = obstacle, kept in the state; valid
// tables never change it) in two ping-pong HBM buffers.
//
// Work decomposition: one CTA of 32 warps per SM. A warp owns a 512-column
// band (16 sites per lane: one 128-bit load and one 128-bit store per lane and
// row) and a segment of rows it streams top to bottom, keeping rows r-1, r,
// r+1 in registers so every source row is read from HBM once. A CTA covers
// up to kBandsPerCta adjacent bands x kWarps / bands segments.
//
// Per row: motion = byte permutes (PRMT, the +-1 column shifts, neighbour
// lane edge bytes via SHFL) and LOP3 bit-select merges; collision = one LDS
// per site from a lane-private copy of the LUT (one PRMT forms the address
// state*256 + lane*4, so lane l always hits bank l). The LUT entry holds the
// chirality-0 outcome (byte 0) and the XOR to the chirality-1 outcome (byte
// 2), whose bit 7 flags "depends on chirality". Rows go to a per-warp smem
// stage. Byte moves that would be ALU shifts are written as multiplies (FMA
// pipe) because the ALU pipe is the binding resource.
//
// Every kBatch rows the warp resolves the chirality-dependent sites with a
// load-balanced walk (prefix sum over lanes, each lane takes an equal slice of
// the batch's dep-site list), evaluating the RNG only there (rng.hpp:25-33;
// key = per-column key staged in smem + global row) and patching the staged
// bytes with shared-memory atomics. Forcing (step.cpp:79-88) is resolved the
// same way on the patched rows. Then the batch leaves with 128-bit streaming
// stores.
#include <cstdint>
#include <type_traits>

#include "fhpg_common.cuh"
#include "fhpg_kernels.cuh"

namespace fhpg {
namespace {

constexpr unsigned kFull = 0xFFFFFFFFu;
constexpr int kThreads = 640;
constexpr int kWarps = kThreads / 32;
constexpr int kBandsPerCta = 4;
constexpr int kBatch = 4;
// Shared memory map (bytes). The LUT uses the first 128 B of every 256-B
// entry row; the second halves hold the column keys of the CTA's 2048
// columns (chirality keys in rows 0-127, forcing keys in rows 128-255).
constexpr int kLutBytes = 256 * 256;
constexpr int kStageOut = 0;                 // [kBatch][512] bytes
constexpr int kStageDep = kBatch * 512;      // [kBatch][512] bytes
constexpr int kStageMask = 2 * kBatch * 512; // [32 lanes][2] u32 dep masks
constexpr int kWarpStage = 2 * kBatch * 512 + 32 * kBatch * 4;
// Request: worst-case gap before the 64 KB-aligned LUT + LUT + all stages
// that do not fit in the gap (see step_fast_kernel).
constexpr int kSmem = 65536 + kLutBytes + kWarps * kWarpStage - (65536 / kWarpStage - 1) * kWarpStage;

template <int B, int E, typename F>
__device__ __forceinline__ void static_for(F&& f) {
  if constexpr (B < E) {
    f(std::integral_constant<int, B>{});
    static_for<B + 1, E>(f);
  }
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint32_t lds32(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ uint32_t lds8(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ uint64_t lds64(uint32_t a) {
  uint64_t v;
  asm volatile("ld.shared.u64 %0, [%1];" : "=l"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ uint4 lds128(uint32_t a) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts32(uint32_t a, uint32_t v) {
  asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(v));
}
__device__ __forceinline__ void sts64(uint32_t a, uint64_t v) {
  asm volatile("st.shared.u64 [%0], %1;" ::"r"(a), "l"(v));
}
__device__ __forceinline__ void sts128(uint32_t a, uint32_t x, uint32_t y, uint32_t z, uint32_t w) {
  asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(a), "r"(x), "r"(y), "r"(z), "r"(w));
}
__device__ __forceinline__ void atoms_xor(uint32_t a, uint32_t v) {
  asm volatile("red.shared.xor.b32 [%0], %1;" ::"r"(a), "r"(v));
}
__device__ __forceinline__ uint4 ldg128(const uint8_t* p) {
  return __ldg(reinterpret_cast<const uint4*>(p));
}
__device__ __forceinline__ uint32_t ldg32(const uint8_t* p) {
  return __ldg(reinterpret_cast<const uint32_t*>(p));
}
__device__ __forceinline__ void stg128_cs(uint8_t* p, uint4 v) {
  __stcs(reinterpret_cast<uint4*>(p), v);
}

struct Raw {
  uint4 v;     // this lane's 16 sites
  uint32_t e;  // lane 0: word left of the band; last lane: word right of it
};

// A source row as the motion needs it: its 16 bytes and the same bytes
// shifted by one column either way (computed once per row and reused by the
// three destination rows that read it).
struct Row {
  uint32_t w[4];
  uint32_t sl[4];  // column x-1 at every byte
  uint32_t sr[4];  // column x+1 at every byte
};

struct Konst {  // run-time copies of StepArgs::k1 ... k2p24
  uint32_t k1, k2, k4, k16, k32, k256, k2p24;
};

// Bit 0 of fin64(z) (fhpg_common.cuh fin64_bit0) with every shift written as
// a multiply so that it issues on the FMA pipe: x >> s == hi(x * 2^(32-s)),
// x << s == x * 2^s; only the four XORs use the (saturated) ALU pipe.
__device__ __forceinline__ uint32_t chir_bit(uint64_t z, const Konst& K) {
  const uint32_t lo = static_cast<uint32_t>(z), hi = static_cast<uint32_t>(z >> 32);
  const uint32_t t_lo = lo ^ (__umulhi(lo, K.k4) + hi * K.k4);  // lo32(z ^ (z >> 30))
  const uint32_t t_hi = hi ^ __umulhi(hi, K.k4);                // hi32(z ^ (z >> 30))
  const uint64_t w = static_cast<uint64_t>(t_lo) * static_cast<uint32_t>(kC1);
  const uint32_t z1_lo = static_cast<uint32_t>(w);
  const uint32_t z1_hi = static_cast<uint32_t>(w >> 32) + t_lo * static_cast<uint32_t>(kC1 >> 32) +
                         t_hi * static_cast<uint32_t>(kC1);
  const uint32_t u = z1_lo ^ (__umulhi(z1_lo, K.k32) + z1_hi * K.k32);  // lo32(z1 ^ (z1 >> 27))
  const uint32_t p = u * static_cast<uint32_t>(kC2);
  return (p ^ __umulhi(p, K.k2)) & 1u;  // bit0 ^ bit31
}

// key + y as one IMAD.WIDE (FMA pipe) instead of a carry chain on the ALU
// pipe: `one` is a run-time 1.
__device__ __forceinline__ uint64_t add_wide(uint64_t key, uint32_t y, uint32_t one) {
  uint64_t z;
  asm("mad.wide.u32 %0, %1, %2, %3;" : "=l"(z) : "r"(y), "r"(one), "l"(key));
  return z;
}

struct Lane {
  int lane, last;
  uint32_t x0;    // first column of the lane (clamped to 0 for inactive lanes)
  uint32_t eoff;  // column of the edge word this lane loads
  bool active;
};

__device__ __forceinline__ Raw load_raw(const uint8_t* row, const Lane& ln) {
  return Raw{ldg128(row + ln.x0), ldg32(row + ln.eoff)};
}

__device__ __forceinline__ Row finish(const Raw& r, const Lane& ln) {
  Row o;
  o.w[0] = r.v.x;
  o.w[1] = r.v.y;
  o.w[2] = r.v.z;
  o.w[3] = r.v.w;
  const uint32_t up = __shfl_up_sync(kFull, r.v.w, 1);
  const uint32_t dn = __shfl_down_sync(kFull, r.v.x, 1);
  const uint32_t L = ln.lane == 0 ? r.e : up;         // top byte = column x0-1
  const uint32_t R = ln.lane == ln.last ? r.e : dn;   // low byte = column x0+16
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    o.sl[j] = __byte_perm(j == 0 ? L : o.w[j - 1], o.w[j], 0x6543);
    o.sr[j] = __byte_perm(o.w[j], j == 3 ? R : o.w[j + 1], 0x4321);
  }
  return o;
}

// Column x-1 / x+1 at every byte of word j.
__device__ __forceinline__ uint32_t shl1(const Row& r, int j) { return r.sl[j]; }
__device__ __forceinline__ uint32_t shr1(const Row& r, int j) {
  return r.sr[j];
}
// (a & m) | (b & ~m) as one LOP3 (the compiler otherwise splits the chain
// into AND + OR-AND pairs).
template <uint32_t M>
__device__ __forceinline__ uint32_t mux(uint32_t a, uint32_t b) {
  uint32_t d;
  asm("lop3.b32 %0, %1, %2, %3, 0xE4;" : "=r"(d) : "r"(a), "r"(b), "n"(M));
  return d;
}

// One destination row. Pull sources (backends.cpp:64-73): k0 (x+q, r+1),
// k1 (x+q-1, r+1), k2 (x-1, r), k3 (x+q-1, r-1), k4 (x+q, r-1), k5 (x+1, r);
// rest bit stays, bit 7 = own obstacle bit. Returns the packed dep-site mask
// (bit 8b + 7 - j <-> byte b of word j).
template <int Q>
__device__ __forceinline__ uint32_t row_update(const Row& P, const Row& C, const Row& N,
                                               uint32_t lut, uint32_t laneoff, const Konst& K,
                                               uint32_t out0[4],
                                               uint32_t dep[4]) {
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const uint32_t n0 = Q ? shr1(N, j) : N.w[j];
    const uint32_t n1 = Q ? N.w[j] : shl1(N, j);
    const uint32_t p3 = Q ? P.w[j] : shl1(P, j);
    const uint32_t p4 = Q ? shr1(P, j) : P.w[j];
    uint32_t m = mux<0xC0C0C0C0u>(C.w[j], n0);  // bit 0 correct, 1-5 overwritten below
    m = mux<0x02020202u>(n1, m);
    m = mux<0x04040404u>(shl1(C, j), m);
    m = mux<0x08080808u>(p3, m);
    m = mux<0x10101010u>(p4, m);
    m = mux<0x20202020u>(shr1(C, j), m);
    // laneoff = LUT base (64 KB aligned) | lane * 4: [laneoff.b0, m.bk,
    // laneoff.b2, laneoff.b3] is the full address of the lane's entry.
    (void)lut;
    const uint32_t v0 = lds32(__byte_perm(laneoff, m, 0x3240));
    const uint32_t v1 = lds32(__byte_perm(laneoff, m, 0x3250));
    const uint32_t v2 = lds32(__byte_perm(laneoff, m, 0x3260));
    const uint32_t v3 = lds32(__byte_perm(laneoff, m, 0x3270));
    // Entries are out | xor << 16 with both < 256, so v0 + 256 v1 packs
    // [out_0, out_1, xor_0, xor_1] without carries (IMAD on the FMA pipe).
    const uint32_t A = v1 * K.k256 + v0;
    const uint32_t B = v3 * K.k256 + v2;
    out0[j] = __byte_perm(A, B, 0x5410);
    dep[j] = __byte_perm(A, B, 0x7632);
  }
  // Dep mask: bit 8b + 7 - j <-> byte b of word j (the flag bits shifted
  // into the high nibble of each byte; a second row goes to the low nibbles).
  const uint32_t FK = 0x80808080u;
  return (dep[0] & FK) | ((dep[1] >> 1) & (FK >> 1)) | ((dep[2] >> 2) & (FK >> 2)) |
         ((dep[3] >> 3) & (FK >> 3));
}

// One dep site handed to a walk callback.
struct Site {
  uint32_t row;   // row inside the batch
  uint32_t sh;    // 8 * byte index inside the staged word
  uint32_t key;   // smem address of the site's column key
  uint32_t word;  // smem address of the site's staged out word
};

// Bit index of the highest set bit (PTX bfind: one FLO).
__device__ __forceinline__ uint32_t top_bit(uint32_t m) {
  uint32_t p;
  asm("bfind.u32 %0, %1;" : "=r"(p) : "r"(m));
  return p;
}

// Load-balanced walk over the dep sites of a batch. Each lane holds two
// masks, M01 (rows 0, 1) and M23 (rows 2, 3): bit 8b + 7 - (4r' + j) <->
// row 2k+r', byte b of word j of the lane's 16 sites (the first row of a
// pair in the high nibbles of the bytes, the second in the low nibbles).
// Phase 1: every lane takes floor(T/32) of its own sites (T = the warp's
// total), a uniform trip count with no owner lookup. Phase 2: the sites left
// over on busier lanes are numbered lane-major and every lane takes an equal
// contiguous slice of that list (prefix sum + binary search over lanes).
// fn(site0, valid0, site1, valid1) handles two sites per call.
template <typename Fn>
__device__ __forceinline__ void balanced_walk(uint32_t M01, uint32_t M23, uint32_t smask,
                                              uint32_t stage, uint32_t keys, int lane, Fn&& fn);

template <typename Fn>
__device__ __forceinline__ void warp_walk(uint32_t M01, uint32_t M23, uint32_t smask,
                                          uint32_t stage, uint32_t keys, int lane, Fn&& fn) {
  // Phase 1 measured slower (v11: 1207 vs 1267 GSUPS, same instruction
  // count per site): the per-site overhead is the same whether the site is
  // the lane's own or another lane's. Keep the single balanced phase.
  constexpr bool kOwnPhase = false;
  const int T = kOwnPhase ? static_cast<int>(__reduce_add_sync(kFull, __popc(M01) + __popc(M23))) : 0;
  const int M = T >> 5;
  const uint32_t kown = keys + static_cast<uint32_t>(lane) * 256u;
  const uint32_t wown = stage + static_cast<uint32_t>(lane) * 16u;
  auto own_next = [&](bool& valid) {
    const bool useA = M01 != 0u;
    const uint32_t m = useA ? M01 : M23;
    valid = m != 0u;
    const uint32_t p = top_bit(m);  // p = 8b + 7 - (4 r1 + j); 0xFFFFFFFF if m == 0
    const uint32_t bit = valid ? (1u << p) : 0u;
    if (useA) M01 ^= bit;
    else M23 ^= bit;
    const uint32_t np = ~p;
    const uint32_t j = np & 3u;
    const uint32_t r1 = (np >> 2) & 1u;
    const uint32_t pr = useA ? 0u : 1u;
    Site t;
    t.row = pr * 2u + r1;
    t.sh = p & 0x18u;
    t.key = kown + j * 32u + t.sh;
    t.word = wown + pr * 1024u + r1 * 512u + j * 4u;
    return t;
  };
  for (int it = 0; it < M; it += 2) {  // M is warp-uniform
    bool v0, v1 = false;
    const Site t0 = own_next(v0);
    const Site t1 = it + 1 < M ? own_next(v1) : t0;
    fn(t0, v0, t1, v1);
  }
  balanced_walk(M01, M23, smask, stage, keys, lane, fn);
}

template <typename Fn>
__device__ __forceinline__ void balanced_walk(uint32_t M01, uint32_t M23, uint32_t smask,
                                              uint32_t stage, uint32_t keys, int lane, Fn&& fn) {
  const int cnt = __popc(M01) + __popc(M23);
  int incl = cnt;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const int v = __shfl_up_sync(kFull, incl, d);
    if (lane >= d) incl += v;
  }
  const int T = __shfl_sync(kFull, incl, 31);
  if (T == 0) return;
  asm volatile("st.shared.v2.u32 [%0], {%1,%2};" ::"r"(smask + lane * 8), "r"(M01), "r"(M23));
  const int s = (lane * T) >> 5;
  const int e = ((lane + 1) * T) >> 5;
  int o = 0;
#pragma unroll
  for (int step = 16; step; step >>= 1) {
    const int v = __shfl_sync(kFull, incl, o + step - 1);
    if (v <= s) o += step;
  }
  const int excl_o = __shfl_sync(kFull, incl - cnt, o);
  __syncwarp();
  if (s < e) {
    int k = s - excl_o;
    uint32_t off = static_cast<uint32_t>(o) * 8u;  // byte offset of the current mask
    uint32_t mask = lds32(smask + off);
    for (;;) {
      const int c = __popc(mask);
      if (k < c) break;
      k -= c;
      off += 4u;
      mask = lds32(smask + off);
    }
    for (; k > 0; --k) mask ^= 1u << top_bit(mask);
    // Per-owner bases, refreshed when the walk moves to the next mask.
    uint32_t kbase = keys + (off >> 3) * 256u;
    uint32_t wbase = stage + (off >> 3) * 16u + (off & 4u) * 256u;
    uint32_t rbase = (off >> 1) & 2u;
    auto next = [&]() {
      while (mask == 0u) {
        off += 4u;
        mask = lds32(smask + off);
        kbase = keys + (off >> 3) * 256u;
        wbase = stage + (off >> 3) * 16u + (off & 4u) * 256u;
        rbase = (off >> 1) & 2u;
      }
      const uint32_t p = top_bit(mask);  // p = 8b + 7 - k, k = 4 * r1 + j
      mask ^= 1u << p;
      const uint32_t np = ~p;
      const uint32_t j = np & 3u;         // word in the lane's 16 bytes
      const uint32_t r1 = (np >> 2) & 1u;  // second row of the pair
      Site t;
      t.row = rbase + r1;
      t.sh = p & 0x18u;                    // 8 * byte
      t.key = kbase + j * 32u + t.sh;      // column 4j + b, 8 bytes per key
      t.word = wbase + r1 * 512u + j * 4u;
      return t;
    };
    // Two sites per iteration: two independent RNG chains in flight per lane.
    for (int it = s; it < e; it += 2) {
      const Site t0 = next();
      const bool has1 = it + 1 < e;
      const Site t1 = has1 ? next() : t0;
      fn(t0, true, t1, has1);
    }
  }
  __syncwarp();
}

template <int P0, bool FORCE, bool FULL>
__device__ __forceinline__ void run_batch(const StepArgs& a, uint32_t lut, uint32_t keys,
                                          uint32_t stage, const Lane& ln, int rb, int nb,
                                          Row (&win)[kBatch + 2], Raw (&pre)[2],
                                          const uint8_t*& nxt, uint8_t*& out, unsigned& swaps) {
  const size_t pitch = a.pitch;
  const uint32_t smask = stage + kStageMask;
  const uint32_t my = stage + ln.lane * 16;  // this lane's 16 bytes of a staged row
  const uint32_t laneoff = lut | (ln.lane * 4u);  // lut is 64 KB aligned
  const Konst K{a.k1, a.k2, a.k4, a.k16, a.k32, a.k256, a.k2p24};
  uint32_t F[kBatch];
  static_for<0, kBatch>([&](auto ic) {
    constexpr int i = decltype(ic)::value;
    F[i] = 0u;
    if (FULL || i < nb) {
      win[i + 2] = finish(pre[i & 1], ln);
      pre[i & 1] = load_raw(nxt, ln);
      nxt += pitch;
      uint32_t o[4], d[4];
      F[i] = row_update<(P0 + i) & 1>(win[i], win[i + 1], win[i + 2], lut, laneoff, K, o, d);
      sts128(my + i * 512, o[0], o[1], o[2], o[3]);
      sts128(my + kStageDep + i * 512, d[0], d[1], d[2], d[3]);
    }
  });
  uint32_t M01 = F[0] | (F[1] >> 4), M23 = F[2] | (F[3] >> 4);
  if (!ln.active) M01 = M23 = 0u;
  __syncwarp();
  const uint64_t ybase = static_cast<uint64_t>(a.row0 + rb);
  const uint32_t y32 = static_cast<uint32_t>(a.row0 + rb);  // global rows < 2^31
  // Chirality: sites whose two outcomes differ (rng.hpp:25-33 keyed by the
  // 1-based storage column and global row, step.cpp:73-76).
  warp_walk(M01, M23, smask, stage, keys, ln.lane,
            [&](const Site& t0, bool has0, const Site& t1, bool has1) {
    // (chir_bit, the all-FMA-pipe variant, measured 4% slower: more issue slots.)
    const uint32_t c0 = fin64_bit0(add_wide(lds64(t0.key), y32 + t0.row, K.k1)) & (has0 ? 1u : 0u);
    const uint32_t c1 = fin64_bit0(add_wide(lds64(t1.key), y32 + t1.row, K.k1)) & (has1 ? 1u : 0u);
    const uint32_t d0 = lds32(t0.word + kStageDep) & (0x7Fu << t0.sh);
    const uint32_t d1 = lds32(t1.word + kStageDep) & (0x7Fu << t1.sh);
    atoms_xor(t0.word, d0 * c0);  // select by multiply (FMA pipe)
    atoms_xor(t1.word, d1 * c1);
  });
  if (FORCE) {
    // Forcing on the post-collision state (step.cpp:79-88): fluid, W set, E clear.
    uint32_t G[kBatch];
    static_for<0, kBatch>([&](auto ic) {
      constexpr int i = decltype(ic)::value;
      G[i] = 0u;
      if (FULL || i < nb) {
        const uint4 f = lds128(my + i * 512);
        const uint32_t w[4] = {f.x, f.y, f.z, f.w};
        uint32_t g = 0;
#pragma unroll
        for (int j = 0; j < 4; ++j)
          g |= (((w[j] >> 5) & ~(w[j] >> 2) & ~(w[j] >> 7)) & 0x01010101u) << (7 - j);
        G[i] = g;
      }
    });
    uint32_t G01 = G[0] | (G[1] >> 4), G23 = G[2] | (G[3] >> 4);
    if (!ln.active) G01 = G23 = 0u;
    warp_walk(G01, G23, smask, stage, keys + 128u * 256u, ln.lane,
              [&](const Site& t0, bool has0, const Site& t1, bool has1) {
      const bool f0 = has0 && (fin64(lds64(t0.key) + ybase + t0.row) >> 32) < a.thr;
      const bool f1 = has1 && (fin64(lds64(t1.key) + ybase + t1.row) >> 32) < a.thr;
      atoms_xor(t0.word, f0 ? 0x24u << t0.sh : 0u);
      atoms_xor(t1.word, f1 ? 0x24u << t1.sh : 0u);
      swaps += static_cast<unsigned>(f0) + static_cast<unsigned>(f1);
    });
  }
  static_for<0, kBatch>([&](auto ic) {
    constexpr int i = decltype(ic)::value;
    if ((FULL || i < nb) && ln.active) stg128_cs(out + i * pitch, lds128(my + i * 512));
  });
  out += kBatch * pitch;
  // The window of the next batch: rows rb+3, rb+4.
  win[0] = win[kBatch];
  win[1] = win[kBatch + 1];
  __syncwarp();
}

template <int P0, bool FORCE>
__device__ __forceinline__ void run_segment(const StepArgs& a, uint32_t lut, uint32_t keys,
                                            uint32_t stage, const Lane& ln, int r_begin,
                                            int r_end, unsigned& swaps) {
  const size_t pitch = a.pitch;
  Row win[kBatch + 2];  // rows rb-1 .. rb+kBatch
  win[0] = finish(load_raw(a.src + (r_begin - 1) * (long long)pitch, ln), ln);
  win[1] = finish(load_raw(a.src + r_begin * (long long)pitch, ln), ln);
  const uint8_t* nxt = a.src + (r_begin + 1) * (long long)pitch;
  Raw pre[2];
  pre[0] = load_raw(nxt, ln);
  nxt += pitch;
  pre[1] = load_raw(nxt, ln);
  nxt += pitch;  // buffers carry 2 spare zero rows below the halo: over-prefetch is safe
  uint8_t* out = a.dst + r_begin * (long long)pitch + ln.x0;
  int rb = r_begin;
  for (; rb + kBatch <= r_end; rb += kBatch)
    run_batch<P0, FORCE, true>(a, lut, keys, stage, ln, rb, kBatch, win, pre, nxt, out, swaps);
  if (rb < r_end)
    run_batch<P0, FORCE, false>(a, lut, keys, stage, ln, rb, r_end - rb, win, pre, nxt, out, swaps);
}

template <bool FORCE>
__global__ void __launch_bounds__(kThreads, 1) step_fast_kernel(StepArgs a) {
  extern __shared__ __align__(16) uint8_t smem[];
  const uint32_t sbase = smem_u32(smem);
  // The LUT sits on a 64 KB boundary of the shared window, so one PRMT builds
  // the complete LDS address (base bytes 2-3 | state << 8 | lane * 4) with no
  // add. Warp stages fill the space before and after it.
  const uint32_t lut_abs = (sbase + 0xFFFFu) & ~0xFFFFu;
  const uint32_t kpre = (lut_abs - sbase) / kWarpStage;
  const int warp = threadIdx.x >> 5;
  const int band_group = blockIdx.x % a.nbands_groups;
  const int seg_group = blockIdx.x / a.nbands_groups;
  const int cta_x0 = band_group * a.bpc * 512;
  if (threadIdx.x == 0 &&
      lut_abs + kLutBytes + (kWarps - umin(kpre, kWarps)) * kWarpStage > sbase + kSmem)
    __trap();  // shared-memory map does not fit the request
  // The prologue is latency-bound on small lattices: every global load is
  // issued before the first dependent shared store.
  // Column keys of this CTA's columns (up to 2048) into the LUT rows' second
  // halves: column c at row c >> 4, +128 + (c & 15) * 8 (a lane's 16 keys
  // share a row); forcing keys 128 rows further.
  constexpr int kKeyIters = (kBandsPerCta * 512 + kThreads - 1) / kThreads;
  uint64_t kc[kKeyIters], kf[kKeyIters];
#pragma unroll
  for (int j = 0; j < kKeyIters; ++j) {
    const int c = threadIdx.x + j * kThreads;
    const bool ok = c < a.bpc * 512 && cta_x0 + c < a.W;
    kc[j] = ok ? a.zc[cta_x0 + c] : 0;
    kf[j] = ok && FORCE ? a.zf[cta_x0 + c] : 0;
  }
  // The 512-byte table goes through shared memory once (warp 0's stage,
  // free until the second barrier).
  const uint32_t tab = kpre > 0 ? sbase : lut_abs + kLutBytes;
  if (threadIdx.x < 128)
    sts32(tab + threadIdx.x * 4, reinterpret_cast<const uint32_t*>(a.table)[threadIdx.x]);
#pragma unroll
  for (int j = 0; j < kKeyIters; ++j) {
    const int c = threadIdx.x + j * kThreads;
    if (c < a.bpc * 512 && cta_x0 + c < a.W) {
      sts64(lut_abs + (c >> 4) * 256 + 128 + (c & 15) * 8, kc[j]);
      if (FORCE) sts64(lut_abs + (128 + (c >> 4)) * 256 + 128 + (c & 15) * 8, kf[j]);
    }
  }
  __syncthreads();
  // LUT: lane-private words (e*256 + 4l) = out(ch0) | flagged XOR(ch0, ch1) << 16.
  for (int i = threadIdx.x; i < 256 * 32; i += blockDim.x) {
    const int e = i >> 5, l = i & 31;
    const uint32_t o0 = lds8(tab + e), o1 = lds8(tab + 256 + e);
    const uint32_t x = o0 ^ o1;
    sts32(lut_abs + e * 256 + l * 4, o0 | ((x | (x ? 0x80u : 0u)) << 16));
  }
  __syncthreads();
  // Next step's column keys (read by the next launch only).
  if (a.zc_next) {
    const int n = gridDim.x * blockDim.x;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < a.W; i += n) {
      a.zc_next[i] = column_key(a.kc_next, static_cast<uint64_t>(i) + 1);
      if (a.zf_next) a.zf_next[i] = column_key(a.kf_next, static_cast<uint64_t>(i) + 1);
    }
  }

  const int bic = warp % a.bpc;
  const int band = band_group * a.bpc + bic;
  const int seg = seg_group * a.spc + warp / a.bpc;
  const int r_begin = a.row_lo + seg * a.seg_rows;
  if (warp >= a.bpc * a.spc || band >= a.nbands || r_begin >= a.row_hi) return;  // whole warp
  const int r_end = min(a.row_hi, r_begin + a.seg_rows);

  Lane ln;
  ln.lane = threadIdx.x & 31;
  const int band_x = band * 512;
  const int x0 = band_x + ln.lane * 16;
  ln.active = x0 < a.W;
  ln.x0 = ln.active ? x0 : 0;
  ln.last = min(31, (a.W - band_x) / 16 - 1);
  ln.eoff = ln.lane == 0 ? (x0 == 0 ? a.W - 4 : x0 - 4)
                         : (ln.lane == ln.last ? (x0 + 16 == a.W ? 0 : x0 + 16) : ln.x0);
  const uint32_t lut = lut_abs;
  const uint32_t keys = lut_abs + bic * 32 * 256 + 128;  // a band's 512 keys: 32 LUT rows
  const uint32_t stage = static_cast<uint32_t>(warp) < kpre
                             ? sbase + warp * kWarpStage
                             : lut_abs + kLutBytes + (warp - kpre) * kWarpStage;
  unsigned swaps = 0;
  if ((a.row0 + r_begin) & 1)
    run_segment<1, FORCE>(a, lut, keys, stage, ln, r_begin, r_end, swaps);
  else
    run_segment<0, FORCE>(a, lut, keys, stage, ln, r_begin, r_end, swaps);

  if (FORCE) {
    unsigned long long s = swaps;
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(kFull, s, o);
    if (ln.lane == 0 && s) atomicAdd(a.swaps, s);
  }
}

}  // namespace

int launch_step_fast(const StepArgs& a0, int num_sms, cudaStream_t st) {
  StepArgs a = a0;
  ensure_smem_optin(reinterpret_cast<const void*>(step_fast_kernel<true>), kSmem);
  ensure_smem_optin(reinterpret_cast<const void*>(step_fast_kernel<false>), kSmem);
  const int rows = a.row_hi - a.row_lo;
  a.k1 = 1u;
  a.k2 = 2u;
  a.k4 = 4u;
  a.k32 = 32u;
  a.k16 = 16u;
  a.k256 = 256u;
  a.k2p24 = 1u << 24;
  a.nbands = (a.W + 511) / 512;
  // Narrow lattices put fewer bands and more row segments in a CTA so that
  // all 20 warps stay busy.
  a.bpc = a.nbands < kBandsPerCta ? a.nbands : kBandsPerCta;
  a.spc = kWarps / a.bpc;
  a.nbands_groups = (a.nbands + a.bpc - 1) / a.bpc;
  // One wave: at most num_sms CTAs (one per SM), each a.spc segments deep.
  int seg_groups = num_sms / a.nbands_groups;
  if (seg_groups < 1) seg_groups = 1;
  int seg = (rows + seg_groups * a.spc - 1) / (seg_groups * a.spc);
  if (seg < kBatch) seg = kBatch;
  a.seg_rows = seg;
  const int nseg = (rows + seg - 1) / seg;
  seg_groups = (nseg + a.spc - 1) / a.spc;
  const int grid = a.nbands_groups * seg_groups;
  if (a.thr != 0) step_fast_kernel<true><<<grid, kThreads, kSmem, st>>>(a);
  else step_fast_kernel<false><<<grid, kThreads, kSmem, st>>>(a);
  return 1;
}

}  // namespace fhpg
