// TEST INFRASTRUCTURE: exercises the C++ host layer (namespace fhp_b200)
// the way the reference's doctest suites exercise proj/core
// (test_collision.cpp, test_lattice.cpp, test_step.cpp, test_bench.cpp),
// checking the device path against the C oracle (oracle/fhp_oracle.c).
//
//   test_host_api cpu   # host-only checks (no GPU needed)
//   test_host_api gpu   # device checks (B200)
#include <cstdio>
#include <cstring>
#include <fstream>
#include <functional>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "fhp_b200/fhp.hpp"
#include "fhp_oracle.h"

using namespace fhp_b200;

static int g_fail = 0, g_checks = 0;
#define CHECK(c)                                                          \
  do {                                                                    \
    ++g_checks;                                                           \
    if (!(c)) {                                                           \
      ++g_fail;                                                           \
      std::printf("FAIL %s:%d  %s\n", __FILE__, __LINE__, #c);            \
    }                                                                     \
  } while (0)
#define CHECK_THROWS_AS(expr, T)                                          \
  do {                                                                    \
    bool thrown = false;                                                  \
    try {                                                                 \
      expr;                                                               \
    } catch (const T&) {                                                  \
      thrown = true;                                                      \
    } catch (...) {                                                       \
    }                                                                     \
    CHECK(thrown);                                                        \
  } while (0)

// ---------------------------------------------------------------- helpers
static std::vector<uint8_t> interior(const Lattice& lat) {
  std::vector<uint8_t> v(static_cast<size_t>(lat.width()) * lat.height());
  for (int r = 0; r < lat.height(); ++r)
    for (int x = 1; x <= lat.width(); ++x) v[static_cast<size_t>(r) * lat.width() + x - 1] = lat.node(r, x);
  return v;
}

// Scrambled lattice (fo_scramble: particles on walls and obstacles too).
static Lattice scrambled(int W, int H, uint64_t seed, std::vector<uint8_t>& state,
                         std::vector<uint8_t>& mask) {
  state.assign(static_cast<size_t>(W) * H, 0);
  mask.assign(static_cast<size_t>(W) * H, 0);
  fo_scramble(W, H, seed, state.data(), mask.data());
  Lattice lat(W, H);
  for (int r = 0; r < H; ++r)
    for (int x = 1; x <= W; ++x)
      if (mask[static_cast<size_t>(r) * W + x - 1]) lat.set_obstacle(r, x, true);
  for (int r = 0; r < H; ++r)
    for (int x = 1; x <= W; ++x) lat.set_node(r, x, state[static_cast<size_t>(r) * W + x - 1]);
  sync_ghost_columns(lat);
  return lat;
}

// ---------------------------------------------------------------- cpu
static void cpu_tests() {
  // test_collision.cpp equivalents
  const auto t = build_table();
  CHECK(collide_node(t, 0b00001001, 1) == 0b00010010);
  CHECK(collide_node(t, 0b00001001, 0) == 0b00100100);
  CHECK(collide_node(t, 0b00010101, 0) == 0b00101010);
  CHECK(collide_node(t, 0b01000100, 0) == 0b00001010);
  CHECK(validate_table(t).valid());
  CHECK(validate_table(build_table(RuleVariant::FhpI)).valid());
  CHECK(validate_table(build_table(RuleVariant::FhpIII)).valid());
  uint8_t ref[512];
  fo_build_default_table(ref);
  CHECK(std::memcmp(ref, t.entries.data(), 512) == 0);
  auto bad = t;
  bad.entries[1] = 0;
  const auto rep = validate_table(bad);
  CHECK(!rep.valid() && rep.issues[0].index == 1 && rep.issues[0].kind == ValidationIssue::Kind::Mass);
  bad = t;
  bad.entries[1] = 0b10;
  CHECK(validate_table(bad).issues.size() == 1 &&
        validate_table(bad).issues[0].kind == ValidationIssue::Kind::Momentum);
  const auto bytes = save_table(t);
  CHECK(bytes.size() == 520);
  CHECK(load_table(bytes).entries == t.entries);
  auto tr = bytes;
  tr.pop_back();
  CHECK_THROWS_AS(load_table(tr), std::runtime_error);
  auto bm = bytes;
  bm[0] = 'X';
  CHECK_THROWS_AS(load_table(bm), std::runtime_error);
  auto cor = bytes;
  cor[9] = 0;
  CHECK_THROWS_AS(load_table(cor), std::runtime_error);
  bool ok = true;
  try {
    load_table(cor, true);
  } catch (...) {
    ok = false;
  }
  CHECK(ok);
  write_table_file("/tmp/fhp_b200_test.tab", build_table(RuleVariant::FhpIII));
  CHECK(load_table(read_table_file("/tmp/fhp_b200_test.tab")).entries ==
        build_table(RuleVariant::FhpIII).entries);

  // test_lattice.cpp equivalents
  CHECK(neighbor_of(5, 2, Direction::E) == (Coord{6, 2}));
  CHECK(neighbor_of(5, 2, Direction::NE) == (Coord{5, 1}));
  CHECK(neighbor_of(5, 3, Direction::NE) == (Coord{6, 2}));
  CHECK(opposite(Direction::E) == Direction::W);
  Lattice g(4, 5);
  for (int r = 0; r < 5; ++r) {
    g.set_node(r, 1, static_cast<NodeState>(0x10 + r));
    g.set_node(r, 4, static_cast<NodeState>(0x20 + r));
  }
  sync_ghost_columns(g);
  for (int r = 0; r < 5; ++r) CHECK(g.node(r, 5) == 0x10 + r && g.node(r, 0) == 0x20 + r);
  Lattice a(8, 5), b(8, 5);
  CHECK(state_digest(a) == state_digest(b));
  b.set_node(2, 3, 0x04);
  CHECK(state_digest(a) != state_digest(b));
  b.set_node(2, 3, 0);
  b.set_node(2, 0, 0x3F);
  CHECK(state_digest(a) == state_digest(b));
  {
    std::ofstream f("/tmp/fhp_b200_geom.txt");
    f << "######\n#....#\n\n#.##.#\r\n#....#\n######\n";
  }
  const auto rows = read_geometry_file("/tmp/fhp_b200_geom.txt");
  CHECK(rows.size() == 5 && rows[2] == "#.##.#");
  {
    std::ofstream f("/tmp/fhp_b200_geom_bad.txt");
    f << "..x.\n";
  }
  CHECK_THROWS_AS(read_geometry_file("/tmp/fhp_b200_geom_bad.txt"), std::runtime_error);
  CHECK_THROWS_AS(read_geometry_file("/tmp/does_not_exist_fhp"), std::runtime_error);
  CHECK_THROWS_AS(Lattice(0, 5), std::invalid_argument);
  CHECK_THROWS_AS(Lattice(5, 2), std::invalid_argument);
  const auto cyl = cylinder_geometry(64, 32, 16, 16, 2);
  uint8_t m[64 * 32];
  fo_cylinder(64, 32, 16, 16, 2, m);
  bool same = true;
  for (int r = 0; r < 32; ++r)
    for (int x = 0; x < 64; ++x) same = same && ((cyl[r][x] == '#') == (m[r * 64 + x] != 0));
  CHECK(same);

  // config / bench harness (test_bench.cpp, acceptance.cpp:239-258)
  SimConfig cfg;
  cfg.width = 0;
  CHECK_THROWS_AS(cfg.validate(), std::invalid_argument);
  cfg = SimConfig{};
  cfg.lanes = 33;
  CHECK_THROWS_AS(cfg.validate(), std::invalid_argument);
  cfg = SimConfig{};
  cfg.gpus = 0;
  CHECK_THROWS_AS(cfg.validate(), std::invalid_argument);
  cfg = SimConfig{};
  cfg.gpus = 2;
  cfg.devices = {0};
  CHECK_THROWS_AS(cfg.validate(), std::invalid_argument);
  cfg = SimConfig{};
  cfg.height = 5;
  cfg.gpus = 4;  // 3 interior rows (make_strip_plan)
  CHECK_THROWS_AS(cfg.validate(), std::invalid_argument);
  CHECK(std::string(backend_name(Backend::Cuda)) == "cuda");
  CHECK(compute_mups(1000, 1000, 100, 0.1) == 1000.0);
  CHECK_THROWS_AS(compute_mups(1, 1, 1, 0.0), std::invalid_argument);
  BenchRecord rec;
  rec.backend = "cuda";
  rec.mups = 1.5;
  CHECK(to_json_line(rec).find("\"backend\":\"cuda\"") != std::string::npos);
  CHECK(ascii_table({rec}).find("cuda") != std::string::npos);

  // host observables (test_observables.cpp:32-50)
  Lattice e(8, 6);
  CHECK(total_mass(e) == 0);
  e.set_node(2, 3, 0x04);
  e.set_node(3, 5, 0x20);
  CHECK((total_momentum(e) == MomentumVec{0, 0}));
  e.set_node(3, 5, 0x00);
  e.set_node(4, 4, 0x02);
  CHECK((total_momentum(e) == MomentumVec{3, 1}));
  std::ostringstream pgm(std::ios::binary);
  Lattice east(8, 10);
  for (int r = 1; r < 9; ++r)
    for (int x = 1; x <= 8; ++x) east.set_node(r, x, 0x04);
  write_density_pgm(pgm, coarse_grain(east, 4));
  CHECK(pgm.str().size() == 15 && static_cast<unsigned char>(pgm.str()[11]) == 36);
}

// ---------------------------------------------------------------- gpu
static void gpu_tests() {
  const auto t3 = build_table(RuleVariant::FhpIII);
  SimConfig cfg;
  cfg.backend = Backend::Cuda;
  // advance drop-in on adversarial uploads, fast (W%16==0) and generic widths
  for (int W : {64, 48, 37, 512, 1056}) {
    std::vector<uint8_t> s, m;
    Lattice lat = scrambled(W, 29, 1000 + W, s, m);
    cfg.seed = 77 + W;
    cfg.force_p = 0.25;
    const uint64_t sw = advance(lat, t3, cfg, 11, 9);
    const uint64_t rsw = fo_advance(W, 29, s.data(), m.data(), t3.entries.data(), cfg.seed,
                                    fo_bernoulli_threshold(cfg.force_p), 11, 9);
    CHECK(interior(lat) == s);
    CHECK(sw == rsw);
  }
  // steps <= 0 leaves the lattice untouched, bit 7 included
  {
    std::vector<uint8_t> s, m;
    Lattice lat = scrambled(40, 12, 5, s, m);
    lat.set_node(3, 3, lat.node(3, 3) | 0x80);
    const auto before = interior(lat);
    CHECK(advance(lat, t3, cfg, 0, 0) == 0);
    CHECK(interior(lat) == before);
  }
  // other backends are not provided here
  {
    Lattice lat(16, 8);
    SimConfig c2 = cfg;
    c2.backend = Backend::Scalar;
    CHECK_THROWS_AS(advance(lat, t3, c2, 0, 1), std::invalid_argument);
  }
  // init_lattice == oracle init
  {
    SimConfig c;
    c.width = 333;
    c.height = 97;
    c.seed = 5;
    c.fill_density = 0.45;
    const auto geom = cylinder_geometry(c.width, c.height, c.width / 4.0, c.height / 2.0, c.height / 16.0);
    Lattice lat = init_lattice(c, geom);
    std::vector<uint8_t> mask(static_cast<size_t>(c.width) * c.height), ref(mask.size());
    fo_cylinder(c.width, c.height, c.width / 4.0, c.height / 2.0, c.height / 16.0, mask.data());
    fo_init(c.width, c.height, c.seed, c.fill_density, mask.data(), ref.data());
    CHECK(interior(lat) == ref);
    CHECK(lat.obstacle(0, 1) && lat.obstacle(c.height - 1, 7));
  }
  // run(): digest + series + device dumps vs the oracle, DEFAULT and FHP-III
  for (RuleVariant v : {RuleVariant::Default, RuleVariant::FhpIII}) {
    SimConfig c;
    c.width = 96;
    c.height = 40;
    c.steps = 77;
    c.fill_density = 0.3;
    c.force_p = 0.05;
    c.seed = 9;
    c.dump_every = 20;
    c.rules = v;
    const auto table = build_table(v);
    int dumps = 0;
    const auto res = run(c, table, {}, [&](int, const Engine& e) {
      ++dumps;
      const auto f = coarse_grain(e, 4);
      CHECK(f.cells_x == 24 && f.cells_y == 10);
    });
    std::vector<uint8_t> ref(static_cast<size_t>(c.width) * c.height);
    fo_init(c.width, c.height, c.seed, c.fill_density, nullptr, ref.data());
    const uint64_t rsw = fo_advance(c.width, c.height, ref.data(), nullptr, table.entries.data(),
                                    c.seed, fo_bernoulli_threshold(c.force_p), 0, c.steps);
    CHECK(interior(res.lattice) == ref);
    CHECK(res.forcing_swaps == rsw);
    CHECK(state_digest(res.lattice) == fo_digest(c.width, c.height, ref.data()));
    CHECK(dumps == 4);  // 20, 40, 60, final 77
    CHECK(res.series.size() == 5 && res.series.front().mass == res.series.back().mass);
    // observables: device reductions == host recomputation
    Engine e(c.width, c.height);
    e.upload(res.lattice);
    const auto fd = coarse_grain(e, 5), fh = coarse_grain(res.lattice, 5);
    bool eq = fd.cells.size() == fh.cells.size();
    for (size_t i = 0; eq && i < fd.cells.size(); ++i)
      eq = fd.cells[i].rho == fh.cells[i].rho && fd.cells[i].ux == fh.cells[i].ux &&
           fd.cells[i].uy == fh.cells[i].uy && fd.cells[i].nodes == fh.cells[i].nodes;
    CHECK(eq);
    const auto pd = velocity_profile(e), ph = velocity_profile(res.lattice);
    bool peq = pd.size() == ph.size();
    for (size_t i = 0; peq && i < pd.size(); ++i)
      peq = pd[i].mean_ux == ph[i].mean_ux && pd[i].sample_count == ph[i].sample_count;
    CHECK(peq);
    CHECK(total_mass(e) == total_mass(res.lattice));
    CHECK(total_momentum(e) == total_momentum(res.lattice));
  }
  // cfg.gpus: the same run over 3 row strips (all on device 0 here), and the
  // asynchronous cell-dump pipeline: identical lattice, swaps and dumps
  {
    SimConfig c;
    c.width = 2048;
    c.height = 131;
    c.steps = 50;
    c.fill_density = 0.25;
    c.force_p = 0.02;
    c.seed = 21;
    c.dump_every = 20;
    c.rules = RuleVariant::FhpIII;
    const auto table = build_table(RuleVariant::FhpIII);
    std::vector<FlowField> sync_dumps;
    const auto one = run(c, table, {}, [&](int, const Engine& e) { sync_dumps.push_back(coarse_grain(e, 16)); });
    SimConfig c3 = c;
    c3.gpus = 3;
    c3.devices = {0, 0, 0};
    std::vector<int> steps_seen;
    std::vector<FlowField> async_dumps;
    const auto three = run_cell_dumps(c3, table, 16, [&](int s, const FlowField& f) {
      steps_seen.push_back(s);
      async_dumps.push_back(f);
    });
    CHECK(interior(three.lattice) == interior(one.lattice));
    CHECK(three.forcing_swaps == one.forcing_swaps);
    CHECK((steps_seen == std::vector<int>{20, 40, 50}));
    bool same = async_dumps.size() == sync_dumps.size();
    for (size_t k = 0; same && k < async_dumps.size(); ++k)
      for (size_t i = 0; same && i < async_dumps[k].cells.size(); ++i)
        same = async_dumps[k].cells[i].rho == sync_dumps[k].cells[i].rho &&
               async_dumps[k].cells[i].ux == sync_dumps[k].cells[i].ux &&
               async_dumps[k].cells[i].uy == sync_dumps[k].cells[i].uy;
    CHECK(same);
    CHECK(three.series.size() == one.series.size() &&
          three.series.back().mass == one.series.back().mass);
    // the drop-in keeps its engine between calls; a new table is picked up
    std::vector<uint8_t> s0, m0;
    Lattice lat = scrambled(2048, 40, 99, s0, m0);
    SimConfig cd;
    cd.seed = 5;
    cd.force_p = 0.1;
    uint64_t sw = advance(lat, table, cd, 0, 4);
    const auto tdef = build_table(RuleVariant::Default);
    sw += advance(lat, tdef, cd, 4, 3);
    std::vector<uint8_t> ref = s0;
    uint64_t rsw = fo_advance(2048, 40, ref.data(), m0.data(), table.entries.data(), cd.seed,
                              fo_bernoulli_threshold(cd.force_p), 0, 4);
    rsw += fo_advance(2048, 40, ref.data(), m0.data(), tdef.entries.data(), cd.seed,
                      fo_bernoulli_threshold(cd.force_p), 4, 3);
    CHECK(interior(lat) == ref);
    CHECK(sw == rsw);
  }
  // run_bench with an injected clock (acceptance.cpp:239-258)
  {
    SimConfig c;
    c.width = 1000;
    c.height = 1000;
    c.steps = 100;
    c.warmup_steps = 0;
    c.fill_density = 0.3;
    double tt = 0.0;
    const auto res = run_bench(c, 1, [&tt]() {
      const double now = tt;
      tt += 0.1;
      return now;
    });
    CHECK(res.median.mups == 1000.0);
  }
}

int main(int argc, char** argv) {
  const std::string mode = argc > 1 ? argv[1] : "cpu";
  try {
    if (mode == "cpu" || mode == "all") cpu_tests();
    if (mode == "gpu" || mode == "all") gpu_tests();
  } catch (const std::exception& e) {
    std::printf("FAIL uncaught exception: %s\n", e.what());
    ++g_fail;
  }
  std::printf("%s: %d checks, %d failures\n", mode.c_str(), g_checks, g_fail);
  return g_fail ? 1 : 0;
}
