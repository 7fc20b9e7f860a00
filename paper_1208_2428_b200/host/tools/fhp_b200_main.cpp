// fhp_b200 — command-line front end with the reference CLI's subcommands,
// flags and exit codes (proj/tools/fhp_main.cpp:18-183): run, bench,
// tablegen, validate; std::invalid_argument -> exit 2, std::runtime_error ->
// exit 3. Additions: --rules default|fhp1|fhp3, --clear-rest, --device,
// tablegen --rules, geometry --cylinder generator. Dumps (coarse_grain(4),
// velocity profile, density PGM) are reduced on the GPU; the lattice stays
// in HBM.
#include <cstdio>
#include <cstdlib>
#include <iostream>
#include <stdexcept>
#include <string>
#include <vector>

#include "fhp_b200/bench.hpp"
#include "fhp_b200/checkpoint.hpp"
#include "fhp_b200/collision.hpp"
#include "fhp_b200/observables.hpp"
#include "fhp_b200/step.hpp"

using namespace fhp_b200;

namespace {

[[noreturn]] void usage(const std::string& why) {
  throw std::invalid_argument(why +
                              "\nusage: fhp_b200 run|bench [--width W] [--height H] [--steps N] "
                              "[--density d] [--force-p p] [--seed s] [--rules default|fhp1|fhp3] "
                              "[--table-file F] [--geometry-file F] [--clear-rest] [--device D] "
                              "[--dump-every K --out-prefix P] [--repeats R --warmup W]\n"
                              "       [--checkpoint-file F [--checkpoint-every K]] [--resume F]\n"
                              "       fhp_b200 tablegen OUTPUT [--rules ...]\n"
                              "       fhp_b200 validate FILE\n"
                              "       fhp_b200 geometry OUTPUT --width W --height H --cylinder");
}

RuleVariant parse_rules(const std::string& s) {
  if (s == "default") return RuleVariant::Default;
  if (s == "fhp1") return RuleVariant::FhpI;
  if (s == "fhp3") return RuleVariant::FhpIII;
  usage("unknown --rules " + s);
}

struct Args {
  std::vector<std::string> pos;
  SimConfig cfg;
  bool cylinder = false;
};

Args parse(int argc, char** argv) {
  Args a;
  a.cfg.backend = Backend::Cuda;
  for (int i = 2; i < argc; ++i) {
    const std::string k = argv[i];
    auto val = [&]() -> std::string {
      if (i + 1 >= argc) usage("missing value for " + k);
      return argv[++i];
    };
    if (k == "--width") a.cfg.width = std::stoi(val());
    else if (k == "--height") a.cfg.height = std::stoi(val());
    else if (k == "--steps") a.cfg.steps = std::stoi(val());
    else if (k == "--density") a.cfg.fill_density = std::stod(val());
    else if (k == "--force-p") a.cfg.force_p = std::stod(val());
    else if (k == "--seed") a.cfg.seed = std::stoull(val());
    else if (k == "--rules") a.cfg.rules = parse_rules(val());
    else if (k == "--table-file") a.cfg.table_file = val();
    else if (k == "--geometry-file") a.cfg.geometry_file = val();
    else if (k == "--dump-every") a.cfg.dump_every = std::stoi(val());
    else if (k == "--out-prefix") a.cfg.out_prefix = val();
    else if (k == "--repeats") a.cfg.repeats = std::stoi(val());
    else if (k == "--warmup") a.cfg.warmup_steps = std::stoi(val());
    else if (k == "--device") a.cfg.device = std::stoi(val());
    else if (k == "--clear-rest") a.cfg.clear_rest = true;
    else if (k == "--checkpoint-file") a.cfg.checkpoint_file = val();
    else if (k == "--checkpoint-every") a.cfg.checkpoint_every = std::stoi(val());
    else if (k == "--resume") a.cfg.resume_file = val();
    else if (k == "--cylinder") a.cylinder = true;
    else if (k == "--backend") {
      if (val() != "cuda") usage("fhp_b200 provides --backend cuda only");
    } else if (!k.empty() && k[0] == '-') usage("unknown option " + k);
    else a.pos.push_back(k);
  }
  return a;
}

void dump_outputs(const SimConfig& cfg, int step, const Engine& e) {
  if (cfg.out_prefix.empty()) return;
  const std::string tag = cfg.out_prefix + "_step" + std::to_string(step);
  const auto field = coarse_grain(e, 4);
  write_flow_csv_file(tag + "_flow.csv", field);
  write_profile_csv_file(tag + "_profile.csv", velocity_profile(e));
  write_density_pgm_file(tag + "_density.pgm", field);
}

int cmd_run(SimConfig cfg) {
  CollisionTable table;
  if (!cfg.resume_file.empty()) {
    // --resume: size, seed, force-p and table come from the checkpoint.
    const Checkpoint ck = read_checkpoint_file(cfg.resume_file);
    cfg.width = ck.width;
    cfg.height = ck.height;
    cfg.seed = ck.seed;
    cfg.force_p = ck.force_p;
    table = ck.table;
  } else {
    table = table_for(cfg);
  }
  const auto result = run(cfg, table, {},
                          [&cfg](int step, const Engine& e) { dump_outputs(cfg, step, e); });
  const auto& last = result.series.back();
  std::cout << "steps " << cfg.steps << "  mass " << last.mass << "  momentum ("
            << last.momentum.px << "," << last.momentum.py << ")  digest 0x" << std::hex
            << state_digest(result.lattice) << std::dec << "  forcing_swaps "
            << result.forcing_swaps << '\n';
  return 0;
}

int cmd_bench(const SimConfig& cfg) {
  const auto res = run_bench(cfg, cfg.repeats);
  for (const auto& r : res.repeats) std::cout << to_json_line(r) << '\n';
  std::cout << ascii_table({res.median});
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  try {
    if (argc < 2) usage("missing subcommand");
    const std::string cmd = argv[1];
    Args a = parse(argc, argv);
    if (cmd == "run") {
      a.cfg.validate();
      return cmd_run(a.cfg);
    }
    if (cmd == "bench") {
      a.cfg.validate();
      return cmd_bench(a.cfg);
    }
    if (cmd == "tablegen") {
      if (a.pos.size() != 1) usage("tablegen needs OUTPUT");
      write_table_file(a.pos[0], build_table(a.cfg.rules));
      return 0;
    }
    if (cmd == "validate") {
      if (a.pos.size() != 1) usage("validate needs FILE");
      const auto t = load_table(read_table_file(a.pos[0]), /*force=*/true);
      const auto rep = validate_table(t);
      std::cout << rep.summary() << '\n';
      return rep.valid() ? 0 : 1;
    }
    if (cmd == "geometry") {
      if (a.pos.size() != 1 || !a.cylinder) usage("geometry needs OUTPUT and --cylinder");
      write_geometry_file(a.pos[0], cylinder_geometry(a.cfg.width, a.cfg.height,
                                                      a.cfg.width / 4.0, a.cfg.height / 2.0,
                                                      a.cfg.height / 16.0));
      return 0;
    }
    usage("unknown subcommand " + cmd);
  } catch (const std::logic_error& e) {  // invalid_argument, out_of_range (bad numbers)
    std::cerr << "error: " << e.what() << '\n';
    return 2;
  } catch (const std::runtime_error& e) {
    std::cerr << "error: " << e.what() << '\n';
    return 3;
  }
}
