// yb_bench — the bench-cli of the reference (SPEC.md bench-cli, flags
// SPEC.md:528; harness bench.hpp:41-391) on the B200 path: a cube PEC cavity
// with the reference's default point source and six probes, run through the
// drop-in shim (include/yeeb200/yeeblock.hpp) and libyeeb200.
//
//   yb_bench --case cube --size N --steps S --variant fused,tb2,naive
//            --mode measure|verify|energy|predict [--out PATH] [--format csv|md]
//            [--split auto] [--threads LIST] [--precision single]
//            [--source-steps K] [--sigma-dt X] [--amplitude A] [--probe-stride P]
//            [--quiescent-skip on|off] [--machine FILE] [--hbm-gbs G] [--probes PATH]
//
// measure: one BenchRecord per variant (bench.hpp:134-175): MC/s =
//   N^3 * steps / total_s / 1e6; total_s = host wall time of Simulation::run;
//   vol_s = device time of the sweep kernels (the "volume passes").
// verify:  every variant from the same initial state; final-field checksum
//   and probe text compared with the first variant (bench.hpp:186-246);
//   exit status 1 iff any FAIL.
// energy:  max relative drift of the leapfrog invariant after the source
//   switches off (measure_energy_drift, bench.hpp:273-303), on the device.
// predict: HBM-bandwidth bounds per variant from the algorithmic bytes per
//   cell-update (the B200 analogue of predict_table, bench.hpp:366-391).
// The GPU tiles itself: --split and --threads are accepted and recorded,
// not used; only single precision exists (--precision double is an error).
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <iostream>
#include <sstream>
#include <string>
#include <vector>

#include "yeeb200/yeeblock.hpp"

using namespace yeeb200;

namespace {

constexpr double kVacuumLightSpeed = 299792458.0;  // grid.hpp:12

struct Config {
  std::string case_name = "cube";
  int size = 128;
  long long steps = 300;
  std::string split = "auto";
  std::vector<std::string> variants = {"fused", "tb2", "naive"};
  std::string threads = "1";
  std::string precision = "single";
  std::string mode = "measure";
  std::string out, format, probes_out;
  double safety = 0.99, amplitude = 1.0, sigma_dt = 8.0;
  long long source_steps = 50;
  int probe_stride = 20;
  bool quiescent_skip = true;
  double hbm_gbs = 6550.7;  // MEASURED_PEAKS.json hbm_gbs on this pool's B200s
};

int variant_id(const std::string& v) {
  if (v == "fused" || v == "standard") return YB_VARIANT_FUSED;
  if (v == "tb2" || v == "twostep") return YB_VARIANT_TB2;
  if (v == "naive") return YB_VARIANT_NAIVE;
  throw std::invalid_argument("unknown variant " + v + " (fused, tb2, naive)");
}

std::vector<std::string> split_list(const std::string& s) {
  std::vector<std::string> out;
  std::stringstream ss(s);
  std::string item;
  while (std::getline(ss, item, ','))
    if (!item.empty()) out.push_back(item);
  return out;
}

// default_probes / default_source (bench.hpp:68-86)
std::vector<ProbeSpec> default_probes(int n, int stride) {
  auto at = [&](double fx, double fy, double fz) {
    ProbeSpec p;
    p.i = static_cast<int>(fx * n);
    p.j = static_cast<int>(fy * n);
    p.k = static_cast<int>(fz * n);
    p.component = Comp::Ez;
    p.stride = stride;
    return p;
  };
  return {at(0.50, 0.50, 0.50), at(0.25, 0.25, 0.25), at(0.75, 0.75, 0.75),
          at(0.25, 0.75, 0.50), at(0.75, 0.25, 0.50), at(0.50, 0.25, 0.75)};
}

SourceSpec default_source(int n, double dt, const Config& cfg) {
  SourceSpec s;
  s.i = s.j = s.k = n / 2;
  s.component = Comp::Ez;
  s.waveform = Waveform::pulse(cfg.amplitude, cfg.sigma_dt * dt);
  s.active_steps = cfg.source_steps;
  return s;
}

struct CaseResult {
  std::string checksum, probe_text;
  RunStats stats;
  double vol_s = 0.0;
  int ctas = 0;
};

// run_case (bench.hpp:105-127) on one variant
CaseResult run_case(const Config& cfg, int variant) {
  const GridSpec<float> grid = make_uniform_grid<float>(cfg.size, 1.0f, static_cast<float>(kVacuumLightSpeed), cfg.safety);
  RunOptions<float> opts;
  opts.sources = {default_source(cfg.size, static_cast<double>(grid.dt), cfg)};
  opts.probes = default_probes(cfg.size, cfg.probe_stride);
  opts.quiescent_skip = cfg.quiescent_skip;
  opts.kernel = variant;
  Simulation<float> sim(grid, opts);
  yb_set_kernel_timing(sim.handle(), 1);
  const auto records = sim.run(cfg.steps);
  CaseResult r;
  r.checksum = field_digest_hex(sim.fields());
  r.probe_text = format_probe_records(records, 9);  // max_digits10 of float
  r.stats = sim.stats();
  yb_info inf{};
  if (yb_get_info(sim.handle(), &inf) == YB_OK) {
    r.vol_s = inf.main_kernel_ms * 1e-3;
    r.ctas = inf.grid_x;
  }
  return r;
}

struct Record {
  std::string case_name, split, precision, variant, checksum;
  int cores = 0;
  double mcs = 0, total_s = 0, vol_s = 0, vol_pct = 0;
};

std::string emit_csv(const std::vector<Record>& rs) {  // bench.hpp:319-333
  std::string out = "case,split,cores,precision,variant,mcs,total_s,vol_s,vol_pct,checksum\n";
  char buf[256];
  for (const Record& r : rs) {
    std::snprintf(buf, sizeof(buf), "%s,%s,%d,%s,%s,%.2f,%.6f,%.6f,%.1f,%s\n", r.case_name.c_str(),
                  r.split.c_str(), r.cores, r.precision.c_str(), r.variant.c_str(), r.mcs, r.total_s, r.vol_s,
                  r.vol_pct, r.checksum.c_str());
    out += buf;
  }
  return out;
}

std::string emit_markdown(const std::vector<Record>& rs) {  // bench.hpp:335-351
  std::string out =
      "| case | split | cores | precision | variant | MC/s | total (s) | vol (s) | V/T % | checksum |\n"
      "|------|-------|-------|-----------|---------|------|-----------|---------|-------|----------|\n";
  char buf[256];
  for (const Record& r : rs) {
    std::snprintf(buf, sizeof(buf), "| %s | %s | %d | %s | %s | %.2f | %.3f | %.3f | %.1f | %s |\n",
                  r.case_name.c_str(), r.split.c_str(), r.cores, r.precision.c_str(), r.variant.c_str(), r.mcs,
                  r.total_s, r.vol_s, r.vol_pct, r.checksum.c_str());
    out += buf;
  }
  return out;
}

void emit(const Config& cfg, const std::string& text) {
  if (cfg.out.empty()) {
    std::cout << text;
    return;
  }
  std::ofstream f(cfg.out, std::ios::binary);
  if (!f) throw std::runtime_error("emit_tables: cannot write " + cfg.out);
  f << text;
}

int mode_measure(const Config& cfg) {
  std::vector<Record> rs;
  const double cells = static_cast<double>(cfg.size) * cfg.size * cfg.size;
  for (const std::string& v : cfg.variants) {
    const CaseResult c = run_case(cfg, variant_id(v));
    Record r;
    r.case_name = cfg.case_name;
    r.split = cfg.split == "auto" ? "gpu-128x8" : cfg.split;
    r.cores = c.ctas;
    r.precision = "single";
    r.variant = v;
    r.total_s = c.stats.total_seconds;
    r.vol_s = c.vol_s;
    r.vol_pct = r.total_s > 0 ? 100.0 * r.vol_s / r.total_s : 0.0;
    r.mcs = r.total_s > 0 ? cells * cfg.steps / r.total_s / 1e6 : 0.0;
    r.checksum = c.checksum;
    rs.push_back(r);
  }
  const std::string fmt = !cfg.format.empty() ? cfg.format
                          : (cfg.out.size() > 3 && cfg.out.substr(cfg.out.size() - 3) == ".md") ? "md"
                                                                                                  : "csv";
  if (fmt == "csv")
    emit(cfg, emit_csv(rs));
  else if (fmt == "md" || fmt == "markdown")
    emit(cfg, emit_markdown(rs));
  else
    throw std::invalid_argument("emit_tables: unknown format " + fmt);
  return 0;
}

int mode_verify(const Config& cfg) {  // verify_equivalence (bench.hpp:222-246)
  if (cfg.variants.size() < 2) throw std::invalid_argument("verify_equivalence: need >= 2 variants");
  if (cfg.size < 8) throw std::invalid_argument("verify: N >= 8 required");
  bool all = true;
  std::string text;
  CaseResult ref;
  std::string ref_label;
  for (size_t q = 0; q < cfg.variants.size(); ++q) {
    const CaseResult r = run_case(cfg, variant_id(cfg.variants[q]));
    const std::string label = cfg.variants[q] + "/gpu/single";
    if (q == 0) {
      ref = r;
      ref_label = label;
      continue;
    }
    const bool fe = r.checksum == ref.checksum, pe = r.probe_text == ref.probe_text;
    all = all && fe && pe;
    text += (fe && pe) ? "PASS" : "FAIL";
    text += "  " + ref_label + " vs " + label;
    if (!fe) text += "  [fields differ]";
    if (!pe) text += "  [probes differ]";
    text += "\n";
  }
  text += all ? "verify: PASS\n" : "verify: FAIL\n";
  text += "checksum " + ref.checksum + "\n";
  if (!cfg.probes_out.empty()) {
    std::ofstream f(cfg.probes_out, std::ios::binary);
    if (!f) throw std::runtime_error("cannot write " + cfg.probes_out);
    f << ref.probe_text;
  }
  emit(cfg, text);
  return all ? 0 : 1;
}

int mode_energy(const Config& cfg) {  // measure_energy_drift (bench.hpp:273-303)
  if (cfg.source_steps >= cfg.steps) throw std::invalid_argument("energy_report: source never switches off");
  const GridSpec<float> grid = make_uniform_grid<float>(cfg.size, 1.0f, static_cast<float>(kVacuumLightSpeed), cfg.safety);
  RunOptions<float> opts;
  opts.sources = {default_source(cfg.size, static_cast<double>(grid.dt), cfg)};
  opts.kernel = variant_id(cfg.variants.front());
  Simulation<float> sim(grid, opts);
  double reference = 0.0, max_drift = 0.0;
  bool have = false;
  for (long long s = 0; s < cfg.steps; ++s) {
    sim.snapshot_h();
    sim.run(1);
    if (s + 1 <= cfg.source_steps) continue;
    const double e = sim.total_energy();
    if (!have) {
      reference = e;
      have = true;
      continue;
    }
    max_drift = std::max(max_drift, reference != 0.0 ? std::abs(e - reference) / std::abs(reference) : std::abs(e));
  }
  char buf[128];
  std::snprintf(buf, sizeof(buf), "single: max relative energy drift %.3e\n", max_drift);
  emit(cfg, buf);
  return 0;
}

int mode_predict(const Config& cfg) {
  // algorithmic HBM bytes per cell-update of the vacuum cube (no per-cell
  // coefficient arrays): fused 6 fields read + 6 written; tb2 the same per
  // two steps; naive: the E pass reads 6 and writes 3, PEC re-touches the
  // faces (ignored), the H pass reads 6 and writes 3.
  std::string out;
  char buf[256];
  std::snprintf(buf, sizeof(buf), "machine: B200, HBM %.1f GB/s (measured copy peak), fp32\n", cfg.hbm_gbs);
  out += buf;
  out += "variant      bytes/cell  bw-bound Gcell/s  bw-bound MC/s\n";
  const double cells = static_cast<double>(cfg.size) * cfg.size * cfg.size;
  for (const std::string& v : cfg.variants) {
    const int id = variant_id(v);
    const double bytes = id == YB_VARIANT_TB2 ? 24.0 : (id == YB_VARIANT_NAIVE ? 72.0 : 48.0);
    const double g = cfg.hbm_gbs / bytes;
    std::snprintf(buf, sizeof(buf), "%-12s %10.1f  %16.1f  %13.0f\n", v.c_str(), bytes, g, g * 1e3);
    out += buf;
  }
  std::snprintf(buf, sizeof(buf), "working set: %.1f MB state (two buffers: %.1f MB) vs 126 MB L2\n",
                cells * 24.0 / 1e6, cells * 48.0 / 1e6);
  out += buf;
  emit(cfg, out);
  return 0;
}

double machine_hbm(const std::string& path, double fallback) {
  std::ifstream f(path);
  if (!f) throw std::invalid_argument("--machine: cannot read " + path);
  std::stringstream ss;
  ss << f.rdbuf();
  const std::string s = ss.str();
  const size_t k = s.find("\"hbm_gbs\"");
  if (k == std::string::npos) return fallback;
  const size_t c = s.find(':', k);
  return c == std::string::npos ? fallback : std::strtod(s.c_str() + c + 1, nullptr);
}

void usage() {
  std::fprintf(stderr,
               "usage: yb_bench [--case cube] [--size N] [--steps S] [--split auto|SXxSYxSZ] "
               "[--variant LIST] [--threads LIST] [--precision single] [--machine FILE] "
               "[--mode measure|verify|energy|predict] [--out PATH] [--format csv|md] "
               "[--source-steps K] [--sigma-dt X] [--amplitude A] [--probe-stride P] "
               "[--quiescent-skip on|off] [--hbm-gbs G] [--probes PATH (verify: probe text)]\n");
}

}  // namespace

int main(int argc, char** argv) {
  Config cfg;
  try {
    for (int a = 1; a < argc; ++a) {
      const std::string k = argv[a];
      if (k == "-h" || k == "--help") {
        usage();
        return 0;
      }
      if (a + 1 >= argc) throw std::invalid_argument("missing value for " + k);
      const std::string v = argv[++a];
      if (k == "--case") {
        if (v != "cube") throw std::invalid_argument("only --case cube exists (SPEC.md bench-cli non-goals)");
        cfg.case_name = v;
      } else if (k == "--size") {
        cfg.size = std::stoi(v);
      } else if (k == "--steps") {
        cfg.steps = std::stoll(v);
      } else if (k == "--split") {
        cfg.split = v;
      } else if (k == "--variant") {
        cfg.variants = split_list(v);
      } else if (k == "--threads") {
        cfg.threads = v;
      } else if (k == "--precision") {
        if (v != "single") throw std::invalid_argument("the B200 path is fp32: --precision single only");
        cfg.precision = v;
      } else if (k == "--machine") {
        cfg.hbm_gbs = machine_hbm(v, cfg.hbm_gbs);
      } else if (k == "--hbm-gbs") {
        cfg.hbm_gbs = std::stod(v);
      } else if (k == "--mode") {
        cfg.mode = v;
      } else if (k == "--out") {
        cfg.out = v;
      } else if (k == "--probes") {
        cfg.probes_out = v;
      } else if (k == "--format") {
        cfg.format = v;
      } else if (k == "--source-steps") {
        cfg.source_steps = std::stoll(v);
      } else if (k == "--sigma-dt") {
        cfg.sigma_dt = std::stod(v);
      } else if (k == "--amplitude") {
        cfg.amplitude = std::stod(v);
      } else if (k == "--probe-stride") {
        cfg.probe_stride = std::stoi(v);
      } else if (k == "--quiescent-skip") {
        cfg.quiescent_skip = v == "on" || v == "1" || v == "true";
      } else {
        throw std::invalid_argument("unknown flag " + k);
      }
    }
    if (cfg.steps < 1) throw std::invalid_argument("BenchConfig: steps < 1");
    if (cfg.size < 8) throw std::invalid_argument("BenchConfig: size < 8");
    if (cfg.variants.empty()) throw std::invalid_argument("no variants");
    for (const std::string& v : cfg.variants) variant_id(v);
    if (cfg.mode == "measure") return mode_measure(cfg);
    if (cfg.mode == "verify") return mode_verify(cfg);
    if (cfg.mode == "energy") return mode_energy(cfg);
    if (cfg.mode == "predict") return mode_predict(cfg);
    throw std::invalid_argument("unknown mode " + cfg.mode);
  } catch (const std::exception& e) {
    std::fprintf(stderr, "yb_bench: %s\n", e.what());
    usage();
    return 2;
  }
}
