// yb_e2e — one BASELINE config end to end through the C++ drop-in
// (include/yeeb200/yeeblock.hpp) with the reference's own host storage: the
// state is a FieldSet<float> (Array3 = std::vector, array3.hpp:120 — plain
// pageable memory) and the per-cell coefficients are std::vector<float>.
// This is what a reference caller that switches to the shim gets, with no
// pinned buffers of its own.
//
//   yb_e2e --config c1..c5 [--steps N] [--kernel tb2|fused] [--reps R]
//          [--quiescent-skip on|off]
//
// Timed region (host steady_clock), per repetition, on a fresh Simulation:
//   set_cell_coefficients (h2d) -> run(steps) (uploads the dirty host
//   FieldSet first: h2d; configs 2 and 4 start from the zero FieldSet the
//   Simulation constructs, as the reference does, so nothing to upload) ->
//   const fields() (d2h of all six components into the FieldSet).
// The Simulation is constructed and its host FieldSet filled before the
// clock starts (the reference's RunStats also exclude construction,
// runner.hpp:245-263). Prints one JSON object with the best repetition and
// the phase split.
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <utility>
#include <vector>

#include "yeeb200/yeeblock.hpp"
#include "yeeb200_inputs.h"

using namespace yeeb200;

namespace {

struct Cfg {
  const char* name;
  int nx, ny, nz;
  long long eps_seed, sigma_seed, field_seed;  // < 0: none (vacuum / zero fields)
  bool source;
  long long steps;
};

// BASELINE.json configs (config 5 at one GPU: 1024 x 1024 x 256)
const Cfg kCfgs[] = {
    {"c1", 128, 128, 128, -1, -1, -1, true, 200},   {"c2", 256, 256, 256, 1, -1, -1, true, 500},
    {"c3", 512, 512, 512, 2, 2, 3, false, 100},     {"c4", 1024, 1024, 512, 4, -1, -1, true, 200},
    {"c5", 1024, 1024, 256, 5, 5, 6, false, 100},
};

double now() { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); }

}  // namespace

int main(int argc, char** argv) {
  std::string cname = "c4", kernel = "tb2";
  long long steps = -1;
  int reps = 2;
  bool qskip = false;
  for (int a = 1; a + 1 < argc; a += 2) {
    const std::string k = argv[a], v = argv[a + 1];
    if (k == "--config") cname = v;
    else if (k == "--steps") steps = std::atoll(v.c_str());
    else if (k == "--kernel") kernel = v;
    else if (k == "--reps") reps = std::atoi(v.c_str());
    else if (k == "--quiescent-skip") qskip = v == "on";
    else {
      std::fprintf(stderr, "usage: yb_e2e --config c1..c5 [--steps N] [--kernel tb2|fused] [--reps R] "
                           "[--quiescent-skip on|off]\n");
      return 2;
    }
  }
  const Cfg* cfg = nullptr;
  for (const Cfg& c : kCfgs)
    if (cname == c.name) cfg = &c;
  if (!cfg) {
    std::fprintf(stderr, "yb_e2e: unknown config %s\n", cname.c_str());
    return 2;
  }
  if (steps < 0) steps = cfg->steps;
  try {
    // unit grid, dt = (float)(0.99/sqrt(3)) (make_uniform_grid semantics, grid.hpp:63-74)
    GridSpec<float> grid;
    grid.nx = cfg->nx;
    grid.ny = cfg->ny;
    grid.nz = cfg->nz;
    grid.dx.assign(cfg->nx, 1.0f);
    grid.dy.assign(cfg->ny, 1.0f);
    grid.dz.assign(cfg->nz, 1.0f);
    grid.c = 1.0f;
    grid.dt = static_cast<float>(stable_dt(grid, 0.99));
    const TileLayout layout = make_layout(grid.dims(), Split{1, 16, 16});
    RunOptions<float> opts;
    opts.quiescent_skip = qskip;
    opts.kernel = kernel == "fused" ? YB_VARIANT_FUSED : YB_VARIANT_TB2;
    if (cfg->source) {  // the configs' Gaussian exp(-((n-40)/12)^2) at the centre Ez
      SourceSpec s;
      s.i = cfg->nx / 2;
      s.j = cfg->ny / 2;
      s.k = cfg->nz / 2;
      s.component = Comp::Ez;
      s.table.resize(static_cast<std::size_t>(steps));
      for (long long n = 0; n < steps; ++n) s.table[static_cast<std::size_t>(n)] = yb_gauss_pulse(n, 40.0, 12.0);
      opts.sources.push_back(s);
    }

    // host inputs (cell order (k*ny+j)*nx+i, include/yeeb200_inputs.h)
    const long long ncell = static_cast<long long>(cfg->nx) * cfg->ny * cfg->nz;
    const float S = grid.dt;
    std::vector<std::pair<CellCoeff, std::vector<float>>> cells;
    if (cfg->eps_seed >= 0) {
      const bool lossy = cfg->sigma_seed >= 0;
      std::vector<float> ca(lossy ? ncell : 0), cb(ncell), da(lossy ? ncell : 0), db(lossy ? ncell : 0);
#pragma omp parallel for schedule(static)
      for (long long q = 0; q < ncell; ++q) {
        const yb_cell_coeffs c = yb_cell_coeffs_at(cfg->eps_seed, cfg->sigma_seed, static_cast<uint64_t>(q), S);
        cb[q] = c.cb;
        if (lossy) {
          ca[q] = c.ca;
          da[q] = c.da;
          db[q] = c.db;
        }
      }
      if (lossy) cells.emplace_back(CellCoeff::Ca, std::move(ca));
      cells.emplace_back(CellCoeff::Cb, std::move(cb));
      if (lossy) {
        cells.emplace_back(CellCoeff::Da, std::move(da));
        cells.emplace_back(CellCoeff::Db, std::move(db));
      }
    }
    // configs 2, 4 (medium, zero fields): the reference's Simulation flow — run from the zero
    // FieldSet the Simulation constructs; the others hand their initial state over (config 1:
    // vacuum, so the state is its only input; configs 3, 5: seeded fields)
    const bool upload = cfg->field_seed >= 0 || cfg->eps_seed < 0;
    FieldSet<float> init;
    if (upload) init.allocate(grid.dims());
    if (cfg->field_seed >= 0)
      for (Comp c : kAllComps) {
        Array3<float>& A = init.field(c);
        float* p = A.data();
        const long long n = static_cast<long long>(A.size());
        const int ci = comp_index(c);
#pragma omp parallel for schedule(static)
        for (long long q = 0; q < n; ++q) p[q] = yb_field_value(static_cast<uint64_t>(cfg->field_seed), ci,
                                                                static_cast<uint64_t>(q));
      }
    long long field_bytes = 0;
    for (Comp c : kAllComps) {
      const IndexBox b = comp_extents(grid.dims(), c);
      field_bytes += 4LL * (b.x.hi - b.x.lo) * (b.y.hi - b.y.lo) * (b.z.hi - b.z.lo);
    }
    const long long coef_bytes = static_cast<long long>(cells.size()) * ncell * 4;

    double best = 1e300, b_coef = 0, b_run = 0, b_down = 0;
    std::string digest;
    for (int r = 0; r < reps; ++r) {
      Simulation<float> sim(grid, layout, Variant::Standard, opts);
      if (upload) sim.fields() = init;  // marked dirty: run() uploads it
      const double t0 = now();
      for (auto& c : cells) sim.set_cell_coefficients(c.first, c.second);
      const double t1 = now();
      sim.run(steps);
      const double t2 = now();
      const FieldSet<float>& out = std::as_const(sim).fields();
      const double t3 = now();
      if (t3 - t0 < best) {
        best = t3 - t0;
        b_coef = t1 - t0;
        b_run = t2 - t1;
        b_down = t3 - t2;
      }
      if (r == reps - 1) digest = field_digest_hex(out);
    }
    const double v = static_cast<double>(ncell) * steps / best / 1e9;
    std::printf(
        "{\"config\": \"%s\", \"grid\": [%d, %d, %d], \"steps\": %lld, \"kernel\": \"%s\", \"quiescent_skip\": %s, "
        "\"value\": %.4f, \"unit\": \"Gcell/s\", \"wall_s\": %.6f, \"h2d_bytes_per_step\": %.1f, "
        "\"d2h_bytes_per_step\": %.1f, \"phases_s\": {\"set_cell_coefficients\": %.6f, "
        "\"run_incl_field_upload\": %.6f, \"fields_readback\": %.6f}, \"reps\": %d, \"digest\": \"%s\", "
        "\"host_memory\": \"pageable (std::vector: FieldSet<float> + coefficient vectors)\"}\n",
        cfg->name, cfg->nx, cfg->ny, cfg->nz, steps, kernel.c_str(), qskip ? "true" : "false", v, best,
        static_cast<double>((upload ? field_bytes : 0) + coef_bytes) / steps, static_cast<double>(field_bytes) / steps, b_coef,
        b_run, b_down, reps, digest.c_str());
  } catch (const std::exception& e) {
    std::fprintf(stderr, "yb_e2e: %s\n", e.what());
    return 1;
  }
  return 0;
}
