// ref_driver.cpp — builds the UNMODIFIED reference (header-only yeeblock,
// /root/reference/proj/include) into oracle/_ref/libyeeref.so so the C oracle
// can be pinned against it and bench.py can time it as the CPU baseline.
// Test infrastructure only (see oracle/yee_oracle.h). Nothing here restates
// the algorithm: every call goes into the reference's own functions.
//
// Entry points:
//   yr_run_kernels  - the Standard step order (schedule.hpp:171-210) driven
//                     directly through apply_ampere_range / apply_pec_boundary
//                     / apply_faraday_range (kernels.hpp:129-155), with an
//                     optional config-style additive source table injected
//                     after PEC and before Faraday (the injection point of
//                     plan_standard, schedule.hpp:184-199).
//   yr_simulation   - yeeblock::Simulation<float>::run (runner.hpp:205-266)
//                     for any Variant/split/worker count with a reference
//                     SourceSpec (source.hpp:15-68).
//   yr_total_energy - total_energy against an HSnapshot (fields.hpp:68-146).
//   yr_run_case     - the reference bench harness's run_case (bench.hpp:105-127):
//                     cube cavity, default source and probes -> checksum + probe text.
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>

#include "yeeblock/yeeblock.hpp"

using namespace yeeblock;

namespace {

thread_local std::string g_err;

GridSpec<float> make_grid(int nx, int ny, int nz, const float* dx, const float* dy,
                          const float* dz, float dt, float c) {
  GridSpec<float> g;
  g.nx = nx;
  g.ny = ny;
  g.nz = nz;
  g.dx.assign(dx, dx + nx);
  g.dy.assign(dy, dy + ny);
  g.dz.assign(dz, dz + nz);
  g.dt = dt;
  g.c = c;
  return g;
}

void load(FieldSet<float>& f, float* const* fields) {
  for (Comp c : kAllComps) {
    Array3<float>& a = f.field(c);
    std::memcpy(a.data(), fields[comp_index(c)], a.size_bytes());
  }
}

void store(const FieldSet<float>& f, float* const* fields) {
  for (Comp c : kAllComps) {
    const Array3<float>& a = f.field(c);
    std::memcpy(fields[comp_index(c)], a.data(), a.size_bytes());
  }
}

}  // namespace

extern "C" {

const char* yr_last_error() { return g_err.c_str(); }

float yr_uniform_dt(int n, float h, float c, double safety) {
  return make_uniform_grid<float>(n, h, c, safety).dt;
}

double yr_stable_dt(int nx, int ny, int nz, const float* dx, const float* dy,
                    const float* dz, float c, double safety) {
  try {
    return stable_dt(make_grid(nx, ny, nz, dx, dy, dz, 0.0f, c), safety);
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1.0;
  }
}

int yr_build_coefficients(int nx, int ny, int nz, const float* dx, const float* dy,
                          const float* dz, float dt, float c, float* cdx, float* cdy,
                          float* cdz) {
  try {
    Coefficients<float> co = build_coefficients(make_grid(nx, ny, nz, dx, dy, dz, dt, c));
    std::memcpy(cdx, co.cdx.data(), sizeof(float) * nx);
    std::memcpy(cdy, co.cdy.data(), sizeof(float) * ny);
    std::memcpy(cdz, co.cdz.data(), sizeof(float) * nz);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

// Standard step order through the reference range kernels. fields[6] are
// dense Array3 buffers (in/out). src_table may be null (no source).
int yr_run_kernels(int nx, int ny, int nz, const float* dx, const float* dy,
                   const float* dz, float dt, float c, float* const* fields,
                   std::int64_t step0, std::int64_t nsteps, int src_comp, int si,
                   int sj, int sk, const float* src_table, std::int64_t src_n,
                   int phases) {
  try {
    GridSpec<float> g = make_grid(nx, ny, nz, dx, dy, dz, dt, c);
    Coefficients<float> co = build_coefficients(g);
    FieldSet<float> f(g.dims());
    load(f, fields);
    const IndexBox all = detail::node_box(g.dims());
    for (std::int64_t t = 0; t < nsteps; ++t) {
      const std::int64_t step = step0 + t;
      if (phases & 1) apply_ampere_range(f, co, all);
      if (phases & 2) apply_pec_boundary(f);
      if (src_table && step >= 0 && step < src_n)
        f.field(static_cast<Comp>(src_comp))(si, sj, sk) += src_table[step];
      if (phases & 4) apply_faraday_range(f, co, all);
    }
    store(f, fields);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

// Simulation<float> on a uniform cube-spaced grid (unit h, wave speed c,
// dt = stable_dt * safety, make_uniform_grid semantics but nx/ny/nz free).
// has_src: one SourceSpec with a differentiated Gaussian (amp, sigma, t0).
int yr_simulation(int nx, int ny, int nz, float h, float c, double safety, int variant,
                  int sx, int sy, int sz, int workers, int quiescent_skip, int has_src,
                  int src_comp, int si, int sj, int sk, double amp, double sigma,
                  double t0, std::int64_t active_steps, float* const* fields,
                  std::int64_t step0, std::int64_t nsteps, double* seconds,
                  std::uint64_t* digest) {
  try {
    GridSpec<float> g;
    g.nx = nx;
    g.ny = ny;
    g.nz = nz;
    g.dx.assign(nx, h);
    g.dy.assign(ny, h);
    g.dz.assign(nz, h);
    g.c = c;
    g.dt = static_cast<float>(stable_dt(g, safety));
    TileLayout layout = make_layout(g.dims(), Split{sx, sy, sz});
    RunOptions<float> opts;
    if (has_src) {
      SourceSpec s;
      s.i = si;
      s.j = sj;
      s.k = sk;
      s.component = static_cast<Comp>(src_comp);
      s.waveform = Waveform{amp, sigma, t0};
      s.active_steps = active_steps;
      opts.sources.push_back(s);
    }
    opts.quiescent_skip = quiescent_skip != 0;
    opts.exec.workers = workers;
    Simulation<float> sim(g, layout, static_cast<Variant>(variant), std::move(opts));
    load(sim.fields(), fields);
    sim.fields().step_index = step0;
    sim.run(nsteps);
    if (seconds) *seconds = sim.stats().total_seconds;
    if (digest) *digest = field_digest(sim.fields());
    store(sim.fields(), fields);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

// The increment inject_current adds at `step` (source.hpp:61-68):
// (Real)(-dt * J(step*dt)) with J the reference Waveform. Returns the number
// of leading steps at which the source is active (active_at, source.hpp:38-40).
std::int64_t yr_source_table(int nx, int ny, int nz, int comp, int si, int sj, int sk,
                             double amp, double sigma, double t0,
                             std::int64_t active_steps, double dt, std::int64_t n,
                             float* out) {
  try {
    SourceSpec s;
    s.i = si;
    s.j = sj;
    s.k = sk;
    s.component = static_cast<Comp>(comp);
    s.waveform = Waveform{amp, sigma, t0};
    s.active_steps = active_steps;
    s.validate(GridDims{nx, ny, nz});
    std::int64_t t = 0;
    for (; t < n && s.active_at(t); ++t)
      out[t] = static_cast<float>(-dt * s.waveform.value(static_cast<double>(t) * dt));
    return t;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

std::uint64_t yr_digest(int nx, int ny, int nz, float* const* fields) {
  FieldSet<float> f(GridDims{nx, ny, nz});
  load(f, fields);
  return field_digest(f);
}

// total_energy (fields.hpp:116-146) of `fields` against an HSnapshot holding
// prev_h[0..2] (hx, hy, hz).
double yr_total_energy(int nx, int ny, int nz, const float* dx, const float* dy, const float* dz,
                       float* const* fields, float* const* prev_h) {
  const GridSpec<float> g = make_grid(nx, ny, nz, dx, dy, dz, 0.0f, 1.0f);
  FieldSet<float> f(GridDims{nx, ny, nz}), p(GridDims{nx, ny, nz});
  load(f, fields);
  for (Comp c : kHComps) {
    Array3<float>& a = p.field(c);
    std::memcpy(a.data(), prev_h[comp_index(c) - 3], a.size_bytes());
  }
  return total_energy(g, f, HSnapshot<float>(p));
}

// run_case<float>(cfg, Standard, split 1x1x1, 1 thread) of the reference
// bench harness (bench.hpp:105-127). checksum: 17-byte buffer (16 hex + NUL);
// probes: the format_probe_records text (probe.hpp:56-66), NUL-terminated;
// returns its length, or -1 on error / -2 if `cap` is too small.
std::int64_t yr_run_case(int size, std::int64_t steps, std::int64_t source_steps, double sigma_dt,
                         double amplitude, int probe_stride, int quiescent_skip, char* checksum,
                         char* probes, std::int64_t cap) {
  try {
    BenchConfig cfg;
    cfg.size = size;
    cfg.steps = steps;
    cfg.source_steps = source_steps;
    cfg.source_sigma_dt = sigma_dt;
    cfg.source_amplitude = amplitude;
    cfg.probe_stride = probe_stride;
    cfg.quiescent_skip = quiescent_skip != 0;
    const CaseResult r = run_case<float>(cfg, Variant::Standard, Split{1, 1, 1}, 1);
    std::snprintf(checksum, 17, "%s", r.checksum.c_str());
    if ((std::int64_t)r.probe_text.size() + 1 > cap) return -2;
    std::memcpy(probes, r.probe_text.c_str(), r.probe_text.size() + 1);
    return (std::int64_t)r.probe_text.size();
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

}  // extern "C"
