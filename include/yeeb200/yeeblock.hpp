// yeeb200/yeeblock.hpp — C++ drop-in shim over libyeeb200.so (include/yeeb200.h).
//
// Re-exposes the reference yeeblock API for the Standard leapfrog path
// (/root/reference/proj/include/yeeblock, header-only CPU library) with the
// same names, argument meanings and exception types, backed by the B200
// kernels: grid setup (grid.hpp), coefficient and field arrays (grid.hpp,
// fields.hpp, array3.hpp), step/advance (runner.hpp) and field readout
// (fields.hpp, probe.hpp). Single precision only (the GPU path is fp32).
//
// Namespace yeeb200; define YEEB200_AS_YEEBLOCK before including to also get
// `namespace yeeblock = yeeb200;` so unmodified caller code compiles.
//
// Not mirrored (out of the hot-path scope): the CPU tilers and
// schedulers (tiling.hpp, schedule.hpp, parallel.hpp), the perf model and
// bench harness (perf_model.hpp, bench.hpp). The GPU has its own tiling;
// Simulation accepts and ignores the reference's variant/layout arguments.
#pragma once

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <functional>
#include <limits>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <vector>

#include "../yeeb200.h"

namespace yeeb200 {

// ---------------------------------------------------------------- errors
namespace detail {
inline void check(int rc) {
  if (rc == YB_OK) return;
  const std::string msg = yb_last_error();
  if (rc == YB_INVALID_ARGUMENT) throw std::invalid_argument(msg);
  if (rc == YB_OUT_OF_RANGE) throw std::out_of_range(msg);
  throw std::runtime_error(msg);
}
}  // namespace detail

// ------------------------------------------------ index boxes (array3.hpp)
struct Interval {
  int lo = 0, hi = 0;
  constexpr int length() const { return hi > lo ? hi - lo : 0; }
  constexpr bool empty() const { return hi <= lo; }
  constexpr bool contains(int v) const { return v >= lo && v < hi; }
};

struct IndexBox {
  Interval x, y, z;
  constexpr bool empty() const { return x.empty() || y.empty() || z.empty(); }
  constexpr long long volume() const {
    return empty() ? 0 : static_cast<long long>(x.length()) * y.length() * z.length();
  }
  constexpr bool contains(int i, int j, int k) const {
    return x.contains(i) && y.contains(j) && z.contains(k);
  }
  Interval& axis(int a) { return a == 0 ? x : (a == 1 ? y : z); }
  const Interval& axis(int a) const { return a == 0 ? x : (a == 1 ? y : z); }
};

/// Dense 3D array, x fastest, index (k*ny + j)*nx + i (array3.hpp:84-121).
template <class T>
class Array3 {
 public:
  Array3() = default;
  Array3(int nx, int ny, int nz)
      : nx_(nx), ny_(ny), nz_(nz), data_(static_cast<std::size_t>(nx) * ny * nz, T(0)) {}
  int nx() const { return nx_; }
  int ny() const { return ny_; }
  int nz() const { return nz_; }
  IndexBox full_box() const { return {{0, nx_}, {0, ny_}, {0, nz_}}; }
  std::size_t size() const { return data_.size(); }
  std::size_t size_bytes() const { return data_.size() * sizeof(T); }
  T* data() { return data_.data(); }
  const T* data() const { return data_.data(); }
  std::size_t index(int i, int j, int k) const {
    return (static_cast<std::size_t>(k) * ny_ + j) * nx_ + i;
  }
  T& operator()(int i, int j, int k) { return data_[index(i, j, k)]; }
  const T& operator()(int i, int j, int k) const { return data_[index(i, j, k)]; }
  void fill(T v) { data_.assign(data_.size(), v); }
  bool same_extents(const Array3& o) const { return nx_ == o.nx_ && ny_ == o.ny_ && nz_ == o.nz_; }

 private:
  int nx_ = 0, ny_ = 0, nz_ = 0;
  std::vector<T> data_;
};

// ------------------------------------------------ staggering (staggering.hpp)
enum class Comp : std::uint8_t { Ex = 0, Ey, Ez, Hx, Hy, Hz };
constexpr Comp kEComps[3] = {Comp::Ex, Comp::Ey, Comp::Ez};
constexpr Comp kHComps[3] = {Comp::Hx, Comp::Hy, Comp::Hz};
constexpr Comp kAllComps[6] = {Comp::Ex, Comp::Ey, Comp::Ez, Comp::Hx, Comp::Hy, Comp::Hz};
constexpr bool is_electric(Comp c) { return c <= Comp::Ez; }
constexpr int comp_index(Comp c) { return static_cast<int>(c); }
constexpr int comp_axis(Comp c) { return comp_index(c) % 3; }
constexpr bool is_node_axis(Comp c, int axis) {
  return is_electric(c) ? (axis != comp_axis(c)) : (axis == comp_axis(c));
}

struct GridDims {
  int nx = 0, ny = 0, nz = 0;
  int cells(int axis) const { return axis == 0 ? nx : (axis == 1 ? ny : nz); }
  long long cell_count() const { return static_cast<long long>(nx) * ny * nz; }
  bool operator==(const GridDims& o) const { return nx == o.nx && ny == o.ny && nz == o.nz; }
  bool operator!=(const GridDims& o) const { return !(*this == o); }
};

inline IndexBox comp_extents(const GridDims& g, Comp c) {
  IndexBox b;
  for (int a = 0; a < 3; ++a) b.axis(a) = {0, g.cells(a) + (is_node_axis(c, a) ? 1 : 0)};
  return b;
}

inline IndexBox curl_updatable_box(const GridDims& g, Comp c) {
  IndexBox b = comp_extents(g, c);
  if (is_electric(c))
    for (int a = 0; a < 3; ++a)
      if (is_node_axis(c, a)) b.axis(a) = {1, g.cells(a)};
  return b;
}

// ------------------------------------------------ grid (grid.hpp)
inline constexpr double kVacuumLightSpeed = 299792458.0;

template <class Real>
struct GridSpec {
  static_assert(std::is_same<Real, float>::value, "the B200 path is single precision");
  int nx = 0, ny = 0, nz = 0;
  std::vector<Real> dx, dy, dz;
  Real dt = Real(0);
  Real c = Real(kVacuumLightSpeed);
  GridDims dims() const { return {nx, ny, nz}; }
  const std::vector<Real>& spacing(int axis) const { return axis == 0 ? dx : (axis == 1 ? dy : dz); }
  void validate() const {
    if (nx < 1 || ny < 1 || nz < 1)
      throw std::invalid_argument("GridSpec: cell counts must be positive");
    if (static_cast<int>(dx.size()) != nx || static_cast<int>(dy.size()) != ny ||
        static_cast<int>(dz.size()) != nz)
      throw std::invalid_argument("GridSpec: spacing array length mismatch");
    for (int a = 0; a < 3; ++a)
      for (Real h : spacing(a))
        if (!(h > Real(0))) throw std::invalid_argument("GridSpec: spacings must be positive");
    if (!(c > Real(0))) throw std::invalid_argument("GridSpec: wave speed must be positive");
  }
};

/// safety / (c * sqrt(sum 1/min(d)^2)), in double (grid.hpp:48-60).
template <class Real>
double stable_dt(const GridSpec<Real>& g, double safety) {
  g.validate();
  if (!(safety > 0.0) || safety > 1.0) throw std::invalid_argument("stable_dt: safety must be in (0, 1]");
  double inv_sq = 0.0;
  for (int a = 0; a < 3; ++a) {
    double hmin = static_cast<double>(g.spacing(a)[0]);
    for (Real h : g.spacing(a)) hmin = std::min(hmin, static_cast<double>(h));
    inv_sq += 1.0 / (hmin * hmin);
  }
  return safety / (static_cast<double>(g.c) * std::sqrt(inv_sq));
}

template <class Real>
GridSpec<Real> make_uniform_grid(int n, Real h, Real c, double safety = 0.99) {
  GridSpec<Real> g;
  g.nx = g.ny = g.nz = n;
  g.dx.assign(n, h);
  g.dy.assign(n, h);
  g.dz.assign(n, h);
  g.c = c;
  g.dt = static_cast<Real>(stable_dt(g, safety));
  return g;
}

template <class Real>
struct Coefficients {
  std::vector<Real> cdx, cdy, cdz;
  const std::vector<Real>& axis(int a) const { return a == 0 ? cdx : (a == 1 ? cdy : cdz); }
};

/// One division c*dt/d per entry (grid.hpp:88-103).
template <class Real>
Coefficients<Real> build_coefficients(const GridSpec<Real>& g) {
  g.validate();
  Coefficients<Real> co;
  const Real cdt = g.c * g.dt;
  auto fill = [cdt](const std::vector<Real>& d, std::vector<Real>& out) {
    out.resize(d.size());
    for (std::size_t i = 0; i < d.size(); ++i) out[i] = cdt / d[i];
  };
  fill(g.dx, co.cdx);
  fill(g.dy, co.cdy);
  fill(g.dz, co.cdz);
  return co;
}

// ------------------------------------------------ fields (fields.hpp)
template <class Real>
struct FieldSet {
  Array3<Real> ex, ey, ez, hx, hy, hz;
  long long step_index = 0;
  FieldSet() = default;
  explicit FieldSet(const GridDims& g) { allocate(g); }
  void allocate(const GridDims& g) {
    dims_ = g;
    auto alloc = [&](Comp c) {
      const IndexBox b = comp_extents(g, c);
      return Array3<Real>(b.x.hi, b.y.hi, b.z.hi);
    };
    ex = alloc(Comp::Ex);
    ey = alloc(Comp::Ey);
    ez = alloc(Comp::Ez);
    hx = alloc(Comp::Hx);
    hy = alloc(Comp::Hy);
    hz = alloc(Comp::Hz);
    step_index = 0;
  }
  const GridDims& dims() const { return dims_; }
  Array3<Real>& field(Comp c) {
    switch (c) {
      case Comp::Ex: return ex;
      case Comp::Ey: return ey;
      case Comp::Ez: return ez;
      case Comp::Hx: return hx;
      case Comp::Hy: return hy;
      default: return hz;
    }
  }
  const Array3<Real>& field(Comp c) const { return const_cast<FieldSet*>(this)->field(c); }
  void zero() {
    for (Comp c : kAllComps) field(c).fill(Real(0));
    step_index = 0;
  }

 private:
  GridDims dims_;
};

/// FNV-1a-64 over raw bytes Ex..Hz (fields.hpp:151-166).
template <class Real>
std::uint64_t field_digest(const FieldSet<Real>& f) {
  std::uint64_t h = 1469598103934665603ull;
  for (Comp c : kAllComps) {
    const unsigned char* b = reinterpret_cast<const unsigned char*>(f.field(c).data());
    for (std::size_t i = 0; i < f.field(c).size_bytes(); ++i) {
      h ^= b[i];
      h *= 1099511628211ull;
    }
  }
  return h;
}

template <class Real>
std::string field_digest_hex(const FieldSet<Real>& f) {
  char buf[17];
  std::snprintf(buf, sizeof(buf), "%016llx", static_cast<unsigned long long>(field_digest(f)));
  return std::string(buf);
}

// ------------------------------------------------ sources (source.hpp)
struct Waveform {
  double amplitude = 1.0, sigma = 1.0, t0 = 4.0;
  static Waveform pulse(double amplitude, double sigma) { return {amplitude, sigma, 4.0 * sigma}; }
  double value(double t) const {
    const double u = (t - t0) / sigma;
    return amplitude * u * std::exp(-0.5 * u * u);
  }
};

struct SourceSpec {
  int i = 0, j = 0, k = 0;
  Comp component = Comp::Ez;
  Waveform waveform;
  long long active_steps = std::numeric_limits<long long>::max();
  /// Optional explicit per-step increments (extension, e.g. the config
  /// Gaussian); when non-empty it replaces -dt*J(step*dt).
  std::vector<float> table;
  bool active_at(long long step) const {
    if (!table.empty()) return step >= 0 && step < static_cast<long long>(table.size());
    return step < active_steps && waveform.amplitude != 0.0;
  }
  void validate(const GridDims& g) const {
    if (!is_electric(component)) throw std::invalid_argument("SourceSpec: component must be electric");
    IndexBox interior = curl_updatable_box(g, component);
    for (int a = 0; a < 3; ++a) {
      Interval r = interior.axis(a);
      if (!is_node_axis(component, a)) r = {r.lo + 1, r.hi - 1};
      const int idx = a == 0 ? i : (a == 1 ? j : k);
      if (!r.contains(idx)) throw std::invalid_argument("SourceSpec: position not interior");
    }
  }
  /// The float increment inject_current adds at `step` (source.hpp:61-68).
  float increment(long long step, double dt) const {
    if (!table.empty()) return table[static_cast<std::size_t>(step)];
    return static_cast<float>(-dt * waveform.value(static_cast<double>(step) * dt));
  }
};

// ------------------------------------------------ probes (probe.hpp)
struct ProbeSpec {
  int i = 0, j = 0, k = 0;
  Comp component = Comp::Ez;
  int stride = 1;
  bool fires_at(long long step) const { return step % stride == 0; }
  void validate(const GridDims& g) const {
    if (stride < 1) throw std::invalid_argument("ProbeSpec: stride must be >= 1");
    if (!comp_extents(g, component).contains(i, j, k))
      throw std::invalid_argument("ProbeSpec: position outside grid");
  }
};

struct ProbeRecord {
  long long step = 0;
  double time = 0.0;
  int probe = 0;
  double value = 0.0;
};

/// One line per sample: step<TAB>time<TAB>probe<TAB>value, the value at
/// `value_digits` significant digits (format_probe_records, probe.hpp:56-66).
inline std::string format_probe_records(const std::vector<ProbeRecord>& records, int value_digits) {
  std::string out;
  char line[128];
  for (const ProbeRecord& r : records) {
    std::snprintf(line, sizeof(line), "%lld\t%.17g\t%d\t%.*g\n", r.step, r.time, r.probe, value_digits, r.value);
    out += line;
  }
  return out;
}

// ------------------------------------------------ runner (runner.hpp)
struct RunStats {
  long long steps = 0;
  double total_seconds = 0.0;
  double volume_seconds = 0.0;
  long long skipped_tiles = 0;
  int fallback_tiles = 0;
  long long single_steps = 0;
};

template <class Real>
struct RunOptions {
  std::vector<SourceSpec> sources;
  std::vector<ProbeSpec> probes;
  bool quiescent_skip = true;  // skip all-zero work items (runner.hpp:60-73); results unchanged
  int device = 0;
  int variant = YB_VARIANT_TB2;
  std::function<void(const FieldSet<Real>&, long long)> after_step;
};

/// Per-cell coefficient selector (extension; the reference has none).
enum class CellCoeff { Ca = YB_CA, Cb = YB_CB, Da = YB_DA, Db = YB_DB };

/// Device-resident state + Standard-step driver (runner.hpp:205-266).
/// fields() returns a host mirror: it is read back on access, and a
/// non-const access marks it dirty so the next run() uploads it.
template <class Real>
class Simulation {
 public:
  explicit Simulation(const GridSpec<Real>& grid, RunOptions<Real> opts = {})
      : grid_(grid), opts_(std::move(opts)), coeffs_(build_coefficients(grid)), mirror_(grid.dims()) {
    grid_.validate();
    if (!(static_cast<double>(grid_.dt) > 0.0) ||
        static_cast<double>(grid_.dt) > stable_dt(grid_, 1.0) * (1.0 + 1e-9))
      throw std::invalid_argument("Simulation: dt violates the stability bound");
    for (const SourceSpec& s : opts_.sources) s.validate(grid_.dims());
    for (const ProbeSpec& p : opts_.probes) p.validate(grid_.dims());
    yb_desc d{};
    d.nx = grid_.nx;
    d.ny = grid_.ny;
    d.nz = grid_.nz;
    d.device = opts_.device;
    d.variant = opts_.variant;
    detail::check(yb_create(&d, &h_));
    detail::check(yb_set_axis_coeffs(h_, coeffs_.cdx.data(), coeffs_.cdy.data(), coeffs_.cdz.data()));
    detail::check(yb_set_quiescent_skip(h_, opts_.quiescent_skip ? 1 : 0));
    if (!opts_.probes.empty()) {  // sampled on the device (sample_probes, probe.hpp:36-51)
      std::vector<int> c, i, j, k, st;
      for (const ProbeSpec& p : opts_.probes) {
        c.push_back(comp_index(p.component));
        i.push_back(p.i);
        j.push_back(p.j);
        k.push_back(p.k);
        st.push_back(p.stride);
      }
      detail::check(yb_set_probes(h_, static_cast<int>(c.size()), c.data(), i.data(), j.data(), k.data(),
                                  st.data()));
    }
  }
  ~Simulation() {
    if (h_) yb_destroy(h_);
  }
  Simulation(const Simulation&) = delete;
  Simulation& operator=(const Simulation&) = delete;

  FieldSet<Real>& fields() {
    sync_mirror();
    dirty_ = true;
    return mirror_;
  }
  const FieldSet<Real>& fields() const {
    const_cast<Simulation*>(this)->sync_mirror();
    return mirror_;
  }
  const GridSpec<Real>& grid() const { return grid_; }
  const Coefficients<Real>& coeffs() const { return coeffs_; }
  const RunStats& stats() const { return stats_; }
  /// The C-ABI handle (extension: timing, info, halo exchange).
  yb_sim* handle() const { return h_; }

  /// Per-cell coefficients (extension): `cells` nx*ny*nz in cell order, or
  /// empty to fall back to the uniform/per-axis default.
  void set_cell_coefficients(CellCoeff which, const std::vector<float>& cells, float uniform = 1.0f) {
    if (!cells.empty() && static_cast<long long>(cells.size()) != grid_.dims().cell_count())
      throw std::invalid_argument("set_cell_coefficients: size mismatch");
    detail::check(yb_set_cell_coeffs(h_, static_cast<int>(which), cells.empty() ? nullptr : cells.data(), uniform));
  }
  /// The pinned seeded medium (include/yeeb200_inputs.h), generated on device.
  void generate_medium(long long eps_seed, long long sigma_seed) {
    detail::check(yb_generate_medium(h_, eps_seed, sigma_seed));
  }

  /// Advances n_steps time levels and returns all probe samples.
  std::vector<ProbeRecord> run(long long n_steps) {
    if (n_steps < 0) throw std::invalid_argument("run: negative step count");
    push_if_dirty();
    const double t0 = now();
    std::vector<ProbeRecord> records;
    long long t = step_;
    const long long t_end = t + n_steps;
    const bool per_step = static_cast<bool>(opts_.after_step);
    while (t < t_end) {
      long long n = t_end - t;
      if (per_step) n = 1;
      load_sources(t, n);
      detail::check(yb_advance(h_, n));
      t += n;
      step_ = t;
      if (opts_.after_step) {
        have_mirror_ = false;
        sync_mirror();
        opts_.after_step(mirror_, t);
      }
    }
    if (!opts_.probes.empty()) drain_probes(records);
    detail::check(yb_synchronize(h_));
    have_mirror_ = false;
    stats_.total_seconds += now() - t0;
    stats_.steps += n_steps;
    yb_info inf{};
    detail::check(yb_get_info(h_, &inf));
    stats_.skipped_tiles = inf.skipped_items;
    return records;
  }

  /// HSnapshot of the device-resident H (fields.hpp:71-82); pair with
  /// total_energy() after advancing (the reference's measure_energy_drift
  /// pattern, bench.hpp:273-303).
  void snapshot_h() {
    push_if_dirty();
    detail::check(yb_snapshot_h(h_));
  }
  /// Leapfrog invariant on the device (total_energy, fields.hpp:116-146).
  double total_energy() {
    push_if_dirty();
    std::vector<double> d[3];
    for (int a = 0; a < 3; ++a)
      for (Real v : grid_.spacing(a)) d[a].push_back(static_cast<double>(v));
    double e = 0.0;
    detail::check(yb_total_energy(h_, d[0].data(), d[1].data(), d[2].data(), &e));
    return e;
  }

  /// The reference range ops on the device-resident state (kernels.hpp:129-155).
  void apply_ampere_range(const IndexBox& b) { range_op(b, true); }
  void apply_faraday_range(const IndexBox& b) { range_op(b, false); }
  void apply_pec_boundary() {
    push_if_dirty();
    detail::check(yb_apply_pec_boundary(h_));
    have_mirror_ = false;
  }

 private:
  static double now() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
  }
  void range_op(const IndexBox& b, bool ampere) {
    push_if_dirty();
    const int box[6] = {b.x.lo, b.x.hi, b.y.lo, b.y.hi, b.z.lo, b.z.hi};
    detail::check(ampere ? yb_apply_ampere_range(h_, box) : yb_apply_faraday_range(h_, box));
    have_mirror_ = false;
  }
  void sync_mirror() {
    if (have_mirror_) return;
    float* d6[6];
    for (Comp c : kAllComps) d6[comp_index(c)] = mirror_.field(c).data();
    detail::check(yb_download_fields(h_, d6));
    mirror_.step_index = step_;
    have_mirror_ = true;
  }
  void push_if_dirty() {
    if (!dirty_) return;
    const float* u6[6];
    for (Comp c : kAllComps) u6[comp_index(c)] = mirror_.field(c).data();
    detail::check(yb_upload_fields(h_, u6));
    step_ = mirror_.step_index;
    detail::check(yb_set_step_index(h_, step_));
    dirty_ = false;
  }
  // per-step increments for steps [t, t+n) as tables indexed by absolute step
  void load_sources(long long t, long long n) {
    detail::check(yb_clear_sources(h_));
    const double dt = static_cast<double>(grid_.dt);
    for (const SourceSpec& s : opts_.sources) {
      std::vector<float> tab(static_cast<std::size_t>(t + n), 0.0f);
      long long last = -1;
      for (long long q = t; q < t + n; ++q)
        if (s.active_at(q)) {
          tab[static_cast<std::size_t>(q)] = s.increment(q, dt);
          last = q;
        }
      if (last < 0) continue;  // active_at is monotone: steps t..last are all active
      detail::check(yb_add_source(h_, comp_index(s.component), s.i, s.j, s.k, tab.data(), last + 1));
    }
  }
  // Appends the device-recorded samples (step order, then probe order).
  void drain_probes(std::vector<ProbeRecord>& records) {
    const double dt = static_cast<double>(grid_.dt);
    constexpr long long kChunk = 1 << 16;
    std::vector<int64_t> steps(kChunk);
    std::vector<int> probe(kChunk);
    std::vector<float> vals(kChunk);
    for (;;) {
      int64_t n = 0;
      detail::check(yb_read_probes(h_, steps.data(), probe.data(), vals.data(), kChunk, &n));
      for (int64_t q = 0; q < n; ++q)
        records.push_back({steps[q], static_cast<double>(steps[q]) * dt, probe[q], static_cast<double>(vals[q])});
      if (n < kChunk) break;
    }
  }

  GridSpec<Real> grid_;
  RunOptions<Real> opts_;
  Coefficients<Real> coeffs_;
  FieldSet<Real> mirror_;
  yb_sim* h_ = nullptr;
  long long step_ = 0;
  bool have_mirror_ = false, dirty_ = false;
  RunStats stats_;
};

/// Copy-in / advance / copy-out (runner.hpp:349-362).
template <class Real>
std::vector<ProbeRecord> run_simulation(const GridSpec<Real>& grid, long long n_steps,
                                        FieldSet<Real>& state, RunOptions<Real> opts = {},
                                        RunStats* stats_out = nullptr) {
  Simulation<Real> sim(grid, std::move(opts));
  sim.fields() = state;
  auto records = sim.run(n_steps);
  state = sim.fields();
  if (stats_out) *stats_out = sim.stats();
  return records;
}

/// Source-free single Standard step with explicit coefficients (runner.hpp:394-398).
template <class Real>
void step_standard(const GridSpec<Real>& g, FieldSet<Real>& f, const Coefficients<Real>& c) {
  if (static_cast<double>(g.dt) > stable_dt(g, 1.0) * (1.0 + 1e-9))
    throw std::invalid_argument("step: dt violates the stability bound");
  yb_desc d{};
  d.nx = g.nx;
  d.ny = g.ny;
  d.nz = g.nz;
  yb_sim* h = nullptr;
  detail::check(yb_create(&d, &h));
  struct Guard {
    yb_sim* h;
    ~Guard() { yb_destroy(h); }
  } guard{h};
  detail::check(yb_set_axis_coeffs(h, c.cdx.data(), c.cdy.data(), c.cdz.data()));
  {
    const float* u6[6];
    for (Comp q : kAllComps) u6[comp_index(q)] = f.field(q).data();
    detail::check(yb_upload_fields(h, u6));
  }
  detail::check(yb_set_step_index(h, f.step_index));
  detail::check(yb_advance(h, 1));
  {
    float* d6[6];
    for (Comp q : kAllComps) d6[comp_index(q)] = f.field(q).data();
    detail::check(yb_download_fields(h, d6));
  }
  f.step_index += 1;
}

}  // namespace yeeb200

#ifdef YEEB200_AS_YEEBLOCK
namespace yeeblock = yeeb200;
#endif
