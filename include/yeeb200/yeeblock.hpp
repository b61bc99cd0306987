// yeeb200/yeeblock.hpp — C++ drop-in shim over libyeeb200.so (include/yeeb200.h).
//
// Re-exposes the reference yeeblock API (/root/reference/proj/include/yeeblock,
// a header-only CPU library templated on Real) with the same names,
// signatures, argument meanings and exception types, backed by the B200
// kernels:
//   array3.hpp      Interval, IndexBox, intersect, overlaps, contains, box_difference, Array3
//   staggering.hpp  Comp, comp_* helpers, GridDims, comp_extents, curl_updatable_box, pec_boxes
//   grid.hpp        GridSpec, stable_dt, make_uniform_grid, Coefficients, build_coefficients
//   fields.hpp      FieldSet, HSnapshot, total_energy (on the device), field_digest(_hex)
//   kernels.hpp     update_e_box, update_h_box, zero_box, apply_ampere_range,
//                   apply_faraday_range, apply_pec_boundary (per-DoF device kernels
//                   on the caller's host FieldSet, float or double: yb_fs_apply)
//   source.hpp      Waveform, SourceSpec, inject_current
//   probe.hpp       ProbeSpec, ProbeRecord, sample_probes, format_probe_records
//   tiling.hpp      Split, Tile, TileLayout, make_layout       (accepted; inert on the GPU)
//   schedule.hpp    Variant, variant_name, parse_variant, ...  (accepted; inert on the GPU)
//   parallel.hpp    ExecConfig                                 (accepted; inert on the GPU)
//   runner.hpp      RunStats, RunOptions, Simulation(grid, layout, variant, opts),
//                   run_simulation(grid, layout, variant, n, state, opts, stats),
//                   step_standard / step_tiled / step_interleaved / step_planewise /
//                   step_twostep
//
// The time loop (Simulation, run_simulation, step_*) is the device-resident
// fp32 path (Simulation<float>; a static_assert rejects other Real). The
// per-box operations and total_energy accept FieldSet<float> and
// FieldSet<double>. Every reference variant computes bit-identical fields
// (schedule.hpp:13-15), so the GPU runs its own schedule whatever Variant and
// TileLayout the caller passes; the layout must still match the grid, as in
// the reference. The reference's own unit tests (proj/tests/kernel_test.cpp,
// grid_test.cpp) compile unmodified against include/yeeb200/compat/ and pass
// on the GPU (tests/cpp/Makefile, tests/test_shim_reference.py).
//
// Namespace yeeb200; include/yeeb200/compat/yeeblock/*.hpp (or defining
// YEEB200_AS_YEEBLOCK) adds `namespace yeeblock = yeeb200;`.
//
// Not mirrored: the CPU plan IR and executor (schedule.hpp StepPlan /
// build_plan, runner.hpp execute_plan, parallel.hpp WorkerPool /
// assign_tiles), the tile-interface bookkeeping of TileLayout, the per-DoF
// update_e_dof / update_h_dof (subsumed by the box operations), the perf model
// and bench harness (perf_model.hpp, bench.hpp; yb_bench is the B200
// analogue).
#pragma once

#include <algorithm>
#include <array>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <limits>
#include <optional>
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
template <class Real>
constexpr int dtype_of() {
  static_assert(std::is_same<Real, float>::value || std::is_same<Real, double>::value,
                "Real must be float or double");
  return std::is_same<Real, float>::value ? YB_F32 : YB_F64;
}
}  // namespace detail

// ------------------------------------------------ index boxes (array3.hpp)
/// Half-open [lo, hi).
struct Interval {
  int lo = 0, hi = 0;
  constexpr int length() const { return hi > lo ? hi - lo : 0; }
  constexpr bool empty() const { return hi <= lo; }
  constexpr bool contains(int v) const { return v >= lo && v < hi; }
};

constexpr Interval intersect(Interval a, Interval b) {
  return {a.lo > b.lo ? a.lo : b.lo, a.hi < b.hi ? a.hi : b.hi};
}

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

inline IndexBox intersect(const IndexBox& a, const IndexBox& b) {
  return {intersect(a.x, b.x), intersect(a.y, b.y), intersect(a.z, b.z)};
}
inline bool overlaps(const IndexBox& a, const IndexBox& b) { return !intersect(a, b).empty(); }
/// An empty inner box lies inside anything (array3.hpp:47-52).
inline bool contains(const IndexBox& outer, const IndexBox& inner) {
  if (inner.empty()) return true;
  for (int a = 0; a < 3; ++a)
    if (inner.axis(a).lo < outer.axis(a).lo || inner.axis(a).hi > outer.axis(a).hi) return false;
  return true;
}

/// a \ b as at most six disjoint boxes, slabs peeled per axis low side then
/// high side, x then y then z (array3.hpp:57-82 order).
template <class Sink>
inline void box_difference(const IndexBox& a, const IndexBox& b, Sink&& emit) {
  const IndexBox cut = intersect(a, b);
  if (cut.empty()) {
    if (!a.empty()) emit(a);
    return;
  }
  IndexBox rest = a;
  for (int ax = 0; ax < 3; ++ax) {
    const Interval keep = cut.axis(ax), have = rest.axis(ax);
    for (const Interval side : {Interval{have.lo, keep.lo}, Interval{keep.hi, have.hi}}) {
      IndexBox slab = rest;
      slab.axis(ax) = side;
      if (!slab.empty()) emit(slab);
    }
    rest.axis(ax) = keep;
  }
}

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
constexpr std::array<Comp, 3> kEComps = {Comp::Ex, Comp::Ey, Comp::Ez};
constexpr std::array<Comp, 3> kHComps = {Comp::Hx, Comp::Hy, Comp::Hz};
constexpr std::array<Comp, 6> kAllComps = {Comp::Ex, Comp::Ey, Comp::Ez, Comp::Hx, Comp::Hy, Comp::Hz};
constexpr bool is_electric(Comp c) { return c <= Comp::Ez; }
constexpr int comp_index(Comp c) { return static_cast<int>(c); }
inline const char* comp_name(Comp c) {
  static const char* names[6] = {"ex", "ey", "ez", "hx", "hy", "hz"};
  return names[comp_index(c)];
}
constexpr int comp_axis(Comp c) { return comp_index(c) % 3; }
/// E is node-centred off its own axis, H on its own axis (staggering.hpp:44-47).
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

/// E DoFs off the PEC faces; H over its full extents (staggering.hpp:70-77).
inline IndexBox curl_updatable_box(const GridDims& g, Comp c) {
  IndexBox b = comp_extents(g, c);
  if (is_electric(c))
    for (int a = 0; a < 3; ++a)
      if (is_node_axis(c, a)) b.axis(a) = {1, g.cells(a)};
  return b;
}

/// The PEC-forced DoFs of an E component as disjoint boxes (staggering.hpp:81-86).
inline void pec_boxes(const GridDims& g, Comp c, std::vector<IndexBox>& out) {
  if (!is_electric(c)) return;
  box_difference(comp_extents(g, c), curl_updatable_box(g, c), [&](const IndexBox& b) { out.push_back(b); });
}

// ------------------------------------------------ grid (grid.hpp)
inline constexpr double kVacuumLightSpeed = 299792458.0;

template <class Real>
struct GridSpec {
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

/// Copy of the three magnetic arrays for the leapfrog energy (fields.hpp:71-82).
template <class Real>
struct HSnapshot {
  Array3<Real> hx, hy, hz;
  HSnapshot() = default;
  explicit HSnapshot(const FieldSet<Real>& f) : hx(f.hx), hy(f.hy), hz(f.hz) {}
  const Array3<Real>& field(Comp c) const { return c == Comp::Hx ? hx : (c == Comp::Hy ? hy : hz); }
};

namespace detail {
/// Dual spacing at node i: half the adjacent cells, halved at the ends (fields.hpp:86-93).
template <class Real>
double dual_spacing(const std::vector<Real>& d, int i) {
  const int n = static_cast<int>(d.size());
  if (i == 0) return 0.5 * static_cast<double>(d[0]);
  if (i == n) return 0.5 * static_cast<double>(d[n - 1]);
  return 0.5 * (static_cast<double>(d[i - 1]) + static_cast<double>(d[i]));
}
template <class Real>
double dof_volume(const GridSpec<Real>& g, Comp c, int i, int j, int k) {
  const int idx[3] = {i, j, k};
  double v = 1.0;
  for (int a = 0; a < 3; ++a) {
    const std::vector<Real>& d = g.spacing(a);
    v *= is_node_axis(c, a) ? dual_spacing(d, idx[a]) : static_cast<double>(d[idx[a]]);
  }
  return v;
}
inline int current_device() {
  // the device a host-FieldSet operation runs on (YB_DEVICE, default 0)
  const char* e = std::getenv("YB_DEVICE");
  return e ? std::atoi(e) : 0;
}
}  // namespace detail

/// Leapfrog invariant sum_E V*E^2 + sum_H V*Hprev*Hnow (fields.hpp:116-146),
/// accumulated in double on the device (yb_fs_total_energy; deterministic,
/// its summation order differs from the reference's serial loop).
template <class Real>
double total_energy(const GridSpec<Real>& g, const FieldSet<Real>& f, const HSnapshot<Real>& prev_h) {
  if (f.dims() != g.dims()) throw std::invalid_argument("total_energy: grid/field extents mismatch");
  for (Comp c : kHComps)
    if (!f.field(c).same_extents(prev_h.field(c)))
      throw std::invalid_argument("total_energy: H snapshot extents mismatch");
  std::vector<double> d[3];
  for (int a = 0; a < 3; ++a)
    for (Real h : g.spacing(a)) d[a].push_back(static_cast<double>(h));
  const void* f6[6];
  for (Comp c : kAllComps) f6[comp_index(c)] = f.field(c).data();
  const void* p3[3] = {prev_h.hx.data(), prev_h.hy.data(), prev_h.hz.data()};
  double e = 0.0;
  detail::check(yb_fs_total_energy(detail::current_device(), detail::dtype_of<Real>(), g.nx, g.ny, g.nz, f6, p3,
                                   d[0].data(), d[1].data(), d[2].data(), &e));
  return e;
}

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

// ------------------------------------------------ per-box operations (kernels.hpp)
// On the caller's host FieldSet: the components the operation reads go to the
// device, per-DoF kernels update them in the reference's operand order
// (bit-identical), the written components come back (yb_fs_apply).
namespace detail {
inline IndexBox node_box(const GridDims& g) { return {{0, g.nx + 1}, {0, g.ny + 1}, {0, g.nz + 1}}; }

inline void check_range(const GridDims& g, const IndexBox& box, const char* what) {
  if (!contains(node_box(g), box)) throw std::out_of_range(std::string(what) + ": range out of bounds");
}

template <class Real>
void fs_apply(FieldSet<Real>& f, const Coefficients<Real>* c, int op, Comp comp, const IndexBox& b) {
  const GridDims g = f.dims();
  void* f6[6];
  for (Comp q : kAllComps) f6[comp_index(q)] = f.field(q).data();
  const void* cd[3] = {nullptr, nullptr, nullptr};
  if (c) {
    if (static_cast<int>(c->cdx.size()) != g.nx || static_cast<int>(c->cdy.size()) != g.ny ||
        static_cast<int>(c->cdz.size()) != g.nz)
      throw std::invalid_argument("Coefficients: array lengths do not match the field extents");
    cd[0] = c->cdx.data();
    cd[1] = c->cdy.data();
    cd[2] = c->cdz.data();
  }
  const int box[6] = {b.x.lo, b.x.hi, b.y.lo, b.y.hi, b.z.lo, b.z.hi};
  check(yb_fs_apply(current_device(), dtype_of<Real>(), g.nx, g.ny, g.nz, f6, c ? cd : nullptr, op,
                    comp_index(comp), box));
}
}  // namespace detail

/// One E component over `box` (kernels.hpp:78-88); box must lie inside curl_updatable_box.
template <class Real>
void update_e_box(FieldSet<Real>& f, const Coefficients<Real>& c, Comp comp, const IndexBox& box) {
  detail::fs_apply(f, &c, YB_OP_UPDATE_E, comp, box);
}
/// One H component over `box` (kernels.hpp:92-101); box must lie inside the component's extents.
template <class Real>
void update_h_box(FieldSet<Real>& f, const Coefficients<Real>& c, Comp comp, const IndexBox& box) {
  detail::fs_apply(f, &c, YB_OP_UPDATE_H, comp, box);
}
/// Exact zeros over `box` of one component (kernels.hpp:104-111).
template <class Real>
void zero_box(FieldSet<Real>& f, Comp comp, const IndexBox& box) {
  detail::fs_apply<Real>(f, nullptr, YB_OP_ZERO, comp, box);
}
/// Ampere over `box` (node index space) intersected with each E component's
/// updatable box (kernels.hpp:129-135).
template <class Real>
void apply_ampere_range(FieldSet<Real>& f, const Coefficients<Real>& c, const IndexBox& box) {
  detail::fs_apply(f, &c, YB_OP_AMPERE, Comp::Ex, box);
}
/// Faraday over `box` intersected with each H component's extents (kernels.hpp:138-144).
template <class Real>
void apply_faraday_range(FieldSet<Real>& f, const Coefficients<Real>& c, const IndexBox& box) {
  detail::fs_apply(f, &c, YB_OP_FARADAY, Comp::Hx, box);
}
/// Tangential E := +0 on the six outer faces (kernels.hpp:147-155).
template <class Real>
void apply_pec_boundary(FieldSet<Real>& f) {
  detail::fs_apply<Real>(f, nullptr, YB_OP_PEC, Comp::Ex, IndexBox{});
}

// ------------------------------------------------ sources (source.hpp)
/// Differentiated Gaussian J(t) = A (t-t0)/s exp(-(t-t0)^2/(2 s^2)) (source.hpp:15-31).
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
  /// Extension: explicit per-step increments (e.g. the configs' Gaussian);
  /// when non-empty it replaces -dt*J(step*dt) and is active for its length.
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
  /// The increment inject_current adds at `step` (source.hpp:61-68), in Real.
  template <class Real = float>
  Real increment(long long step, double dt) const {
    if (!table.empty()) return static_cast<Real>(table[static_cast<std::size_t>(step)]);
    return static_cast<Real>(-dt * waveform.value(static_cast<double>(step) * dt));
  }
};

/// Soft source on the caller's FieldSet: the one DoF += (Real)(-dt*J(step*dt))
/// (source.hpp:61-68). A single scalar update of host memory; the device
/// time loop applies sources inside its sweep kernels.
template <class Real>
void inject_current(FieldSet<Real>& f, const SourceSpec& s, long long step, double dt) {
  if (step < 0) throw std::invalid_argument("inject_current: negative step");
  if (!s.active_at(step)) return;
  f.field(s.component)(s.i, s.j, s.k) += s.increment<Real>(step, dt);
}

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

/// Samples of a host FieldSet, every probe whose stride divides `step` (probe.hpp:36-51).
template <class Real>
std::vector<ProbeRecord> sample_probes(const FieldSet<Real>& f, const std::vector<ProbeSpec>& probes,
                                       long long step, double dt) {
  if (step < 0) throw std::invalid_argument("sample_probes: negative step");
  std::vector<ProbeRecord> out;
  for (std::size_t p = 0; p < probes.size(); ++p) {
    const ProbeSpec& q = probes[p];
    if (!q.fires_at(step)) continue;
    out.push_back({step, static_cast<double>(step) * dt, static_cast<int>(p),
                   static_cast<double>(f.field(q.component)(q.i, q.j, q.k))});
  }
  return out;
}

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

// ------------------------------------------------ tiling / schedules (inert on the GPU)
struct Split {
  int sx = 1, sy = 1, sz = 1;
  int axis(int a) const { return a == 0 ? sx : (a == 1 ? sy : sz); }
  int count() const { return sx * sy * sz; }
  bool operator==(const Split& o) const { return sx == o.sx && sy == o.sy && sz == o.sz; }
};

struct Tile {
  int id = 0;
  IndexBox cells;
  std::array<int, 6> neighbor = {};  // -x,+x,-y,+y,-z,+z; -1 at domain faces
};

/// The reference's CPU tile decomposition (tiling.hpp:76-118), kept so that
/// callers building one compile and validate unchanged. The GPU tiles the
/// grid itself; the interface sets of the CPU schedulers are not built.
struct TileLayout {
  GridDims dims;
  Split split;
  std::array<std::vector<int>, 3> breaks;
  std::vector<Tile> tiles;
  int tile_id(int a, int b, int c) const { return (c * split.sy + b) * split.sx + a; }
  const Tile& tile_at(int a, int b, int c) const { return tiles[tile_id(a, b, c)]; }
};

/// Near-equal tiles, remainder to the leading ones (tiling.hpp:121-128, :208-239).
inline TileLayout make_layout(const GridDims& dims, const Split& split) {
  for (int a = 0; a < 3; ++a)
    if (split.axis(a) < 1 || split.axis(a) > dims.cells(a))
      throw std::invalid_argument("make_layout: invalid split for grid");
  TileLayout L;
  L.dims = dims;
  L.split = split;
  for (int a = 0; a < 3; ++a) {
    const int n = dims.cells(a), p = split.axis(a), base = n / p, rem = n % p;
    L.breaks[a].assign(static_cast<std::size_t>(p) + 1, 0);
    for (int t = 0; t < p; ++t) L.breaks[a][t + 1] = L.breaks[a][t] + base + (t < rem ? 1 : 0);
  }
  L.tiles.resize(static_cast<std::size_t>(split.count()));
  for (int c = 0; c < split.sz; ++c)
    for (int b = 0; b < split.sy; ++b)
      for (int a = 0; a < split.sx; ++a) {
        Tile& t = L.tiles[static_cast<std::size_t>(L.tile_id(a, b, c))];
        t.id = L.tile_id(a, b, c);
        t.cells = {{L.breaks[0][a], L.breaks[0][a + 1]},
                   {L.breaks[1][b], L.breaks[1][b + 1]},
                   {L.breaks[2][c], L.breaks[2][c + 1]}};
        t.neighbor = {a > 0 ? L.tile_id(a - 1, b, c) : -1, a + 1 < split.sx ? L.tile_id(a + 1, b, c) : -1,
                      b > 0 ? L.tile_id(a, b - 1, c) : -1, b + 1 < split.sy ? L.tile_id(a, b + 1, c) : -1,
                      c > 0 ? L.tile_id(a, b, c - 1) : -1, c + 1 < split.sz ? L.tile_id(a, b, c + 1) : -1};
      }
  return L;
}

/// The reference's five update orderings (schedule.hpp:16-37). All produce
/// bit-identical fields; on the GPU they select nothing but the after_step
/// cadence of TwoStep (gathered pairs).
enum class Variant { Standard, Tiled, Interleaved, Planewise, TwoStep };
constexpr std::array<Variant, 5> kAllVariants = {Variant::Standard, Variant::Tiled, Variant::Interleaved,
                                                 Variant::Planewise, Variant::TwoStep};
inline const char* variant_name(Variant v) {
  static const char* names[5] = {"standard", "tiled", "interleaved", "planewise", "twostep"};
  return names[static_cast<int>(v)];
}
inline std::optional<Variant> parse_variant(const std::string& s) {
  for (Variant v : kAllVariants)
    if (s == variant_name(v)) return v;
  return std::nullopt;
}
constexpr int variant_substeps(Variant v) { return v == Variant::TwoStep ? 2 : 1; }

/// Worker-pool settings of the CPU executor (parallel.hpp:19-23); accepted, unused.
struct ExecConfig {
  int workers = 1;
  bool pin = false;
  int chunk = 0;
};

// ------------------------------------------------ runner (runner.hpp)
struct RunStats {
  long long steps = 0;
  double total_seconds = 0.0;
  double volume_seconds = 0.0;
  long long skipped_tiles = 0;  // work items skipped as quiescent (device count)
  int fallback_tiles = 0;
  long long single_steps = 0;
};

template <class Real>
struct RunOptions {
  std::vector<SourceSpec> sources;
  std::vector<ProbeSpec> probes;
  bool quiescent_skip = true;  // skip all-zero work items (runner.hpp:60-73); results unchanged
  ExecConfig exec;
  std::function<void(const FieldSet<Real>&, long long)> after_step;
  // extensions: the CUDA device and the step kernel (YB_VARIANT_*; TB2 = the fastest)
  int device = 0;
  int kernel = YB_VARIANT_TB2;
  /// When run() brings the state back into the host FieldSet that fields() returns. The reference's
  /// FieldSet is the live state (runner.hpp:236); here it is a mirror of the device state.
  /// Lazy: on the first fields() access after a run. Eager: as part of run() (yb_run_to_host: the
  /// readback overlaps the last sweeps, also into this pageable storage). Auto (default): eager
  /// for runs of at least 64 steps where that overlap is possible (two-step kernel, no probes,
  /// quiescent_skip off), until a readback was paid for and never looked at.
  enum class Readback { Lazy, Eager, Auto };
  Readback readback = Readback::Auto;
};

/// Per-cell coefficient selector (extension; the reference has none).
enum class CellCoeff { Ca = YB_CA, Cb = YB_CB, Da = YB_DA, Db = YB_DB };

/// Device-resident state + time loop (runner.hpp:205-266).
/// fields() returns a host mirror: it is read back on access, and a
/// non-const access marks it dirty so the next run() uploads it.
template <class Real>
class Simulation {
  static_assert(std::is_same<Real, float>::value,
                "yeeb200::Simulation: the device time loop is single precision (use float)");

 public:
  /// The reference constructor (runner.hpp:208-234): validates the layout
  /// against the grid, dt, sources and probes with the reference's errors.
  Simulation(const GridSpec<Real>& grid, const TileLayout& layout, Variant v, RunOptions<Real> opts)
      : Simulation(checked(grid, layout), std::move(opts), v) {}
  /// Extension: no CPU layout needed.
  explicit Simulation(const GridSpec<Real>& grid, RunOptions<Real> opts = {}, Variant v = Variant::Standard)
      : grid_(grid), variant_(v), opts_(std::move(opts)), mirror_(grid.dims()) {
    grid_.validate();
    coeffs_ = build_coefficients(grid_);
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
    d.variant = opts_.kernel;
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
  Variant variant() const { return variant_; }
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

  /// Advances n_steps time levels and returns all probe samples (runner.hpp:243-266).
  std::vector<ProbeRecord> run(long long n_steps) {
    if (n_steps < 0) throw std::invalid_argument("run: negative step count");
    push_if_dirty();
    if (eager_unread_) auto_lazy_ = true;  // the last eager readback was never looked at
    using RB = typename RunOptions<Real>::Readback;
    // Auto: only where the readback can overlap the run (yb_run_to_host streams with the two-step
    // kernel, no probes, quiescent skip off); elsewhere an eager readback is just an early one
    const bool streams = opts_.kernel == YB_VARIANT_TB2 && opts_.probes.empty() && !opts_.quiescent_skip;
    const bool eager = !opts_.after_step && n_steps > 0 &&
                       (opts_.readback == RB::Eager ||
                        (opts_.readback == RB::Auto && streams && n_steps >= 64 && !auto_lazy_));
    const double t0 = now();
    std::vector<ProbeRecord> records;
    long long t = step_;
    const long long t_end = t + n_steps;
    while (t < t_end) {
      long long n = t_end - t;
      if (opts_.after_step) {
        // the reference's cadence: every step, or gathered TwoStep pairs (runner.hpp:249-262, :280-284)
        n = (variant_ == Variant::TwoStep && can_gather(t, t_end)) ? 2 : 1;
      } else if (variant_ == Variant::TwoStep) {
        for (long long q = t; q < t_end;) {  // RunStats::single_steps as the reference counts it
          if (can_gather(q, t_end)) {
            q += 2;
          } else {
            ++stats_.single_steps;
            ++q;
          }
        }
      }
      load_sources(t, n);
      if (eager) {  // one chunk (no after_step): advance and read back in one overlapped call
        float* d6[6];
        for (Comp c : kAllComps) d6[comp_index(c)] = mirror_.field(c).data();
        detail::check(yb_run_to_host(h_, n, d6));
      } else {
        detail::check(yb_advance(h_, n));
      }
      t += n;
      step_ = t;
      if (opts_.after_step) {
        if (variant_ == Variant::TwoStep && n == 1) ++stats_.single_steps;
        have_mirror_ = false;
        sync_mirror();
        opts_.after_step(mirror_, t);
      }
    }
    if (!opts_.probes.empty()) drain_probes(records);
    detail::check(yb_synchronize(h_));
    have_mirror_ = eager;
    eager_unread_ = eager;
    if (eager) mirror_.step_index = step_;
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
  // the reference's first two checks (runner.hpp:217-220), before any device work
  static const GridSpec<Real>& checked(const GridSpec<Real>& grid, const TileLayout& layout) {
    grid.validate();
    if (layout.dims != grid.dims()) throw std::invalid_argument("Simulation: layout built for another grid");
    return grid;
  }
  static double now() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
  }
  bool source_injects(long long step) const {
    for (const SourceSpec& s : opts_.sources)
      if (s.active_at(step)) return true;
    return false;
  }
  bool probe_fires(long long step) const {
    for (const ProbeSpec& p : opts_.probes)
      if (p.fires_at(step)) return true;
    return false;
  }
  // runner.hpp:280-284
  bool can_gather(long long t, long long t_end) const {
    return t + 2 <= t_end && !probe_fires(t + 1) && !source_injects(t) && !source_injects(t + 1);
  }
  void range_op(const IndexBox& b, bool ampere) {
    push_if_dirty();
    const int box[6] = {b.x.lo, b.x.hi, b.y.lo, b.y.hi, b.z.lo, b.z.hi};
    detail::check(ampere ? yb_apply_ampere_range(h_, box) : yb_apply_faraday_range(h_, box));
    have_mirror_ = false;
  }
  void sync_mirror() {
    eager_unread_ = false;  // the caller looks at the state after its runs
    if (have_mirror_) return;
    auto_lazy_ = false;
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
          tab[static_cast<std::size_t>(q)] = s.increment<float>(q, dt);
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
  Variant variant_ = Variant::Standard;
  RunOptions<Real> opts_;
  Coefficients<Real> coeffs_;
  FieldSet<Real> mirror_;
  yb_sim* h_ = nullptr;
  long long step_ = 0;
  bool have_mirror_ = false, dirty_ = false;
  bool eager_unread_ = false, auto_lazy_ = false;  // RunOptions::Readback::Auto bookkeeping
  RunStats stats_;
};

/// Copy-in / advance / copy-out (runner.hpp:349-362), the reference signature.
template <class Real>
std::vector<ProbeRecord> run_simulation(const GridSpec<Real>& grid, const TileLayout& layout, Variant v,
                                        long long n_steps, FieldSet<Real>& state, RunOptions<Real> opts = {},
                                        RunStats* stats_out = nullptr) {
  Simulation<Real> sim(grid, layout, v, std::move(opts));
  sim.fields() = state;
  auto records = sim.run(n_steps);
  state = sim.fields();
  if (stats_out) *stats_out = sim.stats();
  return records;
}

/// Extension: the same without a CPU layout.
template <class Real>
std::vector<ProbeRecord> run_simulation(const GridSpec<Real>& grid, long long n_steps, FieldSet<Real>& state,
                                        RunOptions<Real> opts = {}, RunStats* stats_out = nullptr) {
  Simulation<Real> sim(grid, std::move(opts));
  sim.fields() = state;
  auto records = sim.run(n_steps);
  state = sim.fields();
  if (stats_out) *stats_out = sim.stats();
  return records;
}

namespace detail {
/// Source-free single invocation advancing `levels` steps (runner.hpp:365-386).
template <class Real>
void one_step(const GridSpec<Real>& g, FieldSet<Real>& f, const Coefficients<Real>& c, const TileLayout* layout,
              int levels) {
  static_assert(std::is_same<Real, float>::value, "yeeb200::step_*: the device time loop is single precision");
  if (static_cast<double>(g.dt) > stable_dt(g, 1.0) * (1.0 + 1e-9))
    throw std::invalid_argument("step: dt violates the stability bound");
  if (layout && layout->dims != g.dims()) throw std::invalid_argument("step: layout built for another grid");
  yb_desc d{};
  d.nx = g.nx;
  d.ny = g.ny;
  d.nz = g.nz;
  d.device = current_device();
  yb_sim* h = nullptr;
  check(yb_create(&d, &h));
  struct Guard {
    yb_sim* h;
    ~Guard() { yb_destroy(h); }
  } guard{h};
  check(yb_set_axis_coeffs(h, c.cdx.data(), c.cdy.data(), c.cdz.data()));
  {
    const float* u6[6];
    for (Comp q : kAllComps) u6[comp_index(q)] = f.field(q).data();
    check(yb_upload_fields(h, u6));
  }
  check(yb_set_step_index(h, f.step_index));
  check(yb_advance(h, levels));
  {
    float* d6[6];
    for (Comp q : kAllComps) d6[comp_index(q)] = f.field(q).data();
    check(yb_download_fields(h, d6));
  }
  f.step_index += levels;
}
}  // namespace detail

/// Source-free single steps with explicit coefficients (runner.hpp:391-420);
/// all variants are bit-identical, step_twostep advances two levels.
template <class Real>
void step_standard(const GridSpec<Real>& g, FieldSet<Real>& f, const Coefficients<Real>& c) {
  detail::one_step(g, f, c, nullptr, 1);
}
template <class Real>
void step_tiled(const GridSpec<Real>& g, FieldSet<Real>& f, const Coefficients<Real>& c, const TileLayout& L) {
  detail::one_step(g, f, c, &L, 1);
}
template <class Real>
void step_interleaved(const GridSpec<Real>& g, FieldSet<Real>& f, const Coefficients<Real>& c,
                      const TileLayout& L) {
  detail::one_step(g, f, c, &L, 1);
}
template <class Real>
void step_planewise(const GridSpec<Real>& g, FieldSet<Real>& f, const Coefficients<Real>& c,
                    const TileLayout& L) {
  detail::one_step(g, f, c, &L, 1);
}
template <class Real>
void step_twostep(const GridSpec<Real>& g, FieldSet<Real>& f, const Coefficients<Real>& c, const TileLayout& L) {
  detail::one_step(g, f, c, &L, 2);
}

}  // namespace yeeb200

#ifdef YEEB200_AS_YEEBLOCK
namespace yeeblock = yeeb200;
#endif
