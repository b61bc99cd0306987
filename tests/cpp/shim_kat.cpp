// shim_kat.cpp — the reference's own known-answer tests
// (/root/reference/proj/tests/kernel_test.cpp, grid_test.cpp) restated as
// plain asserts against the C++ drop-in shim (include/yeeb200/yeeblock.hpp),
// i.e. executed by the B200 kernels through the C-ABI. Catch2 is absent.
#define YEEB200_AS_YEEBLOCK
#include "yeeb200/yeeblock.hpp"

#include <cstdio>
#include <utility>
#include <cstdlib>

using namespace yeeblock;

static int failures = 0;
#define CHECK(cond)                                                      \
  do {                                                                   \
    if (!(cond)) {                                                       \
      std::fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond); \
      ++failures;                                                        \
    }                                                                    \
  } while (0)
#define CHECK_THROWS_AS(expr, T)         \
  do {                                   \
    bool caught = false;                 \
    try {                                \
      expr;                              \
    } catch (const T&) {                 \
      caught = true;                     \
    }                                    \
    CHECK(caught && #expr);              \
  } while (0)

// kernel_test.cpp:14-24 unit_grid with c*dt/h fixed (float here)
static GridSpec<float> unit_grid(int n, float cdt_over_h) {
  GridSpec<float> g;
  g.nx = g.ny = g.nz = n;
  g.dx.assign(n, 1.0f);
  g.dy.assign(n, 1.0f);
  g.dz.assign(n, 1.0f);
  g.c = 1.0f;
  g.dt = cdt_over_h;
  return g;
}

static bool identical(const FieldSet<float>& a, const FieldSet<float>& b) {
  for (Comp c : kAllComps)
    if (std::memcmp(a.field(c).data(), b.field(c).data(), a.field(c).size_bytes()) != 0) return false;
  return true;
}

int main() {
  // grid_test.cpp:7-36: build_coefficients is one division per entry
  {
    GridSpec<float> g;
    g.nx = 2;
    g.ny = 3;
    g.nz = 1;
    g.dx = {1.0f, 1.0f};
    g.dy = {0.1f, 0.2f, 0.4f};
    g.dz = {2.0f};
    g.c = 1.0f;
    g.dt = 0.5f;
    CHECK(build_coefficients(g).cdx == (std::vector<float>{0.5f, 0.5f}));
    g.dt = 1.0f;
    CHECK(build_coefficients(g).cdz == (std::vector<float>{0.5f}));
    g.dz = {-1.0f};
    CHECK_THROWS_AS(build_coefficients(g), std::invalid_argument);
  }
  // grid_test.cpp:91-97 + the pinned Courant constant
  {
    auto gf = make_uniform_grid<float>(8, 1.0f, 1.0f, 0.99);
    CHECK(static_cast<double>(gf.dt) <= stable_dt(gf, 1.0) * (1 + 1e-7));
    float s;
    const unsigned bits = 0x3f1252dbu;
    std::memcpy(&s, &bits, 4);
    CHECK(gf.dt == s);
  }
  // kernel_test.cpp:43-63 staggered extents
  {
    FieldSet<float> f({3, 4, 5});
    CHECK(f.ex.nx() == 3 && f.ex.ny() == 5 && f.ex.nz() == 6);
    CHECK(f.ey.nx() == 4 && f.ey.ny() == 4 && f.ey.nz() == 6);
    CHECK(f.ez.nx() == 4 && f.ez.ny() == 5 && f.ez.nz() == 5);
    CHECK(f.hx.nx() == 4 && f.hx.ny() == 4 && f.hx.nz() == 5);
    CHECK(f.hy.nx() == 3 && f.hy.ny() == 5 && f.hy.nz() == 5);
    CHECK(f.hz.nx() == 3 && f.hz.ny() == 4 && f.hz.nz() == 6);
  }
  const IndexBox node{{0, 5}, {0, 5}, {0, 5}};
  // kernel_test.cpp:84-106: one hz face feeds its four edges with +-0.5
  {
    Simulation<float> sim(unit_grid(4, 0.5f));
    sim.fields().hz(2, 2, 2) = 1.0f;
    sim.apply_ampere_range(node);
    const FieldSet<float>& f = sim.fields();
    CHECK(f.ex(2, 2, 2) == 0.5f);
    CHECK(f.ex(2, 3, 2) == -0.5f);
    CHECK(f.ey(2, 2, 2) == -0.5f);
    CHECK(f.ey(3, 2, 2) == 0.5f);
    int nonzero = 0;
    for (Comp c : kEComps) {
      const auto& a = f.field(c);
      for (std::size_t q = 0; q < a.size(); ++q) nonzero += a.data()[q] != 0.0f;
    }
    CHECK(nonzero == 4);
  }
  // kernel_test.cpp:108-130 faraday single-edge excitations
  {
    Simulation<float> sim(unit_grid(4, 0.5f));
    sim.fields().ey(1, 1, 2) = 1.0f;
    sim.apply_faraday_range(node);
    CHECK(sim.fields().hx(1, 1, 1) == 0.5f);
    Simulation<float> sim2(unit_grid(4, 0.5f));
    sim2.fields().ez(1, 2, 1) = 1.0f;
    sim2.apply_faraday_range(node);
    CHECK(sim2.fields().hx(1, 1, 1) == -0.5f);
  }
  // kernel_test.cpp:132-141 range ops reject out-of-bounds boxes
  {
    Simulation<float> sim(unit_grid(4, 0.5f));
    const IndexBox bad = {{0, 6}, {0, 4}, {0, 4}};
    CHECK_THROWS_AS(sim.apply_ampere_range(bad), std::out_of_range);
    CHECK_THROWS_AS(sim.apply_faraday_range(bad), std::out_of_range);
  }
  // kernel_test.cpp:143-165 PEC zeroes exactly the shell
  {
    Simulation<float> sim(unit_grid(4, 0.5f));
    for (Comp c : kEComps) sim.fields().field(c).fill(1.0f);
    sim.apply_pec_boundary();
    const FieldSet<float>& f = sim.fields();
    for (Comp c : kEComps) {
      const auto& a = f.field(c);
      const IndexBox inner = curl_updatable_box(f.dims(), c);
      for (int k = 0; k < a.nz(); ++k)
        for (int j = 0; j < a.ny(); ++j)
          for (int i = 0; i < a.nx(); ++i) CHECK(a(i, j, k) == (inner.contains(i, j, k) ? 1.0f : 0.0f));
    }
  }
  // kernel_test.cpp:181-228 soft source: increment exactly (float)(-dt*J(step*dt))
  {
    auto g = unit_grid(8, 0.5f);
    RunOptions<float> opts;
    SourceSpec s;
    s.i = s.j = s.k = 4;
    s.component = Comp::Ez;
    s.waveform = Waveform::pulse(2.0, 3.0);
    opts.sources = {s};
    Simulation<float> sim(g, opts);
    sim.fields().step_index = 7;
    // Ampere+PEC on zero fields is zero, so after one step ez(4,4,4) is the increment
    sim.run(1);
    CHECK(sim.fields().ez(4, 4, 4) == static_cast<float>(-0.5 * s.waveform.value(7 * 0.5)));
    SourceSpec bad = s;
    bad.j = 0;
    CHECK_THROWS_AS(bad.validate(g.dims()), std::invalid_argument);
    RunOptions<float> o2;
    o2.sources = {bad};
    CHECK_THROWS_AS(Simulation<float>(g, o2), std::invalid_argument);
  }
  // kernel_test.cpp:230-258 probes fire on the stride and read exact values
  {
    auto g = unit_grid(8, 0.5f);
    RunOptions<float> opts;
    opts.probes = {{4, 4, 4, Comp::Ez, 2}, {1, 1, 1, Comp::Hx, 3}};
    SourceSpec s;
    s.i = s.j = s.k = 4;
    s.component = Comp::Ez;
    s.waveform = Waveform::pulse(1.0, 2.0);
    opts.sources = {s};
    Simulation<float> sim(g, opts);
    auto recs = sim.run(6);
    int at6 = 0;
    for (auto& r : recs) at6 += r.step == 6;
    CHECK(recs.size() == 5 && at6 == 2);  // probe 0 at 2,4,6; probe 1 at 3,6
  }
  // kernel_test.cpp:289-298 digest distinguishes any bit flip
  {
    FieldSet<float> a({4, 4, 4}), b({4, 4, 4});
    CHECK(field_digest(a) == field_digest(b));
    b.hy(1, 2, 3) = -0.0f;
    CHECK(field_digest(a) != field_digest(b));
  }
  // run_simulation == step_standard x n == Simulation::run (bit-exact)
  {
    auto g = make_uniform_grid<float>(12, 1.0f, 1.0f, 0.99);
    FieldSet<float> f(g.dims());
    for (Comp c : kAllComps)
      for (std::size_t q = 0; q < f.field(c).size(); ++q)
        f.field(c).data()[q] = std::sin(0.37f * q + comp_index(c));
    FieldSet<float> a = f, b = f;
    run_simulation(g, 5, a);
    const auto co = build_coefficients(g);
    for (int t = 0; t < 5; ++t) step_standard(g, b, co);
    CHECK(identical(a, b));
    CHECK(a.step_index == 5 && b.step_index == 5);
    CHECK(field_digest_hex(a) == field_digest_hex(b));
  }
  // kernel_test.cpp:265-283 total_energy KATs, on the device
  {
    auto g = unit_grid(4, 0.5f);
    Simulation<float> sim(g);
    sim.snapshot_h();
    CHECK(sim.total_energy() == 0.0);
    sim.fields().ez(2, 2, 1) = 2.0f;
    CHECK(sim.total_energy() == 4.0);
    sim.fields().zero();
    sim.fields().hx(2, 1, 1) = 3.0f;
    sim.snapshot_h();
    sim.fields().hx(2, 1, 1) = 0.5f;
    CHECK(sim.total_energy() == 1.5);
  }
  // RunOptions::Readback (extension): the host FieldSet after run() is the same whether it is read
  // back lazily (first fields() access), eagerly inside run() (the streamed readback into this
  // pageable storage) or by the Auto policy — across consecutive runs, with and without a look at
  // the fields in between, and after host-side writes.
  {
    GridSpec<float> g;
    g.nx = 96, g.ny = 40, g.nz = 24;
    g.dx.assign(g.nx, 1.0f), g.dy.assign(g.ny, 1.0f), g.dz.assign(g.nz, 1.0f);
    g.dt = static_cast<float>(stable_dt(g, 0.99));
    FieldSet<float> init(g.dims());
    for (Comp c : kAllComps)
      for (std::size_t q = 0; q < init.field(c).size(); ++q)
        init.field(c).data()[q] = std::sin(0.11f * q + comp_index(c));
    using RB = RunOptions<float>::Readback;
    std::string digest[3][3];
    int p = 0;
    for (RB mode : {RB::Lazy, RB::Eager, RB::Auto}) {
      RunOptions<float> o;
      o.quiescent_skip = false;
      o.readback = mode;
      Simulation<float> sim(g, o);
      sim.fields() = init;
      sim.run(70);
      digest[p][0] = field_digest_hex(std::as_const(sim).fields());
      sim.run(66);  // no look at the fields after this one ...
      sim.run(64);  // ... so Auto stops reading back eagerly here
      digest[p][1] = field_digest_hex(std::as_const(sim).fields());
      sim.fields().ez(5, 6, 7) += 1.0f;  // host-side write: uploaded by the next run
      sim.run(65);
      digest[p][2] = field_digest_hex(std::as_const(sim).fields());
      CHECK(std::as_const(sim).fields().step_index == 70 + 66 + 64 + 65);
      ++p;
    }
    for (int q = 0; q < 3; ++q) {
      CHECK(digest[0][q] == digest[1][q]);
      CHECK(digest[0][q] == digest[2][q]);
    }
    CHECK(digest[0][0] != digest[0][1]);
  }
  if (failures) {
    std::fprintf(stderr, "%d failure(s)\n", failures);
    return 1;
  }
  std::printf("shim KATs ok\n");
  return 0;
}
