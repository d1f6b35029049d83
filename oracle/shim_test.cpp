// shim_test.cpp -- TEST INFRASTRUCTURE: drives include/sgweno_gpu.hpp (the C++
// drop-in over libsgwg.so) side by side with the unmodified reference on the
// same CombinationSet, through the reference's own public API:
// make_family + initialize_family, then sgweno::evolve_family / combine on one
// copy and sgweno::gpu::evolve_family / combine on the other.  Built by
// oracle/Makefile into oracle/_ref/shim_test (needs the reference headers at
// build time; runs on the GPU box).  Exit 0 iff bitwise equal.
#include <cstdio>
#include <cstring>
#include <numbers>

#include "sgweno/io.hpp"
#include "sgweno/runner.hpp"
#include "sgweno_gpu.hpp"

using namespace sgweno;

static bool same(const std::vector<double>& a, const std::vector<double>& b) {
  return a.size() == b.size() && std::memcmp(a.data(), b.data(), a.size() * 8) == 0;
}

int main() {
  using std::numbers::pi;
  int bad = 0;
  // BASELINE C2 family at reduced level: 2D Burgers, CFL 0.5, stop at 0.02
  {
    ProblemSpec spec;
    spec.kind = ModelKind::burgers;
    spec.box = DomainBox::cube(0.0, 2.0, 2);
    spec.boundary.assign(2, BoundaryKind::periodic);
    spec.law = {ModelKind::burgers, {}};
    spec.initial = [](std::span<const double> x) { return 0.5 + std::sin(pi * (x[0] + x[1])); };
    CombinationSet ref = make_family(spec.box, {16, 16}, spec.boundary, 4);
    initialize_family(ref, spec);
    CombinationSet dev = ref;
    StepPolicy pol;
    pol.mode = DtMode::cfl;
    pol.cfl_number = 0.5;
    const WenoParams wp{1e-6, WenoMode::nonlinear};
    FamilyModel model(spec, ref, wp, 1);
    std::vector<GridField> ref_stops, dev_stops;
    auto dts_ref = evolve_family(ref, model, pol, 0.05, {0.02}, [&](double) {
      ref_stops.push_back(combine(ref, InterpMode::weno, 1e-6));
    });
    auto dts_dev = gpu::evolve_family(dev, spec, wp, pol, 0.05, {0.02}, [&](double) {
      dev_stops.push_back(gpu::combine(dev, InterpMode::weno, 1e-6));
    });
    bool ok = same(dts_ref, dts_dev) && ref_stops.size() == 2 && dev_stops.size() == 2;
    for (size_t m = 0; ok && m < ref.members.size(); ++m)
      ok = same(ref.members[m].state, dev.members[m].state);
    for (size_t s = 0; ok && s < 2; ++s) ok = same(ref_stops[s].values, dev_stops[s].values);
    std::printf("C2-family (N_L=4) Burgers via shim: %zu steps, bitwise %s\n", dts_dev.size(),
                ok ? "EQUAL" : "DIFFERENT");
    bad += !ok;
  }
  // 3D advection (BASELINE C3 shape, reduced), accuracy-mode dt
  {
    ProblemSpec spec;
    spec.kind = ModelKind::advection;
    spec.box = DomainBox::cube(0.0, 2.0, 3);
    spec.boundary.assign(3, BoundaryKind::periodic);
    spec.law = {ModelKind::advection, {1.0, 1.0, 1.0}};
    spec.initial = [](std::span<const double> x) { return std::sin(pi * (x[0] + x[1] + x[2])); };
    CombinationSet ref = make_family(spec.box, {8, 8, 8}, spec.boundary, 3);
    initialize_family(ref, spec);
    CombinationSet dev = ref;
    StepPolicy pol;
    pol.mode = DtMode::accuracy;
    pol.reference_spacing = 2.0 / 64;
    const WenoParams wp{1e-6, WenoMode::nonlinear};
    FamilyModel model(spec, ref, wp, 1);
    auto dts_ref = evolve_family(ref, model, pol, 0.01);
    auto dts_dev = gpu::evolve_family(dev, spec, wp, pol, 0.01);
    bool ok = same(dts_ref, dts_dev);
    for (size_t m = 0; ok && m < ref.members.size(); ++m)
      ok = same(ref.members[m].state, dev.members[m].state);
    ok = ok && same(combine(ref, InterpMode::weno, 1e-6).values,
                    gpu::combine(dev, InterpMode::weno, 1e-6).values);
    std::printf("3D advection (N_L=3) via shim: %zu steps, bitwise %s\n", dts_dev.size(),
                ok ? "EQUAL" : "DIFFERENT");
    bad += !ok;
  }
  // reduced Vlasov-Maxwell (paper ex6 at reduced size): states carry E1, E2, B3
  {
    ExampleDefaults ex = make_example(ExampleId::ex6);
    const ProblemSpec& spec = ex.problem;
    CombinationSet ref = make_family(spec.box, {8, 8, 8}, spec.boundary, 2);
    initialize_family(ref, spec);
    CombinationSet dev = ref;
    StepPolicy pol;
    pol.mode = DtMode::cfl;
    pol.cfl_number = 0.4;
    const WenoParams wp{1e-6, WenoMode::nonlinear};
    FamilyModel model(spec, ref, wp, 1);
    auto dts_ref = evolve_family(ref, model, pol, 0.5, {0.2});
    auto dts_dev = gpu::evolve_family(dev, spec, wp, pol, 0.5, {0.2});
    bool ok = same(dts_ref, dts_dev) && !dts_dev.empty();
    for (size_t m = 0; ok && m < ref.members.size(); ++m)
      ok = same(ref.members[m].state, dev.members[m].state);
    ok = ok && same(combine(ref, InterpMode::weno, 1e-6).values,
                    gpu::combine(dev, InterpMode::weno, 1e-6).values);
    std::printf("Vlasov-Maxwell (ex6, N_L=2) via shim: %zu steps, bitwise %s\n", dts_dev.size(),
                ok ? "EQUAL" : "DIFFERENT");
    bad += !ok;
  }
  // runner outputs from the device: quadrature_mass / field_min / field_max of
  // the combination, and the SGW5 dump read back with read_field_dump
  {
    ExampleDefaults ex = make_example(ExampleId::ex1);
    CombinationSet set = make_family(ex.problem.box, {10, 10}, ex.problem.boundary, 3);
    initialize_family(set, ex.problem);
    GridField f = combine(set, InterpMode::lagrange, 1e-6);
    const sgwg_field_stats st = gpu::combined_stats(set, InterpMode::lagrange, 1e-6);
    const double mass = quadrature_mass(f);
    bool ok = st.min == detail::field_min(f) && st.max == detail::field_max(f) &&
              std::abs(st.mass - mass) <= 1e-13 * std::abs(mass);
    const std::string path = "/tmp/sgwg_shim_snapshot.sgw5";
    gpu::write_field_dump(path, set, InterpMode::lagrange, 1e-6);
    const FieldDump d = read_field_dump(path);
    ok = ok && same(d.values, f.values) && d.extents[0] == f.geom.points[0];
    std::printf("runner outputs via shim (stats, SGW5 dump): %s\n", ok ? "EQUAL" : "DIFFERENT");
    bad += !ok;
  }
  // failure propagation: FamilyIntegratorFailure{level, step, stage}
  {
    ProblemSpec spec;
    spec.kind = ModelKind::burgers;
    spec.box = DomainBox::cube(0.0, 2.0, 2);
    spec.boundary.assign(2, BoundaryKind::periodic);
    spec.law = {ModelKind::burgers, {}};
    spec.initial = [](std::span<const double> x) { return 1e150 * std::sin(pi * x[0]); };
    CombinationSet ref = make_family(spec.box, {8, 8}, spec.boundary, 2);
    initialize_family(ref, spec);
    CombinationSet dev = ref;
    StepPolicy pol;
    pol.mode = DtMode::cfl;
    pol.cfl_number = 0.5;
    const WenoParams wp{};
    FamilyModel model(spec, ref, wp, 1);
    LevelIndex lr, ld;
    long long sr = -1, sd = -2;
    int gr = -1, gd = -2;
    try {
      evolve_family(ref, model, pol, 0.01);
    } catch (const FamilyIntegratorFailure& e) {
      lr = e.level, sr = e.step, gr = e.stage;
    }
    try {
      gpu::evolve_family(dev, spec, wp, pol, 0.01);
    } catch (const FamilyIntegratorFailure& e) {
      ld = e.level, sd = e.step, gd = e.stage;
    }
    const bool ok = (lr == ld) && sr == sd && gr == gd && sr >= 0;
    std::printf("failure propagation: reference (step %lld, stage %d), gpu (step %lld, stage %d) %s\n",
                sr, gr, sd, gd, ok ? "EQUAL" : "DIFFERENT");
    bad += !ok;
  }
  return bad == 0 ? 0 : 1;
}
