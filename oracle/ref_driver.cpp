// ref_driver.cpp -- thin extern "C" driver over the UNMODIFIED reference headers
// (/root/reference/proj/include/sgweno/*.hpp, included in place, never copied).
//
// TEST INFRASTRUCTURE ONLY.  Built by oracle/Makefile into oracle/_ref/libsgwref.so
// (git-ignored, travels to the GPU box with the snapshot).  Used to pin the C
// restatement (oracle/sgw_oracle.c), to generate tests/golden/ fixtures, and as
// bench.py's CPU baseline ("kind": "reference").  It contains no algorithm of
// its own: every entry point calls the reference's public API:
//   make_family (combine.hpp:69-83), initialize_family (models.hpp:855-871),
//   FamilyModel (models.hpp:754-851), evolve_family (timestep.hpp:126-174),
//   combine (combine.hpp:95-122), prolong (interp.hpp:197-250),
//   conservation_law_rhs_into (models.hpp:184-198), vb_rhs_into (334-363),
//   weno_derivative_line / advect_derivative_line (weno.hpp:118-192).
// The only glue is evolve_scaled(): the BASELINE C1 dt rule 0.5*h^(5/3) has
// no StepPolicy slot, so it replays evolve_family's control flow
// with that dt; with scale == 1 it is checked bitwise against evolve_family.
#include <chrono>
#include <cmath>
#include <cstring>
#include <numbers>
#include <vector>

#include "sgw_oracle.h"  // struct layouts only (sgwo_domain/model/policy)
#include "sgweno/combine.hpp"
#include "sgweno/interp.hpp"
#include "sgweno/models.hpp"
#include "sgweno/timestep.hpp"
#include "sgweno/weno.hpp"

using namespace sgweno;

namespace {

DomainBox box_of(const sgwo_domain* d) {
  return DomainBox::make(std::vector<double>(d->lower, d->lower + d->d),
                         std::vector<double>(d->upper, d->upper + d->d));
}
std::vector<BoundaryKind> bc_of(const sgwo_domain* d) {
  std::vector<BoundaryKind> b;
  for (int k = 0; k < d->d; ++k)
    b.push_back(d->bc[k] == SGWO_ZERO ? BoundaryKind::zero : BoundaryKind::periodic);
  return b;
}
std::vector<int> root_of(const sgwo_domain* d) {
  return std::vector<int>(d->root_cells, d->root_cells + d->d);
}

double preset_value(int preset, std::span<const double> x) {
  using std::numbers::pi;
  switch (preset) {
    case SGWO_IC_C1: return std::sin(pi * (x[0] + x[1]));
    case SGWO_IC_C2: return 0.5 + std::sin(pi * (x[0] + x[1]));
    case SGWO_IC_C3: return std::sin(pi * (x[0] + x[1] + x[2]));
    case SGWO_IC_C4:
      return (1.0 + 0.01 * std::cos(0.5 * x[0])) / std::sqrt(2.0 * pi) *
             std::exp(-0.5 * (x[1] * x[1]));
    case SGWO_IC_C5:
      return (1.0 + 0.05 * (std::cos(0.5 * x[0]) + std::cos(0.5 * x[1]))) / (2.0 * pi) *
             std::exp(-0.5 * (x[2] * x[2] + x[3] * x[3]));
    default: break;
  }
  return 0.0;
}

ProblemSpec make_spec(const sgwo_domain* d, const sgwo_model* m, int preset) {
  ProblemSpec p;
  p.box = box_of(d);
  p.boundary = bc_of(d);
  switch (m->kind) {
    case SGWO_ADVECTION:
      p.kind = ModelKind::advection;
      p.law = {ModelKind::advection, std::vector<double>(m->speeds, m->speeds + d->d)};
      break;
    case SGWO_BURGERS:
      p.kind = ModelKind::burgers;
      p.law = {ModelKind::burgers, {}};
      break;
    case SGWO_VLASOV_MAXWELL:
      p.kind = ModelKind::vlasov_maxwell;
      p.vm = VlasovMaxwellSpec{};
      p.init_b3 = make_example(ExampleId::ex6).problem.init_b3;
      break;
    default:
      p.kind = ModelKind::vlasov_boltzmann;
      p.vb = VlasovBoltzmannSpec{m->space_dim, m->theta, m->tau};
      break;
  }
  // presets that exist in the reference are taken from make_example verbatim
  switch (preset) {
    case SGWO_IC_EX1: p.initial = make_example(ExampleId::ex1).problem.initial; break;
    case SGWO_IC_EX2: p.initial = make_example(ExampleId::ex2).problem.initial; break;
    case SGWO_IC_EX3: p.initial = make_example(ExampleId::ex3a).problem.initial; break;
    case SGWO_IC_EX5A:
      p.initial = make_example(ExampleId::ex5a).problem.initial;
      p.normalize_initial_mass = true;
      break;
    case SGWO_IC_EX5B:
      p.initial = make_example(ExampleId::ex5b).problem.initial;
      p.normalize_initial_mass = true;
      break;
    case SGWO_IC_EX6: p.initial = make_example(ExampleId::ex6).problem.initial; break;
    default: p.initial = [preset](std::span<const double> x) { return preset_value(preset, x); };
  }
  return p;
}

WenoParams weno_of(const sgwo_model* m) {
  return WenoParams{m->epsilon, m->weno_mode == SGWO_WENO_LINEAR ? WenoMode::linear
                                                                 : WenoMode::nonlinear};
}
InterpMode interp_of(int mode) {
  return mode == SGWO_INTERP_LAGRANGE ? InterpMode::lagrange : InterpMode::weno;
}

CombinationSet family_of(const sgwo_domain* d) {
  return make_family(box_of(d), root_of(d), bc_of(d), d->nl);
}
// member states sized for the model (Vlasov-Maxwell: f + E1, E2, B3 lines)
CombinationSet family_of(const sgwo_domain* d, const sgwo_model* m) {
  CombinationSet set = family_of(d);
  if (m->kind == SGWO_VLASOV_MAXWELL)
    for (auto& mm : set.members)
      mm.state.assign(mm.geom.total_points() + 3 * static_cast<std::size_t>(mm.geom.points[0]), 0.0);
  return set;
}

void load_states(CombinationSet& set, const double* states) {
  std::size_t off = 0;
  for (auto& m : set.members) {
    std::memcpy(m.state.data(), states + off, sizeof(double) * m.state.size());
    off += m.state.size();
  }
}
void store_states(const CombinationSet& set, double* states) {
  std::size_t off = 0;
  for (auto& m : set.members) {
    std::memcpy(states + off, m.state.data(), sizeof(double) * m.state.size());
    off += m.state.size();
  }
}

// evolve_family (timestep.hpp:126-174) control flow with dt = scale * pow(h, 5/3).
template <class Model>
std::vector<double> evolve_scaled(CombinationSet& set, Model& model, const StepPolicy& policy,
                                  double scale, double tfinal, std::vector<double> stops,
                                  const std::function<void(double)>& on_stop) {
  const GridGeometry finest = finest_geometry(set);
  const double eps_dedupe = 1e-12 * std::max(1.0, tfinal);
  stops.push_back(tfinal);
  std::sort(stops.begin(), stops.end());
  stops.erase(std::remove_if(stops.begin(), stops.end(),
                             [&](double s) { return s <= 0.0 || s > tfinal + eps_dedupe; }),
              stops.end());
  stops.erase(std::unique(stops.begin(), stops.end(),
                          [&](double a, double b) { return std::abs(a - b) <= eps_dedupe; }),
              stops.end());
  if (stops.empty()) stops.push_back(tfinal);
  std::vector<SspRk3> rk(set.members.size());
  std::vector<double> dts;
  double t = 0.0;
  long long step_index = 0;
  const double eps_t = 1e-12 * std::max(1.0, tfinal);
  for (double stop : stops) {
    if (stop > tfinal + eps_t) break;
    while (stop - t > eps_t) {
      const auto speeds = model.family_wave_speeds();
      double dt = compute_dt(policy, speeds, finest.spacing, stop - t);
      if (policy.mode == DtMode::accuracy) dt = std::min(scale * std::pow(policy.reference_spacing, 5.0 / 3.0), stop - t);
      if (stop - (t + dt) <= eps_t) dt = stop - t;
      for (std::size_t mi = 0; mi < set.members.size(); ++mi) {
        auto& member = set.members[mi];
        try {
          rk[mi].step(member.state, [&](const std::vector<double>& s, std::vector<double>& k) {
            model.rhs(mi, s, k);
          }, dt);
        } catch (const IntegratorFailure& e) {
          throw FamilyIntegratorFailure(member.geom.level, step_index, e.stage);
        }
      }
      t += dt;
      dts.push_back(dt);
      ++step_index;
    }
    t = stop;
    if (on_stop) on_stop(t);
  }
  return dts;
}

}  // namespace

extern "C" {

int sgwref_enumerate_levels(int d, int nl, int* out, int cap) {
  try {
    auto lv = enumerate_combination_levels(d, nl);
    std::sort(lv.begin(), lv.end());
    int n = static_cast<int>(lv.size());
    for (int i = 0; i < n && i < cap; ++i)
      for (int k = 0; k < d; ++k) out[i * d + k] = lv[i].levels[k];
    return n;
  } catch (...) {
    return -1;
  }
}

double sgwref_weno5_flux_positive(const double* s, double eps, int mode) {
  return weno5_flux_positive({s[0], s[1], s[2], s[3], s[4]},
                             WenoParams{eps, mode == SGWO_WENO_LINEAR ? WenoMode::linear
                                                                      : WenoMode::nonlinear});
}

// flux_kind 0: advect_derivative_line(c); 1: Burgers generic; 2: c*u generic with alpha.
int sgwref_weno_derivative_line(const double* u, int n, int flux_kind, double c, double alpha,
                                double dx, int bc, double eps, int mode, double* out) {
  try {
    WenoParams p{eps, mode == SGWO_WENO_LINEAR ? WenoMode::linear : WenoMode::nonlinear};
    BoundaryKind b = bc == SGWO_ZERO ? BoundaryKind::zero : BoundaryKind::periodic;
    std::span<const double> us(u, n);
    std::span<double> os(out, n);
    if (flux_kind == 0)
      advect_derivative_line(us, c, dx, b, p, os);
    else if (flux_kind == 1)
      weno_derivative_line(us, [](double v) { return 0.5 * v * v; }, alpha, dx, b, p, os);
    else
      weno_derivative_line(us, [c](double v) { return c * v; }, alpha, dx, b, p, os);
    return 0;
  } catch (...) {
    return SGWO_EINVAL;
  }
}

int sgwref_rhs(const sgwo_domain* dom, const int* level, const sgwo_model* m, const double* state,
               double* out) {
  try {
    auto g = GridGeometry::make(box_of(dom), LevelIndex{std::vector<int>(level, level + dom->d)},
                                root_of(dom), bc_of(dom));
    const std::size_t n = g.total_points();
    std::span<const double> s(state, n);
    std::span<double> o(out, n);
    if (m->kind == SGWO_ADVECTION || m->kind == SGWO_BURGERS) {
      ScalarConservationLaw law{m->kind == SGWO_BURGERS ? ModelKind::burgers : ModelKind::advection,
                                std::vector<double>(m->speeds, m->speeds + dom->d)};
      conservation_law_rhs_into(g, s, law, weno_of(m), 1, o);
    } else if (m->kind == SGWO_VLASOV_BOLTZMANN) {
      VlasovBoltzmannSpec vb{m->space_dim, m->theta, m->tau};
      auto ws = VbWorkspace::make(g, vb);
      vb_rhs_into(g, ws, s, vb, weno_of(m), 1, o);
    } else if (m->kind == SGWO_VLASOV_MAXWELL) {
      VlasovMaxwellSpec vm{};
      auto ws = VmWorkspace::make(g, vm);
      vm_rhs_into(g, ws, std::span<const double>(state, ws.state_size()), vm, weno_of(m), 1,
                  std::span<double>(out, ws.state_size()));
    } else {
      return SGWO_EINVAL;  // Vlasov-Poisson has no reference implementation
    }
    return 0;
  } catch (...) {
    return SGWO_EINVAL;
  }
}

int sgwref_upsample_line(const double* src, int n_src, double* dst, int n_dst, int m, int bc,
                         int mode, double eps) {
  try {
    auto tab = detail::OffsetTable::make(m, interp_of(mode));
    detail::upsample_line(std::span<const double>(src, n_src), std::span<double>(dst, n_dst), tab,
                          bc == SGWO_ZERO ? BoundaryKind::zero : BoundaryKind::periodic,
                          interp_of(mode), eps);
    return 0;
  } catch (...) {
    return SGWO_EINVAL;
  }
}

int sgwref_prolong(const sgwo_domain* dom, const int* level, const double* src, int mode,
                   double eps, double* dst) {
  try {
    GridField f;
    f.geom = GridGeometry::make(box_of(dom), LevelIndex{std::vector<int>(level, level + dom->d)},
                                root_of(dom), bc_of(dom));
    f.values.assign(src, src + f.geom.total_points());
    GridField p = prolong(f, dom->nl, interp_of(mode), eps);
    std::memcpy(dst, p.values.data(), sizeof(double) * p.values.size());
    return 0;
  } catch (...) {
    return SGWO_EINVAL;
  }
}

int sgwref_combine(const sgwo_domain* dom, const double* states, int mode, double eps, double* out,
                   int threads) {
  try {
    CombinationSet set = family_of(dom);
    load_states(set, states);
    GridField acc = combine(set, interp_of(mode), eps, threads);
    std::memcpy(out, acc.values.data(), sizeof(double) * acc.values.size());
    return 0;
  } catch (...) {
    return SGWO_EINVAL;
  }
}

int sgwref_init_family(int preset, const sgwo_domain* dom, const sgwo_model* m, double* states) {
  try {
    CombinationSet set = family_of(dom);
    ProblemSpec spec = make_spec(dom, m, preset);
    initialize_family(set, spec);
    store_states(set, states);
    return 0;
  } catch (...) {
    return SGWO_EINVAL;
  }
}

typedef void (*sgwref_stop_cb)(double t, const double* states, void* user);

// evolve_family over caller-supplied member states (packed in sorted member
// order).  cb (may be NULL) sees the packed states at every stop.  Timing of
// the evolve loop (including callbacks) is returned in *seconds.
int sgwref_evolve(const sgwo_domain* dom, const sgwo_model* m, const sgwo_policy* pol,
                  double* states, double tfinal, const double* stops, int nstops,
                  sgwref_stop_cb cb, void* user, int threads, double* dts, long cap, long* nsteps,
                  int* fail_member, long* fail_step, int* fail_stage, double* seconds) {
  try {
    CombinationSet set = family_of(dom, m);
    load_states(set, states);
    ProblemSpec spec = make_spec(dom, m, -1);
    FamilyModel model(spec, set, weno_of(m), threads);
    StepPolicy policy;
    policy.mode = pol->mode == SGWO_DT_CFL ? DtMode::cfl : DtMode::accuracy;
    policy.cfl_number = pol->cfl;
    policy.reference_spacing = pol->reference_spacing;
    std::vector<double> st(stops, stops + nstops);
    std::vector<double> packed(states, states + 0);
    auto on_stop = [&](double t) {
      if (!cb) return;
      std::vector<double> tmp;
      std::size_t tot = 0;
      for (auto& mm : set.members) tot += mm.state.size();
      tmp.resize(tot);
      store_states(set, tmp.data());
      cb(t, tmp.data(), user);
    };
    const auto t0 = std::chrono::steady_clock::now();
    std::vector<double> d;
    int status = 0;
    try {
      if (pol->mode == SGWO_DT_ACCURACY && pol->dt_scale != 1.0)
        d = evolve_scaled(set, model, policy, pol->dt_scale, tfinal, st, on_stop);
      else
        d = evolve_family(set, model, policy, tfinal, st, on_stop);
    } catch (const FamilyIntegratorFailure& e) {
      status = SGWO_ENONFINITE;
      for (std::size_t i = 0; i < set.members.size(); ++i)
        if (set.members[i].geom.level == e.level && fail_member) *fail_member = static_cast<int>(i);
      if (fail_step) *fail_step = e.step;
      if (fail_stage) *fail_stage = e.stage;
    }
    const auto t1 = std::chrono::steady_clock::now();
    if (seconds) *seconds = std::chrono::duration<double>(t1 - t0).count();
    store_states(set, states);
    if (nsteps) *nsteps = static_cast<long>(d.size());
    for (std::size_t i = 0; i < d.size() && static_cast<long>(i) < cap; ++i) dts[i] = d[i];
    return status;
  } catch (...) {
    return SGWO_EINVAL;
  }
}

// Same as sgwref_evolve but forcing the replayed loop (checks evolve_scaled
// against evolve_family bitwise when scale == 1).
int sgwref_evolve_replay(const sgwo_domain* dom, const sgwo_model* m, const sgwo_policy* pol,
                         double* states, double tfinal, const double* stops, int nstops,
                         double* dts, long cap, long* nsteps) {
  try {
    CombinationSet set = family_of(dom, m);
    load_states(set, states);
    ProblemSpec spec = make_spec(dom, m, -1);
    FamilyModel model(spec, set, weno_of(m), 1);
    StepPolicy policy;
    policy.mode = pol->mode == SGWO_DT_CFL ? DtMode::cfl : DtMode::accuracy;
    policy.cfl_number = pol->cfl;
    policy.reference_spacing = pol->reference_spacing;
    auto d = evolve_scaled(set, model, policy, pol->dt_scale, tfinal,
                           std::vector<double>(stops, stops + nstops), nullptr);
    store_states(set, states);
    if (nsteps) *nsteps = static_cast<long>(d.size());
    for (std::size_t i = 0; i < d.size() && static_cast<long>(i) < cap; ++i) dts[i] = d[i];
    return 0;
  } catch (...) {
    return SGWO_EINVAL;
  }
}

// Timed CPU baseline: evolve `nsteps_max` lockstep steps (or to tfinal) of a
// preset family with the reference threads setting, returning evolve seconds.
int sgwref_time_prefix(const sgwo_domain* dom, const sgwo_model* m, const sgwo_policy* pol,
                       int preset, double tfinal, int threads, double* seconds, long* nsteps,
                       double* combine_seconds, int interp_mode) {
  try {
    CombinationSet set = family_of(dom);
    ProblemSpec spec = make_spec(dom, m, preset);
    initialize_family(set, spec);
    FamilyModel model(spec, set, weno_of(m), threads);
    StepPolicy policy;
    policy.mode = pol->mode == SGWO_DT_CFL ? DtMode::cfl : DtMode::accuracy;
    policy.cfl_number = pol->cfl;
    policy.reference_spacing = pol->reference_spacing;
    const auto t0 = std::chrono::steady_clock::now();
    std::vector<double> d;
    if (pol->mode == SGWO_DT_ACCURACY && pol->dt_scale != 1.0)
      d = evolve_scaled(set, model, policy, pol->dt_scale, tfinal, {}, nullptr);
    else
      d = evolve_family(set, model, policy, tfinal, {}, nullptr);
    const auto t1 = std::chrono::steady_clock::now();
    *seconds = std::chrono::duration<double>(t1 - t0).count();
    *nsteps = static_cast<long>(d.size());
    if (combine_seconds) {
      const auto c0 = std::chrono::steady_clock::now();
      GridField acc = combine(set, interp_of(interp_mode), m->epsilon, threads);
      const auto c1 = std::chrono::steady_clock::now();
      *combine_seconds = std::chrono::duration<double>(c1 - c0).count();
      (void)acc;
    }
    return 0;
  } catch (...) {
    return SGWO_EINVAL;
  }
}

}  // extern "C"
