// sgweno_gpu.hpp -- header-only C++ shim with the reference's signatures over
// the C ABI (include/sgwg.h).  A maintainer of the reference adds this header
// next to proj/include/sgweno/ and links libsgwg.so; call sites switch from
// sgweno::evolve_family / sgweno::combine to sgweno::gpu::evolve_family /
// sgweno::gpu::combine with unchanged arguments and semantics:
//
//   evolve_family  timestep.hpp:126-174   (stop list, exact landing, on_stop,
//                                           returns the dt sequence, throws
//                                           FamilyIntegratorFailure{level,step,stage})
//   combine        combine.hpp:95-122     (returns the finest-grid GridField)
//   prolong        interp.hpp:197-250
//
// The model is taken from the ProblemSpec + WenoParams that the reference's
// FamilyModel (models.hpp:754-851) is constructed from.  Member states stay in
// the host CombinationSet between calls (uploaded at entry, downloaded before
// every on_stop and at exit), exactly the reference's ownership.
#pragma once

#include <cstring>
#include <functional>
#include <stdexcept>
#include <string>
#include <vector>

#include "sgweno/combine.hpp"
#include "sgweno/models.hpp"
#include "sgweno/timestep.hpp"
#include "sgwg.h"

namespace sgweno::gpu {

struct Error : std::runtime_error {
  int status;
  Error(int s, const std::string& m) : std::runtime_error(m), status(s) {}
};

inline void check(int st) {
  if (st == SGWG_OK) return;
  const std::string msg = sgwg_last_error();
  if (st == SGWG_EINVAL) throw std::invalid_argument(msg);
  throw Error(st, msg);
}

// One device per process; arith = SGWG_ARITH_EXACT reproduces the reference
// bit for bit, SGWG_ARITH_FAST is the throughput build (<= 1e-10).
class Device {
 public:
  explicit Device(int device = 0, int arith = SGWG_ARITH_EXACT) {
    check(sgwg_init(device, &ctx_));
    check(sgwg_set_arith(ctx_, arith));
  }
  ~Device() { sgwg_shutdown(ctx_); }
  Device(const Device&) = delete;
  Device& operator=(const Device&) = delete;
  sgwg_ctx* get() const { return ctx_; }

 private:
  sgwg_ctx* ctx_ = nullptr;
};

inline Device& default_device() {
  static Device d(0, SGWG_ARITH_EXACT);
  return d;
}

namespace detail {

inline sgwg_domain domain_of(const CombinationSet& set) {
  if (set.members.empty()) throw std::invalid_argument("empty family");
  const GridGeometry& g = set.members.front().geom;
  sgwg_domain d{};
  d.d = g.dim();
  d.nl = set.finest_level;
  for (int k = 0; k < d.d; ++k) {
    d.lower[k] = g.box.lower[k];
    d.upper[k] = g.box.upper[k];
    d.root_cells[k] = g.root_cells[k];
    d.bc[k] = (g.boundary[k] == BoundaryKind::zero) ? SGWG_ZERO : SGWG_PERIODIC;
  }
  return d;
}

inline sgwg_model model_of(const ProblemSpec& spec, const WenoParams& p) {
  sgwg_model m{};
  m.epsilon = p.epsilon;
  m.weno_mode = (p.mode == WenoMode::linear) ? SGWG_WENO_LINEAR : SGWG_WENO_NONLINEAR;
  switch (spec.kind) {
    case ModelKind::advection:
      m.kind = SGWG_ADVECTION;
      for (size_t k = 0; k < spec.law.speeds.size() && k < SGWG_MAXD; ++k)
        m.speeds[k] = spec.law.speeds[k];
      break;
    case ModelKind::burgers: m.kind = SGWG_BURGERS; break;
    case ModelKind::vlasov_boltzmann:
      m.kind = SGWG_VLASOV_BOLTZMANN;
      m.space_dim = spec.vb.space_dim;
      m.theta = spec.vb.theta;
      m.tau = spec.vb.tau;
      break;
    case ModelKind::vlasov_maxwell: m.kind = SGWG_VLASOV_MAXWELL; break;
    default: throw std::invalid_argument("model not on the B200 path");
  }
  return m;
}

// RAII device family mirroring a host CombinationSet
// (member states are the reference's: the grid field followed by any model
// state -- the Vlasov-Maxwell field lines -- once the model is set)
class Family {
 public:
  Family(sgwg_ctx* ctx, const CombinationSet& set) {
    const sgwg_domain d = domain_of(set);
    check(sgwg_family_create(ctx, &d, &fam_));
    check(sgwg_family_sizes(fam_, &npts_, &nfine_));
  }
  ~Family() { sgwg_family_destroy(fam_); }
  void set_model(const sgwg_model& m) {
    check(sgwg_set_model(fam_, &m));
    check(sgwg_family_sizes(fam_, &npts_, &nfine_));
  }
  // whole member states when the device family carries the model state, the
  // grid fields only otherwise (e.g. a combination of Vlasov-Maxwell states)
  bool whole(const CombinationSet& set) const {
    size_t field = 0, state = 0;
    for (const auto& m : set.members) {
      field += m.field_size();
      state += m.state.size();
    }
    if (npts_ == state) return true;
    if (npts_ == field) return false;
    throw std::invalid_argument("member states do not match the device family");
  }
  void upload(const CombinationSet& set) {
    const bool all = whole(set);
    std::vector<double> buf;
    buf.reserve(npts_);
    for (const auto& m : set.members)
      buf.insert(buf.end(), m.state.begin(),
                 all ? m.state.end() : m.state.begin() + m.field_size());
    check(sgwg_family_upload(fam_, buf.data(), buf.size()));
  }
  void download(CombinationSet& set) const {
    const bool all = whole(set);
    std::vector<double> buf(npts_);
    check(sgwg_family_download(fam_, buf.data(), buf.size()));
    size_t off = 0;
    for (auto& m : set.members) {
      const size_t n = all ? m.state.size() : m.field_size();
      std::memcpy(m.state.data(), buf.data() + off, sizeof(double) * n);
      off += n;
    }
  }
  sgwg_family* get() const { return fam_; }
  size_t finest_points() const { return nfine_; }

 private:
  sgwg_family* fam_ = nullptr;
  size_t npts_ = 0, nfine_ = 0;
};

}  // namespace detail

// Drop-in for evolve_family(set, FamilyModel(spec, set, params, threads), policy, T, stops, on_stop)
inline std::vector<double> evolve_family(CombinationSet& set, const ProblemSpec& spec,
                                         const WenoParams& params, const StepPolicy& policy,
                                         double tfinal, std::vector<double> stops = {},
                                         const std::function<void(double)>& on_stop = nullptr,
                                         Device& dev = default_device(), double dt_scale = 1.0) {
  detail::Family fam(dev.get(), set);
  fam.set_model(detail::model_of(spec, params));
  fam.upload(set);
  sgwg_policy pol{};
  pol.mode = (policy.mode == DtMode::cfl) ? SGWG_DT_CFL : SGWG_DT_ACCURACY;
  pol.cfl = policy.cfl_number;
  pol.reference_spacing = policy.reference_spacing;
  pol.dt_scale = dt_scale;
  struct Cb {
    CombinationSet* set;
    detail::Family* fam;
    const std::function<void(double)>* fn;
  } cb{&set, &fam, &on_stop};
  auto tramp = [](double t, void* user) {
    auto* c = static_cast<Cb*>(user);
    if (*c->fn) {
      c->fam->download(*c->set);  // the callback sees the states at the stop
      (*c->fn)(t);
    }
  };
  std::vector<double> dts(1u << 22);
  size_t n = 0;
  sgwg_failure fail{};
  const int st = sgwg_evolve(fam.get(), &pol, tfinal, stops.data(), (int)stops.size(), tramp, &cb,
                             dts.data(), dts.size(), &n, &fail);
  if (st == SGWG_ENONFINITE) {
    fam.download(set);
    const auto levels = enumerate_combination_levels(set.members.front().geom.dim(),
                                                     set.finest_level);
    auto sorted = levels;
    std::sort(sorted.begin(), sorted.end());
    throw FamilyIntegratorFailure(fail.member >= 0 ? sorted[fail.member] : LevelIndex{},
                                  fail.step, fail.stage);
  }
  check(st);
  fam.download(set);
  dts.resize(std::min(n, dts.size()));
  return dts;
}

// Drop-in for combine(set, mode, eps, threads)
inline GridField combine(const CombinationSet& set, InterpMode mode, double epsilon,
                         Device& dev = default_device()) {
  detail::Family fam(dev.get(), set);
  fam.upload(set);
  GridField out = GridField::zeros(finest_geometry(set));
  check(sgwg_combine(fam.get(), mode == InterpMode::weno ? SGWG_INTERP_WENO : SGWG_INTERP_LAGRANGE,
                     epsilon, out.values.data(), out.values.size(), 0));
  return out;
}

// Runner-level outputs from the device (runner.hpp:330-366): diagnostics of
// the combination without downloading it, and the SGW5 dump streamed in slabs.
inline sgwg_field_stats combined_stats(const CombinationSet& set, InterpMode mode, double epsilon,
                                       int exact_preset = -1, double t = 0.0,
                                       const ProblemSpec* spec = nullptr,
                                       Device& dev = default_device()) {
  detail::Family fam(dev.get(), set);
  if (spec != nullptr) fam.set_model(detail::model_of(*spec, WenoParams{epsilon, WenoMode::nonlinear}));
  fam.upload(set);
  sgwg_field_stats st{};
  check(sgwg_combined_stats(fam.get(), mode == InterpMode::weno ? SGWG_INTERP_WENO
                                                                 : SGWG_INTERP_LAGRANGE,
                            epsilon, exact_preset, t, &st));
  return st;
}

inline void write_field_dump(const std::string& path, const CombinationSet& set, InterpMode mode,
                             double epsilon, Device& dev = default_device()) {
  detail::Family fam(dev.get(), set);
  fam.upload(set);
  check(sgwg_write_snapshot(fam.get(), mode == InterpMode::weno ? SGWG_INTERP_WENO
                                                                 : SGWG_INTERP_LAGRANGE,
                            epsilon, path.c_str()));
}

}  // namespace sgweno::gpu
