// sgwg_api.cu -- host runtime of the C ABI (include/sgwg.h).
//
// Owns the device family (packed member states, step-control block, pass
// task tables), sequences the batched WENO pass kernels into SSP-RK3 steps,
// captures chunks of steps into CUDA graphs with device-side dt and stop
// landing (no host sync per step), and runs prolongation + combination.
// Reference interfaces replaced: make_family (combine.hpp:69-83),
// FamilyModel (models.hpp:754-851), evolve_family (timestep.hpp:126-174),
// prolong (interp.hpp:197-250), combine (combine.hpp:95-122).
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <array>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "../../include/sgwg.h"
#include "sgwg_internal.h"

using namespace sgwg;

namespace {

thread_local std::string g_err;

int fail_with(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define CK(call)                                                                         \
  do {                                                                                   \
    cudaError_t e_ = (call);                                                             \
    if (e_ != cudaSuccess)                                                               \
      return fail_with(SGWG_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
  } while (0)

#define CKN(call)                                                                    \
  do {                                                                               \
    ncclResult_t r_ = (call);                                                        \
    if (r_ != ncclSuccess)                                                           \
      return fail_with(SGWG_ENCCL, std::string(#call) + ": " + ncclGetErrorString(r_)); \
  } while (0)

#define TRY(call)          \
  do {                     \
    int s_ = (call);       \
    if (s_ != SGWG_OK) return s_; \
  } while (0)

long long binomial(int n, int k) {  // combine.hpp:27-32
  if (k < 0 || k > n) return 0;
  long long r = 1;
  for (int i = 1; i <= k; ++i) r = r * (n - k + i) / i;
  return r;
}

// enumerate_combination_levels (grid.hpp:57-79): lexicographic by construction
void enum_rec(int d, int nl, int lo, int k, int used, std::array<int, 4>& cur,
              std::vector<std::array<int, 4>>& out) {
  if (k == d - 1) {
    for (int last = std::max(0, lo - used); last + used <= nl; ++last) {
      cur[k] = last;
      if (used + last >= lo) out.push_back(cur);
    }
    return;
  }
  for (int l = 0; l + used <= nl; ++l) {
    cur[k] = l;
    enum_rec(d, nl, lo, k + 1, used + l, cur, out);
  }
}

std::vector<std::array<int, 4>> enumerate_levels(int d, int nl) {
  std::vector<std::array<int, 4>> out;
  std::array<int, 4> cur{0, 0, 0, 0};
  enum_rec(d, nl, std::max(0, nl - d + 1), 0, 0, cur, out);
  std::sort(out.begin(), out.end());  // combine.hpp:71-72 (already sorted)
  return out;
}

struct PassCfg {
  int S, P, W, pitch;
};

// tiling of one line direction of length n: segments of <= 64 points, runs of
// <= kMaxRun points per thread, as many lines per CTA as the 256 threads allow.
// Runs are 4 points on short lines (C5's 8/9-point lines) and 8 otherwise;
// the padded segment is long enough for whole runs (the fast kernel computes
// full runs and discards outputs past the segment).
PassCfg pass_cfg(int n) {
  PassCfg c;
  c.S = std::min(n, 64);
  c.P = (n <= 16) ? 4 : 8;
  const int R = (c.S + c.P - 1) / c.P;
  c.W = kPassThreads / R;
  c.pitch = R * c.P + 6;
  if (c.pitch % 2 == 0) c.pitch += 1;
  return c;
}

}  // namespace

struct sgwg_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  int arith = SGWG_ARITH_EXACT;
  int profile = 0;
  int sm_count = 148;
  int families = 0;      // open families created on this context
  bool closing = false;  // sgwg_shutdown called while families were open
};

struct StageBufs {
  const double* uin;
  const double* un;
  double* out;
};

struct PassDesc {
  int kdim;
  int flux;
  double c_const;
};

struct ProlongPlan {
  // per dimension k in 0..d-2: slot tables of members with refinement > 0
  struct Dim {
    int nslots = 0;
    int ntasks = 0;
    int2* tasks = nullptr;
    const double** src = nullptr;
    double** dst = nullptr;
    int* slot_member = nullptr;
    long long* slot_n = nullptr;
    int* slot_ext = nullptr;
    long long* item0 = nullptr;  // fast chunked form: first work item of each slot
    long long nitems = 0;        // 0: generic upsample kernel
    int nrows0 = 0;              // dimension-0 pass: output rows of the slab
  } dims[kMaxD];
  std::vector<double*> owned;
  // final pass
  const double** fsrc = nullptr;
  double* fcoef = nullptr;
  int* fext = nullptr;
  int* fref = nullptr;
  std::vector<int> href;  // host copy of fref (launch-time kernel choice)
  int nm = 0;
  long long row_a = 0, row_b = 0;  // dimension-0 fine rows covered
};

struct sgwg_family {
  sgwg_ctx* ctx = nullptr;
  sgwg_domain dom{};
  int d = 0, nl = 0;
  int nm = 0;   // local members
  int nfull = 0;
  std::vector<int> gidx;
  std::vector<std::array<int, 4>> levels;
  std::vector<MemberDesc> hmem;
  MemberDesc* dmem = nullptr;
  long long total = 0;        // distribution points of the local members
  long long state_total = 0;  // member state doubles (Vlasov-Maxwell: + 3 field lines each)
  long long finest = 0;
  int fine_ext[kMaxD] = {1, 1, 1, 1};
  double fine_h[kMaxD] = {0, 0, 0, 0};
  double *u = nullptr, *A = nullptr, *B = nullptr, *K = nullptr;
  int4* dtasks[kMaxD] = {nullptr, nullptr, nullptr, nullptr};
  int ntasks[kMaxD] = {0, 0, 0, 0};
  int smem_doubles[kMaxD] = {0, 0, 0, 0};
  int maxW[kMaxD] = {0, 0, 0, 0};
  int2* dmax_tasks = nullptr;
  int nmax_tasks = 0;
  unsigned long long* amax = nullptr;  // 3 slots x nm
  unsigned long long* fail = nullptr;  // nm
  StepCtl* ctl = nullptr;
  StepCtl* hctl = nullptr;  // pinned mirror
  double* dts = nullptr;
  long long dts_cap = 0;
  sgwg_model model{};
  bool has_model = false;
  // Vlasov-Poisson
  double *rho = nullptr, *E = nullptr, *emax = nullptr;
  // Vlasov-Maxwell field lines (E1, E2, B3 per member) of u^n / stage A / stage B
  double *Fu = nullptr, *FA = nullptr, *FB = nullptr, *vmspd = nullptr;
  long long nx_total = 0;
  int2* dmtasks = nullptr;  // moment kernel work list
  int nmtasks = 0;
  double* fe = nullptr;     // per-step sum of |E_combined|^2 h (Vlasov-Poisson diagnostic)
  long long fe_cap = 0;
  double* dcoef = nullptr;  // combination coefficient of each local member
  FieldParams energy_fp{};  // the stage-1 field parameters of the current step
  int4* degrp = nullptr;     // field-energy groups (members sharing an x-grid)
  int2* degrp_m = nullptr;
  int* degrp_mem = nullptr;
  int negrp = 0, ngx = 0;
  double* egrid = nullptr;
  int egrp_tsum = 0;               // energy_rows_kernel: 2 x sum of group x2 extents
  double* eparts = nullptr;        // energy_rows_kernel: per finest x row partial sums
  unsigned int* edone = nullptr;   // energy_rows_kernel: CTAs done (self-resetting)
  // batched energy record of captured step chunks (energy_rows_batch_kernel)
  double* ering = nullptr;         // kEnergyRing step-start fields
  long long ering_stride = 0;      // doubles of one field (space_dim x total x points)
  long long* erecorded = nullptr;  // steps recorded so far
  double* egrid_b = nullptr;       // the groups' combined fields of a chunk's steps
  int ecls_n = 0;                  // groups classed by x2 extent (ascending), 0: not usable
  int ecls_n1[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  unsigned char egrp_cls[64] = {0};
  long long egrid_stride = 0;
  bool ering_step = false;         // the step being enqueued keeps its field in the ring
  // graphs: steps per chunk -> exec
  std::map<int, cudaGraphExec_t> graphs;
  long long graph_key_policy = -1;
  // prolongation plans
  ProlongPlan* full_plan = nullptr;
  // row-slab plans of the whole family over slab_arena, by (row_a, row_b): built
  // once (a plan is ~30 small device tables) and reused by every later combination
  std::map<std::pair<long long, long long>, ProlongPlan*> slab_plans;
  // option B for sharded families (gather_view): every member's state on every rank,
  // combined in dimension-0 row slabs split over the ranks
  std::vector<int> gsel;                   // global member index of each local member
  bool gview = false;
  std::vector<MemberDesc> ghmem;           // all members in family order, offsets into gu
  MemberDesc* gdmem = nullptr;
  double* gu = nullptr;
  std::vector<long long> grank_off, grank_cnt;  // per-rank block of gu (doubles)
  std::map<std::pair<long long, long long>, ProlongPlan*> gslab_plans;
  double* fine_buf = nullptr;
  double* diag_slab = nullptr;     // combined-field slab for diagnostics / snapshots
  long long diag_slab_doubles = 0;
  double* diag_scratch = nullptr;  // stats partials + result
  double* slab_arena = nullptr;  // row-slab combination intermediates
  long long slab_arena_doubles = 0;
  double* slab_out = nullptr;
  long long slab_out_doubles = 0;
  // multi-GPU
  ncclComm_t comm = nullptr;
  int nranks = 1, rank = 0;
  sgwg_stats stats{};
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  cudaEvent_t evs0 = nullptr, evs1 = nullptr;  // whole combined_stats span (ev0/ev1 time each slab)
  cudaStream_t side = nullptr;                 // off-critical-path work (energy record)
  cudaEvent_t evfork = nullptr, evjoin = nullptr;
  cudaStream_t side2 = nullptr;        // x pass concurrent with the VP field solve
  // timing experiments only (SGWG_STAMPS=file): device-clock stamps between the kernels
  // of the captured steps, dumped at the end of sgwg_evolve
  long long* tl = nullptr;
  std::vector<int> tl_labels;
  cudaEvent_t evfork2 = nullptr, evjoin2 = nullptr;
  bool p4x_forked = false;
  // current policy for graph building
  DtParams dtp{};
  DtParams* d_dtp = nullptr;       // device copy (fused dt)
  unsigned int* counter = nullptr;  // CTA-done counter (fused dt)
  // 2D fused-stage tiles
  int4* dtiles2d = nullptr;
  int ntiles2d = 0;
  int smem2d = 0;
  int4* dtiles2d_fast = nullptr;
  int ntiles2d_fast = 0;
  int4* dtiles2d_half = nullptr;  // 1024-point tiles of the stage kernel (two CTAs per SM)
  int ntiles2d_half = 0;
  int smem2d_half = 0;
  int4* dtiles2d_q = nullptr;     // 512-point tiles (four CTAs per SM)
  int ntiles2d_q = 0;
  int smem2d_q = 0;
  int smem2d_fast = 0;
  int4* dtiles3d_fast = nullptr;  // fast 3D stage tiles (advection)
  int ntiles3d_fast = 0;
  int smem3d_fast = 0;
  int tiles3d_half = 0;  // 1024-point 3D tiles (pipelined kernel, two CTAs per SM)
  PlaneTile* dptiles[2] = {nullptr, nullptr};  // fast 4D plane tiles (pairs (0,1), (2,3))
  int nptiles[2] = {0, 0};
  int psmem = 0;
  // fast build, state magnitude >= kOverflowGuard: the step kernels of this
  // call run in the reference arithmetic (overflow_guard)
  bool exact_override = false;
  // profile mode: per-kernel event times and algorithmic counts (sgwg_kernel_profile)
  std::map<std::string, sgwg_kernel_timing> kprof;
  int4* dp4tiles[2] = {nullptr, nullptr};  // whole-plane 4D tiles (plane4d.cuh): x pass, v pass
  int np4tiles[2] = {0, 0};
  int p4smem[2] = {0, 0};                  // dynamic shared memory (doubles) per pass
  int p4vpitch = 0;                        // > 0: persistent v pass, slot pitch (doubles)
  int p4xpitch = 0;                        // > 0: persistent x pass, slot pitch (doubles)
  P4VTile* dp4vtiles = nullptr;            // persistent v pass: tile descriptors
  unsigned int* dp4sched = nullptr;        // persistent v pass: dynamic tile counter (2 words)
  P4XTile* dp4xtiles = nullptr;            // persistent x pass: tile descriptors
  unsigned int* dp4xsched = nullptr;       // persistent x pass: dynamic tile counter
  double* rho_parts = nullptr;      // Vlasov-Poisson charge-density partial sums
  double* twid = nullptr;           // FFT twiddle table (2 x hmax)
  int hmax = 1;
  const double* parts_of = nullptr; // the state rho_parts currently describes (or null)
  bool no_fused2d = false;  // SGWG_NO_FUSED2D=1: use the per-dimension pass kernels
  bool single = false;      // single-grid mode (runner.hpp:106-115): combine = the grid itself
};

namespace {

int arith_of(const sgwg_family* f) {
  return f->exact_override ? SGWG_ARITH_EXACT : f->ctx->arith;
}

cudaError_t do_launch_pass(const sgwg_family* f, const PassParams& p, int kdim) {
  // split-flux arrays (+ a du array in the fast kernel) + coefficients + line bases
  const size_t nsplit = ((p.flux == kFluxBurgers) ? 2 : 1) + 1;
  const size_t smem =
      (nsplit * (size_t)f->smem_doubles[kdim] + 2 * (size_t)f->maxW[kdim]) * sizeof(double);
  if (arith_of(f) == SGWG_ARITH_FAST) return fast::launch_pass(p, f->ntasks[kdim], smem, f->ctx->stream);
  return exact::launch_pass(p, f->ntasks[kdim], smem, f->ctx->stream);
}

std::vector<PassDesc> pass_order(const sgwg_family* f) {
  std::vector<PassDesc> v;
  const sgwg_model& m = f->model;
  if (m.kind == SGWG_ADVECTION || m.kind == SGWG_BURGERS) {
    for (int k = 0; k < f->d; ++k)
      v.push_back({k, m.kind == SGWG_BURGERS ? (int)kFluxBurgers : (int)kFluxAdvect,
                   m.kind == SGWG_ADVECTION ? m.speeds[k] : 0.0});
  } else if (m.kind == SGWG_VLASOV_MAXWELL) {  // vm_rhs_into: x2, xi1, xi2 (models.hpp:455-480)
    v.push_back({0, (int)kFluxVM0, 0.0});
    v.push_back({1, (int)kFluxVM1, 0.0});
    v.push_back({2, (int)kFluxVM2, 0.0});
  } else {  // vb_rhs_into order: x_0, v_0, x_1, v_1 (models.hpp:339-350)
    const int dx = m.space_dim;
    for (int j = 0; j < dx; ++j) {
      v.push_back({j, (int)kFluxKinX, 0.0});
      v.push_back({dx + j, m.kind == SGWG_VLASOV_POISSON ? (int)kFluxKinVP : (int)kFluxKinVB, 0.0});
    }
  }
  return v;
}

void account_kernel(sgwg_family* f, const char* name, double ms, double flops, double bytes) {
  sgwg_kernel_timing& k = f->kprof[name];
  std::snprintf(k.name, sizeof(k.name), "%s", name);
  k.ms_sum += ms;
  k.launches += 1;
  k.flops_per_launch = flops;
  k.bytes_per_launch = bytes;
}

void account_timed(sgwg_family* f, int stage, int npass_dims, bool last, float ms) {
  f->stats.pass_ms_sum += ms;
  f->stats.pass_launches++;
  // algorithmic counts: per point and direction
  // advective 70 flops, Burgers 142; RK stage update 2/5/5 flops;
  // stage bytes 16 (stage 1) / 24 (stages 2, 3) per point.
  const double pts = (double)f->total;
  const bool burgers = f->model.kind == SGWG_BURGERS;
  f->stats.pass_flops += pts * (burgers ? 142.0 : 70.0) * npass_dims;
  if (last && stage > 0) {
    f->stats.pass_flops += pts * (stage == 1 ? 2.0 : 5.0);
    f->stats.pass_bytes += pts * (stage == 1 ? 16.0 : 24.0);
  }
}

// tile size of the fast 2D stage kernel: 512 points, four CTAs per SM (measured:
// S2 stage 358 -> 319 us, C4 3.17 -> 2.90 s against 1024-point tiles, two per
// SM); SGWG_TILE2D=1024 / 2048 select the larger tiles
int stage_tile_code() {
  const char* e = std::getenv("SGWG_TILE2D");
  if (e != nullptr && std::string(e) == "2048") return 0;
  if (e != nullptr && std::string(e) == "1024") return 1;
  return 2;
}

// fast 4D plane path (kernels.cuh plane_fast_kernel)
bool plane_path(const sgwg_family* f) {
  return f->d == 4 && f->nptiles[0] > 0 && f->nptiles[1] > 0 && arith_of(f) == SGWG_ARITH_FAST;
}
// fast 4D whole-plane path (plane4d.cuh), preferred when the family qualifies
bool plane4_path(const sgwg_family* f) {
  return f->d == 4 && f->np4tiles[0] > 0 && f->np4tiles[1] > 0 &&
         arith_of(f) == SGWG_ARITH_FAST;
}

// Vlasov-Poisson field of `state`.  The charge density comes from the
// partial sums the plane kernel left for its stage output when they describe
// `state`; otherwise the moment kernel recomputes them.
int launch_field_for(sgwg_family* f, const double* state, int stage, bool with_energy = false) {
  const sgwg_model& m = f->model;
  FieldParams fp{};
  fp.mem = f->dmem;
  fp.f = state;
  fp.rho = f->rho;
  fp.efield = f->E;
  fp.emax = f->emax;
  fp.space_dim = m.space_dim;
  fp.stage = stage;
  fp.L[0] = f->dom.upper[0] - f->dom.lower[0];
  fp.L[1] = (m.space_dim == 2) ? f->dom.upper[1] - f->dom.lower[1] : 1.0;
  fp.ctl = f->ctl;
  fp.mtasks = f->dmtasks;
  fp.nmtasks = f->nmtasks;
  fp.nmembers = f->nm;
  fp.rho_parts = f->rho_parts;
  fp.twid = f->twid;
  fp.hmax = f->hmax;
  fp.egrp = f->degrp;
  fp.egrp_m = f->degrp_m;
  fp.egrp_mem = f->degrp_mem;
  // members grouped by x-grid when the per-point member loop would be large
  const long long fine_x = (long long)f->fine_ext[0] * ((m.space_dim == 2) ? f->fine_ext[1] : 1);
  bool groups = fine_x * f->nm > (1LL << 20);
  if (const char* e = std::getenv("SGWG_ENERGY_GROUPS")) groups = (e[0] == '1');
  fp.negrp = groups ? f->negrp : 0;
  fp.ngx = f->ngx;
  fp.egrid = f->egrid;
  if (with_energy && f->ering_step) {
    fp.ering = f->ering;
    fp.ering_stride = f->ering_stride;
    fp.ering_slots = kEnergyRing;
    fp.ncls = f->ecls_n;
    for (int k = 0; k < 8; ++k) fp.cls_n1[k] = f->ecls_n1[k];
    std::memcpy(fp.grp_cls, f->egrp_cls, sizeof(fp.grp_cls));
  }
  const bool with_moment = (f->parts_of != state);
  CK(launch_field(fp, f->nm, with_moment, f->ctx->stream));
  f->parts_of = state;
  f->stats.kernel_launches += with_moment ? 2 : 1;
  if (with_energy) f->energy_fp = fp;  // recorded after the dt (launch_step)
  return SGWG_OK;
}

constexpr int kStampSlots = 4096;
int stamp(sgwg_family* f, cudaStream_t s, int label) {
  static const bool on = std::getenv("SGWG_STAMPS") != nullptr;
  if (!on) return SGWG_OK;
  if (f->tl == nullptr) return SGWG_OK;
  if ((int)f->tl_labels.size() >= kStampSlots) return SGWG_OK;
  CK(launch_stamp(f->tl, (int)f->tl_labels.size(), s));
  f->tl_labels.push_back(label);
  return SGWG_OK;
}
int dump_stamps(sgwg_family* f) {
  const char* path = std::getenv("SGWG_STAMPS");
  if (path == nullptr || f->tl == nullptr) return SGWG_OK;
  std::vector<long long> h(f->tl_labels.size());
  CK(cudaMemcpy(h.data(), f->tl, sizeof(long long) * h.size(), cudaMemcpyDeviceToHost));
  if (FILE* fp = std::fopen(path, "w")) {
    for (size_t i = 0; i < h.size(); ++i) std::fprintf(fp, "%d %lld\n", f->tl_labels[i], h[i]);
    std::fclose(fp);
  }
  return SGWG_OK;
}

// The energy record of captured step chunks is batched: the step-start fields go to a ring
// and one launch at the end of the chunk records all its steps (energy_rows_batch_kernel).
// Eligible: the one-kernel row form's cases (2D x-grids with member groups, C5).
bool energy_rows_form(const sgwg_family* f) {
  const long long fine_x = (long long)f->fine_ext[0] * ((f->model.space_dim == 2) ? f->fine_ext[1] : 1);
  bool groups = fine_x * f->nm > (1LL << 20);
  if (const char* e = std::getenv("SGWG_ENERGY_GROUPS")) groups = (e[0] == '1');
  return f->model.space_dim == 2 && groups && f->negrp > 0 && f->negrp < 64 &&
         f->egrp_tsum <= 4096 && f->eparts != nullptr &&
         std::getenv("SGWG_ENERGY_LEGACY") == nullptr;
}
// small families without member groups: a CTA per step (energy_direct_batch_kernel)
bool energy_direct_form(const sgwg_family* f) {
  const long long fine_x = (long long)f->fine_ext[0] * ((f->model.space_dim == 2) ? f->fine_ext[1] : 1);
  bool groups = fine_x * f->nm > (1LL << 20);
  if (const char* e = std::getenv("SGWG_ENERGY_GROUPS")) groups = (e[0] == '1');
  return !groups && fine_x * f->nm <= (1LL << 17);
}
bool energy_batched(const sgwg_family* f, bool timed) {
  if (timed || f->fe == nullptr || f->ering == nullptr || f->comm != nullptr ||
      f->model.kind != SGWG_VLASOV_POISSON)
    return false;
  if (!(energy_rows_form(f) && f->ecls_n > 0) && !energy_direct_form(f)) return false;
  if (const char* e = std::getenv("SGWG_NO_ENERGY"))  // timing experiments only
    if (e[0] == '1') return false;
  const char* e = std::getenv("SGWG_ENERGY_BATCH");
  return e == nullptr || e[0] != '0';
}
int launch_energy_batch(sgwg_family* f, int nsteps) {
  const FieldParams& fp = f->energy_fp;
  if (!(energy_rows_form(f) && f->ecls_n > 0)) {
    const int dx = f->model.space_dim;
    const int fine1 = (dx == 2) ? f->fine_ext[1] : 1;
    const double hv = f->fine_h[0] * ((dx == 2) ? f->fine_h[1] : 1.0);
    CK(launch_field_energy_batch_direct(fp, f->dcoef, f->fine_ext[0], fine1, hv, f->fe, f->fe_cap,
                                        nsteps, f->edone, f->erecorded, f->ctx->stream));
    f->stats.kernel_launches++;
    return SGWG_OK;
  }
  const double hvol = f->fine_h[0] * f->fine_h[1];
  CK(launch_field_energy_batch(fp, f->dcoef, f->fine_ext[0], f->fine_ext[1], hvol, f->fe, f->fe_cap,
                               nsteps, f->eparts, f->edone, f->erecorded, f->egrid_b,
                               f->egrid_stride, f->ctx->stream));
  f->stats.kernel_launches += 2;
  return SGWG_OK;
}

// ||E||_2 of u^n for the step record, on the side stream: forked after the
// step's dt kernel, joined before stage 2's field solve overwrites E, so it
// runs concurrently with stage 1
int launch_energy_side(sgwg_family* f) {
  if (f->fe == nullptr) return SGWG_OK;
  if (const char* e = std::getenv("SGWG_NO_ENERGY"))  // timing experiments only
    if (e[0] == '1') return SGWG_OK;
  const FieldParams& fp = f->energy_fp;
  const int dx = f->model.space_dim;
  const int fine1 = (dx == 2) ? f->fine_ext[1] : 1;
  const double hvol = f->fine_h[0] * ((dx == 2) ? f->fine_h[1] : 1.0);
  CK(cudaEventRecord(f->evfork, f->ctx->stream));
  CK(cudaStreamWaitEvent(f->side, f->evfork, 0));
  // one-kernel row form for 2D x-grids with member groups (C5), else group + point kernels
  const bool rows = (dx == 2 && fp.negrp > 0 && fp.negrp < 64 && f->egrp_tsum <= 4096 &&
                     f->eparts != nullptr);
  CK(launch_field_energy(fp, f->dcoef, f->fine_ext[0], fine1, hvol, f->fe, f->fe_cap, f->side,
                         rows ? f->eparts : nullptr, rows ? f->edone : nullptr));
  TRY(stamp(f, f->side, 11));
  CK(cudaEventRecord(f->evjoin, f->side));
  f->stats.kernel_launches += rows ? 1 : (fp.negrp > 0) ? 2 : 1;
  return SGWG_OK;
}

// Vlasov-Maxwell field lines belonging to a distribution buffer
double* fields_of(const sgwg_family* f, const double* state) {
  if (state == f->A) return f->FA;
  if (state == f->B) return f->FB;
  return f->Fu;
}

// One RK stage (stage 1..3) or a bare tendency evaluation (stage 0).
// fuse_dt: the stage-3 kernel also computes the next step's dt (last CTA).
// one pass of the whole-plane 4D stage (plane4d.cuh) on stream s
int launch_p4_pass(sgwg_family* f, int stage, const StageBufs& b, int pass, cudaStream_t s,
                   bool timed, const DtParams* dtp) {
  const sgwg_model& m = f->model;
  const bool vp = (m.kind == SGWG_VLASOV_POISSON);
  Plane4Params p{};
  p.mem = f->dmem;
  p.stage = stage;
  p.linear = (m.weno_mode == SGWG_WENO_LINEAR);
  p.eps = m.epsilon;
  p.space_dim = m.space_dim;
  p.uin = b.uin;
  p.un = b.un;
  p.out = b.out;
  p.kbuf = f->K;
  p.efield = f->E;
  p.ctl = f->ctl;
  p.fail = f->fail;
  p.counter = f->counter;
  p.rpt = 1;
  if (const char* e = std::getenv("SGWG_P4_RPT")) p.rpt = std::max(1, std::atoi(e));
  if (const char* e = std::getenv("SGWG_P4_DBG")) p.dbg = std::atoi(e);
  p.masked = 1;
  if (const char* e = std::getenv("SGWG_P4_MASKED")) p.masked = std::atoi(e);
  p.tiles = f->dp4tiles[pass];
  if (vp) {
    p.flux_a = p.flux_b = (pass == 0) ? kFluxKinX : kFluxKinVP;
  } else {
    p.flux_a = p.flux_b = kFluxAdvect;
    p.c_a = m.speeds[2 * pass];
    p.c_b = m.speeds[2 * pass + 1];
  }
  p.rho_parts = (pass == 1 && vp) ? f->rho_parts : nullptr;
  p.dtp = dtp;
  if (timed) CK(cudaEventRecord(f->ev0, s));
  int nblk = f->np4tiles[pass];
  p.ntiles = nblk;
  if (pass == 1 && f->p4vpitch > 0) {
    p.vpitch = f->p4vpitch;
    p.vtiles = f->dp4vtiles;
    p.sched = f->dp4sched;
    nblk = std::min(nblk, 2 * f->ctx->sm_count);
  }
  if (pass == 0 && f->p4xpitch > 0) {
    p.xpitch = f->p4xpitch;
    p.xtiles = f->dp4xtiles;
    p.sched = f->dp4xsched;
    nblk = std::min(nblk, 2 * f->ctx->sm_count);
  }
  CK(fast::launch_plane4(p, pass, nblk, (size_t)f->p4smem[pass] * sizeof(double), s));
  if (timed) {
    CK(cudaEventRecord(f->ev1, s));
    CK(cudaEventSynchronize(f->ev1));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, f->ev0, f->ev1));
    account_timed(f, stage, 2, pass == 1, ms);
    // algorithmic counts per launch: 70 flops per point and
    // direction; x pass + K (1), v pass + accumulate (2) + RK stage (2/5/5) +
    // charge density (2); HBM: u^(s) in, K out | u^(s), K, (u^n) in, out out
    const double pts = (double)f->total;
    const double rk = (stage == 0) ? 0.0 : (stage == 1 ? 2.0 : 5.0);
    if (pass == 0)
      account_kernel(f, f->p4xpitch > 0 ? "xpass4d_persist_kernel" : "xpass4d_kernel", ms,
                     pts * 141.0, pts * 16.0);
    else
      account_kernel(f, f->p4vpitch > 0 ? "vpass4d_persist_kernel" : "vpass4d_kernel", ms,
                     pts * (142.0 + rk + (vp ? 2.0 : 0.0)), pts * (stage > 1 ? 32.0 : 24.0));
  }
  f->stats.kernel_launches++;
  return SGWG_OK;
}

// Vlasov-Poisson on the whole-plane 4D path: the stage's x pass does not read the
// field, so it runs on a second stream concurrently with the field solve (and,
// for stage 1, the dt and energy kernels); the v pass joins it.  Graph-captured
// steps only (timed launches stay serial for the per-kernel clock).
bool p4_overlap(const sgwg_family* f, bool timed) {
  if (timed || !plane4_path(f) || f->model.kind != SGWG_VLASOV_POISSON) return false;
  const char* e = std::getenv("SGWG_P4_OVERLAP");
  return e == nullptr || e[0] != '0';
}
// the fork point (before the field solve), then -- after the field kernels have been
// enqueued, so they are dispatched first -- the x pass on the low-priority stream
int mark_x_fork(sgwg_family* f) {
  CK(cudaEventRecord(f->evfork2, f->ctx->stream));
  return SGWG_OK;
}
int fork_x_pass(sgwg_family* f, int stage, const StageBufs& b) {
  CK(cudaStreamWaitEvent(f->side2, f->evfork2, 0));
  TRY(launch_p4_pass(f, stage, b, 0, f->side2, false, nullptr));
  TRY(stamp(f, f->side2, 20 + stage));
  CK(cudaEventRecord(f->evjoin2, f->side2));
  f->p4x_forked = true;
  return SGWG_OK;
}

int launch_stage(sgwg_family* f, int stage, const StageBufs& b, bool timed, bool with_field = true,
                 bool fuse_dt = false) {
  const sgwg_model& m = f->model;
  const bool burgers = (m.kind == SGWG_BURGERS);
  if (m.kind == SGWG_VLASOV_POISSON && with_field) {
    const bool ovl = p4_overlap(f, timed) && !f->p4x_forked;
    if (ovl) TRY(mark_x_fork(f));
    TRY(launch_field_for(f, b.uin, stage));
    TRY(stamp(f, f->ctx->stream, 30 + stage));
    if (ovl) TRY(fork_x_pass(f, stage, b));
  }
  const auto order = pass_order(f);
  const int in_slot = (stage == 0) ? 0 : stage - 1;
  const int out_slot = (stage == 0) ? 0 : stage % 3;
  // stage s clears the slot stage s+1 will write: it was last read one stage ago
  unsigned long long* zero_slot =
      (burgers && stage > 0) ? f->amax + (size_t)((stage + 1) % 3) * f->nm : nullptr;
  const DtParams* dtp = (fuse_dt && stage == 3) ? f->d_dtp : nullptr;
  const bool vm = (m.kind == SGWG_VLASOV_MAXWELL);
  if (vm) {  // field lines: currents, characteristic WENO derivatives, RK stage
    VmParams vp{};
    vp.mem = f->dmem;
    vp.f = b.uin;
    vp.fin = fields_of(f, b.uin);
    vp.fun = f->Fu;
    vp.fout = fields_of(f, b.out);
    vp.stage = stage;
    vp.linear = (m.weno_mode == SGWG_WENO_LINEAR);
    vp.eps = m.epsilon;
    vp.ctl = f->ctl;
    vp.fail = f->fail;
    int nxmax = 1;
    for (const auto& M : f->hmem) nxmax = std::max(nxmax, M.nx);
    const int smem = 4 * nxmax * (int)sizeof(double);
    CK(arith_of(f) == SGWG_ARITH_FAST ? fast::launch_vm_fields(vp, f->nm, smem, f->ctx->stream)
                                       : exact::launch_vm_fields(vp, f->nm, smem, f->ctx->stream));
    f->stats.kernel_launches++;
  }
  // every path below but the plane path writes a state without its rho partials
  if (stage > 0 && !plane_path(f) && !plane4_path(f)) f->parts_of = nullptr;
  if (plane4_path(f)) {  // fast 4D on whole planes: x pass -> K, v pass + RK stage + rho
    const bool vp = (m.kind == SGWG_VLASOV_POISSON);
    const bool xdone = f->p4x_forked;  // the x pass already runs on the side stream
    f->p4x_forked = false;
    if (xdone) CK(cudaStreamWaitEvent(f->ctx->stream, f->evjoin2, 0));
    if (!timed) TRY(stamp(f, f->ctx->stream, 40 + stage));
    for (int pass = xdone ? 1 : 0; pass < 2; ++pass)
      TRY(launch_p4_pass(f, stage, b, pass, f->ctx->stream, timed, (pass == 1) ? dtp : nullptr));
    if (!timed) TRY(stamp(f, f->ctx->stream, 50 + stage));
    if (stage > 0) f->parts_of = vp ? b.out : nullptr;
    return SGWG_OK;
  }
  if (plane_path(f)) {  // fast 4D: dims (0,1) -> K, dims (2,3) + RK stage
    const bool vp = (m.kind == SGWG_VLASOV_POISSON);
    PlaneParams p{};
    p.mem = f->dmem;
    p.stage = stage;
    p.linear = (m.weno_mode == SGWG_WENO_LINEAR);
    p.eps = m.epsilon;
    p.space_dim = m.space_dim;
    p.uin = b.uin;
    p.un = b.un;
    p.out = b.out;
    p.kbuf = f->K;
    p.efield = f->E;
    p.ctl = f->ctl;
    p.fail = f->fail;
    p.counter = f->counter;
    for (int pr = 0; pr < 2; ++pr) {
      p.pr = pr;
      p.tiles = f->dptiles[pr];
      if (vp) {
        p.flux_a = p.flux_b = (pr == 0) ? kFluxKinX : kFluxKinVP;
      } else {
        p.flux_a = p.flux_b = kFluxAdvect;
        p.c_a = m.speeds[2 * pr];
        p.c_b = m.speeds[2 * pr + 1];
      }
      p.rho_parts = (pr == 1 && vp) ? f->rho_parts : nullptr;
      p.dtp = (pr == 1) ? dtp : nullptr;
      if (timed) CK(cudaEventRecord(f->ev0, f->ctx->stream));
      CK(fast::launch_plane(p, f->nptiles[pr], (size_t)f->psmem * sizeof(double),
                            f->ctx->stream));
      if (timed) {
        CK(cudaEventRecord(f->ev1, f->ctx->stream));
        CK(cudaEventSynchronize(f->ev1));
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, f->ev0, f->ev1));
        account_timed(f, stage, 2, pr == 1, ms);
      }
      f->stats.kernel_launches++;
    }
    if (stage > 0) f->parts_of = vp ? b.out : nullptr;
    return SGWG_OK;
  }
  if (f->d == 3 && f->ntiles3d_fast > 0 && arith_of(f) == SGWG_ARITH_FAST &&
      m.kind == SGWG_ADVECTION) {  // fused 3D stage (all three sweeps + RK, one launch)
    Stage2DParams p{};
    p.mem = f->dmem;
    p.tiles = f->dtiles3d_fast;
    p.flux0 = p.flux1 = p.flux2 = kFluxAdvect;
    p.c0 = m.speeds[0];
    p.c1 = m.speeds[1];
    p.c2 = m.speeds[2];
    p.stage = stage;
    p.linear = (m.weno_mode == SGWG_WENO_LINEAR);
    p.eps = m.epsilon;
    p.uin = b.uin;
    p.un = b.un;
    p.out = b.out;
    p.ctl = f->ctl;
    p.nmembers = f->nm;
    p.fail = f->fail;
    p.dtp = dtp;
    p.counter = f->counter;
    p.half_tiles = f->tiles3d_half;
    if (timed) CK(cudaEventRecord(f->ev0, f->ctx->stream));
    CK(fast::launch_stage3d(p, f->ntiles3d_fast, (size_t)f->smem3d_fast * sizeof(double),
                            f->ctx->stream));
    if (timed) {
      CK(cudaEventRecord(f->ev1, f->ctx->stream));
      CK(cudaEventSynchronize(f->ev1));
      float ms = 0.f;
      CK(cudaEventElapsedTime(&ms, f->ev0, f->ev1));
      account_timed(f, stage, 3, true, ms);
    }
    f->stats.kernel_launches++;
    return SGWG_OK;
  }
  if (f->d == 2 && f->ntiles2d > 0) {
    Stage2DParams p{};
    const bool fastk = arith_of(f) == SGWG_ARITH_FAST;
    p.mem = f->dmem;
    p.tiles = fastk ? f->dtiles2d_fast : f->dtiles2d;
    int nt = fastk ? f->ntiles2d_fast : f->ntiles2d;
    size_t smem = (size_t)(fastk ? f->smem2d_fast : f->smem2d) * sizeof(double);
    if (fastk && stage_tile_code() == 2) {
      p.tiles = f->dtiles2d_q;
      p.half_tiles = 2;
      nt = f->ntiles2d_q;
      smem = (size_t)f->smem2d_q * sizeof(double);
    } else if (fastk && stage_tile_code() == 1) {
      p.tiles = f->dtiles2d_half;
      p.half_tiles = 1;
      nt = f->ntiles2d_half;
      smem = (size_t)f->smem2d_half * sizeof(double);
    }
    p.burgers = burgers;
    // large Burgers families (never co-resident: no persistent kernel) take the Newton /
    // direct-difference form of the reconstructions (fast_rcp); a property of the family
    p.newton = (burgers && f->total > (1LL << 21)) ? 1 : 0;
    p.flux0 = order[0].flux;
    p.flux1 = order[1].flux;
    p.c0 = order[0].c_const;
    p.c1 = order[1].c_const;
    p.stage = stage;
    p.linear = (m.weno_mode == SGWG_WENO_LINEAR);
    p.eps = m.epsilon;
    p.space_dim = m.space_dim;
    p.uin = b.uin;
    p.un = b.un;
    p.out = b.out;
    p.efield = f->E;
    p.ctl = f->ctl;
    p.amax_in = f->amax + (size_t)in_slot * f->nm;
    p.amax_out = f->amax + (size_t)out_slot * f->nm;
    p.amax_zero = zero_slot;
    p.nmembers = f->nm;
    p.track_max = burgers && stage != 0;
    p.fail = f->fail;
    p.dtp = dtp;
    p.counter = f->counter;
    if (timed) CK(cudaEventRecord(f->ev0, f->ctx->stream));
    CK(fastk ? fast::launch_stage2d(p, nt, smem, f->ctx->stream)
             : exact::launch_stage2d(p, nt, smem, f->ctx->stream));
    if (timed) {
      CK(cudaEventRecord(f->ev1, f->ctx->stream));
      CK(cudaEventSynchronize(f->ev1));
      float ms = 0.f;
      CK(cudaEventElapsedTime(&ms, f->ev0, f->ev1));
      account_timed(f, stage, 2, true, ms);
    }
    f->stats.kernel_launches++;
    return SGWG_OK;
  }
  for (size_t pi = 0; pi < order.size(); ++pi) {
    const PassDesc& pd = order[pi];
    PassParams p{};
    p.mem = f->dmem;
    p.tasks = f->dtasks[pd.kdim];
    p.kdim = pd.kdim;
    p.flux = pd.flux;
    p.first = (pi == 0);
    p.last = (pi + 1 == order.size());
    p.stage = stage;
    p.linear = (m.weno_mode == SGWG_WENO_LINEAR);
    p.eps = m.epsilon;
    p.c_const = pd.c_const;
    p.space_dim = m.space_dim;
    p.uin = b.uin;
    p.un = b.un;
    p.out = b.out;
    p.kbuf = f->K;
    p.efield = vm ? fields_of(f, b.uin) : f->E;
    p.ctl = f->ctl;
    p.amax_in = f->amax + (size_t)in_slot * f->nm;
    p.amax_out = f->amax + (size_t)out_slot * f->nm;
    p.amax_zero = (pi == 0) ? zero_slot : nullptr;
    p.nmembers = f->nm;
    p.track_max = burgers && stage != 0;
    p.fail = f->fail;
    p.dyn_smem_doubles = f->smem_doubles[pd.kdim];
    p.dtp = p.last ? dtp : nullptr;
    p.counter = f->counter;
    if (timed) CK(cudaEventRecord(f->ev0, f->ctx->stream));
    CK(do_launch_pass(f, p, pd.kdim));
    if (timed) {
      CK(cudaEventRecord(f->ev1, f->ctx->stream));
      CK(cudaEventSynchronize(f->ev1));
      float ms = 0.f;
      CK(cudaEventElapsedTime(&ms, f->ev0, f->ev1));
      account_timed(f, stage, 1, p.last, ms);
    }
    f->stats.kernel_launches++;
  }
  return SGWG_OK;
}

int launch_member_max_slot0(sgwg_family* f) {
  CK(cudaMemsetAsync(f->amax, 0, sizeof(unsigned long long) * 3 * f->nm, f->ctx->stream));
  CK(launch_member_max(f->dmem, f->nm, f->dmax_tasks, f->nmax_tasks, f->u, f->amax,
                       f->ctx->stream));
  return SGWG_OK;
}

// Overflow guard of the fast build.  Its reconstructions put the three WENO
// weights over one common denominator (one reciprocal instead of four
// divides), which overflows for |u| >~ 1e36 where the reference's separate
// divides (weno.hpp:60-72) stay finite.  Every evolve / rk3_step / rhs call
// first reduces max|u| over the family (one small kernel); at or above 1e30
// the step kernels of the call run in the reference arithmetic instead, so the
// fast build never reports a non-finite tendency the reference would not.
// (The 4D whole-plane and combination kernels also re-run an overflowed window
// in the reference form themselves.)
constexpr double kOverflowGuard = 1e30;
void clear_graphs(sgwg_family* f);
int overflow_guard(sgwg_family* f) {
  bool on = false;
  if (f->ctx->arith == SGWG_ARITH_FAST && f->nm > 0) {
    TRY(launch_member_max_slot0(f));
    std::vector<unsigned long long> mx(f->nm);
    CK(cudaMemcpyAsync(mx.data(), f->amax, sizeof(unsigned long long) * f->nm,
                       cudaMemcpyDeviceToHost, f->ctx->stream));
    CK(cudaStreamSynchronize(f->ctx->stream));
    for (unsigned long long b : mx) {
      double v;
      std::memcpy(&v, &b, sizeof(v));
      if (!(v < kOverflowGuard)) on = true;  // (NaN included: the reference path reports it)
    }
  }
  if (on != f->exact_override) {
    f->exact_override = on;
    clear_graphs(f);
  }
  return SGWG_OK;
}

// dt of the next step can be fused into the stage-3 kernel when nothing has to
// happen between the end of a step and the dt (no field solve, no all-reduce)
bool dt_fusable(const sgwg_family* f) {
  return f->comm == nullptr && f->model.kind != SGWG_VLASOV_POISSON &&
         f->model.kind != SGWG_VLASOV_MAXWELL;
}

// the (unfused) dt of a step: speeds (+ NCCL all-reduce(max)), dt kernel
int launch_dt_step(sgwg_family* f) {
  DtParams dp = f->dtp;
  if (f->comm != nullptr) {
    CK(launch_local_speeds(dp, f->ctx->stream));
    CKN(ncclAllReduce(f->ctl->speeds, f->ctl->speeds, kMaxD + 1, ncclDouble, ncclMax, f->comm,
                      f->ctx->stream));
    dp.use_reduced = 1;
    f->stats.kernel_launches++;
  }
  CK(launch_dt(dp, f->ctx->stream));
  f->stats.kernel_launches++;
  return SGWG_OK;
}

// one full step.  Unfused: (VP field of u^n), speeds (+ all-reduce), dt, three
// stages.  Fused (dt_fusable): three stages, the dt of this step having been
// computed by the previous step's stage-3 kernel (or the segment's first dt).
int launch_step(sgwg_family* f, bool timed) {
  const bool vp = f->model.kind == SGWG_VLASOV_POISSON;
  const bool fused = dt_fusable(f);
  if (!fused) {
    const bool ovl = vp && p4_overlap(f, timed);
    f->ering_step = vp && energy_batched(f, timed);
    if (!timed) TRY(stamp(f, f->ctx->stream, 0));
    if (ovl) TRY(mark_x_fork(f));
    if (vp) TRY(launch_field_for(f, f->u, 1, /*with_energy=*/true));
    if (!timed) TRY(stamp(f, f->ctx->stream, 31));
    if (f->model.kind == SGWG_VLASOV_MAXWELL) {  // family_wave_speeds of u^n
      VmParams sp{};
      sp.mem = f->dmem;
      sp.fin = f->Fu;
      sp.ctl = f->ctl;
      sp.speeds = f->vmspd;
      CK(launch_vm_speeds(sp, f->nm, f->ctx->stream));
      f->stats.kernel_launches++;
    }
    TRY(launch_dt_step(f));
    if (!timed) TRY(stamp(f, f->ctx->stream, 1));
    if (ovl) TRY(fork_x_pass(f, 1, StageBufs{f->u, f->u, f->A}));
    if (vp && !f->ering_step) TRY(launch_energy_side(f));
  }
  // stage 1: u -> A; stage 2: (A, u) -> B; stage 3: (B, u) -> u (timestep.hpp:91-103)
  StageBufs s1{f->u, f->u, f->A}, s2{f->A, f->u, f->B}, s3{f->B, f->u, f->u};
  // VP: the stage-1 field was computed above (it feeds dt); stages 2, 3 recompute it
  TRY(launch_stage(f, 1, s1, timed, /*with_field=*/!vp));
  if (vp && !fused && f->fe != nullptr && !f->ering_step)
    CK(cudaStreamWaitEvent(f->ctx->stream, f->evjoin, 0));
  TRY(launch_stage(f, 2, s2, timed));
  TRY(launch_stage(f, 3, s3, timed, true, fused));
  return SGWG_OK;
}

int build_tasks(sgwg_family* f) {
  for (int k = 0; k < f->d; ++k) {
    std::vector<int4> t;
    int smax = 0, wmax = 0;
    for (int mi = 0; mi < f->nm; ++mi) {
      MemberDesc& M = f->hmem[mi];
      const int n = M.ext[k];
      const PassCfg c = pass_cfg(n);
      M.segS[k] = c.S;
      M.runP[k] = c.P;
      M.linesW[k] = c.W;
      M.pitch[k] = c.pitch;
      smax = std::max(smax, c.W * c.pitch);
      wmax = std::max(wmax, c.W);
      const long long nlines = M.npts / n;
      for (long long L0 = 0; L0 < nlines; L0 += c.W)
        for (int s0 = 0; s0 < n; s0 += c.S) t.push_back(make_int4(mi, (int)L0, s0, 0));
    }
    f->ntasks[k] = (int)t.size();
    f->smem_doubles[k] = smax;
    f->maxW[k] = wmax;
    CK(cudaMalloc(&f->dtasks[k], sizeof(int4) * std::max<size_t>(1, t.size())));
    CK(cudaMemcpy(f->dtasks[k], t.data(), sizeof(int4) * t.size(), cudaMemcpyHostToDevice));
  }
  if (f->d == 2 && !f->no_fused2d) {  // fused 2D stage tiles: TX x TY = 256 points
    std::vector<int4> t;
    int smax = 0;
    for (int mi = 0; mi < f->nm; ++mi) {
      MemberDesc& M = f->hmem[mi];
      M.ty = (M.ext[1] >= 32) ? 32 : (M.ext[1] >= 16 ? 16 : 8);
      M.tx = 256 / M.ty;
      const int sm = 2 * (M.tx + 6) * (M.ty + 6) + (M.tx + 1) * M.ty + M.tx * (M.ty + 1) +
                     M.tx + M.ty;
      smax = std::max(smax, sm);
      for (int i0 = 0; i0 < M.ext[0]; i0 += M.tx)
        for (int j0 = 0; j0 < M.ext[1]; j0 += M.ty) t.push_back(make_int4(mi, i0, j0, 0));
    }
    f->ntiles2d = (int)t.size();
    f->smem2d = smax;
    CK(cudaMalloc(&f->dtiles2d, sizeof(int4) * std::max<size_t>(1, t.size())));
    CK(cudaMemcpy(f->dtiles2d, t.data(), sizeof(int4) * t.size(), cudaMemcpyHostToDevice));
    // fast build: 2048-point tiles of shape (TX, TY) in {(32,64),(64,32),(16,128),(128,16)},
    // the one that wastes least on this member (kernels.cuh stage2d_fast_kernel)
    static const int shp[4][2] = {{32, 64}, {64, 32}, {16, 128}, {128, 16}};
    std::vector<int4> tf;
    int sfmax = 0;
    for (int mi = 0; mi < f->nm; ++mi) {
      const MemberDesc& M = f->hmem[mi];
      int best = 0;
      long long bw = -1;
      for (int s = 0; s < 4; ++s) {
        const long long cov = (long long)((M.ext[0] + shp[s][0] - 1) / shp[s][0]) * shp[s][0] *
                              ((M.ext[1] + shp[s][1] - 1) / shp[s][1]) * shp[s][1];
        if (bw < 0 || cov < bw) {
          bw = cov;
          best = s;
        }
      }
      const int TX = shp[best][0], TY = shp[best][1];
      const int PY = ((TY + 6) % 2 == 0) ? TY + 7 : TY + 6;
      const int sm = 2 * (TX + 6) * PY + 2 * TX * (TY + 1) + TX + TY;
      sfmax = std::max(sfmax, sm);
      for (int i0 = 0; i0 < M.ext[0]; i0 += TX)
        for (int j0 = 0; j0 < M.ext[1]; j0 += TY) tf.push_back(make_int4(mi, i0, j0, best));
    }
    f->ntiles2d_fast = (int)tf.size();
    f->smem2d_fast = sfmax;
    CK(cudaMalloc(&f->dtiles2d_fast, sizeof(int4) * std::max<size_t>(1, tf.size())));
    CK(cudaMemcpy(f->dtiles2d_fast, tf.data(), sizeof(int4) * tf.size(), cudaMemcpyHostToDevice));
    // stage-kernel tiles: 1024 points in {(32,32),(16,64),(64,16),(8,128),(128,8)}
    // (kernels.cuh tile_body_half, shape codes 4..8)
    static const int shh[5][2] = {{32, 32}, {16, 64}, {64, 16}, {8, 128}, {128, 8}};
    std::vector<int4> th;
    int shmax = 0;
    for (int mi = 0; mi < f->nm; ++mi) {
      const MemberDesc& M = f->hmem[mi];
      int best = 0;
      long long bw = -1;
      for (int s = 0; s < 5; ++s) {
        const long long cov = (long long)((M.ext[0] + shh[s][0] - 1) / shh[s][0]) * shh[s][0] *
                              ((M.ext[1] + shh[s][1] - 1) / shh[s][1]) * shh[s][1];
        if (bw < 0 || cov < bw) {
          bw = cov;
          best = s;
        }
      }
      const int TX = shh[best][0], TY = shh[best][1];
      const int PY = ((TY + 6) % 2 == 0) ? TY + 7 : TY + 6;
      const int sm = 2 * (TX + 6) * PY + 2 * TX * (TY + 1) + TX + TY;
      shmax = std::max(shmax, sm);
      for (int i0 = 0; i0 < M.ext[0]; i0 += TX)
        for (int j0 = 0; j0 < M.ext[1]; j0 += TY) th.push_back(make_int4(mi, i0, j0, 4 + best));
    }
    f->ntiles2d_half = (int)th.size();
    f->smem2d_half = shmax;
    CK(cudaMalloc(&f->dtiles2d_half, sizeof(int4) * std::max<size_t>(1, th.size())));
    CK(cudaMemcpy(f->dtiles2d_half, th.data(), sizeof(int4) * th.size(), cudaMemcpyHostToDevice));
    static const int shq[4][2] = {{16, 32}, {32, 16}, {8, 64}, {64, 8}};
    std::vector<int4> tq;
    int sqmax = 0;
    for (int mi = 0; mi < f->nm; ++mi) {
      const MemberDesc& M = f->hmem[mi];
      int best = 0;
      long long bw = -1;
      for (int s = 0; s < 4; ++s) {
        const long long cov = (long long)((M.ext[0] + shq[s][0] - 1) / shq[s][0]) * shq[s][0] *
                              ((M.ext[1] + shq[s][1] - 1) / shq[s][1]) * shq[s][1];
        if (bw < 0 || cov < bw) {
          bw = cov;
          best = s;
        }
      }
      const int TX = shq[best][0], TY = shq[best][1];
      const int PY = ((TY + 6) % 2 == 0) ? TY + 7 : TY + 6;
      const int sm = 2 * (TX + 6) * PY + 2 * TX * (TY + 1) + TX + TY;
      sqmax = std::max(sqmax, sm);
      for (int i0 = 0; i0 < M.ext[0]; i0 += TX)
        for (int j0 = 0; j0 < M.ext[1]; j0 += TY) tq.push_back(make_int4(mi, i0, j0, 8 + best));
    }
    f->ntiles2d_q = (int)tq.size();
    f->smem2d_q = sqmax;
    CK(cudaMalloc(&f->dtiles2d_q, sizeof(int4) * std::max<size_t>(1, tq.size())));
    CK(cudaMemcpy(f->dtiles2d_q, tq.data(), sizeof(int4) * tq.size(), cudaMemcpyHostToDevice));
  }
  if (f->d == 3 && !f->no_fused2d) {  // fast 3D stage tiles, 3 shapes
    // default 512-point tiles (8x8x8, shape code 6), one per CTA, four CTAs per SM
    // (measured: C3 165.3 -> 155.3 ms, S3 stage 1246 -> 1066 us against the pipelined kernel
    // on 1024-point tiles, two CTAs per SM, shape codes 3..5: SGWG_3D_TILE=1024; 2048-point
    // tiles, one CTA per SM: SGWG_3D_TILE=2048)
    static const int shp3f[3][3] = {{8, 16, 16}, {16, 8, 16}, {16, 16, 8}};
    static const int shp3h[3][3] = {{8, 8, 16}, {8, 16, 8}, {16, 8, 8}};
    static const int shp3q[3][3] = {{8, 8, 8}, {8, 8, 8}, {8, 8, 8}};
    const char* e3 = std::getenv("SGWG_3D_TILE");
    f->tiles3d_half = 2;
    if (e3 != nullptr && std::string(e3) == "1024") f->tiles3d_half = 1;
    if (e3 != nullptr && std::string(e3) == "2048") f->tiles3d_half = 0;
    const int(*shp3)[3] = (f->tiles3d_half == 2) ? shp3q : f->tiles3d_half ? shp3h : shp3f;
    std::vector<int4> t3;
    int smax = 0;
    bool ok = true;
    for (int mi = 0; mi < f->nm; ++mi) {
      const MemberDesc& M = f->hmem[mi];
      if (M.ext[0] >= 65536 || M.ext[1] >= 65536) ok = false;
      if (M.npts >= (1LL << 31)) ok = false;  // 32-bit member-local offsets in the kernel
      int best = 0;
      long long bw = -1;
      for (int s = 0; s < 3; ++s) {
        long long cov = 1;
        for (int k = 0; k < 3; ++k)
          cov *= (long long)((M.ext[k] + shp3[s][k] - 1) / shp3[s][k]) * shp3[s][k];
        if (bw < 0 || cov < bw) {
          bw = cov;
          best = s;
        }
      }
      const int TX = shp3[best][0], TY = shp3[best][1], TZ = shp3[best][2];
      const int PZ = ((TZ + 6) % 2 == 0) ? TZ + 7 : TZ + 6;
      const int sm = (TX + 6) * (TY + 6) * PZ + 3 * TX * TY * (TZ + 1) + TY * TZ + TX * TZ + TX * TY;
      smax = std::max(smax, sm);
      for (int i0 = 0; i0 < M.ext[0]; i0 += TX)
        for (int j0 = 0; j0 < M.ext[1]; j0 += TY)
          for (int l0 = 0; l0 < M.ext[2]; l0 += TZ)
            t3.push_back(make_int4(mi, (i0 << 16) | j0,
                                   (l0 << 8) | (f->tiles3d_half == 2 ? 6 : best + 3 * f->tiles3d_half), 0));
    }
    if (ok) {
      f->ntiles3d_fast = (int)t3.size();
      f->smem3d_fast = smax;
      CK(cudaMalloc(&f->dtiles3d_fast, sizeof(int4) * std::max<size_t>(1, t3.size())));
      CK(cudaMemcpy(f->dtiles3d_fast, t3.data(), sizeof(int4) * t3.size(),
                    cudaMemcpyHostToDevice));
    }
  }
  std::vector<int2> mt;
  for (int mi = 0; mi < f->nm; ++mi)
    for (long long c = 0; c * 4096 < f->hmem[mi].npts; ++c) mt.push_back(make_int2(mi, (int)c));
  f->nmax_tasks = (int)mt.size();
  CK(cudaMalloc(&f->dmax_tasks, sizeof(int2) * std::max<size_t>(1, mt.size())));
  CK(cudaMemcpy(f->dmax_tasks, mt.data(), sizeof(int2) * mt.size(), cudaMemcpyHostToDevice));
  return SGWG_OK;
}

int check_domain(const sgwg_domain* dom) {
  if (dom == nullptr) return fail_with(SGWG_EINVAL, "null domain");
  if (dom->d < 1 || dom->d > 4)
    return fail_with(SGWG_EINVAL, "enumerate_combination_levels: d must be 1..4");
  if (dom->nl < dom->d - 1)
    return fail_with(SGWG_EINVAL, "enumerate_combination_levels: need N_L >= d-1");
  for (int k = 0; k < dom->d; ++k) {
    if (!(dom->upper[k] > dom->lower[k]))
      return fail_with(SGWG_EINVAL, "DomainBox: upper must exceed lower");
    if (dom->root_cells[k] < 1)
      return fail_with(SGWG_EINVAL, "GridGeometry: root cells must be >= 1");
    if (dom->bc[k] != SGWG_PERIODIC && dom->bc[k] != SGWG_ZERO)
      return fail_with(SGWG_EINVAL, "unknown boundary kind");
  }
  return SGWG_OK;
}

// geometry of the component grid at levels lv (GridGeometry::make, grid.hpp:110-133),
// its state at `off` in a packed buffer
MemberDesc geom_desc(const sgwg_domain* dom, const std::array<int, 4>& lv, long long off) {
  const int d = dom->d;
  MemberDesc M{};
  M.offset = off;
  M.npts = 1;
  for (int k = 0; k < kMaxD; ++k) {
    M.ext[k] = 1;
    M.h[k] = 1.0;
    M.inv_h[k] = 1.0;
  }
  for (int k = 0; k < d; ++k) {
    const int cells = dom->root_cells[k] << lv[k];
    M.ext[k] = cells + (dom->bc[k] == SGWG_ZERO ? 1 : 0);
    M.bc[k] = dom->bc[k];
    M.level[k] = lv[k];
    M.h[k] = std::ldexp((dom->upper[k] - dom->lower[k]) / dom->root_cells[k], -lv[k]);
    M.inv_h[k] = 1.0 / M.h[k];
    M.lower[k] = dom->lower[k];
    M.npts *= M.ext[k];
  }
  M.stride[d - 1] = 1;
  for (int k = d - 2; k >= 0; --k) M.stride[k] = M.stride[k + 1] * M.ext[k + 1];
  for (int k = d; k < kMaxD; ++k) M.stride[k] = 1;
  return M;
}

int family_create(sgwg_ctx* ctx, const sgwg_domain* dom, const int* members, int count,
                  sgwg_family** out, bool single = false) {
  if (ctx == nullptr || out == nullptr) return fail_with(SGWG_EINVAL, "null argument");
  if (single) {  // make_single_grid (runner.hpp:106-115): one grid at (N_L, ..., N_L)
    if (dom == nullptr || dom->d < 1 || dom->d > 4 || dom->nl < 0)
      return fail_with(SGWG_EINVAL, "single grid: bad domain");
  } else {
    TRY(check_domain(dom));
  }
  CK(cudaSetDevice(ctx->device));
  std::vector<std::array<int, 4>> all;
  if (single) {
    std::array<int, 4> lv{0, 0, 0, 0};
    for (int k = 0; k < dom->d; ++k) lv[k] = dom->nl;
    all.push_back(lv);
  } else {
    all = enumerate_levels(dom->d, dom->nl);
  }
  std::vector<int> sel;
  if (members == nullptr) {
    for (int i = 0; i < (int)all.size(); ++i) sel.push_back(i);
  } else {
    for (int i = 0; i < count; ++i) {
      if (members[i] < 0 || members[i] >= (int)all.size() || (i > 0 && members[i] <= members[i - 1]))
        return fail_with(SGWG_EINVAL, "shard members must be ascending valid indices");
      sel.push_back(members[i]);
    }
  }
  sgwg_family* f = new sgwg_family();
  f->ctx = ctx;
  ++ctx->families;
  f->dom = *dom;
  f->d = dom->d;
  f->nl = dom->nl;
  f->nfull = (int)all.size();
  f->nm = (int)sel.size();
  f->single = single;
  const int d = f->d;
  for (int k = 0; k < d; ++k) {  // finest_geometry (combine.hpp:85-91)
    const int cells = dom->root_cells[k] << dom->nl;
    f->fine_ext[k] = cells + (dom->bc[k] == SGWG_ZERO ? 1 : 0);
    f->fine_h[k] = std::ldexp((dom->upper[k] - dom->lower[k]) / dom->root_cells[k], -dom->nl);
  }
  f->finest = 1;
  for (int k = 0; k < d; ++k) f->finest *= f->fine_ext[k];
  long long off = 0;
  for (int gi : sel) {
    const auto& lv = all[gi];
    const MemberDesc M = geom_desc(dom, lv, off);
    f->hmem.push_back(M);
    f->gidx.push_back(gi);
    f->levels.push_back(lv);
    off += M.npts;
  }
  f->total = off;
  f->state_total = off;
  f->no_fused2d = std::getenv("SGWG_NO_FUSED2D") != nullptr;
  CK(cudaEventCreate(&f->ev0));
  CK(cudaEventCreate(&f->ev1));
  CK(cudaEventCreate(&f->evs0));
  CK(cudaEventCreate(&f->evs1));
  CK(cudaStreamCreateWithFlags(&f->side, cudaStreamNonBlocking));
  CK(cudaEventCreateWithFlags(&f->evfork, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&f->evjoin, cudaEventDisableTiming));
  {
    int lo = 0, hi = 0;  // the x pass's stream at the lowest priority
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    CK(cudaStreamCreateWithPriority(&f->side2, cudaStreamNonBlocking, lo));
  }
  CK(cudaEventCreateWithFlags(&f->evfork2, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&f->evjoin2, cudaEventDisableTiming));
  int st = build_tasks(f);
  if (st != SGWG_OK) return st;
  CK(cudaMalloc(&f->dmem, sizeof(MemberDesc) * std::max(1, f->nm)));
  CK(cudaMemcpy(f->dmem, f->hmem.data(), sizeof(MemberDesc) * f->nm, cudaMemcpyHostToDevice));
  // (+2 doubles: the whole-plane 4D pass stages 16-byte-aligned spans that may
  // round one double past a member's end)
  const size_t bytes = sizeof(double) * (std::max<long long>(1, f->total) + 2);
  CK(cudaMalloc(&f->u, bytes));
  CK(cudaMalloc(&f->A, bytes));
  CK(cudaMalloc(&f->B, bytes));
  CK(cudaMalloc(&f->K, bytes));
  CK(cudaMemset(f->u, 0, bytes));  // make_family: zero states (combine.hpp:79)
  CK(cudaMalloc(&f->amax, sizeof(unsigned long long) * 3 * std::max(1, f->nm)));
  CK(cudaMalloc(&f->fail, sizeof(unsigned long long) * std::max(1, f->nm)));
  CK(cudaMalloc(&f->ctl, sizeof(StepCtl)));
  CK(cudaMalloc(&f->d_dtp, sizeof(DtParams)));
  CK(cudaMalloc(&f->counter, sizeof(unsigned int)));
  CK(cudaMemset(f->counter, 0, sizeof(unsigned int)));
  CK(cudaMallocHost(&f->hctl, sizeof(StepCtl)));
  std::memset(f->hctl, 0, sizeof(StepCtl));
  *out = f;
  return SGWG_OK;
}

template <class T>
int upload_vec(T** dptr, const std::vector<T>& v);

int setup_vp(sgwg_family* f) {
  const int dx = f->model.space_dim;
  if (dx < 1 || dx > 2 || f->d != 2 * dx)
    return fail_with(SGWG_EINVAL, "kinetic model: grid rank must be twice the space dimension");
  long long xoff = 0;
  for (auto& M : f->hmem) {
    M.nx = 1;
    for (int k = 0; k < dx; ++k) M.nx *= M.ext[k];
    M.vn = (int)(M.npts / M.nx);
    M.xext[0] = M.ext[0];
    M.xext[1] = (dx == 2) ? M.ext[1] : 1;
    M.xoff = xoff;
    // the charge density in partial sums over up to kRhoParts chunks of the
    // velocity block, so long blocks are integrated by several warps
    M.rparts = std::max(1, std::min(kRhoParts, (M.vn + 127) / 128));
    xoff += M.nx;
    if (f->model.kind == SGWG_VLASOV_POISSON) {
      for (int k = 0; k < dx; ++k)
        if (M.bc[k] != SGWG_PERIODIC)
          return fail_with(SGWG_EINVAL, "Vlasov-Poisson: x directions must be periodic");
      if (M.nx > 2048) return fail_with(SGWG_EUNSUPPORTED, "Vlasov-Poisson: x-grid > 2048 points");
      for (int k = 0; k < dx; ++k)
        if ((M.ext[k] & (M.ext[k] - 1)) != 0)
          return fail_with(SGWG_EUNSUPPORTED, "Vlasov-Poisson: x extents must be powers of two");
    }
  }
  f->nx_total = xoff;
  CK(cudaMemcpy(f->dmem, f->hmem.data(), sizeof(MemberDesc) * f->nm, cudaMemcpyHostToDevice));
  {  // combination coefficients of the local members (combine.hpp:34-43, 116)
    std::vector<double> cf;
    const int d = f->d;
    for (int mi = 0; mi < f->nm; ++mi) {
      int ls = 0;
      for (int k = 0; k < d; ++k) ls += f->levels[mi][k];
      const int j = f->nl - ls;
      cf.push_back(f->single ? 1.0 : (double)((j % 2 == 0 ? 1 : -1) * binomial(d - 1, j)));
    }
    cudaFree(f->dcoef);
    f->dcoef = nullptr;
    TRY(upload_vec(&f->dcoef, cf));
  }
  {  // field-energy groups: members sharing an x-grid, in member order
    std::vector<std::pair<int, int>> keys;
    std::vector<std::vector<int>> mem;
    for (int mi = 0; mi < f->nm; ++mi) {
      const std::pair<int, int> k(f->hmem[mi].xext[0], f->hmem[mi].xext[1]);
      size_t g = 0;
      while (g < keys.size() && keys[g] != k) ++g;
      if (g == keys.size()) {
        keys.push_back(k);
        mem.emplace_back();
      }
      mem[g].push_back(mi);
    }
    std::vector<int4> gd;
    std::vector<int2> gm;
    std::vector<int> gmem;
    int off = 0, gx = 0;
    for (size_t g = 0; g < keys.size(); ++g) {
      const int nxg = keys[g].first * keys[g].second;
      gd.push_back(make_int4(keys[g].first, keys[g].second, off, gx));
      gm.push_back(make_int2((int)gmem.size(), (int)mem[g].size()));
      gmem.insert(gmem.end(), mem[g].begin(), mem[g].end());
      off += nxg * dx;
      gx += nxg;
    }
    cudaFree(f->degrp);
    cudaFree(f->degrp_m);
    cudaFree(f->degrp_mem);
    cudaFree(f->egrid);
    f->degrp = nullptr;
    f->degrp_m = nullptr;
    f->degrp_mem = nullptr;
    f->egrid = nullptr;
    TRY(upload_vec(&f->degrp, gd));
    TRY(upload_vec(&f->degrp_m, gm));
    TRY(upload_vec(&f->degrp_mem, gmem));
    CK(cudaMalloc(&f->egrid, sizeof(double) * std::max(1, off)));
    f->egrp_tsum = 0;  // doubles of one finest row's group interpolants (energy_rows_kernel)
    for (size_t g = 0; g < keys.size(); ++g) f->egrp_tsum += 2 * keys[g].second;
    cudaFree(f->eparts);
    cudaFree(f->edone);
    f->eparts = nullptr;
    f->edone = nullptr;
    CK(cudaMalloc(&f->eparts, sizeof(double) * std::max(1, f->fine_ext[0]) * kEnergyRing));
    CK(cudaMalloc(&f->edone, sizeof(unsigned int) * (kEnergyRing + 1)));
    CK(cudaMemset(f->edone, 0, sizeof(unsigned int) * (kEnergyRing + 1)));
    cudaFree(f->ering);
    cudaFree(f->erecorded);
    f->ering = nullptr;
    f->erecorded = nullptr;
    f->ering_stride = (long long)xoff * dx;
    CK(cudaMalloc(&f->ering, sizeof(double) * std::max<long long>(1, f->ering_stride) * kEnergyRing));
    CK(cudaMalloc(&f->erecorded, sizeof(long long)));
    CK(cudaMemset(f->erecorded, 0, sizeof(long long)));
    {  // classes of groups sharing the x2 extent (energy_row_cls)
      std::vector<int> ext;
      for (const auto& k : keys) ext.push_back(k.second);
      std::sort(ext.begin(), ext.end());
      ext.erase(std::unique(ext.begin(), ext.end()), ext.end());
      int tsum = 0;
      bool ok = ext.size() <= 8 && keys.size() < 64 && dx == 2;
      for (int e : ext) {
        tsum += 2 * e;
        ok = ok && e > 0 && (e & (e - 1)) == 0 && f->fine_ext[1] % e == 0 && f->fine_ext[1] / e <= 128;
      }
      ok = ok && tsum <= 1024;
      f->ecls_n = ok ? (int)ext.size() : 0;
      if (ok) {
        for (size_t k = 0; k < ext.size(); ++k) f->ecls_n1[k] = ext[k];
        for (size_t g = 0; g < keys.size(); ++g)
          f->egrp_cls[g] = (unsigned char)(std::find(ext.begin(), ext.end(), keys[g].second) - ext.begin());
      }
    }
    cudaFree(f->egrid_b);
    f->egrid_b = nullptr;
    f->egrid_stride = std::max(1, off);
    CK(cudaMalloc(&f->egrid_b, sizeof(double) * f->egrid_stride * kEnergyRing));
    f->negrp = (int)keys.size();
    f->ngx = gx;
  }
  if (f->model.kind == SGWG_VLASOV_POISSON && f->rho == nullptr) {
    CK(cudaMalloc(&f->rho, sizeof(double) * std::max<long long>(1, xoff)));
    CK(cudaMalloc(&f->E, sizeof(double) * std::max<long long>(1, xoff * dx)));
    CK(cudaMalloc(&f->emax, sizeof(double) * std::max(1, f->nm * dx)));
    CK(cudaMalloc(&f->rho_parts, sizeof(double) * std::max<long long>(1, xoff) * kRhoParts));
  }
  {  // FFT twiddles for the largest x-grid line of the family
    int hmax = 1;
    for (const auto& M : f->hmem) hmax = std::max(hmax, std::max(M.xext[0], M.xext[1]) / 2);
    cudaFree(f->twid);
    f->twid = nullptr;
    CK(cudaMalloc(&f->twid, sizeof(double) * 2 * hmax));
    CK(launch_twiddles(f->twid, hmax, f->ctx->stream));
    CK(cudaStreamSynchronize(f->ctx->stream));
    f->hmax = hmax;
  }
  f->parts_of = nullptr;
  return SGWG_OK;
}

// moment kernel work: 8 (x point, velocity chunk) items -- one warp each -- per
// CTA; rebuilt whenever the members' partial counts change (plane tiling)
int build_moment_tasks(sgwg_family* f) {
  std::vector<int2> mt;
  for (int mi = 0; mi < f->nm; ++mi) {
    const MemberDesc& M = f->hmem[mi];
    for (int q0 = 0; q0 < M.nx * M.rparts; q0 += 8) mt.push_back(make_int2(mi, q0));
  }
  cudaFree(f->dmtasks);
  f->dmtasks = nullptr;
  f->nmtasks = (int)mt.size();
  TRY(upload_vec(&f->dmtasks, mt));
  return SGWG_OK;
}

// Vlasov-Maxwell: per member nx = x2 points, the (xi1, xi2) block, the packed
// offset of its field lines; the member state is f followed by E1, E2, B3
// (initialize_family, models.hpp:855-871).
int setup_vm(sgwg_family* f) {
  long long xoff = 0;
  for (auto& M : f->hmem) {
    M.nx = M.ext[0];
    M.vn = M.ext[1] * M.ext[2];
    M.xext[0] = M.ext[0];
    M.xext[1] = 1;
    M.xoff = xoff;
    M.rparts = 1;
    xoff += M.nx;
  }
  CK(cudaMemcpy(f->dmem, f->hmem.data(), sizeof(MemberDesc) * f->nm, cudaMemcpyHostToDevice));
  for (double** b : {&f->Fu, &f->FA, &f->FB}) {
    cudaFree(*b);
    *b = nullptr;
    CK(cudaMalloc(b, sizeof(double) * std::max<long long>(1, 3 * xoff)));
    CK(cudaMemset(*b, 0, sizeof(double) * std::max<long long>(1, 3 * xoff)));
  }
  cudaFree(f->vmspd);
  f->vmspd = nullptr;
  CK(cudaMalloc(&f->vmspd, sizeof(double) * 2 * std::max(1, f->nm)));
  f->state_total = f->total + 3 * xoff;
  return SGWG_OK;
}

// Fast 4D plane tiles (kernels.cuh plane_fast_kernel).  Pair pr covers the
// planes of dims (2pr, 2pr+1); a tile holds nv consecutive planes (>= 4 for
// pr = 0, whose planes interleave in memory, so loads use whole sectors), split
// into windows of multiples of 8 (+1) points when a plane exceeds the point
// cap.  Caps: <= 2048 points (8 per thread) and <= 9000 doubles of shared
// memory (3 CTAs per SM).  For Vlasov-Poisson the number of windows of a
// velocity plane is the member's count of charge-density partials.
int build_plane_tiles(sgwg_family* f) {
  for (int pr = 0; pr < 2; ++pr) {
    cudaFree(f->dptiles[pr]);
    f->dptiles[pr] = nullptr;
    f->nptiles[pr] = 0;
  }
  f->psmem = 0;
  const sgwg_model& m = f->model;
  if (f->d != 4 || f->no_fused2d || f->nm == 0) return SGWG_OK;
  if (m.kind != SGWG_ADVECTION && m.kind != SGWG_VLASOV_POISSON) return SGWG_OK;
  if (m.kind == SGWG_VLASOV_POISSON && m.space_dim != 2) return SGWG_OK;
  int cap = 2048;
  if (const char* e = std::getenv("SGWG_PLANE_CAP")) cap = std::max(256, std::min(2048, std::atoi(e)));
  int smem_cap = 9000;
  if (const char* e = std::getenv("SGWG_PLANE_SMEM")) smem_cap = std::max(2000, std::atoi(e));
  auto piece = [](int n, int k) { return std::min(n, ((n + k - 1) / k + 7) / 8 * 8); };
  std::vector<PlaneTile> t[2];
  std::vector<int> rparts(f->nm, 1);
  int smax = 0;
  for (int mi = 0; mi < f->nm; ++mi) {
    const MemberDesc& M = f->hmem[mi];
    if (M.npts >= (1LL << 31)) return SGWG_OK;  // 32-bit member-local offsets
    for (int pr = 0; pr < 2; ++pr) {
      const int na = M.ext[2 * pr], nb = M.ext[2 * pr + 1];
      const int nplanes = (pr == 0) ? M.ext[2] * M.ext[3] : M.ext[0] * M.ext[1];
      const int vmin = (pr == 0) ? std::min(4, nplanes) : 1;
      auto fits = [&](int V, int pa, int pb) {
        return V * pa * pb <= cap && fast::plane_smem_doubles(V, pa, pb) <= smem_cap;
      };
      int ka = 1, kb = 1;
      while (!fits(vmin, piece(na, ka), piece(nb, kb))) {
        const int pa = piece(na, ka), pb = piece(nb, kb);
        if (pa >= pb && pa > 8)
          ++ka;
        else if (pb > 8)
          ++kb;
        else
          return fail_with(SGWG_EINVAL, "plane tiling: no window fits");
      }
      const int pa = piece(na, ka), pb = piece(nb, kb);
      int V = vmin;
      if (pa == na && pb == nb)
        while (V < kPlaneMaxV && V < nplanes && fits(V + 1, na, nb)) ++V;
      int part = 0;
      for (int i0 = 0; i0 < na; i0 += pa)
        for (int j0 = 0; j0 < nb; j0 += pb, ++part) {
          const int tx = std::min(pa, na - i0), ty = std::min(pb, nb - j0);
          for (int p0 = 0; p0 < nplanes; p0 += V) {
            const int nv = std::min(V, nplanes - p0);
            t[pr].push_back(PlaneTile{mi, p0, nv, part, i0, j0, tx, ty});
            smax = std::max(smax, fast::plane_smem_doubles(nv, tx, ty));
          }
        }
      if (pr == 1) {
        if (part > kRhoParts) return SGWG_OK;  // (no such member in the BASELINE families)
        rparts[mi] = part;
      }
    }
  }
  for (int mi = 0; mi < f->nm; ++mi) f->hmem[mi].rparts = rparts[mi];
  CK(cudaMemcpy(f->dmem, f->hmem.data(), sizeof(MemberDesc) * f->nm, cudaMemcpyHostToDevice));
  for (int pr = 0; pr < 2; ++pr) {
    f->nptiles[pr] = (int)t[pr].size();
    TRY(upload_vec(&f->dptiles[pr], t[pr]));
  }
  f->psmem = smax;
  f->parts_of = nullptr;
  return SGWG_OK;
}

// Whole-plane 4D tiles (plane4d.cuh).  The family qualifies when dims (0, 1)
// are periodic with power-of-two extents >= 8 and an x-plane of <= 2048
// points, and dims (2, 3) are zero-ghost lines of 8m + 1 >= 9 points with a
// velocity plane of < 4096 points (every BASELINE C5 member; SGWG_PLANE4=0
// keeps the windowed plane kernels).  x pass: the whole x-plane times C
// consecutive velocity points, X C ~ 4096; v pass: G whole velocity planes,
// G V ~ SGWG_P4_VTARGET (3072) points.  One charge-density partial per x point.
int build_plane4_tiles(sgwg_family* f) {
  for (int pass = 0; pass < 2; ++pass) {
    cudaFree(f->dp4tiles[pass]);
    f->dp4tiles[pass] = nullptr;
    f->np4tiles[pass] = 0;
    f->p4smem[pass] = 0;
  }
  const sgwg_model& m = f->model;
  if (f->d != 4 || f->no_fused2d || f->nm == 0 || arith_of(f) != SGWG_ARITH_FAST) return SGWG_OK;
  if (m.kind != SGWG_ADVECTION && !(m.kind == SGWG_VLASOV_POISSON && m.space_dim == 2))
    return SGWG_OK;
  if (const char* e = std::getenv("SGWG_PLANE4"))
    if (e[0] == '0') return SGWG_OK;
  if (f->dom.bc[0] != SGWG_PERIODIC || f->dom.bc[1] != SGWG_PERIODIC ||
      f->dom.bc[2] != SGWG_ZERO || f->dom.bc[3] != SGWG_ZERO)
    return SGWG_OK;
  auto pow2 = [](int n) { return n >= 8 && (n & (n - 1)) == 0; };
  for (const auto& M : f->hmem) {
    const int X = M.ext[0] * M.ext[1], V = M.ext[2] * M.ext[3];
    if (!pow2(M.ext[0]) || !pow2(M.ext[1]) || X > 2048) return SGWG_OK;
    if (M.ext[2] < 9 || M.ext[3] < 9 || (M.ext[2] & 7) != 1 || (M.ext[3] & 7) != 1 || V >= 4096)
      return SGWG_OK;
  }
  // persistent v pass (SGWG_P4_PERSIST, default on): six tile slots per CTA, two CTAs per SM
  bool persist = true;
  if (const char* e = std::getenv("SGWG_P4_PERSIST")) persist = (e[0] != '0');
  // (2,330: two planes of the 9 x 129 / 17 x 65 / 33 x 33 shapes -- 2 x 1,161 points -- fit)
  int vtarget = persist ? 2330 : 2400;
  if (const char* e = std::getenv("SGWG_P4_VTARGET")) vtarget = std::max(64, std::atoi(e));
  int xtarget = 4096;
  if (const char* e = std::getenv("SGWG_P4_XTARGET")) xtarget = std::max(128, std::atoi(e));
  std::vector<int4> t[2];
  for (int mi = 0; mi < f->nm; ++mi) {
    const MemberDesc& M = f->hmem[mi];
    const int X = M.ext[0] * M.ext[1], V = M.ext[2] * M.ext[3];
    int cs = ((X << 1) <= xtarget) ? 1 : 0;
    while (cs < 6 && (X << (cs + 1)) <= xtarget) ++cs;
    const int C = 1 << cs;
    for (int v0 = 0; v0 < V; v0 += C) t[0].push_back(make_int4(mi, v0, std::min(C, V - v0), cs));
    f->p4smem[0] = std::max(f->p4smem[0], 3 * (X << cs));  // u, d/dx1, d/dx2
    const int G = std::max(1, std::min(kP4MaxG, vtarget / V));
    for (int x0 = 0; x0 < X; x0 += G) {
      const int g = std::min(G, X - x0);
      t[1].push_back(make_int4(mi, x0, g, 0));
      f->p4smem[1] = std::max(f->p4smem[1], 5 * ((g * V + 3) & ~1));  // u, K, u^n, dv1, dv2
    }
  }
  f->p4vpitch = 0;
  f->p4xpitch = 0;
  if (persist) {
    int xp = 0;
    for (const int4& q : t[0]) xp = std::max(xp, (f->hmem[q.x].ext[0] * f->hmem[q.x].ext[1]) << q.w);
    xp = (xp + 1) & ~1;
    // U0, U1, d/dx1 + ~1.2 KB static + 1 KB reserved per CTA, two CTAs in 228 KB.
    // Opt-in (SGWG_P4_XPERSIST=1): measured slower than the one-tile-per-CTA x pass
    // on C5 (150 vs 138 us per launch), unlike the v pass (209 vs 218 us)
    const char* xe = std::getenv("SGWG_P4_XPERSIST");
    if (xe != nullptr && xe[0] == '1' && 3LL * xp * 8 + 1800 <= 115712) {
      f->p4xpitch = xp;
      f->p4smem[0] = 3 * xp;
      std::vector<P4XTile> xt;
      const int sd = m.space_dim;
      for (const int4& q : t[0]) {
        const MemberDesc& M = f->hmem[q.x];
        P4XTile x{};
        x.src = M.offset + q.y;
        x.ih1 = M.inv_h[0];
        x.ih2 = M.inv_h[1];
        if (m.kind == SGWG_VLASOV_POISSON) {  // kinetic x lines: c = v_j (models.hpp:341-344)
          x.ca0 = M.lower[sd + 0];
          x.ca1 = M.h[sd + 0];
          x.cb0 = M.lower[sd + 1];
          x.cb1 = M.h[sd + 1];
        } else {  // advection speeds of dims 0, 1
          x.ca0 = m.speeds[0];
          x.cb0 = m.speeds[1];
        }
        x.V = M.ext[2] * M.ext[3];
        x.cs = q.w;
        x.nc = q.z;
        x.n1 = M.ext[0];
        x.n2 = M.ext[1];
        x.n4 = M.ext[3];
        x.v0 = q.y;
        x.mi = q.x;
        xt.push_back(x);
      }
      cudaFree(f->dp4xtiles);
      f->dp4xtiles = nullptr;
      TRY(upload_vec(&f->dp4xtiles, xt));
      if (f->dp4xsched == nullptr) {
        CK(cudaMalloc(&f->dp4xsched, 2 * sizeof(unsigned int)));
        CK(cudaMemset(f->dp4xsched, 0, 2 * sizeof(unsigned int)));
      }
    }
    int pitch = 0;
    for (const int4& q : t[1]) {
      const int V = f->hmem[q.x].ext[2] * f->hmem[q.x].ext[3];
      pitch = std::max(pitch, (q.z * V + 3) & ~1);
    }
    // 6 slots + ~2.5 KB static + 1 KB reserved per CTA, two CTAs in 228 KB
    if (6LL * pitch * 8 + 2600 <= 115712) {
      f->p4vpitch = pitch;
      f->p4smem[1] = 6 * pitch;
    }
  }
  if (f->p4vpitch > 0) {  // persistent v pass: a descriptor per tile (plane4d.cuh VInfo)
    std::vector<P4VTile> vt;
    for (const int4& q : t[1]) {
      const MemberDesc& M = f->hmem[q.x];
      P4VTile v{};
      v.mi = q.x;
      v.x0 = q.y;
      v.G = q.z;
      v.n3 = M.ext[2];
      v.n4 = M.ext[3];
      v.V = v.n3 * v.n4;
      v.NT = v.G * v.V;
      v.gs = M.offset + (long long)v.x0 * v.V;
      v.ga = v.gs & ~1LL;
      v.shift = (int)(v.gs - v.ga);
      v.nbytes = (unsigned)((((v.gs + v.NT + 1) & ~1LL) - v.ga) * 8);
      v.xoff = M.xoff;
      v.nx = M.nx;
      v.ih3 = M.inv_h[2];
      v.ih4 = M.inv_h[3];
      v.hh = M.h[2] * M.h[3];
      vt.push_back(v);
    }
    cudaFree(f->dp4vtiles);
    f->dp4vtiles = nullptr;
    TRY(upload_vec(&f->dp4vtiles, vt));
    if (f->dp4sched == nullptr) {
      CK(cudaMalloc(&f->dp4sched, 2 * sizeof(unsigned int)));
      CK(cudaMemset(f->dp4sched, 0, 2 * sizeof(unsigned int)));
    }
  }
  for (int mi = 0; mi < f->nm; ++mi) f->hmem[mi].rparts = 1;
  CK(cudaMemcpy(f->dmem, f->hmem.data(), sizeof(MemberDesc) * f->nm, cudaMemcpyHostToDevice));
  for (int pass = 0; pass < 2; ++pass) {
    f->np4tiles[pass] = (int)t[pass].size();
    TRY(upload_vec(&f->dp4tiles[pass], t[pass]));
  }
  f->parts_of = nullptr;
  return SGWG_OK;
}

void clear_graphs(sgwg_family* f) {
  for (auto& kv : f->graphs) cudaGraphExecDestroy(kv.second);
  f->graphs.clear();
}

int get_graph(sgwg_family* f, int nsteps, cudaGraphExec_t* exec) {
  auto it = f->graphs.find(nsteps);
  if (it != f->graphs.end()) {
    *exec = it->second;
    return SGWG_OK;
  }
  cudaGraph_t g;
  const long long saved = f->stats.kernel_launches;
  if (f->tl == nullptr && std::getenv("SGWG_STAMPS") != nullptr) {
    CK(cudaMalloc(&f->tl, sizeof(long long) * kStampSlots));
    CK(cudaMemset(f->tl, 0, sizeof(long long) * kStampSlots));
  }
  CK(cudaStreamBeginCapture(f->ctx->stream, cudaStreamCaptureModeThreadLocal));
  for (int s = 0; s < nsteps; ++s) {
    int st = launch_step(f, false);
    if (st != SGWG_OK) {
      cudaStreamEndCapture(f->ctx->stream, &g);
      return st;
    }
  }
  if (f->ering_step) {  // the chunk's energy records in one launch
    int st = launch_energy_batch(f, nsteps);
    if (st != SGWG_OK) {
      cudaStreamEndCapture(f->ctx->stream, &g);
      return st;
    }
  }
  CK(cudaStreamEndCapture(f->ctx->stream, &g));
  f->stats.kernel_launches = saved;
  cudaGraphExec_t e;
  // per-node priorities (the side streams' kernels below the critical path's): without the
  // flag every node runs at the priority of the stream the graph is launched into
  CK(cudaGraphInstantiate(&e, g, std::getenv("SGWG_NO_NODE_PRIO") ? 0 : cudaGraphInstantiateFlagUseNodePriority));
  CK(cudaGraphDestroy(g));
  f->graphs[nsteps] = e;
  *exec = e;
  return SGWG_OK;
}

int launches_per_step(const sgwg_family* f) {
  const bool fused3d = f->d == 3 && f->ntiles3d_fast > 0 && arith_of(f) == SGWG_ARITH_FAST &&
                       f->model.kind == SGWG_ADVECTION;
  const int np = ((f->d == 2 && f->ntiles2d > 0) || fused3d) ? 1
                 : (plane_path(f) || plane4_path(f))         ? 2
                                                             : (int)pass_order(f).size();
  int n = 3 * np;
  if (!dt_fusable(f)) n += 1;
  if (f->model.kind == SGWG_VLASOV_MAXWELL) n += 3 + 1;  // field lines per stage, speeds
  if (f->model.kind == SGWG_VLASOV_POISSON) {  // (moment +) field per stage, energy per step
    const long long fine_x = (long long)f->fine_ext[0] *
                             ((f->model.space_dim == 2) ? f->fine_ext[1] : 1);
    n += (plane_path(f) || plane4_path(f)) ? 3 : 6;
    // the energy record: per step, or (captured chunks) batched per chunk -- counted there
    if (!energy_batched(f, false))
      n += energy_rows_form(f) ? 1 : ((fine_x * f->nm > (1LL << 20)) ? 2 : 1);
  }
  if (f->comm != nullptr) n += 1;
  return n;
}

int read_failure(sgwg_family* f, sgwg_failure* fail) {
  std::vector<unsigned long long> h(f->nm);
  CK(cudaMemcpy(h.data(), f->fail, sizeof(unsigned long long) * f->nm, cudaMemcpyDeviceToHost));
  // evolve_family steps members serially, so the reported failure is the
  // lowest member index among those failing at the earliest step
  unsigned long long best_step = ULLONG_MAX;
  for (auto c : h)
    if (c != ULLONG_MAX) best_step = std::min(best_step, c / 4);
  for (int mi = 0; mi < f->nm; ++mi)
    if (h[mi] != ULLONG_MAX && h[mi] / 4 == best_step) {
      if (fail) {
        fail->member = f->gidx[mi];
        fail->step = (long long)(h[mi] / 4);
        fail->stage = (int)(h[mi] % 4);
      }
      return fail_with(SGWG_ENONFINITE, "integrator failure at step " + std::to_string(best_step));
    }
  if (fail) {  // failure on another rank (propagated through the all-reduce)
    fail->member = -1;
    fail->step = -1;
    fail->stage = 0;
  }
  return fail_with(SGWG_ENONFINITE, "integrator failure on another rank");
}

// ---- prolongation / combination plans ----

void free_plan(ProlongPlan* pl) {
  if (pl == nullptr) return;
  for (auto& dm : pl->dims) {
    cudaFree(dm.tasks);
    cudaFree(dm.src);
    cudaFree(dm.dst);
    cudaFree(dm.slot_member);
    cudaFree(dm.slot_n);
    cudaFree(dm.slot_ext);
    cudaFree(dm.item0);
  }
  for (double* p : pl->owned) cudaFree(p);
  cudaFree(pl->fsrc);
  cudaFree(pl->fcoef);
  cudaFree(pl->fext);
  cudaFree(pl->fref);
  delete pl;
}

template <class T>
int upload_vec(T** dptr, const std::vector<T>& v) {
  CK(cudaMalloc(dptr, sizeof(T) * std::max<size_t>(1, v.size())));
  if (!v.empty()) CK(cudaMemcpy(*dptr, v.data(), sizeof(T) * v.size(), cudaMemcpyHostToDevice));
  return SGWG_OK;
}

constexpr int kUpsampleChunk = 2048;

// ---------------------------------------------------------------------------
// Option B for sharded families: prolongation is dimension-
// sequential with dimension 0 first (interp.hpp:217-244), so the finest grid
// splits into independent dimension-0 row slabs.  Every rank gathers all
// member states (C5: 96.5 MB) and combines ITS rows for every member, in
// family order -- bitwise the single-GPU result, no all-reduce of the finest
// grid (C5: 34.6 GB).  Used by sgwg_combined_stats (5 doubles reduced across
// ranks), sgwg_eval_points (every rank evaluates all points) and
// sgwg_combine_local (this rank's rows, the result left sharded); forced for a
// one-rank communicator by SGWG_OPTION_B=1, disabled by SGWG_COMBINE_ALLREDUCE=1.
// ---------------------------------------------------------------------------
bool use_option_b(const sgwg_family* f) {
  if (f->comm == nullptr || f->single || f->state_total != f->total || f->d < 2) return false;
  if (std::getenv("SGWG_COMBINE_ALLREDUCE") != nullptr) return false;
  if (f->nranks > 1) return true;
  const char* e = std::getenv("SGWG_OPTION_B");
  return e != nullptr && e[0] == '1';
}

// rows [a, b) of dimension 0 that rank r combines
void option_b_rows(const sgwg_family* f, int r, long long* a, long long* b) {
  const long long rows = f->fine_ext[0];
  *a = rows * r / f->nranks;
  *b = rows * (r + 1) / f->nranks;
}

// the layout of the gathered states (once per family): owners from an NCCL
// all-gather of ownership flags; rank r's block holds its members in family
// order, exactly its local state buffer
int build_gathered_view(sgwg_family* f) {
  if (f->gview) return SGWG_OK;
  const int nfull = f->nfull, R = f->nranks;
  cudaStream_t s = f->ctx->stream;
  std::vector<int> own(nfull, 0), all((size_t)nfull * R, 0);
  for (int g : f->gidx) own[g] = 1;
  int *down = nullptr, *dall = nullptr;
  CK(cudaMalloc(&down, sizeof(int) * nfull));
  CK(cudaMalloc(&dall, sizeof(int) * nfull * R));
  CK(cudaMemcpyAsync(down, own.data(), sizeof(int) * nfull, cudaMemcpyHostToDevice, s));
  ncclResult_t nr = ncclAllGather(down, dall, nfull, ncclInt32, f->comm, s);
  if (nr == ncclSuccess) {
    CK(cudaMemcpyAsync(all.data(), dall, sizeof(int) * nfull * R, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
  }
  cudaFree(down);
  cudaFree(dall);
  if (nr != ncclSuccess) return fail_with(SGWG_ENCCL, ncclGetErrorString(nr));
  const auto levels = enumerate_levels(f->d, f->nl);
  std::vector<int> owner(nfull, -1);
  for (int g = 0; g < nfull; ++g)
    for (int r = 0; r < R; ++r)
      if (all[(size_t)r * nfull + g]) {
        if (owner[g] >= 0) return fail_with(SGWG_EINVAL, "shards overlap: a member on two ranks");
        owner[g] = r;
      }
  for (int g = 0; g < nfull; ++g)
    if (owner[g] < 0) return fail_with(SGWG_EINVAL, "shards do not cover the family");
  f->grank_cnt.assign(R, 0);
  f->ghmem.clear();
  std::vector<long long> local(nfull);
  for (int g = 0; g < nfull; ++g) {
    f->ghmem.push_back(geom_desc(&f->dom, levels[g], 0));
    local[g] = f->grank_cnt[owner[g]];
    f->grank_cnt[owner[g]] += f->ghmem.back().npts;
  }
  f->grank_off.assign(R, 0);
  for (int r = 1; r < R; ++r) f->grank_off[r] = f->grank_off[r - 1] + f->grank_cnt[r - 1];
  const long long total = f->grank_off[R - 1] + f->grank_cnt[R - 1];
  for (int g = 0; g < nfull; ++g) f->ghmem[g].offset = f->grank_off[owner[g]] + local[g];
  if (f->grank_cnt[f->rank] != f->total)
    return fail_with(SGWG_EINVAL, "gathered view: this rank's block differs from its states");
  CK(cudaMalloc(&f->gu, sizeof(double) * std::max(1LL, total)));
  TRY(upload_vec(&f->gdmem, f->ghmem));
  f->gview = true;
  return SGWG_OK;
}

// every rank's member states into gu (grouped broadcasts: blocks differ in size)
int gather_states(sgwg_family* f) {
  TRY(build_gathered_view(f));
  cudaStream_t s = f->ctx->stream;
  CKN(ncclGroupStart());
  for (int r = 0; r < f->nranks; ++r) {
    double* dst = f->gu + f->grank_off[r];
    const void* src = (r == f->rank) ? (const void*)f->u : (const void*)dst;
    ncclResult_t nr = ncclBroadcast(src, dst, (size_t)f->grank_cnt[r], ncclDouble, r, f->comm, s);
    if (nr != ncclSuccess) {
      ncclGroupEnd();
      return fail_with(SGWG_ENCCL, ncclGetErrorString(nr));
    }
  }
  CKN(ncclGroupEnd());
  return SGWG_OK;
}

// doubles of intermediate storage a plan for fine rows [a, b) of dimension 0 needs
// The members a combination reads: the family's own (local) members, or -- for a
// sharded family combined by row slabs (option B) -- every member of the family,
// gathered from all ranks (gview).  partial: the sum covers only this rank's
// members (all-reduced across ranks afterwards).
struct CombView {
  const std::vector<MemberDesc>* hmem;
  const MemberDesc* dmem;
  const double* u;
  std::map<std::pair<long long, long long>, ProlongPlan*>* cache;
  bool partial;
};
CombView local_view(sgwg_family* f) {
  return CombView{&f->hmem, f->dmem, f->u, &f->slab_plans, true};
}
CombView gathered_view(sgwg_family* f) {
  return CombView{&f->ghmem, f->gdmem, f->gu, &f->gslab_plans, false};
}

long long plan_doubles(const sgwg_family* f, const CombView& v, const std::vector<int>& mis,
                       long long a, long long b) {
  const int d = f->d;
  long long tot = 0;
  for (int mi : mis) {
    const MemberDesc& M = (*v.hmem)[mi];
    long long ext[4];
    for (int q = 0; q < 4; ++q) ext[q] = (q < d) ? M.ext[q] : 1;
    for (int k = 0; k + 1 < d; ++k) {
      if (f->nl - M.level[k] == 0) {
        if (k == 0) ext[0] = b - a;  // row view of the member
        continue;
      }
      ext[k] = (k == 0) ? (b - a) : f->fine_ext[k];
      long long n = 1;
      for (int q = 0; q < d; ++q) n *= ext[q];
      tot += n;
    }
  }
  return tot;
}
long long plan_doubles(sgwg_family* f, const std::vector<int>& mis, long long a, long long b) {
  return plan_doubles(f, local_view(f), mis, a, b);
}

// Prolongation plan of members `mis` restricted to fine rows [a, b) of
// dimension 0 (the whole grid for a = 0, b = fine_ext[0]).  Prolongation is
// dimension-sequential with dimension 0 first (interp.hpp:217-244), so after
// the dimension-0 sweep every row of the finest grid is independent: a slab
// of rows needs only its own rows of the intermediates.  Intermediates are
// carved from `arena` (or one owned allocation when arena is null).
int build_plan(sgwg_family* f, const CombView& v, const std::vector<int>& mis, long long a,
               long long b, double* arena, ProlongPlan** out) {
  ProlongPlan* pl = new ProlongPlan();
  const int d = f->d;
  std::vector<long long> coefs(d);
  for (int j = 0; j < d; ++j) coefs[j] = (j % 2 == 0 ? 1 : -1) * binomial(d - 1, j);
  if (arena == nullptr) {
    const long long nd = plan_doubles(f, v, mis, a, b);
    if (nd > 0) {
      CK(cudaMalloc(&arena, sizeof(double) * nd));
      pl->owned.push_back(arena);
    }
  }
  long long carved = 0;
  pl->row_a = a;
  pl->row_b = b;
  // current array and extents per member
  std::vector<const double*> cur(mis.size());
  std::vector<std::array<int, 4>> ext(mis.size());
  for (size_t s = 0; s < mis.size(); ++s) {
    const MemberDesc& M = (*v.hmem)[mis[s]];
    cur[s] = v.u + M.offset;
    for (int q = 0; q < 4; ++q) ext[s][q] = (q < d) ? M.ext[q] : 1;
    if (d > 1 && f->nl - M.level[0] == 0) {  // dimension 0 already finest: row view
      cur[s] += a * (M.npts / M.ext[0]);
      ext[s][0] = (int)(b - a);
    }
  }
  for (int k = 0; k + 1 < d; ++k) {
    std::vector<int2> tasks;
    std::vector<const double*> src;
    std::vector<double*> dst;
    std::vector<int> smember, sext;
    std::vector<long long> sn, item0;
    long long nitems = 0;
    bool chunked = (arith_of(f) == SGWG_ARITH_FAST);
    for (size_t s = 0; s < mis.size(); ++s) {
      const MemberDesc& M = (*v.hmem)[mis[s]];
      if (f->nl - M.level[k] == 0) continue;  // interp.hpp:219
      if (f->nl - M.level[k] > 7) chunked = false;  // kInterpTabMaxM
      {  // chunked work items: 8-point chunks along k x 32-line blocks
        long long outer = 1, inner = 1;
        for (int q = 0; q < d; ++q) {
          if (q < k) outer *= ext[s][q];
          if (q > k) inner *= ext[s][q];
        }
        const long long nch = (k == 0) ? (((b - 1) >> 3) - (a >> 3) + 1)
                                       : ((f->fine_ext[k] + 7) / 8);
        item0.push_back(nitems);
        nitems += nch * ((outer * inner + 31) / 32);
      }
      long long n = 1;
      for (int q = 0; q < d; ++q)
        n *= (q == k) ? (k == 0 ? (b - a) : f->fine_ext[k]) : ext[s][q];
      double* buf = arena + carved;
      carved += n;
      const int slot = (int)src.size();
      src.push_back(cur[s]);
      dst.push_back(buf);
      smember.push_back(mis[s]);
      for (int q = 0; q < 4; ++q) sext.push_back(ext[s][q]);
      sn.push_back(n);
      for (long long c = 0; c * kUpsampleChunk < n; ++c) tasks.push_back(make_int2(slot, (int)c));
      cur[s] = buf;
      ext[s][k] = (k == 0) ? (int)(b - a) : f->fine_ext[k];
    }
    auto& dm = pl->dims[k];
    dm.nslots = (int)src.size();
    dm.ntasks = (int)tasks.size();
    dm.nitems = chunked ? nitems : 0;
    dm.nrows0 = (int)(b - a);
    TRY(upload_vec(&dm.item0, item0));
    TRY(upload_vec(&dm.tasks, tasks));
    TRY(upload_vec(&dm.src, src));
    TRY(upload_vec(&dm.dst, dst));
    TRY(upload_vec(&dm.slot_member, smember));
    TRY(upload_vec(&dm.slot_n, sn));
    TRY(upload_vec(&dm.slot_ext, sext));
  }
  std::vector<const double*> fsrc;
  std::vector<double> fcoef;
  std::vector<int> fext, fref;
  for (size_t s = 0; s < mis.size(); ++s) {
    const MemberDesc& M = (*v.hmem)[mis[s]];
    int lsum = 0;
    for (int q = 0; q < d; ++q) lsum += M.level[q];
    fsrc.push_back(cur[s]);
    fcoef.push_back((double)coefs[f->nl - lsum]);  // combine.hpp:116
    fext.push_back(ext[s][d - 1]);
    fref.push_back(f->nl - M.level[d - 1]);
  }
  pl->nm = (int)mis.size();
  TRY(upload_vec(&pl->fsrc, fsrc));
  TRY(upload_vec(&pl->fcoef, fcoef));
  TRY(upload_vec(&pl->fext, fext));
  TRY(upload_vec(&pl->fref, fref));
  pl->href = fref;
  *out = pl;
  return SGWG_OK;
}

int build_plan(sgwg_family* f, const std::vector<int>& mis, long long a, long long b,
               double* arena, ProlongPlan** out) {
  return build_plan(f, local_view(f), mis, a, b, arena, out);
}

int run_plan(sgwg_family* f, const CombView& v, ProlongPlan* pl, int mode, double eps, int assign,
             double* out) {
  const int d = f->d;
  const bool fast_mode = arith_of(f) == SGWG_ARITH_FAST;
  for (int k = 0; k + 1 < d; ++k) {
    auto& dm = pl->dims[k];
    if (dm.ntasks == 0) continue;
    UpsampleParams p{};
    p.jrow0 = (k == 0) ? (int)pl->row_a : 0;
    p.mem = v.dmem;
    p.tasks = dm.tasks;
    p.src = dm.src;
    p.dst = dm.dst;
    p.slot_member = dm.slot_member;
    p.slot_n = dm.slot_n;
    p.slot_ext = dm.slot_ext;
    p.kdim = k;
    p.nl = f->nl;
    p.fine_ext = f->fine_ext[k];
    p.bc = f->dom.bc[k];
    p.mode = mode;
    p.eps = eps;
    p.chunk = kUpsampleChunk;
    p.slot_item0 = dm.item0;
    p.nitems = std::getenv("SGWG_UPSAMPLE_GENERIC") ? 0 : dm.nitems;
    p.nslots = dm.nslots;
    p.nrows0 = dm.nrows0;
    CK(fast_mode ? fast::launch_upsample(p, dm.ntasks, f->ctx->stream)
                 : exact::launch_upsample(p, dm.ntasks, f->ctx->stream));
    f->stats.combine_launches++;
  }
  FinalParams fp{};
  fp.mem = v.dmem;
  fp.src = pl->fsrc;
  fp.coef = pl->fcoef;
  fp.msrc_ext = pl->fext;
  fp.mrefine = pl->fref;
  fp.nm = pl->nm;
  fp.nm_host = (int)pl->href.size();
  fp.mref_host = pl->href.data();
  fp.d = d;
  fp.nl = f->nl;
  fp.fine_last = f->fine_ext[d - 1];
  // rows of the finest grid flattened over dims 0..d-2; this plan covers
  // dimension-0 rows [row_a, row_b)
  long long per_row0 = 1;  // finest points per dimension-0 row
  for (int q = 1; q < d; ++q) per_row0 *= f->fine_ext[q];
  fp.nfine = (d == 1) ? f->finest : (pl->row_b - pl->row_a) * per_row0;
  fp.row0 = (d == 1) ? 0 : pl->row_a * (per_row0 / f->fine_ext[d - 1]);
  fp.bc_last = f->dom.bc[d - 1];
  fp.mode = mode;
  fp.eps = eps;
  fp.assign = assign;
  fp.out = out;
  CK(fast_mode ? fast::launch_final(fp, f->ctx->stream) : exact::launch_final(fp, f->ctx->stream));
  f->stats.combine_launches++;
  return SGWG_OK;
}

int run_plan(sgwg_family* f, ProlongPlan* pl, int mode, double eps, int assign, double* out) {
  return run_plan(f, local_view(f), pl, mode, eps, assign, out);
}

int copy_out(sgwg_family* f, const double* dev, double* out, size_t n, int out_is_device) {
  if (out_is_device) {
    if (out != dev)
      CK(cudaMemcpyAsync(out, dev, sizeof(double) * n, cudaMemcpyDeviceToDevice, f->ctx->stream));
  } else {
    CK(cudaMemcpyAsync(out, dev, sizeof(double) * n, cudaMemcpyDeviceToHost, f->ctx->stream));
  }
  CK(cudaStreamSynchronize(f->ctx->stream));
  return SGWG_OK;
}

// device memory the combination may use for intermediates (SGWG_COMBINE_BUDGET_GB, default 24)
long long combine_budget_doubles() {
  const char* e = std::getenv("SGWG_COMBINE_BUDGET_GB");
  const double gb = e ? std::atof(e) : 24.0;
  return (long long)(gb * 1e9 / 8.0);
}

// combination of fine rows [a, b) of dimension 0 into out (host or device)
int combine_rows_impl(sgwg_family* f, const CombView& v, const std::vector<int>& mis, int mode,
                      double eps, long long a, long long b, double* out, int out_is_device) {
  const long long need = plan_doubles(f, v, mis, a, b);
  if (f->slab_arena_doubles < need) {
    for (auto* c : {&f->slab_plans, &f->gslab_plans}) {  // carved from the old arena
      for (auto& kv : *c) free_plan(kv.second);
      c->clear();
    }
    cudaFree(f->slab_arena);
    f->slab_arena = nullptr;
    f->slab_arena_doubles = 0;
    if (need > 0) CK(cudaMalloc(&f->slab_arena, sizeof(double) * need));
    f->slab_arena_doubles = need;
  }
  const long long per_row = (long long)(f->finest / f->fine_ext[0]);
  const long long nout = (b - a) * per_row;
  if (f->slab_out_doubles < nout && !out_is_device) {
    cudaFree(f->slab_out);
    f->slab_out = nullptr;
    f->slab_out_doubles = 0;
    CK(cudaMalloc(&f->slab_out, sizeof(double) * nout));
    f->slab_out_doubles = nout;
  }
  double* dst = out_is_device ? out : f->slab_out;
  ProlongPlan* pl = nullptr;
  const bool cache = ((int)mis.size() == (int)v.hmem->size());
  if (cache) {
    auto it = v.cache->find(std::make_pair(a, b));
    if (it != v.cache->end()) pl = it->second;
  }
  if (pl == nullptr) {
    TRY(build_plan(f, v, mis, a, b, f->slab_arena, &pl));
    if (cache) (*v.cache)[std::make_pair(a, b)] = pl;
  }
  CK(cudaEventRecord(f->ev0, f->ctx->stream));
  int st = run_plan(f, v, pl, mode, eps, 0, dst);
  if (st == SGWG_OK && v.partial && f->comm != nullptr && f->nranks > 1) {
    ncclResult_t r = ncclAllReduce(dst, dst, (size_t)nout, ncclDouble, ncclSum, f->comm,
                                   f->ctx->stream);
    if (r != ncclSuccess) st = fail_with(SGWG_ENCCL, ncclGetErrorString(r));
  }
  if (st == SGWG_OK) {
    CK(cudaEventRecord(f->ev1, f->ctx->stream));
    CK(cudaEventSynchronize(f->ev1));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, f->ev0, f->ev1));
    f->stats.combine_ms = ms;
    st = copy_out(f, dst, out, (size_t)nout, out_is_device);
  }
  if (!cache) free_plan(pl);
  return st;
}

int combine_rows_impl(sgwg_family* f, const std::vector<int>& mis, int mode, double eps,
                      long long a, long long b, double* out, int out_is_device) {
  return combine_rows_impl(f, local_view(f), mis, mode, eps, a, b, out, out_is_device);
}

int ensure_fine_buf(sgwg_family* f) {
  if (f->fine_buf == nullptr) CK(cudaMalloc(&f->fine_buf, sizeof(double) * f->finest));
  return SGWG_OK;
}

int require_model(const sgwg_family* f) {
  if (!f->has_model) return fail_with(SGWG_EINVAL, "sgwg_set_model not called");
  return SGWG_OK;
}

}  // namespace

// =========================================================================
// C ABI
// =========================================================================
extern "C" {

const char* sgwg_last_error(void) { return g_err.c_str(); }
int sgwg_version(void) { return 1; }

int sgwg_init(int device, sgwg_ctx** out) {
  if (out == nullptr) return fail_with(SGWG_EINVAL, "null ctx pointer");
  int n = 0;
  CK(cudaGetDeviceCount(&n));
  if (device < 0 || device >= n) return fail_with(SGWG_ECUDA, "no such CUDA device");
  CK(cudaSetDevice(device));
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10)
    return fail_with(SGWG_ECUDA, std::string("sm_100a build needs a Blackwell device, got ") +
                                     prop.name);
  sgwg_ctx* c = new sgwg_ctx();
  c->device = device;
  c->sm_count = prop.multiProcessorCount;
  {
    // the main stream above the default priority: kernels forked to the family's side
    // streams (default = lowest priority) must not be dispatched ahead of the critical path
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    if (const char* e = std::getenv("SGWG_MAIN_PRIO")) hi = std::atoi(e);
    CK(cudaStreamCreateWithPriority(&c->stream, cudaStreamNonBlocking, hi));
  }
  CK(exact::configure());
  CK(fast::configure());
  CK(configure_field());
  *out = c;
  return SGWG_OK;
}

int sgwg_shutdown(sgwg_ctx* ctx) {
  if (ctx == nullptr) return SGWG_OK;
  if (ctx->families > 0) {  // deferred: the last sgwg_family_destroy frees the context
    ctx->closing = true;
    return SGWG_OK;
  }
  cudaStreamDestroy(ctx->stream);
  delete ctx;
  return SGWG_OK;
}

int sgwg_set_arith(sgwg_ctx* ctx, int arith) {
  if (ctx == nullptr || (arith != SGWG_ARITH_EXACT && arith != SGWG_ARITH_FAST))
    return fail_with(SGWG_EINVAL, "bad arith mode");
  ctx->arith = arith;
  return SGWG_OK;
}

int sgwg_set_profile(sgwg_ctx* ctx, int on) {
  if (ctx == nullptr) return fail_with(SGWG_EINVAL, "null ctx");
  ctx->profile = on ? 1 : 0;
  return SGWG_OK;
}

void* sgwg_stream(sgwg_ctx* ctx) { return ctx ? (void*)ctx->stream : nullptr; }

int sgwg_enumerate_levels(int d, int nl, int* levels, int cap, int* count) {
  if (d < 1 || d > 4) return fail_with(SGWG_EINVAL, "enumerate_combination_levels: d must be 1..4");
  if (nl < d - 1) return fail_with(SGWG_EINVAL, "enumerate_combination_levels: need N_L >= d-1");
  auto v = enumerate_levels(d, nl);
  if (count) *count = (int)v.size();
  if (levels)
    for (int i = 0; i < (int)v.size() && i < cap; ++i)
      for (int k = 0; k < d; ++k) levels[i * d + k] = v[i][k];
  return SGWG_OK;
}

int sgwg_family_create(sgwg_ctx* ctx, const sgwg_domain* dom, sgwg_family** out) {
  return family_create(ctx, dom, nullptr, 0, out);
}

int sgwg_family_create_single(sgwg_ctx* ctx, const sgwg_domain* dom, sgwg_family** out) {
  return family_create(ctx, dom, nullptr, 0, out, true);
}

int sgwg_family_create_shard(sgwg_ctx* ctx, const sgwg_domain* dom, const int* members,
                             int count, sgwg_family** out) {
  if (members == nullptr || count < 0) return fail_with(SGWG_EINVAL, "bad shard member list");
  return family_create(ctx, dom, members, count, out);
}

int sgwg_family_destroy(sgwg_family* f) {
  if (f == nullptr) return SGWG_OK;
  cudaSetDevice(f->ctx->device);
  cudaStreamSynchronize(f->ctx->stream);
  clear_graphs(f);
  free_plan(f->full_plan);
  for (auto& kv : f->slab_plans) free_plan(kv.second);
  f->slab_plans.clear();
  for (auto& kv : f->gslab_plans) free_plan(kv.second);
  f->gslab_plans.clear();
  cudaFree(f->gdmem);
  cudaFree(f->gu);
  if (f->comm) ncclCommDestroy(f->comm);
  for (int k = 0; k < kMaxD; ++k) cudaFree(f->dtasks[k]);
  cudaFree(f->dmax_tasks);
  cudaFree(f->dmem);
  cudaFree(f->u);
  cudaFree(f->A);
  cudaFree(f->B);
  cudaFree(f->K);
  cudaFree(f->amax);
  cudaFree(f->fail);
  cudaFree(f->ctl);
  cudaFree(f->d_dtp);
  cudaFree(f->counter);
  cudaFree(f->dtiles2d);
  cudaFree(f->dtiles2d_fast);
  cudaFree(f->dtiles2d_half);
  cudaFree(f->dtiles2d_q);
  cudaFree(f->dtiles3d_fast);
  cudaFree(f->dptiles[0]);
  cudaFree(f->dptiles[1]);
  cudaFree(f->dp4tiles[0]);
  cudaFree(f->dp4tiles[1]);
  cudaFree(f->dp4vtiles);
  cudaFree(f->dp4sched);
  cudaFree(f->dp4xtiles);
  cudaFree(f->dp4xsched);
  cudaFree(f->rho_parts);
  cudaFree(f->twid);
  cudaFree(f->Fu);
  cudaFree(f->FA);
  cudaFree(f->FB);
  cudaFree(f->vmspd);
  cudaFree(f->degrp);
  cudaFree(f->degrp_m);
  cudaFree(f->degrp_mem);
  cudaFree(f->egrid);
  cudaFree(f->eparts);
  cudaFree(f->edone);
  cudaFree(f->ering);
  cudaFree(f->erecorded);
  cudaFree(f->egrid_b);
  cudaFree(f->fe);
  cudaFree(f->dcoef);
  cudaFreeHost(f->hctl);
  cudaFree(f->dts);
  cudaFree(f->rho);
  cudaFree(f->E);
  cudaFree(f->emax);
  cudaFree(f->dmtasks);
  cudaFree(f->fine_buf);
  cudaFree(f->diag_slab);
  cudaFree(f->diag_scratch);
  cudaFree(f->slab_arena);
  cudaFree(f->slab_out);
  cudaEventDestroy(f->ev0);
  cudaEventDestroy(f->ev1);
  cudaEventDestroy(f->evs0);
  cudaEventDestroy(f->evs1);
  cudaEventDestroy(f->evfork);
  cudaEventDestroy(f->evjoin);
  cudaStreamDestroy(f->side);
  cudaFree(f->tl);
  cudaEventDestroy(f->evfork2);
  cudaEventDestroy(f->evjoin2);
  cudaStreamDestroy(f->side2);
  sgwg_ctx* ctx = f->ctx;
  delete f;
  if (--ctx->families == 0 && ctx->closing) {
    cudaStreamDestroy(ctx->stream);
    delete ctx;
  }
  return SGWG_OK;
}

int sgwg_family_num_members(const sgwg_family* f, int* count) {
  if (f == nullptr || count == nullptr) return fail_with(SGWG_EINVAL, "null argument");
  *count = f->nm;
  return SGWG_OK;
}

int sgwg_family_member(const sgwg_family* f, int mi, int* global_index, int* levels, int* points) {
  if (f == nullptr || mi < 0 || mi >= f->nm) return fail_with(SGWG_EINVAL, "bad member index");
  if (global_index) *global_index = f->gidx[mi];
  for (int k = 0; k < f->d; ++k) {
    if (levels) levels[k] = f->levels[mi][k];
    if (points) points[k] = f->hmem[mi].ext[k];
  }
  return SGWG_OK;
}

int sgwg_family_sizes(const sgwg_family* f, size_t* member_points, size_t* finest_points) {
  if (f == nullptr) return fail_with(SGWG_EINVAL, "null family");
  if (member_points) *member_points = (size_t)f->state_total;
  if (finest_points) *finest_points = (size_t)f->finest;
  return SGWG_OK;
}

}  // extern "C"

namespace {

// member states <-> device buffers: one copy, or (Vlasov-Maxwell) the
// distribution and the field lines of every member separately
int copy_states(sgwg_family* f, double* host_or_dev, bool to_device, cudaMemcpyKind kind,
                double* dist = nullptr, double* fields = nullptr) {
  cudaStream_t s = f->ctx->stream;
  if (dist == nullptr) dist = f->u;
  if (fields == nullptr) fields = f->Fu;
  if (f->state_total == f->total) {
    if (to_device)
      CK(cudaMemcpyAsync(dist, host_or_dev, sizeof(double) * f->total, kind, s));
    else
      CK(cudaMemcpyAsync(host_or_dev, dist, sizeof(double) * f->total, kind, s));
  } else {
    long long so = 0;
    for (const auto& M : f->hmem) {
      double* a = host_or_dev + so;
      double* b = host_or_dev + so + M.npts;
      if (to_device) {
        CK(cudaMemcpyAsync(dist + M.offset, a, sizeof(double) * M.npts, kind, s));
        CK(cudaMemcpyAsync(fields + 3 * M.xoff, b, sizeof(double) * 3 * M.nx, kind, s));
      } else {
        CK(cudaMemcpyAsync(a, dist + M.offset, sizeof(double) * M.npts, kind, s));
        CK(cudaMemcpyAsync(b, fields + 3 * M.xoff, sizeof(double) * 3 * M.nx, kind, s));
      }
      so += M.npts + 3 * M.nx;
    }
  }
  CK(cudaStreamSynchronize(s));
  return SGWG_OK;
}

}  // namespace

extern "C" {

int sgwg_family_upload(sgwg_family* f, const double* host, size_t n) {
  if (f == nullptr || host == nullptr || n != (size_t)f->state_total)
    return fail_with(SGWG_EINVAL, "upload: size must equal the packed member states");
  CK(cudaSetDevice(f->ctx->device));
  f->parts_of = nullptr;
  return copy_states(f, const_cast<double*>(host), true, cudaMemcpyHostToDevice);
}

int sgwg_family_download(sgwg_family* f, double* host, size_t n) {
  if (f == nullptr || host == nullptr || n != (size_t)f->state_total)
    return fail_with(SGWG_EINVAL, "download: size must equal the packed member states");
  CK(cudaSetDevice(f->ctx->device));
  return copy_states(f, host, false, cudaMemcpyDeviceToHost);
}

int sgwg_family_upload_device(sgwg_family* f, const double* dev, size_t n) {
  if (f == nullptr || dev == nullptr || n != (size_t)f->state_total)
    return fail_with(SGWG_EINVAL, "upload: size must equal the packed member states");
  f->parts_of = nullptr;
  return copy_states(f, const_cast<double*>(dev), true, cudaMemcpyDeviceToDevice);
}

int sgwg_family_download_device(sgwg_family* f, double* dev, size_t n) {
  if (f == nullptr || dev == nullptr || n != (size_t)f->state_total)
    return fail_with(SGWG_EINVAL, "download: size must equal the packed member states");
  return copy_states(f, dev, false, cudaMemcpyDeviceToDevice);
}

int sgwg_set_model(sgwg_family* f, const sgwg_model* m) {
  if (f == nullptr || m == nullptr) return fail_with(SGWG_EINVAL, "null argument");
  if (m->kind < SGWG_ADVECTION || m->kind > SGWG_VLASOV_MAXWELL)
    return fail_with(SGWG_EINVAL, "unknown model kind");
  if (m->kind == SGWG_VLASOV_MAXWELL &&
      (f->d != 3 || f->dom.bc[0] != SGWG_PERIODIC || f->dom.bc[1] != SGWG_ZERO ||
       f->dom.bc[2] != SGWG_ZERO))  // VmWorkspace::make (models.hpp:389-393)
    return fail_with(SGWG_EINVAL, "VmWorkspace: need rank 3, periodic x2 and zero xi boundaries");
  if (m->kind == SGWG_VLASOV_BOLTZMANN)
    return fail_with(SGWG_EUNSUPPORTED,
                     "Vlasov-Boltzmann relaxation is outside the B200 hot path (SURVEY 2.1)");
  if (!(m->epsilon > 0.0)) return fail_with(SGWG_EINVAL, "WENO epsilon must be positive");
  // weno_derivative_line: periodic lines need >= 6 points (weno.hpp:122-123)
  for (const auto& M : f->hmem)
    for (int k = 0; k < f->d; ++k)
      if (M.bc[k] == SGWG_PERIODIC && M.ext[k] < 6)
        return fail_with(SGWG_EINVAL, "weno_derivative_line: periodic line too short");
  f->model = *m;
  f->has_model = true;
  if (m->kind == SGWG_VLASOV_POISSON) TRY(setup_vp(f));
  if (m->kind == SGWG_VLASOV_MAXWELL) TRY(setup_vm(f));
  TRY(build_plane_tiles(f));
  TRY(build_plane4_tiles(f));
  if (m->kind == SGWG_VLASOV_POISSON) TRY(build_moment_tasks(f));
  clear_graphs(f);
  return SGWG_OK;
}

int sgwg_nccl_unique_id(void* id128) {
  if (id128 == nullptr) return fail_with(SGWG_EINVAL, "null id");
  ncclUniqueId id;
  CKN(ncclGetUniqueId(&id));
  std::memcpy(id128, &id, sizeof(id));
  return SGWG_OK;
}

int sgwg_family_set_comm(sgwg_family* f, const void* id128, int nranks, int rank) {
  if (f == nullptr || id128 == nullptr || nranks < 1 || rank < 0 || rank >= nranks)
    return fail_with(SGWG_EINVAL, "bad communicator arguments");
  CK(cudaSetDevice(f->ctx->device));
  ncclUniqueId id;
  std::memcpy(&id, id128, sizeof(id));
  if (f->comm) ncclCommDestroy(f->comm);
  CKN(ncclCommInitRank(&f->comm, nranks, id, rank));
  f->nranks = nranks;
  f->rank = rank;
  clear_graphs(f);
  return SGWG_OK;
}

int sgwg_evolve(sgwg_family* f, const sgwg_policy* pol, double tfinal, const double* stops_in,
                int nstops, sgwg_stop_cb on_stop, void* user, double* dts, size_t cap,
                size_t* nsteps, sgwg_failure* fail) {
  if (f == nullptr || pol == nullptr) return fail_with(SGWG_EINVAL, "null argument");
  TRY(require_model(f));
  if (tfinal < 0.0) return fail_with(SGWG_EINVAL, "evolve_family: negative final time");
  if (pol->mode == SGWG_DT_ACCURACY && !(pol->reference_spacing > 0.0))
    return fail_with(SGWG_EINVAL, "compute_dt: reference spacing must be positive");
  if (pol->mode == SGWG_DT_CFL && !(pol->cfl > 0.0))
    return fail_with(SGWG_EINVAL, "compute_dt: cfl must be positive");
  CK(cudaSetDevice(f->ctx->device));
  TRY(overflow_guard(f));
  cudaStream_t s = f->ctx->stream;
  // stop list (timestep.hpp:133-142)
  const double eps_dedupe = 1e-12 * std::max(1.0, tfinal);
  std::vector<double> stops(stops_in, stops_in + std::max(0, nstops));
  stops.push_back(tfinal);
  std::sort(stops.begin(), stops.end());
  stops.erase(std::remove_if(stops.begin(), stops.end(),
                             [&](double x) { return x <= 0.0 || x > tfinal + eps_dedupe; }),
              stops.end());
  stops.erase(std::unique(stops.begin(), stops.end(),
                          [&](double a, double b) { return std::abs(a - b) <= eps_dedupe; }),
              stops.end());
  if (stops.empty()) stops.push_back(tfinal);
  const double eps_t = 1e-12 * std::max(1.0, tfinal);

  // dt parameters (compute_dt, timestep.hpp:47-67; family_wave_speeds models.hpp:791-839)
  DtParams dp{};
  dp.ctl = f->ctl;
  dp.kind = f->model.kind;
  dp.mode = pol->mode;
  dp.cfl = pol->cfl;
  if (pol->mode == SGWG_DT_ACCURACY) {
    double b = std::pow(pol->reference_spacing, 5.0 / 3.0);
    if (pol->dt_scale != 1.0) b = pol->dt_scale * b;
    dp.base_dt = b;
  }
  for (int k = 0; k < f->d; ++k) dp.fine_h[k] = f->fine_h[k];
  if (f->model.kind == SGWG_ADVECTION) {
    for (int k = 0; k < f->d; ++k) dp.const_speeds[k] = std::abs(f->model.speeds[k]);
  } else if (f->model.kind == SGWG_VLASOV_MAXWELL) {
    // s0 = max(1, max|xi2|) over the members (models.hpp:825-826)
    double s0 = 0.0;
    for (const auto& M : f->hmem) {
      double m0 = 1.0;
      for (int i = 0; i < M.ext[2]; ++i) m0 = std::max(m0, std::abs(M.lower[2] + i * M.h[2]));
      s0 = std::max(s0, m0);
    }
    dp.const_speeds[0] = s0;
  } else if (f->model.kind == SGWG_VLASOV_POISSON) {
    const int dx = f->model.space_dim;
    for (int j = 0; j < dx; ++j)
      dp.const_speeds[j] =
          std::max(std::abs(f->dom.lower[dx + j]), std::abs(f->dom.upper[dx + j]));
  }
  dp.d = f->d;
  dp.space_dim = f->model.space_dim;
  dp.amax = f->amax;
  dp.emax = f->emax;
  dp.vmspd = f->vmspd;
  dp.nmembers = f->nm;
  dp.fail = f->fail;
  // dt record buffer
  const long long want_cap = (long long)std::max<size_t>(cap, 1);
  if (f->dts_cap < want_cap) {
    cudaFree(f->dts);
    CK(cudaMalloc(&f->dts, sizeof(double) * want_cap));
    f->dts_cap = want_cap;
    clear_graphs(f);
  }
  if (f->model.kind == SGWG_VLASOV_POISSON) {  // per-step ||E||_2 record
    if (f->fe_cap < f->dts_cap) {
      cudaFree(f->fe);
      CK(cudaMalloc(&f->fe, sizeof(double) * f->dts_cap));
      f->fe_cap = f->dts_cap;
      clear_graphs(f);
    }
    CK(cudaMemsetAsync(f->fe, 0, sizeof(double) * f->fe_cap, s));
    if (f->erecorded != nullptr) CK(cudaMemsetAsync(f->erecorded, 0, sizeof(long long), s));
  }
  dp.dts = f->dts;
  dp.dts_cap = f->dts_cap;
  // graphs bake the policy in: rebuild when it changes
  const long long key = (long long)std::hash<std::string>()(
      std::string((const char*)&dp, sizeof(DtParams) - 0));
  if (key != f->graph_key_policy) {
    clear_graphs(f);
    f->graph_key_policy = key;
  }
  f->dtp = dp;
  CK(cudaMemcpyAsync(f->d_dtp, &f->dtp, sizeof(DtParams), cudaMemcpyHostToDevice, s));

  // initial state of the device loop
  std::memset(f->hctl, 0, sizeof(StepCtl));
  f->hctl->t = 0.0;
  f->hctl->eps_t = eps_t;
  f->hctl->active = 1;
  CK(cudaMemcpyAsync(f->ctl, f->hctl, sizeof(StepCtl), cudaMemcpyHostToDevice, s));
  CK(cudaMemsetAsync(f->fail, 0xff, sizeof(unsigned long long) * f->nm, s));
  if (f->model.kind == SGWG_BURGERS) TRY(launch_member_max_slot0(f));

  f->stats.evolve_ms = 0;
  f->stats.steps = 0;
  f->stats.kernel_launches = 0;
  f->stats.pass_ms_sum = 0;
  f->stats.pass_launches = 0;
  f->stats.pass_flops = 0;
  f->stats.pass_bytes = 0;
  const int lps = launches_per_step(f);
  // small 2D families (fast build, single rank): persistent cooperative kernel
  PersistParams pp{};
  int persist_blocks = 0;
  // 1024-point tiles, two CTAs per SM (measured: C2 34.6 -> 34.3 ms against 2048-point
  // tiles, one per SM; 512-point tiles 35.7 ms), 512-point tiles, four per SM, when
  // the family has fewer 1024-point tiles than SMs (C1 30.2 -> 27.6 ms);
  // SGWG_PERSIST_TILE=2048 / 1024 / 512 force one
  int nsm = 148;
  {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  }
  int pcode = (f->ntiles2d_half < nsm) ? 2 : 1;
  if (const char* e = std::getenv("SGWG_PERSIST_TILE")) {
    if (std::string(e) == "2048") pcode = 0;
    if (std::string(e) == "1024") pcode = 1;
    if (std::string(e) == "512") pcode = 2;
  }
  const int pntiles = (pcode == 2) ? f->ntiles2d_q : (pcode == 1) ? f->ntiles2d_half
                                                                  : f->ntiles2d_fast;
  const int pts_tile = 2048 >> pcode;
  // + the resident tile (stage input and u^n)
  const size_t persist_smem =
      ((size_t)((pcode == 2) ? f->smem2d_q : (pcode == 1) ? f->smem2d_half : f->smem2d_fast) +
       2 * pts_tile) * sizeof(double);
  if (arith_of(f) == SGWG_ARITH_FAST && f->d == 2 && pntiles > 0 && dt_fusable(f) &&
      !f->ctx->profile && std::getenv("SGWG_NO_PERSIST") == nullptr) {
    // one tile per CTA (tiles resident in shared memory across stages); larger
    // families run faster as graph-captured stage launches (measured: S2)
    const int maxb =
        fast::persist2d_max_blocks(f->model.kind == SGWG_BURGERS, pcode, persist_smem);
    persist_blocks = (pntiles <= maxb) ? pntiles : 0;
    const auto order = pass_order(f);
    Stage2DParams& p = pp.base;
    p.mem = f->dmem;
    p.tiles = (pcode == 2) ? f->dtiles2d_q : (pcode == 1) ? f->dtiles2d_half : f->dtiles2d_fast;
    p.ntiles = pntiles;
    p.half_tiles = pcode;
    p.burgers = f->model.kind == SGWG_BURGERS;
    p.flux0 = order[0].flux;
    p.flux1 = order[1].flux;
    p.c0 = order[0].c_const;
    p.c1 = order[1].c_const;
    p.linear = (f->model.weno_mode == SGWG_WENO_LINEAR);
    p.eps = f->model.epsilon;
    p.space_dim = f->model.space_dim;
    p.efield = f->E;
    p.ctl = f->ctl;
    p.amax_in = f->amax;
    p.amax_zero = f->amax;
    p.nmembers = f->nm;
    p.track_max = p.burgers;
    p.fail = f->fail;
    p.dtp = f->d_dtp;
    p.resident = (pntiles <= persist_blocks &&
                  std::getenv("SGWG_NO_RESIDENT") == nullptr) ? 1 : 0;
    pp.u = f->u;
    pp.A = f->A;
    pp.B = f->B;
  }
  double t_host = 0.0;
  double last_dt = (pol->mode == SGWG_DT_ACCURACY) ? dp.base_dt : 0.0;
  int status = SGWG_OK;
  for (double stop : stops) {
    if (stop > tfinal + eps_t) break;
    // set stop, reactivate (t, step, failure state persist)
    CK(cudaMemcpyAsync(&f->ctl->stop, &stop, sizeof(double), cudaMemcpyHostToDevice, s));
    f->hctl->active = 1;
    CK(cudaMemcpyAsync(&f->ctl->active, &f->hctl->active, sizeof(int), cudaMemcpyHostToDevice, s));
    CK(cudaEventRecord(f->ev0, s));
    if (dt_fusable(f) && persist_blocks == 0) TRY(launch_dt_step(f));  // then fused
    double seg_ms = 0.0;
    for (;;) {
      // how many steps to launch before looking: exact in accuracy mode,
      // estimated from the last dt in CFL mode (early-exit kernels absorb overshoot)
      long long est = 1;
      if (last_dt > 0.0) est = (long long)std::ceil((stop - t_host) / last_dt) + 1;
      est = std::max(1LL, std::min(est, 256LL));
      if (persist_blocks > 0) {
        pp.nsteps = (int)std::min<long long>(est, 512);
        CK(fast::launch_persist2d(pp, persist_blocks, persist_smem, s));
        f->stats.kernel_launches++;
      } else if (f->ctx->profile) {  // un-captured, every pass bracketed by events
        for (long long q = 0; q < est; ++q) TRY(launch_step(f, true));
      } else {
        long long left = est;
        while (left > 0) {
          int chunk = 1;
          while (chunk * 2 <= left && chunk < 64) chunk *= 2;
          // captured steps take the rho partials of u^n as given
          if (f->model.kind == SGWG_VLASOV_POISSON && (plane_path(f) || plane4_path(f)) &&
              f->parts_of != f->u)
            TRY(launch_field_for(f, f->u, 0));
          cudaGraphExec_t ge;
          TRY(get_graph(f, chunk, &ge));
          CK(cudaGraphLaunch(ge, s));
          f->stats.kernel_launches += (long long)chunk * lps;
          if (energy_batched(f, false))
            f->stats.kernel_launches += (energy_rows_form(f) && f->ecls_n > 0) ? 2 : 1;
          left -= chunk;
        }
      }
      CK(cudaMemcpyAsync(f->hctl, f->ctl, sizeof(StepCtl), cudaMemcpyDeviceToHost, s));
      CK(cudaStreamSynchronize(s));
      t_host = f->hctl->t;
      if (f->hctl->dt > 0.0) last_dt = f->hctl->dt;
      if (f->hctl->failed) {
        status = read_failure(f, fail);
        break;
      }
      if (!f->hctl->active) break;
    }
    CK(cudaEventRecord(f->ev1, s));
    CK(cudaEventSynchronize(f->ev1));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, f->ev0, f->ev1));
    seg_ms += ms;
    f->stats.evolve_ms += seg_ms;
    if (status != SGWG_OK) break;
    // land exactly on the stop (timestep.hpp:170)
    f->hctl->t = stop;
    t_host = stop;
    CK(cudaMemcpyAsync(&f->ctl->t, &stop, sizeof(double), cudaMemcpyHostToDevice, s));
    CK(cudaStreamSynchronize(s));
    if (on_stop) on_stop(stop, user);
  }
  CK(cudaMemcpyAsync(f->hctl, f->ctl, sizeof(StepCtl), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  TRY(dump_stamps(f));
  f->stats.steps = f->hctl->step;
  if (nsteps) *nsteps = (size_t)f->hctl->step;
  if (dts && cap > 0) {
    const size_t nn = std::min<size_t>(cap, (size_t)f->hctl->step);
    if (nn > 0) CK(cudaMemcpy(dts, f->dts, sizeof(double) * nn, cudaMemcpyDeviceToHost));
  }
  return status;
}

int sgwg_rk3_step(sgwg_family* f, double dt, sgwg_failure* fail) {
  if (f == nullptr) return fail_with(SGWG_EINVAL, "null family");
  TRY(require_model(f));
  if (!(dt > 0.0)) return fail_with(SGWG_EINVAL, "ssp_rk3_step: dt must be positive");
  CK(cudaSetDevice(f->ctx->device));
  TRY(overflow_guard(f));
  cudaStream_t s = f->ctx->stream;
  std::memset(f->hctl, 0, sizeof(StepCtl));
  f->hctl->active = 1;
  f->hctl->dt = dt;
  CK(cudaMemcpyAsync(f->ctl, f->hctl, sizeof(StepCtl), cudaMemcpyHostToDevice, s));
  CK(cudaMemsetAsync(f->fail, 0xff, sizeof(unsigned long long) * f->nm, s));
  if (f->model.kind == SGWG_BURGERS) TRY(launch_member_max_slot0(f));
  StageBufs s1{f->u, f->u, f->A}, s2{f->A, f->u, f->B}, s3{f->B, f->u, f->u};
  TRY(launch_stage(f, 1, s1, false));
  TRY(launch_stage(f, 2, s2, false));
  TRY(launch_stage(f, 3, s3, false));
  std::vector<unsigned long long> h(f->nm);
  CK(cudaMemcpyAsync(h.data(), f->fail, sizeof(unsigned long long) * f->nm,
                     cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  for (auto c : h)
    if (c != ULLONG_MAX) return read_failure(f, fail);
  return SGWG_OK;
}

int sgwg_vp_field(sgwg_family* f, double* rho, size_t nrho, double* E, size_t nE) {
  if (f == nullptr || rho == nullptr || E == nullptr) return fail_with(SGWG_EINVAL, "null argument");
  TRY(require_model(f));
  if (f->model.kind != SGWG_VLASOV_POISSON)
    return fail_with(SGWG_EINVAL, "vp_field: model is not Vlasov-Poisson");
  const int dx = f->model.space_dim;
  if (nrho != (size_t)f->nx_total || nE != (size_t)(f->nx_total * dx))
    return fail_with(SGWG_EINVAL, "vp_field: sizes must be (sum of x-points) and space_dim x that");
  CK(cudaSetDevice(f->ctx->device));
  std::memset(f->hctl, 0, sizeof(StepCtl));
  f->hctl->active = 1;
  CK(cudaMemcpyAsync(f->ctl, f->hctl, sizeof(StepCtl), cudaMemcpyHostToDevice, f->ctx->stream));
  TRY(launch_field_for(f, f->u, 0));
  CK(cudaMemcpyAsync(rho, f->rho, sizeof(double) * nrho, cudaMemcpyDeviceToHost, f->ctx->stream));
  CK(cudaMemcpyAsync(E, f->E, sizeof(double) * nE, cudaMemcpyDeviceToHost, f->ctx->stream));
  CK(cudaStreamSynchronize(f->ctx->stream));
  return SGWG_OK;
}

int sgwg_field_energy(sgwg_family* f, double* out, size_t cap, size_t* n) {
  if (f == nullptr || out == nullptr) return fail_with(SGWG_EINVAL, "null argument");
  if (f->model.kind != SGWG_VLASOV_POISSON || f->fe == nullptr)
    return fail_with(SGWG_EINVAL, "field_energy: no Vlasov-Poisson evolve recorded");
  // the record combines E over this rank's members only; the cross-rank sum
  // of the combined field is not formed, so a sharded family has no record
  if (f->comm != nullptr && f->nranks > 1)
    return fail_with(SGWG_EUNSUPPORTED,
                     "field_energy: not available on a sharded family (per-rank partial E)");
  const size_t steps = (size_t)std::min<long long>(f->stats.steps, f->fe_cap);
  const size_t m = std::min(cap, steps);
  if (m > 0) CK(cudaMemcpy(out, f->fe, sizeof(double) * m, cudaMemcpyDeviceToHost));
  for (size_t i = 0; i < m; ++i) out[i] = std::sqrt(out[i]);
  if (n) *n = m;
  return SGWG_OK;
}

int sgwg_time_stage(sgwg_family* f, int reps, double* avg_ms, double* flops, double* bytes) {
  if (f == nullptr || reps < 1 || avg_ms == nullptr) return fail_with(SGWG_EINVAL, "bad argument");
  TRY(require_model(f));
  CK(cudaSetDevice(f->ctx->device));
  cudaStream_t s = f->ctx->stream;
  // RK stage 1 (u -> A) is idempotent: launch it back to back between two events
  std::memset(f->hctl, 0, sizeof(StepCtl));
  f->hctl->active = 1;
  f->hctl->dt = 1e-9;
  CK(cudaMemcpyAsync(f->ctl, f->hctl, sizeof(StepCtl), cudaMemcpyHostToDevice, s));
  CK(cudaMemsetAsync(f->fail, 0xff, sizeof(unsigned long long) * f->nm, s));
  if (f->model.kind == SGWG_BURGERS) TRY(launch_member_max_slot0(f));
  StageBufs s1{f->u, f->u, f->A};
  const long long saved = f->stats.kernel_launches;
  TRY(launch_stage(f, 1, s1, false));  // warm-up
  CK(cudaEventRecord(f->ev0, s));
  for (int r = 0; r < reps; ++r) TRY(launch_stage(f, 1, s1, false));
  CK(cudaEventRecord(f->ev1, s));
  CK(cudaEventSynchronize(f->ev1));
  float ms = 0.f;
  CK(cudaEventElapsedTime(&ms, f->ev0, f->ev1));
  const long long nl = (f->stats.kernel_launches - saved) / (reps + 1);
  f->stats.kernel_launches = saved;
  *avg_ms = ms / reps / std::max(1LL, nl);
  const double pts = (double)f->total;
  const bool burgers = f->model.kind == SGWG_BURGERS;
  const int nd = (int)pass_order(f).size();
  if (flops) *flops = pts * ((burgers ? 142.0 : 70.0) * nd + 2.0) / std::max(1LL, nl);
  if (bytes) *bytes = pts * 16.0 / std::max(1LL, nl);
  return SGWG_OK;
}

int sgwg_rhs(sgwg_family* f, double* out, size_t n, int out_is_device) {
  if (f == nullptr || out == nullptr || n != (size_t)f->state_total)
    return fail_with(SGWG_EINVAL, "rhs: size must equal the packed member states");
  TRY(require_model(f));
  CK(cudaSetDevice(f->ctx->device));
  TRY(overflow_guard(f));
  cudaStream_t s = f->ctx->stream;
  std::memset(f->hctl, 0, sizeof(StepCtl));
  f->hctl->active = 1;
  CK(cudaMemcpyAsync(f->ctl, f->hctl, sizeof(StepCtl), cudaMemcpyHostToDevice, s));
  if (f->model.kind == SGWG_BURGERS) TRY(launch_member_max_slot0(f));
  StageBufs b{f->u, f->u, f->A};
  TRY(launch_stage(f, 0, b, false));
  if (f->state_total != f->total)  // Vlasov-Maxwell: tendency of f and of the field lines
    return copy_states(f, out, false, out_is_device ? cudaMemcpyDeviceToDevice
                                                    : cudaMemcpyDeviceToHost, f->A, f->FA);
  return copy_out(f, f->A, out, n, out_is_device);
}

}  // extern "C"

namespace {

// combination coefficient of each local member (combine.hpp:34-43, 116)
std::vector<double> member_coefs(const sgwg_family* f) {
  std::vector<double> cf;
  for (int mi = 0; mi < f->nm; ++mi) {
    int ls = 0;
    for (int k = 0; k < f->d; ++k) ls += f->levels[mi][k];
    const int j = f->nl - ls;
    cf.push_back(f->single ? 1.0 : (double)((j % 2 == 0 ? 1 : -1) * binomial(f->d - 1, j)));
  }
  return cf;
}

int check_interp(int mode, double eps) {
  if (mode != SGWG_INTERP_WENO && mode != SGWG_INTERP_LAGRANGE)
    return fail_with(SGWG_EINVAL, "unknown interpolation mode");
  if (mode == SGWG_INTERP_WENO && !(eps > 0.0))
    return fail_with(SGWG_EINVAL, "weno_interp5: epsilon must be positive");
  return SGWG_OK;
}

// Visit the combined finest-grid field in dimension-0 row slabs on the device:
// fn(dev, first_linear_index, points).  One slab when the whole grid fits the
// combination budget (or the family is a single grid).
template <class Fn>
int for_each_combined_slab(sgwg_family* f, int mode, double eps, Fn&& fn, bool own_rows = false) {
  CK(cudaSetDevice(f->ctx->device));
  if (f->single) return fn((const double*)f->u, 0LL, f->finest);
  if (own_rows && use_option_b(f)) {  // option B: this rank's rows, every member
    TRY(gather_states(f));
    const CombView v = gathered_view(f);
    std::vector<int> gm(f->nfull);
    for (int i = 0; i < f->nfull; ++i) gm[i] = i;
    long long ra, rb;
    option_b_rows(f, f->rank, &ra, &rb);
    const long long per_row = (long long)(f->finest / f->fine_ext[0]);
    long long slab = std::max(1LL, rb - ra);
    while (slab > 1 && plan_doubles(f, v, gm, 0, slab) > combine_budget_doubles()) slab = (slab + 1) / 2;
    if (f->diag_slab_doubles < slab * per_row) {
      cudaFree(f->diag_slab);
      f->diag_slab = nullptr;
      f->diag_slab_doubles = 0;
      CK(cudaMalloc(&f->diag_slab, sizeof(double) * slab * per_row));
      f->diag_slab_doubles = slab * per_row;
    }
    for (long long a = ra; a < rb; a += slab) {
      const long long b = std::min(rb, a + slab);
      TRY(combine_rows_impl(f, v, gm, mode, eps, a, b, f->diag_slab, 1));
      TRY(fn((const double*)f->diag_slab, a * per_row, (b - a) * per_row));
    }
    return SGWG_OK;
  }
  if (f->nm == 0 && f->comm == nullptr) return fail_with(SGWG_EINVAL, "combine: empty family");
  std::vector<int> mis(f->nm);
  for (int i = 0; i < f->nm; ++i) mis[i] = i;
  const long long rows = (f->d == 1) ? 1 : f->fine_ext[0];
  if (f->d == 1 || plan_doubles(f, mis, 0, rows) <= combine_budget_doubles()) {
    if (f->full_plan == nullptr) TRY(build_plan(f, mis, 0, rows, nullptr, &f->full_plan));
    TRY(ensure_fine_buf(f));
    TRY(run_plan(f, f->full_plan, mode, eps, 0, f->fine_buf));
    if (f->comm != nullptr && f->nranks > 1)
      CKN(ncclAllReduce(f->fine_buf, f->fine_buf, (size_t)f->finest, ncclDouble, ncclSum,
                        f->comm, f->ctx->stream));
    return fn((const double*)f->fine_buf, 0LL, f->finest);
  }
  const long long per_row = (long long)(f->finest / f->fine_ext[0]);
  long long slab = rows;
  while (slab > 1 && plan_doubles(f, mis, 0, slab) > combine_budget_doubles()) slab = (slab + 1) / 2;
  if (f->diag_slab_doubles < slab * per_row) {
    cudaFree(f->diag_slab);
    f->diag_slab = nullptr;
    CK(cudaMalloc(&f->diag_slab, sizeof(double) * slab * per_row));
    f->diag_slab_doubles = slab * per_row;
  }
  for (long long a = 0; a < rows; a += slab) {
    const long long b = std::min(rows, a + slab);
    TRY(combine_rows_impl(f, mis, mode, eps, a, b, f->diag_slab, 1));
    TRY(fn((const double*)f->diag_slab, a * per_row, (b - a) * per_row));
  }
  return SGWG_OK;
}

}  // namespace

extern "C" {

int sgwg_combined_stats(sgwg_family* f, int mode, double eps, int exact_preset, double t,
                        sgwg_field_stats* out) {
  if (f == nullptr || out == nullptr) return fail_with(SGWG_EINVAL, "null argument");
  TRY(check_interp(mode, eps));
  const bool burgers = f->has_model && f->model.kind == SGWG_BURGERS;
  if (exact_preset >= 0) {
    const bool adv_ok = f->has_model && f->model.kind == SGWG_ADVECTION &&
                        (exact_preset == SGWG_IC_C1 || exact_preset == SGWG_IC_C3 ||
                         exact_preset == SGWG_IC_EX1 || exact_preset == SGWG_IC_EX2);
    const bool bur_ok = burgers && ((exact_preset == SGWG_IC_C2 && f->d == 2) ||
                                    exact_preset == SGWG_IC_EX3);
    if (!adv_ok && !bur_ok)
      return fail_with(SGWG_EINVAL, "combined_stats: no exact solution for this model and preset");
  }
  CK(cudaSetDevice(f->ctx->device));
  if (f->diag_scratch == nullptr)
    CK(cudaMalloc(&f->diag_scratch, sizeof(double) * stats_partial_doubles()));
  StatsParams sp{};
  sp.d = f->d;
  for (int k = 0; k < f->d; ++k) {
    sp.ext[k] = f->fine_ext[k];
    sp.bc[k] = (f->dom.bc[k] == SGWG_PERIODIC) ? 0 : 1;
    sp.h[k] = f->fine_h[k];
    sp.lower[k] = f->dom.lower[k];
    sp.a[k] = (exact_preset >= 0 && !burgers) ? f->model.speeds[k] : 0.0;
  }
  sp.exact = exact_preset;
  sp.burgers = burgers ? 1 : 0;
  sp.t = t;
  sp.partial = f->diag_scratch;
  double mass = 0.0, mn = INFINITY, mx = -INFINITY, l1 = 0.0, linf = 0.0;
  f->stats.combine_launches = 0;
  CK(cudaEventRecord(f->evs0, f->ctx->stream));
  TRY(for_each_combined_slab(f, mode, eps, [&](const double* dev, long long first, long long n) -> int {
    StatsParams q = sp;
    q.field = dev;
    q.first = first;
    q.n = n;
    double h5[5];
    CK(launch_stats(q, f->diag_scratch + stats_partial_doubles() - 5, f->ctx->stream));
    f->stats.combine_launches += 2;
    CK(cudaMemcpyAsync(h5, f->diag_scratch + stats_partial_doubles() - 5, sizeof(h5),
                       cudaMemcpyDeviceToHost, f->ctx->stream));
    CK(cudaStreamSynchronize(f->ctx->stream));
    mass += h5[0];
    mn = std::min(mn, h5[1]);
    mx = std::max(mx, h5[2]);
    l1 += h5[3];
    linf = std::max(linf, h5[4]);
    return SGWG_OK;
  }, /*own_rows=*/true));
  if (use_option_b(f) && f->nranks > 1) {  // this rank's rows only: reduce across ranks
    double h[5] = {mass, l1, -mn, mx, linf};
    double* dh = f->diag_scratch;  // the stats partials are consumed
    CK(cudaMemcpyAsync(dh, h, sizeof(h), cudaMemcpyHostToDevice, f->ctx->stream));
    CKN(ncclAllReduce(dh, dh, 2, ncclDouble, ncclSum, f->comm, f->ctx->stream));
    CKN(ncclAllReduce(dh + 2, dh + 2, 3, ncclDouble, ncclMax, f->comm, f->ctx->stream));
    CK(cudaMemcpyAsync(h, dh, sizeof(h), cudaMemcpyDeviceToHost, f->ctx->stream));
    CK(cudaStreamSynchronize(f->ctx->stream));
    mass = h[0];
    l1 = h[1];
    mn = -h[2];
    mx = h[3];
    linf = h[4];
  }
  CK(cudaEventRecord(f->evs1, f->ctx->stream));
  CK(cudaEventSynchronize(f->evs1));
  float cms = 0.f;
  CK(cudaEventElapsedTime(&cms, f->evs0, f->evs1));
  f->stats.combine_ms = cms;
  out->mass = mass;
  out->min = mn;
  out->max = mx;
  out->points = (double)f->finest;
  out->l1 = (exact_preset >= 0) ? l1 / (double)f->finest : NAN;
  out->linf = (exact_preset >= 0) ? linf : NAN;
  return SGWG_OK;
}

int sgwg_kernel_profile(const sgwg_family* f, sgwg_kernel_timing* out, int cap, int* n) {
  if (f == nullptr || n == nullptr || (cap > 0 && out == nullptr))
    return fail_with(SGWG_EINVAL, "null argument");
  int i = 0;
  for (const auto& kv : f->kprof) {
    if (i < cap) out[i] = kv.second;
    ++i;
  }
  *n = i;
  return SGWG_OK;
}

int sgwg_kernel_profile_reset(sgwg_family* f) {
  if (f == nullptr) return fail_with(SGWG_EINVAL, "null argument");
  f->kprof.clear();
  return SGWG_OK;
}

const char* sgwg_stage_kernels(const sgwg_family* f) {
  if (f == nullptr || !f->has_model) return "";
  const bool fast = arith_of(f) == SGWG_ARITH_FAST;
  if (plane4_path(f))
    return f->p4vpitch > 0 ? (f->p4xpitch > 0 ? "xpass4d_persist_kernel + vpass4d_persist_kernel"
                                              : "xpass4d_kernel + vpass4d_persist_kernel")
                           : "xpass4d_kernel + vpass4d_kernel";
  if (plane_path(f)) return "plane_fast_kernel (x2)";
  if (f->d == 3 && f->ntiles3d_fast > 0 && fast && f->model.kind == SGWG_ADVECTION)
    return "stage3d_small_kernel";
  if (f->d == 2 && f->ntiles2d > 0)
    return fast ? "stage2d_quarter_kernel (evolve: evolve2d_persistent_kernel when co-resident)"
                : "stage2d_kernel";
  return "pass_kernel";
}

int sgwg_eval_points(sgwg_family* f, int mode, double eps, const int* idx, size_t npoints,
                     double* out) {
  if (f == nullptr || (npoints > 0 && (idx == nullptr || out == nullptr)))
    return fail_with(SGWG_EINVAL, "null argument");
  TRY(check_interp(mode, eps));
  for (size_t q = 0; q < npoints; ++q)
    for (int k = 0; k < f->d; ++k)
      if (idx[q * f->d + k] < 0 || idx[q * f->d + k] >= f->fine_ext[k])
        return fail_with(SGWG_EINVAL, "eval_points: index outside the finest grid");
  if (npoints == 0) return SGWG_OK;
  CK(cudaSetDevice(f->ctx->device));
  int* didx = nullptr;
  double *dcoef = nullptr, *dout = nullptr;
  // option B: every rank evaluates every point from the gathered states (no all-reduce)
  const bool optb = use_option_b(f);
  if (optb) TRY(gather_states(f));
  std::vector<double> cf = member_coefs(f);
  if (optb) {
    cf.clear();
    for (const MemberDesc& M : f->ghmem) {
      int ls = 0;
      for (int k = 0; k < f->d; ++k) ls += M.level[k];
      const int j = f->nl - ls;
      cf.push_back((double)((j % 2 == 0 ? 1 : -1) * binomial(f->d - 1, j)));  // combine.hpp:116
    }
  }
  const int nmv = optb ? f->nfull : f->nm;
  int st = SGWG_OK;
  auto fail_cuda = [&](cudaError_t e) {
    return (e == cudaSuccess) ? SGWG_OK : fail_with(SGWG_ECUDA, cudaGetErrorString(e));
  };
  st = fail_cuda(cudaMalloc(&didx, sizeof(int) * npoints * f->d));
  if (st == SGWG_OK) st = fail_cuda(cudaMalloc(&dcoef, sizeof(double) * std::max(1, nmv)));
  if (st == SGWG_OK) st = fail_cuda(cudaMalloc(&dout, sizeof(double) * npoints));
  if (st == SGWG_OK)
    st = fail_cuda(cudaMemcpyAsync(didx, idx, sizeof(int) * npoints * f->d,
                                   cudaMemcpyHostToDevice, f->ctx->stream));
  if (st == SGWG_OK && nmv > 0)
    st = fail_cuda(cudaMemcpyAsync(dcoef, cf.data(), sizeof(double) * nmv,
                                   cudaMemcpyHostToDevice, f->ctx->stream));
  if (st == SGWG_OK) {
    EvalParams p{};
    p.mem = optb ? f->gdmem : f->dmem;
    p.u = optb ? f->gu : f->u;
    p.coef = dcoef;
    p.idx = didx;
    p.npts = (long long)npoints;
    p.nm = nmv;
    p.d = f->d;
    p.nl = f->single ? f->levels[0][0] : f->nl;
    p.mode = mode;
    p.eps = eps;
    p.out = dout;
    st = fail_cuda(arith_of(f) == SGWG_ARITH_FAST ? fast::launch_eval_points(p, f->ctx->stream)
                                                   : exact::launch_eval_points(p, f->ctx->stream));
  }
  if (st == SGWG_OK && !optb && f->comm != nullptr && f->nranks > 1) {
    const ncclResult_t r = ncclAllReduce(dout, dout, npoints, ncclDouble, ncclSum, f->comm,
                                         f->ctx->stream);
    if (r != ncclSuccess) st = fail_with(SGWG_ENCCL, ncclGetErrorString(r));
  }
  if (st == SGWG_OK)
    st = fail_cuda(cudaMemcpyAsync(out, dout, sizeof(double) * npoints, cudaMemcpyDeviceToHost,
                                   f->ctx->stream));
  if (st == SGWG_OK) st = fail_cuda(cudaStreamSynchronize(f->ctx->stream));
  cudaFree(didx);
  cudaFree(dcoef);
  cudaFree(dout);
  return st;
}

int sgwg_write_snapshot(sgwg_family* f, int mode, double eps, const char* path) {
  if (f == nullptr || path == nullptr) return fail_with(SGWG_EINVAL, "null argument");
  TRY(check_interp(mode, eps));
  // FieldDumpHeader (io.hpp:17-26): magic, version, rank, extents, pad, spacings
  unsigned char hdr[64];
  std::memset(hdr, 0, sizeof(hdr));
  std::memcpy(hdr, "SGW5", 4);
  const uint32_t version = 1, dim = (uint32_t)f->d;
  std::memcpy(hdr + 4, &version, 4);
  std::memcpy(hdr + 8, &dim, 4);
  for (int k = 0; k < f->d; ++k) {
    const uint32_t e = (uint32_t)f->fine_ext[k];
    std::memcpy(hdr + 12 + 4 * k, &e, 4);
    std::memcpy(hdr + 32 + 8 * k, &f->fine_h[k], 8);
  }
  // sharded family: every rank takes part in the combination's all-reduce, rank 0 writes.
  // The writer's I/O failures are deferred (io_st) so that it still joins every
  // collective of the slab loop -- returning early would leave the other ranks
  // blocked inside ncclAllReduce.
  const bool writer = (f->comm == nullptr || f->rank == 0);
  FILE* fp = writer ? std::fopen(path, "wb") : nullptr;
  int io_st = SGWG_OK;
  if (writer && fp == nullptr)
    io_st = fail_with(SGWG_EINVAL, std::string("write_snapshot: cannot open ") + path);
  if (io_st == SGWG_OK && writer && std::fwrite(hdr, 1, sizeof(hdr), fp) != sizeof(hdr))
    io_st = fail_with(SGWG_EINVAL, "write_snapshot: write failed");
  double* host = nullptr;
  long long host_n = 0;
  int st = for_each_combined_slab(f, mode, eps, [&](const double* dev, long long, long long n) -> int {
    if (!writer || io_st != SGWG_OK) return SGWG_OK;
    if (host_n < n) {
      cudaFreeHost(host);
      host = nullptr;
      host_n = 0;
      if (cudaMallocHost(&host, sizeof(double) * n) != cudaSuccess) {
        io_st = fail_with(SGWG_ECUDA, "write_snapshot: pinned host buffer");
        return SGWG_OK;
      }
      host_n = n;
    }
    if (cudaMemcpyAsync(host, dev, sizeof(double) * n, cudaMemcpyDeviceToHost, f->ctx->stream) !=
            cudaSuccess ||
        cudaStreamSynchronize(f->ctx->stream) != cudaSuccess) {
      io_st = fail_with(SGWG_ECUDA, "write_snapshot: device-to-host copy");
      return SGWG_OK;
    }
    if (std::fwrite(host, sizeof(double), (size_t)n, fp) != (size_t)n)
      io_st = fail_with(SGWG_EINVAL, "write_snapshot: write failed");
    return SGWG_OK;
  });
  cudaFreeHost(host);
  if (fp != nullptr && std::fclose(fp) != 0 && io_st == SGWG_OK)
    io_st = fail_with(SGWG_EINVAL, "write_snapshot: close failed");
  return (st != SGWG_OK) ? st : io_st;
}

int sgwg_combine(sgwg_family* f, int mode, double eps, double* out, size_t n, int out_is_device) {
  if (f == nullptr || out == nullptr || n != (size_t)f->finest)
    return fail_with(SGWG_EINVAL, "combine: output size must equal the finest-grid points");
  if (mode != SGWG_INTERP_WENO && mode != SGWG_INTERP_LAGRANGE)
    return fail_with(SGWG_EINVAL, "unknown interpolation mode");
  if (mode == SGWG_INTERP_WENO && !(eps > 0.0))
    return fail_with(SGWG_EINVAL, "weno_interp5: epsilon must be positive");
  if (f->nm == 0 && f->comm == nullptr) return fail_with(SGWG_EINVAL, "combine: empty family");
  if (f->single) {  // runner.hpp:323-324: the single grid's field is the result
    f->stats.combine_ms = 0.0;
    return copy_out(f, f->u, out, n, out_is_device);
  }
  CK(cudaSetDevice(f->ctx->device));
  std::vector<int> mis(f->nm);
  for (int i = 0; i < f->nm; ++i) mis[i] = i;
  const long long rows = (f->d == 1) ? 1 : f->fine_ext[0];
  const long long full_need = plan_doubles(f, mis, 0, rows);
  f->stats.combine_launches = 0;
  if (f->d == 1 || full_need <= combine_budget_doubles()) {
    // whole finest grid in one plan (cached: pointers are stable for the family)
    if (f->full_plan == nullptr) TRY(build_plan(f, mis, 0, rows, nullptr, &f->full_plan));
    double* dst = out_is_device ? out : nullptr;
    if (dst == nullptr) {
      TRY(ensure_fine_buf(f));
      dst = f->fine_buf;
    }
    CK(cudaEventRecord(f->ev0, f->ctx->stream));
    TRY(run_plan(f, f->full_plan, mode, eps, 0, dst));
    if (f->comm != nullptr && f->nranks > 1)
      CKN(ncclAllReduce(dst, dst, (size_t)f->finest, ncclDouble, ncclSum, f->comm,
                        f->ctx->stream));
    CK(cudaEventRecord(f->ev1, f->ctx->stream));
    CK(cudaEventSynchronize(f->ev1));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, f->ev0, f->ev1));
    f->stats.combine_ms = ms;
    return copy_out(f, dst, out, n, out_is_device);
  }
  // too large for one plan (BASELINE C5: finest grid 4.3e9 points): slabs of
  // dimension-0 rows, each combined into its part of `out`
  const long long per_row = (long long)(f->finest / f->fine_ext[0]);
  long long slab = rows;
  while (slab > 1 && plan_doubles(f, mis, 0, slab) > combine_budget_doubles()) slab = (slab + 1) / 2;
  double ms_total = 0.0;
  for (long long a = 0; a < rows; a += slab) {
    const long long b = std::min(rows, a + slab);
    TRY(combine_rows_impl(f, mis, mode, eps, a, b, out + a * per_row, out_is_device));
    ms_total += f->stats.combine_ms;
  }
  f->stats.combine_ms = ms_total;
  return SGWG_OK;
}

int sgwg_combine_rows(sgwg_family* f, int mode, double eps, long long row_begin,
                      long long row_end, double* out, size_t n, int out_is_device) {
  if (f == nullptr || out == nullptr || f->d < 2 || row_begin < 0 || row_end > f->fine_ext[0] ||
      row_begin >= row_end)
    return fail_with(SGWG_EINVAL, "combine_rows: bad row range (needs d >= 2)");
  const long long per_row = (long long)(f->finest / f->fine_ext[0]);
  if (n != (size_t)((row_end - row_begin) * per_row))
    return fail_with(SGWG_EINVAL, "combine_rows: output size must equal rows x points per row");
  if (mode != SGWG_INTERP_WENO && mode != SGWG_INTERP_LAGRANGE)
    return fail_with(SGWG_EINVAL, "unknown interpolation mode");
  CK(cudaSetDevice(f->ctx->device));
  std::vector<int> mis(f->nm);
  for (int i = 0; i < f->nm; ++i) mis[i] = i;
  f->stats.combine_launches = 0;
  return combine_rows_impl(f, mis, mode, eps, row_begin, row_end, out, out_is_device);
}

int sgwg_combine_local(sgwg_family* f, int mode, double eps, double* out, size_t n,
                       int out_is_device, long long* row_begin, long long* row_end) {
  if (f == nullptr || row_begin == nullptr || row_end == nullptr)
    return fail_with(SGWG_EINVAL, "null argument");
  TRY(check_interp(mode, eps));
  if (f->d < 2) return fail_with(SGWG_EINVAL, "combine_local: needs d >= 2");
  CK(cudaSetDevice(f->ctx->device));
  long long a = 0, b = f->fine_ext[0];
  if (use_option_b(f)) option_b_rows(f, f->rank, &a, &b);
  *row_begin = a;
  *row_end = b;
  const long long per_row = (long long)(f->finest / f->fine_ext[0]);
  if (out == nullptr) return SGWG_OK;  // query of the row range
  if (n != (size_t)((b - a) * per_row))
    return fail_with(SGWG_EINVAL, "combine_local: output size must equal this rank's rows x points per row");
  if (!use_option_b(f)) return sgwg_combine(f, mode, eps, out, n, out_is_device);
  TRY(gather_states(f));
  const CombView v = gathered_view(f);
  std::vector<int> gm(f->nfull);
  for (int i = 0; i < f->nfull; ++i) gm[i] = i;
  long long slab = std::max(1LL, b - a);
  while (slab > 1 && plan_doubles(f, v, gm, 0, slab) > combine_budget_doubles()) slab = (slab + 1) / 2;
  double ms = 0.0;
  for (long long r0 = a; r0 < b; r0 += slab) {
    const long long r1 = std::min(b, r0 + slab);
    TRY(combine_rows_impl(f, v, gm, mode, eps, r0, r1, out + (r0 - a) * per_row, out_is_device));
    ms += f->stats.combine_ms;
  }
  f->stats.combine_ms = ms;
  return SGWG_OK;
}

int sgwg_prolong(sgwg_family* f, int mi, int mode, double eps, double* out, size_t n,
                 int out_is_device) {
  if (f == nullptr || out == nullptr || n != (size_t)f->finest)
    return fail_with(SGWG_EINVAL, "prolong: output size must equal the finest-grid points");
  if (mi < 0 || mi >= f->nm) return fail_with(SGWG_EINVAL, "bad member index");
  if (mode != SGWG_INTERP_WENO && mode != SGWG_INTERP_LAGRANGE)
    return fail_with(SGWG_EINVAL, "unknown interpolation mode");
  CK(cudaSetDevice(f->ctx->device));
  ProlongPlan* pl = nullptr;
  TRY(build_plan(f, std::vector<int>{mi}, 0, (f->d == 1) ? 1 : f->fine_ext[0], nullptr, &pl));
  double* dst = out_is_device ? out : nullptr;
  if (dst == nullptr) {
    int st = ensure_fine_buf(f);
    if (st != SGWG_OK) {
      free_plan(pl);
      return st;
    }
    dst = f->fine_buf;
  }
  int st = run_plan(f, pl, mode, eps, 1, dst);
  if (st == SGWG_OK) st = copy_out(f, dst, out, n, out_is_device);
  free_plan(pl);
  return st;
}

static double preset_value(int preset, const double* x, int d) {
  const double pi = 3.14159265358979323846;  // std::numbers::pi
  switch (preset) {
    case SGWG_IC_C1: return std::sin(pi * (x[0] + x[1]));
    case SGWG_IC_C2: return 0.5 + std::sin(pi * (x[0] + x[1]));
    case SGWG_IC_C3: return std::sin(pi * (x[0] + x[1] + x[2]));
    case SGWG_IC_C4:
      return (1.0 + 0.01 * std::cos(0.5 * x[0])) / std::sqrt(2.0 * pi) *
             std::exp(-0.5 * (x[1] * x[1]));
    case SGWG_IC_C5:
      return (1.0 + 0.05 * (std::cos(0.5 * x[0]) + std::cos(0.5 * x[1]))) / (2.0 * pi) *
             std::exp(-0.5 * (x[2] * x[2] + x[3] * x[3]));
    case SGWG_IC_EX1: return 0.3 + 0.7 * std::sin(0.5 * pi * (x[0] + x[1]));
    case SGWG_IC_EX3: {
      double s = 0.0;
      for (int k = 0; k < d; ++k) s += x[k];
      return 1.0 + 0.5 * std::sin(s);
    }
    case SGWG_IC_EX5A: {
      const double xx = x[0], v = x[1];
      const double s = std::sin(0.5 * xx * xx);
      return s * s * std::exp(-0.5 * (xx * xx + v * v));
    }
    case SGWG_IC_EX5B: {
      const double x1 = x[0], x2 = x[1], v1 = x[2], v2 = x[3];
      const double s = std::sin(0.5 * x1 * x1);
      const double c = std::cos(0.5 * x2 * x2);
      return s * s * c * c * std::exp(-0.5 * (x1 * x1 + x2 * x2 + v1 * v1 + v2 * v2));
    }
    case SGWG_IC_EX2: return 1.0 + 0.5 * std::sin(x[0] + x[1] + x[2]);
  }
  return 0.0;
}

struct PresetIc {
  int preset;
};
// ex6 (models.hpp:722-742), VlasovMaxwellSpec defaults (models.hpp:43-50)
static int g_ex6_marker = 0;
static double ex6_f(const double* x, int, void*) {
  const double pi = 3.14159265358979323846;  // std::numbers::pi
  const double beta = 0.01, delta = 0.5, v01 = 0.3, v02 = 0.3;
  const double xi1 = x[1], xi2 = x[2];
  const double g1 = delta * std::exp(-(xi1 - v01) * (xi1 - v01) / beta);
  const double g2 = (1.0 - delta) * std::exp(-(xi1 + v02) * (xi1 + v02) / beta);
  return std::exp(-xi2 * xi2 / beta) * (g1 + g2) / (pi * beta);
}
static double ex6_b3(double x2) { return 0.001 * std::sin(0.2 * x2); }
static double preset_cb(const double* x, int d, void* user) {
  return preset_value(static_cast<PresetIc*>(user)->preset, x, d);
}

int sgwg_family_init_fn(sgwg_family* f, sgwg_ic_fn ic, void* user, int normalize_mass) {
  if (f == nullptr || ic == nullptr) return fail_with(SGWG_EINVAL, "null argument");
  std::vector<double> host((size_t)std::max<long long>(1, f->state_total));
  const int d = f->d;
  const bool vm = f->state_total != f->total;
  long long so = 0;
  for (int mi = 0; mi < f->nm; ++mi) {
    const MemberDesc& M = f->hmem[mi];
    double* out = host.data() + (vm ? so : M.offset);
    if (vm) {  // field lines: E1 = E2 = 0, B3 = init_b3(x2) (initialize_family, models.hpp:861-867)
      so += M.npts + 3 * M.nx;
      for (int i = 0; i < M.nx; ++i) {
        out[M.npts + i] = 0.0;
        out[M.npts + M.nx + i] = 0.0;
        const double x2 = M.lower[0] + i * M.h[0];
        out[M.npts + 2 * M.nx + i] = (user == &g_ex6_marker) ? ex6_b3(x2) : 0.0;
      }
    }
    int idx[kMaxD] = {0, 0, 0, 0};
    double x[kMaxD];
    for (int k = 0; k < d; ++k) x[k] = M.lower[k];
    for (long long lin = 0; lin < M.npts; ++lin) {  // restrict_to_grid (grid.hpp:166-186)
      out[lin] = ic(x, d, user);
      for (int k = d - 1; k >= 0; --k) {
        if (++idx[k] < M.ext[k]) {
          x[k] = M.lower[k] + idx[k] * M.h[k];
          break;
        }
        idx[k] = 0;
        x[k] = M.lower[k];
      }
    }
    if (normalize_mass) {  // normalize_initial / quadrature_mass (models.hpp:73-102)
      int id2[kMaxD] = {0, 0, 0, 0};
      double sum = 0.0, comp = 0.0;
      for (long long lin = 0; lin < M.npts; ++lin) {
        double wp = 1.0;
        for (int k = 0; k < d; ++k) {
          double w = M.h[k];
          if (M.bc[k] == SGWG_ZERO && (id2[k] == 0 || id2[k] == M.ext[k] - 1)) w *= 0.5;
          wp *= w;
        }
        const double term = wp * out[lin] - comp;
        const double next = sum + term;
        comp = (next - sum) - term;
        sum = next;
        for (int k = d - 1; k >= 0; --k) {
          if (++id2[k] < M.ext[k]) break;
          id2[k] = 0;
        }
      }
      if (!(sum > 0.0)) return fail_with(SGWG_EINVAL, "normalize_initial: nonpositive mass");
      for (long long lin = 0; lin < M.npts; ++lin) out[lin] /= sum;
    }
  }
  return sgwg_family_upload(f, host.data(), (size_t)f->state_total);
}

int sgwg_family_init_preset(sgwg_family* f, int preset) {
  if (preset < SGWG_IC_C1 || preset > SGWG_IC_EX6) return fail_with(SGWG_EINVAL, "unknown preset");
  if (preset == SGWG_IC_EX6) {
    if (f == nullptr || !f->has_model || f->model.kind != SGWG_VLASOV_MAXWELL)
      return fail_with(SGWG_EINVAL, "init_preset: ex6 needs a Vlasov-Maxwell model");
    return sgwg_family_init_fn(f, ex6_f, &g_ex6_marker, 0);
  }
  PresetIc p{preset};
  const int norm = (preset == SGWG_IC_EX5A || preset == SGWG_IC_EX5B) ? 1 : 0;
  return sgwg_family_init_fn(f, preset_cb, &p, norm);
}

int sgwg_get_stats(const sgwg_family* f, sgwg_stats* st) {
  if (f == nullptr || st == nullptr) return fail_with(SGWG_EINVAL, "null argument");
  *st = f->stats;
  return SGWG_OK;
}

int sgwg_fp64_peak(sgwg_ctx* ctx, double* tflops) {
  if (ctx == nullptr || tflops == nullptr) return fail_with(SGWG_EINVAL, "null argument");
  CK(cudaSetDevice(ctx->device));
  double* buf;
  CK(cudaMalloc(&buf, sizeof(double)));
  const int iters = 1 << 16;
  const int blocks = ctx->sm_count * 8;
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  CK(launch_fp64_peak(buf, iters, blocks, ctx->stream));  // warm-up
  float best = 1e30f;
  for (int rep = 0; rep < 5; ++rep) {
    CK(cudaEventRecord(a, ctx->stream));
    CK(launch_fp64_peak(buf, iters, blocks, ctx->stream));
    CK(cudaEventRecord(b, ctx->stream));
    CK(cudaEventSynchronize(b));
    float ms;
    CK(cudaEventElapsedTime(&ms, a, b));
    best = std::min(best, ms);
  }
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaFree(buf);
  const double flops = (double)blocks * 256.0 * iters * 8.0 * 2.0;
  *tflops = flops / (best * 1e-3) / 1e12;
  return SGWG_OK;
}

}  // extern "C"
