// sgwg_internal.h -- device-side data layout shared by the kernel TUs and the
// host runtime (sgwg_api.cu).  Not part of the public C ABI (include/sgwg.h).
//
// HBM layout of a family: every member's state is packed in
// one contiguous fp64 buffer in the reference's sorted member order, each
// member row-major with dimension 0 slowest (grid.hpp:102-108).  Three such
// buffers (u^n, stage A, stage B) plus one tendency buffer K hold a step.
#pragma once
#include <cstdio>
#include <cuda_runtime.h>
#include <stdint.h>

namespace sgwg {

constexpr int kMaxD = 4;
constexpr int kPassThreads = 256;  // threads per WENO pass CTA
constexpr int kMaxRun = 8;         // max points per thread run (registers)

enum FluxKind : int {
  kFluxAdvect = 0,   // c*u with c constant over the member (advection speeds)
  kFluxBurgers = 1,  // 0.5 u^2 with Lax-Friedrichs split, alpha = max|u| of the member
  kFluxKinX = 2,     // kinetic x_j line: c = v_j coordinate      (models.hpp:341-344)
  kFluxKinVB = 3,    // kinetic v_j line: c = -x_j coordinate     (models.hpp:346-349)
  kFluxKinVP = 4,    // kinetic v_j line: c = -E_j(x) (Vlasov-Poisson, new physics)
  kFluxVM0 = 5,      // Vlasov-Maxwell x2 line: c = xi2               (models.hpp:456-460)
  kFluxVM1 = 6,      // Vlasov-Maxwell xi1 line: c = E1(x2) + xi2 B3(x2) (models.hpp:461-470)
  kFluxVM2 = 7       // Vlasov-Maxwell xi2 line: c = E2(x2) - xi1 B3(x2) (models.hpp:471-480)
};

// One component grid on the device (GridGeometry, grid.hpp:85-136).
// Device-side invariant checks of the experiment build -DSGWG_CHECK (compute-sanitizer is not
// available on the GPU pool): a failed check prints its tag and traps.
#ifdef SGWG_CHECK
#define SGWG_DCHECK(cond, tag)                                                          \
  do {                                                                                  \
    if (!(cond)) {                                                                      \
      printf("SGWG_DCHECK failed: %s (block %d thread %d)\n", tag, (int)blockIdx.x,     \
             (int)threadIdx.x);                                                         \
      __trap();                                                                         \
    }                                                                                   \
  } while (0)
#else
#define SGWG_DCHECK(cond, tag) \
  do {                         \
  } while (0)
#endif

struct MemberDesc {
  long long offset;        // first point in the packed state buffers
  long long npts;
  long long stride[kMaxD];
  int ext[kMaxD];          // points per dimension
  int bc[kMaxD];
  int level[kMaxD];
  double h[kMaxD];
  double inv_h[kMaxD];
  double lower[kMaxD];
  // per-dimension WENO pass tiling: segment length S, run length P, lines W, smem pitch
  int segS[kMaxD], runP[kMaxD], linesW[kMaxD], pitch[kMaxD];
  // Vlasov-Poisson: x-grid of the member
  long long xoff;          // offset of this member in the packed x-grid buffers (rho, E)
  int nx;                  // x points
  int vn;                  // points of the velocity block (contiguous)
  int xext[2];             // x extents (dx=1: {n0, 1})
  int tx, ty;              // 2D fused-stage tile (d == 2)
  int rparts;              // Vlasov-Poisson: charge-density partial sums per x point
};

// Vlasov-Poisson charge density in partial-sum form: rho(x) = 1 - sum_t parts[x][t],
// t < MemberDesc::rparts (one partial per velocity-plane tile, fixed order)
constexpr int kRhoParts = 8;
constexpr int kPlaneMaxV = 32;  // planes per fast 4D plane tile
constexpr int kP4MaxG = 64;     // x points per whole-plane 4D v-pass tile (plane4d.cuh)

// Step control block (timestep.hpp:126-174 loop state), device resident.
struct StepCtl {
  double t;          // current time
  double stop;       // current stop
  double eps_t;      // 1e-12 * max(1, T)
  double dt;         // dt of the current step
  long long step;    // number of steps taken (also next step index)
  long long cur_step;
  int active;        // 1 while stop - t > eps_t and no failure
  int failed;        // a member reported a non-finite tendency
  double speeds[kMaxD + 1];  // family wave speeds of the step (+ failure flag slot)
};

struct PassParams {
  const MemberDesc* mem;
  const int4* tasks;       // (member, first line, segment start, -)
  int kdim;                // dimension swept by this pass
  int flux;                // FluxKind
  int first, last;         // first / last pass of the stage (accumulation order)
  int stage;               // 1..3 RK stage when last; 0: rhs only (out = tendency)
  int linear;              // WenoMode::linear
  double eps;
  double c_const;          // advection speed of this dimension
  int space_dim;           // kinetic models
  const double* uin;       // stage input
  const double* un;        // u^n (stages 2, 3)
  double* out;             // stage output
  double* kbuf;            // tendency accumulator
  const double* efield;    // VP: E, packed per member [comp][xi]
  const StepCtl* ctl;      // dt, active, step
  const unsigned long long* amax_in;   // per member max|u_in| (Burgers alpha)
  unsigned long long* amax_out;        // per member max|out| (next stage alpha)
  unsigned long long* amax_zero;       // slot cleared by this pass (or null)
  int nmembers;
  int track_max;
  unsigned long long* fail;            // per member: min(step*4 + stage)
  int dyn_smem_doubles;    // doubles of dynamic smem per array
  const struct DtParams* dtp;  // stage 3, last pass: fused next-step dt (or null)
  unsigned int* counter;       // CTA-done counter for the fused dt
};

struct Stage2DParams {
  const MemberDesc* mem;
  const int4* tiles;       // (member, i0, j0, -)
  int burgers;
  int flux0, flux1;        // FluxKind of the dimension-0 / dimension-1 sweep
  double c0, c1;           // advection speeds
  int flux2;               // 3D stage kernel: dimension-2 sweep
  double c2;
  int stage;               // 1..3, 0 = tendency only
  int linear;
  double eps;
  int space_dim;
  const double* uin;
  const double* un;
  double* out;
  const double* efield;
  const StepCtl* ctl;
  const unsigned long long* amax_in;
  unsigned long long* amax_out;
  unsigned long long* amax_zero;
  int nmembers;
  int track_max;
  unsigned long long* fail;
  const struct DtParams* dtp;
  unsigned int* counter;
  // persistent mode (evolve2d_persistent_kernel): dt from the CTA's own copy of
  // the step control, cache-global loads of data written by other CTAs
  double dt_value;
  unsigned long long cur_step;
  int ntiles;
  int resident;       // one tile per CTA: stage input / u^n kept in shared memory
  int resident_load;  // first stage of the launch: fill the resident copy from HBM
  int trace_ss;       // step * 3 + stage - 1 (phase-trace experiment builds)
  int half_tiles;     // fast stage kernel on 1024-point tiles (two CTAs per SM)
  int newton;         // Burgers families too large for the persistent kernel: fast_rcp<NEWTON> form
};

struct PersistParams {
  Stage2DParams base;      // tiles, physics, amax, fail (stage/uin/un/out set per stage)
  double* u;
  double* A;
  double* B;
  int nsteps;              // steps of this launch (early exit when the stop is reached)
};

// fast 4D stage as two plane launches (kernels.cuh plane_fast_kernel): a tile
// is nv consecutive planes of the pair of dimensions (a, a+1), a = 2*pr, each
// restricted to the window [i0, i0+tx) x [j0, j0+ty).
struct PlaneTile {
  int mi, plane0, nv, part;
  int i0, j0, tx, ty;
};

struct PlaneParams {
  const MemberDesc* mem;
  const PlaneTile* tiles;
  int pr;                  // 0: dims (0,1) -> tendency K; 1: dims (2,3) + RK stage
  int flux_a, flux_b;      // FluxKind of the two sweeps
  double c_a, c_b;         // advection speeds
  int stage;               // 1..3, 0 = tendency only
  int linear;
  double eps;
  int space_dim;
  const double* uin;
  const double* un;
  double* out;
  double* kbuf;
  const double* efield;
  const StepCtl* ctl;
  unsigned long long* fail;
  double* rho_parts;       // pr = 1, Vlasov-Poisson: sum_v w_v out per (x point, part)
  const struct DtParams* dtp;
  unsigned int* counter;
};

// v-pass tile descriptor of the persistent 4D v pass (plane4d.cuh), precomputed on the
// host so a CTA prefetches it with one async copy (no dependent load chain)
struct __align__(16) P4VTile {
  long long gs, ga;  // tile start (doubles) and its 16-byte aligned floor
  long long xoff;    // member's first x point in the packed x-grid buffers
  double ih3, ih4, hh;
  int mi, x0, G, n3, n4, V, NT, shift, nx;
  unsigned nbytes;
  int pad[2];
};
static_assert(sizeof(P4VTile) == 96, "P4VTile is copied in 16-byte pieces");

// x-pass tile descriptor of the persistent 4D x pass (plane4d.cuh): the gather and
// the line coefficients without dependent loads (host-precomputed)
struct __align__(16) P4XTile {
  long long src;           // member offset + v0 (doubles)
  double ih1, ih2;
  double ca0, ca1, cb0, cb1;  // x_j line coefficients: ca0 + i3 ca1, cb0 + i4 cb1 (KinX / advection)
  int V, cs, nc, n1, n2, n4, v0, mi;
};
static_assert(sizeof(P4XTile) == 96, "P4XTile is copied in 16-byte pieces");

// fast 4D stage on whole planes (plane4d.cuh): x pass tiles (mi, v0, nc, log2 C),
// v pass tiles (mi, x0, G, -)
struct Plane4Params {
  const MemberDesc* mem;
  const int4* tiles;
  int flux_a, flux_b;      // FluxKind of the lower / upper dimension of the pass
  double c_a, c_b;         // advection speeds
  int stage;               // 1..3, 0 = tendency only
  int linear;
  double eps;
  int space_dim;
  const double* uin;
  const double* un;
  double* out;
  double* kbuf;
  const double* efield;
  const StepCtl* ctl;
  unsigned long long* fail;
  double* rho_parts;       // v pass, Vlasov-Poisson: sum_v w_v out per x point (part 0)
  const struct DtParams* dtp;
  unsigned int* counter;
  int rpt;                 // runs per warp task (plane4d.cuh P4Sweeps)
  int xpitch;              // > 0: persistent x pass (xpass4d_persist_kernel), slot pitch in doubles
  const P4VTile* vtiles;   // persistent v pass: descriptor per tile
  const P4XTile* xtiles;   // persistent x pass: descriptor per tile
  unsigned int* sched;     // persistent v pass: [next tile counter, CTAs done] (self-resetting)
  int vpitch;              // > 0: persistent v pass (vpass4d_persist_kernel), slot pitch in doubles
  int ntiles;              // v-pass tiles (persistent form)
  int masked;              // 1: one sweep body with runtime ghost masks (default), 0: per-pattern bodies
  int dbg;                 // timing experiments only (SGWG_P4_DBG): 1 no sweeps, 2 no epilogue, 4 no K/u^n copies
};

// Vlasov-Maxwell field lines (vm_rhs_into, models.hpp:437-505): per member the
// packed fields F[3*xoff ...] = (E1[nx], E2[nx], B3[nx]) over its x2 points.
struct VmParams {
  const MemberDesc* mem;
  const double* f;         // stage input distribution (packed)
  const double* fin;       // stage input fields
  const double* fun;       // u^n fields (stages 2, 3)
  double* fout;            // stage output fields (stage 0: field tendencies)
  int stage;
  int linear;
  double eps;
  const StepCtl* ctl;
  unsigned long long* fail;
  double* speeds;          // vm_speeds: per member (s1, s2) of family_wave_speeds
};

struct UpsampleParams {
  const MemberDesc* mem;
  const int2* tasks;       // (member-slot, first output index of the chunk)
  const double* const* src;  // per member-slot source array
  double* const* dst;        // per member-slot destination array
  const int* slot_member;    // member-slot -> member index
  const long long* slot_n;   // member-slot -> dst points
  const int* slot_ext;       // member-slot -> src extents (4 per slot, dims > k original)
  int kdim;
  int nl;
  int fine_ext;            // finest points along kdim
  int bc;
  int mode;                // InterpMode
  double eps;
  int chunk;
  int jrow0;               // dimension-0 slab: fine index of the first output row
  // fast chunked form (upsample_fast_kernel): items = (slot, 8-point chunk, 32 lines)
  const long long* slot_item0;  // first item of each slot (prefix), nslots entries
  long long nitems;        // 0: the generic kernel
  int nslots;
  int nrows0;              // k == 0: output rows of the slab
};

struct FinalParams {
  const MemberDesc* mem;
  const double* const* src;  // per local member: array after dims 0..d-2
  const double* coef;        // per local member combination coefficient
  const int* msrc_ext;       // per local member: source extent along the last dim
  const int* mrefine;        // per local member: refinement exponent along the last dim
  int nm;
  int d;
  int nl;
  int fine_last;           // finest points along the last dim
  long long nfine;         // finest points (or slab points)
  long long row0;          // first finest row (dims 0..d-2 flattened) of this launch
  int bc_last;
  int mode;
  double eps;
  int assign;              // 1: out = p (prolong of one member, no accumulation)
  double* out;
  int nm_host;             // host copy of the refinement exponents (launch-time dispatch)
  const int* mref_host;
};

struct EvalParams {        // combined field at single finest-grid points
  const MemberDesc* mem;
  const double* u;         // packed member states
  const double* coef;      // combination coefficient per member
  const int* idx;          // npts x d finest multi-indices
  long long npts;
  int nm, d, nl, mode;
  double eps;
  double* out;
};

struct StatsParams {       // k_diag.cu: diagnostics of a slab of the combined field
  const double* field;
  long long n;             // points of the slab
  long long first;         // finest-grid linear index of field[0]
  int d;
  int ext[kMaxD];
  int bc[kMaxD];
  double h[kMaxD];
  double lower[kMaxD];
  int exact;               // preset of the exact solution or -1
  int burgers;             // exact solution of the Burgers sine waves (else advection)
  double t;
  double a[kMaxD];         // advection speeds
  double* partial;         // stats_partial_doubles() scratch
};

struct FieldParams {
  const MemberDesc* mem;
  const double* f;         // stage input (packed)
  double* rho;             // packed per member (nx)
  double* efield;          // packed per member (space_dim * nx)
  double* emax;            // per member max|E_j| (space_dim per member), stage 1 only
  int space_dim;
  int stage;
  double L[2];             // periodic x lengths
  const StepCtl* ctl;
  const int2* mtasks;      // moment kernel work: (member, first x point), 8 x points each
  int nmtasks;
  int nmembers;
  double* rho_parts;       // kRhoParts partial sums per x point (see MemberDesc::rparts)
  const double* twid;      // FFT twiddles: cos(pi q/hmax), then sin(pi q/hmax), q < hmax
  int hmax;
  // field-energy diagnostic: members grouped by x-grid
  const int4* egrp;        // (n0, n1, offset in egrid, first group x point)
  const int2* egrp_m;      // (first, count) into egrp_mem
  const int* egrp_mem;     // member indices, sorted order within a group
  int negrp;
  int ngx;                 // total group x points
  double* egrid;           // per group: sum_m c_m E_m on the group's x-grid
  const double* ecoef;     // combination coefficient per member (negrp == 0: no groups)
  // batched energy record (captured step chunks): the step-start field of step k is also
  // kept in slot k % ering_slots of a ring, and one launch per chunk records every step
  double* ering;           // ering_slots x ering_stride doubles (nullptr: off)
  long long ering_stride;
  int ering_slots;
  // groups classed by their x2 extent (the batched record sums a class's groups before the
  // x2 interpolation they share): class extents, each group's class
  int ncls;
  int cls_n1[8];
  unsigned char grp_cls[64];
};
constexpr int kEnergyRing = 64;  // >= the steps of a captured chunk

// launchers: one set per arithmetic TU (k_exact.cu, k_fast.cu)
#define SGWG_DECLARE_LAUNCHERS(NS)                                                        \
  namespace NS {                                                                          \
  cudaError_t configure();                                                                \
  cudaError_t launch_pass(const PassParams& p, int nblocks, size_t smem, cudaStream_t s); \
  cudaError_t launch_stage2d(const Stage2DParams& p, int nblocks, size_t smem, cudaStream_t s); \
  cudaError_t launch_upsample(const UpsampleParams& p, int nblocks, cudaStream_t s);      \
  cudaError_t launch_final(const FinalParams& p, cudaStream_t s);                         \
  cudaError_t launch_eval_points(const EvalParams& p, cudaStream_t s);                    \
  cudaError_t launch_vm_fields(const VmParams& p, int nmembers, int smem, cudaStream_t s);    \
  }
SGWG_DECLARE_LAUNCHERS(exact)
SGWG_DECLARE_LAUNCHERS(fast)
namespace fast {
cudaError_t launch_stage3d(const Stage2DParams& p, int nblocks, size_t smem, cudaStream_t s);
cudaError_t launch_plane(const PlaneParams& p, int nblocks, size_t smem, cudaStream_t s);
int plane_smem_doubles(int nv, int tx, int ty);
cudaError_t launch_plane4(const Plane4Params& p, int pass, int nblocks, size_t smem, cudaStream_t s);
cudaError_t configure_plane4();
cudaError_t launch_persist2d(const PersistParams& p, int nblocks, size_t smem, cudaStream_t s);
int persist2d_max_blocks(int burgers, int half, size_t smem);
}  // namespace fast

// exact-arithmetic scalar kernels (k_exact.cu)
struct DtParams {
  StepCtl* ctl;
  int kind;                // model kind
  int mode;                // DtMode
  double cfl;
  double base_dt;          // accuracy mode: pow(h, 5/3) (x scale), computed on the host
  double fine_h[kMaxD];    // finest spacings (finest_geometry)
  double const_speeds[kMaxD];
  int d;
  int space_dim;
  const unsigned long long* amax;  // Burgers: per member max|u^n| (slot 0)
  const double* emax;              // VP: per member max|E_j|
  const double* vmspd;             // Vlasov-Maxwell: per member (s1, s2)
  int nmembers;
  const unsigned long long* fail;
  double* dts;
  long long dts_cap;
  int use_reduced;         // speeds already reduced across ranks into ctl->speeds
};
cudaError_t launch_local_speeds(const DtParams& p, cudaStream_t s);
cudaError_t launch_dt(const DtParams& p, cudaStream_t s);
cudaError_t launch_stamp(long long* tl, int slot, cudaStream_t s);
cudaError_t launch_member_max(const MemberDesc* mem, int nmembers, const int2* tasks, int ntasks,
                              const double* u, unsigned long long* amax, cudaStream_t s);
cudaError_t configure_field();
cudaError_t launch_field(const FieldParams& p, int nmembers, bool with_moment, cudaStream_t s);
cudaError_t launch_twiddles(double* tw, int hmax, cudaStream_t s);
cudaError_t launch_field_energy_batch_direct(const FieldParams& p, const double* coef, int fine0,
                                             int fine1, double hvol, double* out_base,
                                             long long cap, int nbatch, unsigned int* done,
                                             long long* recorded, cudaStream_t s);
cudaError_t launch_field_energy_batch(const FieldParams& p, const double* coef, int fine0, int fine1,
                                      double hvol, double* out_base, long long cap, int nbatch,
                                      double* part, unsigned int* done, long long* recorded,
                                      double* egrid_b, long long egrid_stride, cudaStream_t s);
cudaError_t launch_field_energy(const FieldParams& p, const double* coef, int fine0, int fine1,
                                double hvol, double* out_base, long long cap, cudaStream_t s,
                                double* part = nullptr, unsigned int* done = nullptr);
cudaError_t launch_fp64_peak(double* out, int iters, int blocks, cudaStream_t s);
cudaError_t launch_vm_speeds(const VmParams& p, int nmembers, cudaStream_t s);
int stats_partial_doubles();
cudaError_t launch_stats(const StatsParams& p, double* out5, cudaStream_t s);

}  // namespace sgwg
