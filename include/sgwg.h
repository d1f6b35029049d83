/*
 * sgwg.h -- C ABI of the B200-native sparse-grid WENO5 hot path.
 *
 * The reference (`sgweno`, header-only C++20, /root/reference/proj/include/sgweno)
 * has no FFI: its operator boundary is the duck-typed Model concept consumed by
 * `evolve_family` plus the free functions `make_family`, `initialize_family`,
 * `prolong` and `combine`.  A GPU backend has to replace the whole
 * evolve + combine pipeline (a per-member, per-stage host `rhs` callback would
 * force a host<->device copy per stage), so this ABI exports exactly the
 * entry points a maintainer would bind to replace those calls.  Each function
 * cites the reference interface it replaces (paths relative to
 * proj/include/sgweno/).  Plain C types only: no torch, no C++.
 *
 * Conventions
 *   - Member order is the reference's: levels sorted lexicographically
 *     (grid.hpp:57-79, combine.hpp:71-72).  Member states are packed one after
 *     another in that order, each row-major with dimension 0 slowest
 *     (grid.hpp:102-108).  This is also the device layout.
 *   - Every function returns SGWG_OK (0) or a nonzero status; the message of
 *     the last failure on the calling thread is sgwg_last_error().  There is no
 *     CPU fallback: without a usable sm_100 device sgwg_init fails.
 */
#ifndef SGWG_H
#define SGWG_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SGWG_MAXD 4

/* status codes (errors of the reference map as noted) */
enum {
  SGWG_OK = 0,
  SGWG_EINVAL = 1,     /* std::invalid_argument / std::out_of_range            */
  SGWG_ENONFINITE = 2, /* FamilyIntegratorFailure{level,step,stage}, timestep.hpp:31-40 */
  SGWG_ECUDA = 3,      /* CUDA runtime error (no device, OOM, launch failure)   */
  SGWG_ENCCL = 4,      /* NCCL error in a sharded family                       */
  SGWG_EUNSUPPORTED = 5
};

/* grid.hpp:14 BoundaryKind */
enum { SGWG_PERIODIC = 0, SGWG_ZERO = 1 };
/* models.hpp:19 ModelKind (+ the Vlasov-Poisson model of BASELINE C4/C5).
 * SGWG_VLASOV_MAXWELL: the reduced (x2, xi1, xi2) system of models.hpp:376-527;
 * a member's state is its distribution followed by the field lines E1, E2, B3
 * over its x2 points (initialize_family, models.hpp:855-871). */
enum {
  SGWG_ADVECTION = 0,
  SGWG_BURGERS = 1,
  SGWG_VLASOV_BOLTZMANN = 2,
  SGWG_VLASOV_POISSON = 3,
  SGWG_VLASOV_MAXWELL = 4
};
/* weno.hpp:17 WenoMode */
enum { SGWG_WENO_NONLINEAR = 0, SGWG_WENO_LINEAR = 1 };
/* interp.hpp:16 InterpMode */
enum { SGWG_INTERP_LAGRANGE = 0, SGWG_INTERP_WENO = 1 };
/* timestep.hpp:15 DtMode */
enum { SGWG_DT_CFL = 0, SGWG_DT_ACCURACY = 1 };
/* arithmetic of the device kernels */
enum {
  SGWG_ARITH_EXACT = 0, /* reference expression order, no FMA contraction, IEEE divides:
                           bitwise equal to the reference built without FMA */
  SGWG_ARITH_FAST = 1   /* FMA contraction, one divide per reconstruction, reciprocal
                           spacings: within 1e-10 of the reference */
};

/* DomainBox + root cells + boundaries + N_L: the arguments of make_family
 * (combine.hpp:69-70, grid.hpp:17-37). */
typedef struct {
  int d;                      /* 1..4 */
  int nl;                     /* finest level N_L (>= d-1) */
  double lower[SGWG_MAXD];
  double upper[SGWG_MAXD];
  int root_cells[SGWG_MAXD];
  int bc[SGWG_MAXD];          /* SGWG_PERIODIC / SGWG_ZERO */
} sgwg_domain;

/* ProblemSpec's physics (models.hpp:23-41, 568-580) + WenoParams (weno.hpp:19-22). */
typedef struct {
  int kind;                   /* SGWG_ADVECTION ... */
  int weno_mode;              /* SGWG_WENO_NONLINEAR / LINEAR */
  double epsilon;             /* WENO epsilon, reference default 1e-6 (weno.hpp:20) */
  double speeds[SGWG_MAXD];   /* advection speeds a_k (models.hpp:25) */
  int space_dim;              /* kinetic models: phase space has 2*space_dim dims */
  double theta, tau;          /* Vlasov-Boltzmann relaxation (models.hpp:37-41) */
} sgwg_model;

/* StepPolicy (timestep.hpp:17-21) + the accuracy-mode multiplier that BASELINE
 * C1 needs (dt = 0.5 h^{5/3}).  dt_scale = 1 is the reference rule. */
typedef struct {
  int mode;                   /* SGWG_DT_CFL / SGWG_DT_ACCURACY */
  double cfl;                 /* cfl_number */
  double reference_spacing;   /* minimum spacing of the finest grid */
  double dt_scale;
} sgwg_policy;

/* FamilyIntegratorFailure (timestep.hpp:31-40): member index (sorted order),
 * step index and RK stage (1..3) of the first non-finite tendency. */
typedef struct {
  int member;
  long long step;
  int stage;
} sgwg_failure;

/* Device-timed statistics of the last sgwg_evolve / sgwg_combine. */
typedef struct {
  double evolve_ms;           /* CUDA-event time of the whole evolve (all stops, no combines) */
  double combine_ms;          /* CUDA-event time of the last combine */
  long long steps;            /* RK steps taken */
  long long kernel_launches;  /* device kernels launched by the last evolve (incl. early-exit) */
  long long combine_launches; /* device kernels launched by the last combine */
  double pass_ms_sum;         /* profile mode: summed event time of the WENO pass kernels */
  long long pass_launches;    /* profile mode: number of timed WENO pass launches */
  double pass_flops;          /* algorithmic flops of those launches (SURVEY 8(d) counting) */
  double pass_bytes;          /* algorithmic HBM bytes of those launches */
} sgwg_stats;

/* profile mode (sgwg_set_profile): per-kernel event time of every launch of
 * the last evolves and the kernel's algorithmic work per launch (SURVEY 8(d)
 * counting), for the roofline of the stage kernels */
typedef struct {
  char name[48];
  double ms_sum;
  long long launches;
  double flops_per_launch;
  double bytes_per_launch;
} sgwg_kernel_timing;

typedef struct sgwg_ctx sgwg_ctx;
typedef struct sgwg_family sgwg_family;

/* on_stop(t) of evolve_family (timestep.hpp:129,171). Called on the host after
 * the device has landed exactly on stop time t; the callback may call
 * sgwg_combine / sgwg_download on the same family. */
typedef void (*sgwg_stop_cb)(double t, void* user);

/* ---- context ------------------------------------------------------------ */
/* Bind a CUDA device (one process per GPU).  Replaces nothing in the
 * reference (it is single-process CPU; parallel.hpp:12-31 thread fan-out). */
int sgwg_init(int device, sgwg_ctx** out);
/* Frees the context.  While families created on it are still open the call is
 * deferred: the context (and its stream) is freed by the last
 * sgwg_family_destroy. */
int sgwg_shutdown(sgwg_ctx* ctx);
const char* sgwg_last_error(void);
int sgwg_version(void);
/* arithmetic mode for families created afterwards (default SGWG_ARITH_EXACT) */
int sgwg_set_arith(sgwg_ctx* ctx, int arith);
/* profile mode: time every WENO pass launch with CUDA events, no CUDA graphs */
int sgwg_set_profile(sgwg_ctx* ctx, int on);
/* the cudaStream_t all work of this context is issued on (as void*) */
void* sgwg_stream(sgwg_ctx* ctx);

/* ---- family: make_family (combine.hpp:69-83) ------------------------------ */
/* Full family: every combination level of (d, nl), sorted. */
int sgwg_family_create(sgwg_ctx* ctx, const sgwg_domain* dom, sgwg_family** out);
/* Shard of a family: only the listed members (indices into the sorted full
 * family, ascending).  Evolve and combine act on these members only; a
 * sharded combine returns this shard's partial combination sum. */
int sgwg_family_create_shard(sgwg_ctx* ctx, const sgwg_domain* dom, const int* members,
                             int count, sgwg_family** out);
/* Single-grid mode: one grid at level (N_L, ..., N_L) -- make_single_grid
 * (runner.hpp:106-115), the reference's full-grid comparison run.  Its
 * "combination" is the grid's own field (runner.hpp:323-324). */
int sgwg_family_create_single(sgwg_ctx* ctx, const sgwg_domain* dom, sgwg_family** out);
int sgwg_family_destroy(sgwg_family* fam);
/* enumerate_combination_levels (grid.hpp:57-79), sorted: count, then levels[count*d] */
int sgwg_enumerate_levels(int d, int nl, int* levels, int cap, int* count);
int sgwg_family_num_members(const sgwg_family* fam, int* count);
/* global (full-family) index, level tuple and point extents of local member mi */
int sgwg_family_member(const sgwg_family* fam, int mi, int* global_index, int* levels,
                       int* points);
/* total packed points of the local members; finest-grid points (finest_geometry,
 * combine.hpp:85-91) */
int sgwg_family_sizes(const sgwg_family* fam, size_t* member_points, size_t* finest_points);

/* ---- state transfer: initialize_family (models.hpp:855-871) / member.state ---- */
/* Upload/download the packed states of all local members (host pointers). */
int sgwg_family_upload(sgwg_family* fam, const double* host, size_t n);
int sgwg_family_download(sgwg_family* fam, double* host, size_t n);
/* Same, device pointers (cudaMemcpyDeviceToDevice on the family stream). */
int sgwg_family_upload_device(sgwg_family* fam, const double* dev, size_t n);
int sgwg_family_download_device(sgwg_family* fam, double* dev, size_t n);

/* ---- physics: FamilyModel (models.hpp:754-851) ---------------------------- */
int sgwg_set_model(sgwg_family* fam, const sgwg_model* model);

/* ---- multi-GPU: NCCL communicator over the shards (one rank per process) ---- */
/* id: 128-byte ncclUniqueId made by sgwg_nccl_unique_id on rank 0 and
 * broadcast by the caller (e.g. torch.distributed).  Used for the per-step
 * family wave-speed all-reduce(max) and the combine reduction. */
int sgwg_nccl_unique_id(void* id128);
int sgwg_family_set_comm(sgwg_family* fam, const void* id128, int nranks, int rank);

/* ---- evolve_family (timestep.hpp:126-174) --------------------------------- */
/* March the (local) family from its current time to tfinal in lockstep with
 * the reference's stop list / landing / dt rules.  dts (capacity cap, may be
 * NULL) receives the dt sequence, *nsteps its length.  On a non-finite
 * tendency returns SGWG_ENONFINITE and fills *fail.  The family's time starts
 * at 0 when it is created / uploaded. */
int sgwg_evolve(sgwg_family* fam, const sgwg_policy* policy, double tfinal, const double* stops,
                int nstops, sgwg_stop_cb on_stop, void* user, double* dts, size_t cap,
                size_t* nsteps, sgwg_failure* fail);

/* ---- combine (combine.hpp:95-122) with prolong (interp.hpp:197-250) -------- */
/* acc = sum over members in sorted order of c_m * P_m(u_m) on the finest grid.
 * out: finest_points doubles, host (out_is_device = 0) or device pointer.  In a
 * sharded family with a communicator the partial sums are all-reduced (sum)
 * so every rank receives the combined field. */
int sgwg_combine(sgwg_family* fam, int interp_mode, double eps, double* out, size_t n,
                 int out_is_device);
/* The same combination restricted to finest-grid rows [row_begin, row_end) of
 * dimension 0 (d >= 2): out holds (row_end-row_begin) x (finest points per
 * row).  Prolongation is dimension-sequential with dimension 0 first
 * (interp.hpp:217-244), so rows are independent after the dimension-0 sweep;
 * this is how sgwg_combine handles finest grids too large for one pass
 * (BASELINE C5: 4.3e9 points) and how a sharded output is produced. */
int sgwg_combine_rows(sgwg_family* fam, int interp_mode, double eps, long long row_begin,
                      long long row_end, double* out, size_t n, int out_is_device);
/* This rank's share of the combination, the result left sharded (option B for a
 * family with a multi-rank communicator): every rank gathers all member
 * states (NCCL broadcasts of the shards) and combines ITS dimension-0 rows
 * [*row_begin, *row_end) -- rows * rank / nranks .. rows * (rank + 1) / nranks -- for
 * every member in family order, so the rows are bitwise those of the one-GPU
 * combine(set, mode, eps) (combine.hpp:95-122).  Without a communicator: all rows.
 * out == NULL only reports the row range; else n = (row_end - row_begin) x points per
 * dimension-0 row.  Collective over the communicator. */
int sgwg_combine_local(sgwg_family* fam, int interp_mode, double eps, double* out, size_t n,
                       int out_is_device, long long* row_begin, long long* row_end);
/* prolong (interp.hpp:197-250) of one local member onto the finest grid. */
int sgwg_prolong(sgwg_family* fam, int mi, int interp_mode, double eps, double* out, size_t n,
                 int out_is_device);

/* ---- combined-field diagnostics and output (runner.hpp) ----- */
/* Diagnostics of the combined finest-grid field (combine(set, mode, eps)),
 * reduced on the device slab by slab (the field is never downloaded):
 *   mass      quadrature_mass (models.hpp:75-94)
 *   min, max  field_min / field_max (runner.hpp:202-211)
 *   l1, linf  error_norms (diag.hpp:30-43) against the exact solution: linear
 *             advection of a periodic preset, u0(x - a t) (exact_preset one of
 *             SGWG_IC_C1, _C3, _EX1, _EX2, SGWG_ADVECTION model), or the Burgers
 *             sine waves before the shock (SGWG_IC_C2 in 2D, SGWG_IC_EX3;
 *             burgers_sine_exact models.hpp:533-560); -1: none (l1 = linf = NaN). */
typedef struct sgwg_field_stats {
  double mass;
  double min, max;
  double l1, linf;
  double points;  /* finest-grid points reduced */
} sgwg_field_stats;
int sgwg_combined_stats(sgwg_family* fam, int interp_mode, double eps, int exact_preset,
                        double t, sgwg_field_stats* out);
/* Combined field at npoints finest-grid multi-indices idx[p*d + k] (cut planes,
 * probes; write_cuts runner.hpp:159-200): each point equals the same point of
 * sgwg_combine (bitwise in the exact build) without forming the finest grid. */
int sgwg_eval_points(sgwg_family* fam, int interp_mode, double eps, const int* idx,
                     size_t npoints, double* out);
/* SGW5 snapshot of the combined field (write_field_dump, io.hpp:17-54): 64-byte
 * header + row-major float64 payload, streamed slab by slab from the device. */
int sgwg_write_snapshot(sgwg_family* fam, int interp_mode, double eps, const char* path);

/* ---- single-stage entry points (unit-level parity) ------------ */
/* FamilyModel::rhs (models.hpp:772-788) of every local member: tendency of the
 * current states into out (packed like the states). */
int sgwg_rhs(sgwg_family* fam, double* out, size_t n, int out_is_device);
/* One SspRk3::step (timestep.hpp:83-108) of every local member with a given dt. */
int sgwg_rk3_step(sgwg_family* fam, double dt, sgwg_failure* fail);

int sgwg_get_stats(const sgwg_family* fam, sgwg_stats* stats);

/* Vlasov-Poisson (new physics): charge density rho = 1 - int f dv and
 * field E (space_dim components) of the current member states, packed per
 * member (rho: x-points of each member; E: component-major per member). */
int sgwg_vp_field(sgwg_family* fam, double* rho, size_t nrho, double* E, size_t nE);
/* Per-step field energy of the last sgwg_evolve (BASELINE C4 "log|E|_2 recorded
 * per step"): out[s] = ||E_c||_2 at the start of step s, E_c = sum_m c_m I_m(E_m)
 * on the finest x-grid (I_m: separable degree-4 Lagrange interpolation,
 * interp.hpp:36-53), ||.||_2 with the finest x-spacings.  SGWG_EUNSUPPORTED on
 * a sharded family (the record would cover the local members only). */
int sgwg_field_energy(sgwg_family* fam, double* out, size_t cap, size_t* n);
/* profile-mode kernel table (entries sorted by name; *n = entries available) */
int sgwg_kernel_profile(const sgwg_family* fam, sgwg_kernel_timing* out, int cap, int* n);
int sgwg_kernel_profile_reset(sgwg_family* fam);
/* the stage kernel(s) the family's evolve launches (fixed at sgwg_set_model) */
const char* sgwg_stage_kernels(const sgwg_family* fam);

/* ---- host-side initial data: initialize_family (models.hpp:855-871) ------- */
/* Initial-condition presets of BASELINE C1-C5 and the paper examples,
 * evaluated with the host libm at the reference's coordinates
 * (restrict_to_grid, grid.hpp:166-186; normalize_initial models.hpp:97-102 for
 * the kinetic examples), then uploaded.  Bitwise equal to initialize_family. */
enum {
  SGWG_IC_C1 = 0,   /* sin(pi(x+y))                                   */
  SGWG_IC_C2 = 1,   /* 0.5 + sin(pi(x+y))                             */
  SGWG_IC_C3 = 2,   /* sin(pi(x+y+z))                                 */
  SGWG_IC_C4 = 3,   /* (1+0.01 cos(x/2)) exp(-v^2/2)/sqrt(2pi)        */
  SGWG_IC_C5 = 4,   /* (1+0.05(cos(x1/2)+cos(x2/2))) exp(-|v|^2/2)/2pi */
  SGWG_IC_EX1 = 5,  /* 0.3 + 0.7 sin(pi/2 (x+y))      models.hpp:605  */
  SGWG_IC_EX3 = 6,  /* 1 + 0.5 sin(sum x)             models.hpp:647  */
  SGWG_IC_EX5A = 7, /* models.hpp:690-694, mass-normalised            */
  SGWG_IC_EX5B = 8, /* models.hpp:709-714, mass-normalised            */
  SGWG_IC_EX2 = 9,  /* 1 + 0.5 sin(x+y+z)             models.hpp:625  */
  SGWG_IC_EX6 = 10  /* Vlasov-Maxwell two-stream + B3 = b sin(k0 x2), models.hpp:722-742 */
};
int sgwg_family_init_preset(sgwg_family* fam, int preset);
/* General initial data: ic(x, d, user) evaluated on the host at every grid
 * point of every local member (restrict_to_grid order), then uploaded. */
typedef double (*sgwg_ic_fn)(const double* x, int d, void* user);
int sgwg_family_init_fn(sgwg_family* fam, sgwg_ic_fn ic, void* user, int normalize_mass);

/* Roofline probe: average device time of one WENO stage kernel launch (RK
 * stage 1 of the current state, launched `reps` times back to back between
 * CUDA events on the family stream), with the algorithmic flops / HBM bytes
 * of one launch (SURVEY.md 8(d) counting). */
int sgwg_time_stage(sgwg_family* fam, int reps, double* avg_ms, double* flops, double* bytes);

/* DFMA throughput probe (TFLOP/s) used as the measured fp64 roofline peak. */
int sgwg_fp64_peak(sgwg_ctx* ctx, double* tflops);

#ifdef __cplusplus
}
#endif
#endif /* SGWG_H */
