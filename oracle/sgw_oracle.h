/*
 * sgw_oracle.h -- CPU restatement of the reference sgweno hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This is the parity oracle for the B200 path; it is
 * linked only by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference leg.  The product (paper_2007_10196_b200/libsgwg.so) never
 * calls it and has no CPU fallback.
 *
 * Every function restates the reference algorithm in plain C99 with the
 * reference's expression order, so that a build with -ffp-contract=off is
 * bitwise identical to the reference headers (pinned by
 * tests/test_oracle_pin.py against oracle/_ref/libsgwref.so and the golden
 * fixtures under tests/golden/).  File:line citations are relative to
 * /root/reference/proj/include/sgweno/.
 *
 * The Vlasov-Poisson model (kind SGWO_VLASOV_POISSON) has NO reference
 * counterpart: it follows the kinetic transport template of
 * vb_rhs_into (models.hpp:334-363) with the prescribed field replaced by a
 * periodic spectral Poisson solve.  Parity for it is UNPINNED w.r.t. the
 * reference.
 */
#ifndef SGW_ORACLE_H
#define SGW_ORACLE_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SGWO_MAXD 4

enum { SGWO_PERIODIC = 0, SGWO_ZERO = 1 };
enum {
  SGWO_ADVECTION = 0,
  SGWO_BURGERS = 1,
  SGWO_VLASOV_BOLTZMANN = 2,
  SGWO_VLASOV_POISSON = 3,
  SGWO_VLASOV_MAXWELL = 4 /* reference only (oracle/ref_driver.cpp); no C restatement */
};
enum { SGWO_WENO_NONLINEAR = 0, SGWO_WENO_LINEAR = 1 };
enum { SGWO_INTERP_LAGRANGE = 0, SGWO_INTERP_WENO = 1 };
enum { SGWO_DT_CFL = 0, SGWO_DT_ACCURACY = 1 };

/* status codes (mirror of the C-ABI's) */
enum { SGWO_OK = 0, SGWO_EINVAL = 1, SGWO_ENONFINITE = 2 };

typedef struct {
  int d;                     /* 1..4 */
  int nl;                    /* finest level N_L */
  double lower[SGWO_MAXD];
  double upper[SGWO_MAXD];
  int root_cells[SGWO_MAXD];
  int bc[SGWO_MAXD];         /* SGWO_PERIODIC / SGWO_ZERO */
} sgwo_domain;

typedef struct {
  int kind;                  /* SGWO_ADVECTION ... */
  int weno_mode;             /* SGWO_WENO_NONLINEAR / LINEAR */
  double epsilon;            /* WENO epsilon (weno.hpp:20) */
  double speeds[SGWO_MAXD];  /* advection speeds */
  int space_dim;             /* kinetic models: phase space has 2*space_dim dims */
  double theta, tau;         /* Vlasov-Boltzmann relaxation */
} sgwo_model;

typedef struct {
  int mode;                  /* SGWO_DT_CFL / SGWO_DT_ACCURACY */
  double cfl;
  double reference_spacing;
  double dt_scale;           /* accuracy-mode multiplier; 1.0 = reference rule */
} sgwo_policy;

typedef void (*sgwo_stop_cb)(double t, void* user);

/* grid.hpp:57-79, sorted lexicographically (combine.hpp:71-72). Returns count, -1 on error. */
int sgwo_enumerate_levels(int d, int nl, int* out, int cap);
/* combine.hpp:34-43 */
int sgwo_combination_coefficients(int d, int nl, long long* coef);
/* grid.hpp:110-133 */
void sgwo_member_geometry(const sgwo_domain* dom, const int* level, int* points, double* spacing);
size_t sgwo_member_points(const sgwo_domain* dom, const int* level);

/* weno.hpp:36-44, 60-72 */
void sgwo_smoothness_indicators(const double* s, double* b);
double sgwo_weno5_flux_positive(const double* s, double eps, int mode);
double sgwo_weno5_flux_negative(const double* s, double eps, int mode);

/* weno.hpp:118-154 (flux_kind 1: Burgers 0.5u^2, 2: linear c*u, generic kernel)
 * weno.hpp:160-192 (flux_kind 0: advect_derivative_line with coefficient c). */
int sgwo_weno_derivative_line(const double* u, int n, int flux_kind, double c, double alpha,
                              double dx, int bc, double eps, int mode, double* out);

/* models.hpp:184-198 / 334-363 (+ VP restatement). out = tendency. */
int sgwo_rhs(const sgwo_domain* dom, const int* level, const sgwo_model* model,
             const double* state, double* out);

/* timestep.hpp:83-108: in-place SSP-RK3 step; returns 0 or failing stage (1..3). */
int sgwo_rk3_step(const sgwo_domain* dom, const int* level, const sgwo_model* model,
                  double* state, double dt);

/* timestep.hpp:47-67 */
double sgwo_compute_dt(const sgwo_policy* p, const double* speeds, const double* spacings, int d,
                       double remaining);

/* models.hpp:791-839 family wave speeds for the packed family states. */
int sgwo_family_wave_speeds(const sgwo_domain* dom, const sgwo_model* model, const double* states,
                            double* speeds);

/* timestep.hpp:126-174 evolve_family over the packed member states (member order =
 * sorted levels).  dts/cap receive the dt sequence; nsteps its length.  On a
 * non-finite tendency returns SGWO_ENONFINITE with fail_{member,step,stage}. */
/* member-level OpenMP threads of sgwo_evolve / sgwo_combine (default 1);
 * results are bitwise independent of the count */
void sgwo_set_threads(int n);
int sgwo_get_threads(void);

int sgwo_evolve(const sgwo_domain* dom, const sgwo_model* model, const sgwo_policy* pol,
                double* states, double tfinal, const double* stops, int nstops, sgwo_stop_cb cb,
                void* user, double* dts, long cap, long* nsteps, int* fail_member,
                long* fail_step, int* fail_stage);

/* interp.hpp:197-250 prolongation of one member onto the finest grid. */
int sgwo_prolong(const sgwo_domain* dom, const int* level, const double* src, int interp_mode,
                 double eps, double* dst);
/* interp.hpp:151-189 one dyadic upsampling line (m = refinement exponent). */
int sgwo_upsample_line(const double* src, int n_src, double* dst, int n_dst, int m, int bc,
                       int interp_mode, double eps);
/* combine.hpp:95-122 */
int sgwo_combine(const sgwo_domain* dom, const double* states, int interp_mode, double eps,
                 double* out);

/* The combined solution on the finest-grid box [lo_k, hi_k) (row-major), each
 * member prolonged only on the lines the box reads: bitwise equal to the same
 * entries of sgwo_combine (cut planes of configurations whose finest grid is
 * too large to materialise). */
int sgwo_combine_box(const sgwo_domain* dom, const double* states, int interp_mode, double eps,
                     const int* lo, const int* hi, double* out);
/* Vlasov-Poisson field-energy record (sgwg_field_energy's definition) of the
 * packed family states, and an optional per-step record filled by sgwo_evolve. */
double sgwo_field_energy(const sgwo_domain* dom, int space_dim, const double* states);
void sgwo_set_energy_record(double* buf, long cap);
/* stop sgwo_evolve after n steps (0 = no limit; bounded CPU baselines) */
void sgwo_set_max_steps(long n);

size_t sgwo_family_total_points(const sgwo_domain* dom);
size_t sgwo_finest_points(const sgwo_domain* dom);

/* Initial-condition presets restricted like restrict_to_grid (grid.hpp:166-186),
 * including normalize_initial (models.hpp:97-102) for the VB presets. */
enum {
  SGWO_IC_C1 = 0,     /* sin(pi(x+y)) */
  SGWO_IC_C2 = 1,     /* 0.5 + sin(pi(x+y)) */
  SGWO_IC_C3 = 2,     /* sin(pi(x+y+z)) */
  SGWO_IC_C4 = 3,     /* 1D1V Landau */
  SGWO_IC_C5 = 4,     /* 2D2V Landau */
  SGWO_IC_EX1 = 5,    /* 0.3 + 0.7 sin(pi/2 (x+y)) */
  SGWO_IC_EX3 = 6,    /* 1 + 0.5 sin(sum x) */
  SGWO_IC_EX5A = 7,   /* sin^2(x^2/2) exp(-(x^2+v^2)/2), normalized */
  SGWO_IC_EX5B = 8,   /* 4D VB, normalized */
  SGWO_IC_EX2 = 9,    /* 1 + 0.5 sin(x+y+z) */
  SGWO_IC_EX6 = 10    /* Vlasov-Maxwell ex6 (reference only) */
};
int sgwo_restrict_preset(int preset, const sgwo_domain* dom, const int* level, double* out);
int sgwo_init_family(int preset, const sgwo_domain* dom, double* states);

/* Vlasov-Poisson field of one member: rho(x) = 1 - int f dv, E = -grad phi,
 * -lap phi = rho (periodic, spectral).  E has space_dim * nx entries (component-major). */
int sgwo_vp_field(const sgwo_domain* dom, const int* level, int space_dim, const double* f,
                  double* rho, double* E);

#ifdef __cplusplus
}
#endif
#endif
