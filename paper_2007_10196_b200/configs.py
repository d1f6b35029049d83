"""BASELINE.json configurations C1-C5 (and reference paper examples) as plain data.

Host-side presets only (the reference keeps these in make_example,
/root/reference/proj/include/sgweno/models.hpp:595-746).  Each config is a
dict consumed by the C-ABI wrapper (paper_2007_10196_b200.sgwg) and by the
test oracle adapters.  Deltas from the reference presets are listed in
SURVEY.md Appendix A.
"""
import math

PERIODIC, ZERO = 0, 1
ADVECTION, BURGERS, VLASOV_BOLTZMANN, VLASOV_POISSON, VLASOV_MAXWELL = 0, 1, 2, 3, 4
NONLINEAR, LINEAR = 0, 1
LAGRANGE, WENO = 0, 1
DT_CFL, DT_ACCURACY = 0, 1

# initial-condition presets (mirror oracle/sgw_oracle.h SGWO_IC_*; the same
# ids are understood by the C-ABI's host-side sgwg_family_init_preset)
IC_C1, IC_C2, IC_C3, IC_C4, IC_C5, IC_EX1, IC_EX3, IC_EX5A, IC_EX5B, IC_EX2, IC_EX6 = range(11)


def _finest_h(cfg):
    return min((cfg["upper"][k] - cfg["lower"][k]) / cfg["root"][k] / (1 << cfg["nl"])
               for k in range(cfg["d"]))


def config(name, **over):
    """Return the named configuration dict (copy); keyword overrides applied last."""
    pi = math.pi
    if name == "C1":
        c = dict(d=2, nl=3, lower=[0.0, 0.0], upper=[2.0, 2.0], root=[16, 16], bc=[PERIODIC] * 2,
                 kind=ADVECTION, speeds=[1.0, 1.0], weno_mode=NONLINEAR, epsilon=1e-6,
                 dt_mode=DT_ACCURACY, cfl=0.4, dt_scale=0.5, tfinal=1.0, stops=[],
                 interp=WENO, ic=IC_C1, space_dim=0)
    elif name == "C2":
        c = dict(d=2, nl=5, lower=[0.0, 0.0], upper=[2.0, 2.0], root=[32, 32], bc=[PERIODIC] * 2,
                 kind=BURGERS, speeds=[0.0, 0.0], weno_mode=NONLINEAR, epsilon=1e-6,
                 dt_mode=DT_CFL, cfl=0.5, dt_scale=1.0, tfinal=0.5, stops=[0.1],
                 interp=WENO, ic=IC_C2, space_dim=0)
    elif name == "C3":
        c = dict(d=3, nl=4, lower=[0.0] * 3, upper=[2.0] * 3, root=[16] * 3, bc=[PERIODIC] * 3,
                 kind=ADVECTION, speeds=[1.0, 1.0, 1.0], weno_mode=NONLINEAR, epsilon=1e-6,
                 dt_mode=DT_ACCURACY, cfl=0.4, dt_scale=1.0, tfinal=0.5, stops=[],
                 interp=WENO, ic=IC_C3, space_dim=0)
    elif name == "C4":
        c = dict(d=2, nl=5, lower=[0.0, -2 * pi], upper=[4 * pi, 2 * pi], root=[32, 32],
                 bc=[PERIODIC, ZERO], kind=VLASOV_POISSON, speeds=[0.0] * 2,
                 weno_mode=NONLINEAR, epsilon=1e-6, dt_mode=DT_CFL, cfl=0.5, dt_scale=1.0,
                 tfinal=40.0, stops=[], interp=WENO, ic=IC_C4, space_dim=1)
    elif name == "C5":
        c = dict(d=4, nl=5, lower=[0.0, 0.0, -6.0, -6.0], upper=[4 * pi, 4 * pi, 6.0, 6.0],
                 root=[8] * 4, bc=[PERIODIC, PERIODIC, ZERO, ZERO], kind=VLASOV_POISSON,
                 speeds=[0.0] * 4, weno_mode=NONLINEAR, epsilon=1e-6, dt_mode=DT_CFL, cfl=0.5,
                 dt_scale=1.0, tfinal=20.0, stops=[], interp=WENO, ic=IC_C5, space_dim=2)
    elif name == "ex1":   # models.hpp:599-618 (Table 1 of the paper)
        c = dict(d=2, nl=3, lower=[0.0, 0.0], upper=[4.0, 4.0], root=[10, 10], bc=[PERIODIC] * 2,
                 kind=ADVECTION, speeds=[1.0, 1.0], weno_mode=LINEAR, epsilon=1e-6,
                 dt_mode=DT_ACCURACY, cfl=0.4, dt_scale=1.0, tfinal=0.5, stops=[],
                 interp=LAGRANGE, ic=IC_EX1, space_dim=0)
    elif name == "ex2":   # models.hpp:619-638 (Table 2): 3D linear advection
        c = dict(d=3, nl=3, lower=[0.0] * 3, upper=[2 * pi] * 3, root=[10] * 3,
                 bc=[PERIODIC] * 3, kind=ADVECTION, speeds=[1.0, 1.0, 1.0], weno_mode=LINEAR,
                 epsilon=1e-6, dt_mode=DT_ACCURACY, cfl=0.4, dt_scale=1.0, tfinal=0.5, stops=[],
                 interp=LAGRANGE, ic=IC_EX2, space_dim=0)
    elif name == "ex3b":  # models.hpp:639-664 (3D Burgers), T = 0.1
        c = dict(d=3, nl=3, lower=[0.0] * 3, upper=[2 * pi] * 3, root=[10] * 3,
                 bc=[PERIODIC] * 3, kind=BURGERS, speeds=[0.0] * 3, weno_mode=NONLINEAR,
                 epsilon=1e-6, dt_mode=DT_ACCURACY, cfl=0.4, dt_scale=1.0, tfinal=0.1, stops=[],
                 interp=WENO, ic=IC_EX3, space_dim=0)
    elif name == "ex3a":  # models.hpp:639-664 (Table 4), paper epsilon 1e-3
        c = dict(d=2, nl=3, lower=[0.0, 0.0], upper=[2 * pi, 2 * pi], root=[10, 10],
                 bc=[PERIODIC] * 2, kind=BURGERS, speeds=[0.0, 0.0], weno_mode=NONLINEAR,
                 epsilon=1e-3, dt_mode=DT_ACCURACY, cfl=0.4, dt_scale=1.0, tfinal=0.3, stops=[],
                 interp=WENO, ic=IC_EX3, space_dim=0)
    elif name == "ex5a":  # models.hpp:683-701 (Vlasov-Boltzmann, E = -x)
        c = dict(d=2, nl=3, lower=[-5.0, -5.0], upper=[5.0, 5.0], root=[10, 10], bc=[ZERO] * 2,
                 kind=VLASOV_BOLTZMANN, speeds=[0.0] * 2, weno_mode=NONLINEAR, epsilon=1e-6,
                 dt_mode=DT_CFL, cfl=0.4, dt_scale=1.0, tfinal=6.0, stops=[0.5, 1.0, 2.0, 3.0],
                 interp=WENO, ic=IC_EX5A, space_dim=1, theta=1.0, tau=1.0)
    elif name == "ex5b":  # models.hpp:702-721
        c = dict(d=4, nl=3, lower=[-5.0] * 4, upper=[5.0] * 4, root=[10] * 4, bc=[ZERO] * 4,
                 kind=VLASOV_BOLTZMANN, speeds=[0.0] * 4, weno_mode=NONLINEAR, epsilon=1e-6,
                 dt_mode=DT_CFL, cfl=0.4, dt_scale=1.0, tfinal=3.0, stops=[0.5, 1.0],
                 interp=WENO, ic=IC_EX5B, space_dim=2, theta=1.0, tau=1.0)
    elif name == "ex6":   # models.hpp:722-742: reduced Vlasov-Maxwell (x2, xi1, xi2), k0 = 0.2
        c = dict(d=3, nl=3, lower=[0.0, -1.2, -1.2], upper=[2 * pi / 0.2, 1.2, 1.2],
                 root=[10] * 3, bc=[PERIODIC, ZERO, ZERO], kind=VLASOV_MAXWELL, speeds=[0.0] * 3,
                 weno_mode=NONLINEAR, epsilon=1e-6, dt_mode=DT_CFL, cfl=0.4, dt_scale=1.0,
                 tfinal=10.0, stops=[10.0], interp=WENO, ic=IC_EX6, space_dim=1)
    elif name == "S2":    # large-problem stress case for the kernel roofline:
        # C2's physics on root 2048, N_L = 1 (3 members, 20.97M points per stage)
        c = dict(d=2, nl=1, lower=[0.0, 0.0], upper=[2.0, 2.0], root=[2048, 2048],
                 bc=[PERIODIC] * 2, kind=BURGERS, speeds=[0.0, 0.0], weno_mode=NONLINEAR,
                 epsilon=1e-6, dt_mode=DT_CFL, cfl=0.5, dt_scale=1.0, tfinal=0.002, stops=[],
                 interp=WENO, ic=IC_C2, space_dim=0)
    elif name == "S3":    # 3D advection stress case: root 128, N_L = 2 (10 members, 8.4M pts)
        c = dict(d=3, nl=2, lower=[0.0] * 3, upper=[2.0] * 3, root=[128] * 3, bc=[PERIODIC] * 3,
                 kind=ADVECTION, speeds=[1.0, 1.0, 1.0], weno_mode=NONLINEAR, epsilon=1e-6,
                 dt_mode=DT_ACCURACY, cfl=0.4, dt_scale=1.0, tfinal=0.0002, stops=[],
                 interp=WENO, ic=IC_C3, space_dim=0)
    else:
        raise KeyError(name)
    c.setdefault("theta", 1.0)
    c.setdefault("tau", 1.0)
    c["name"] = name
    c.update(over)
    c["reference_spacing"] = over.get("reference_spacing", _finest_h(c))
    return c
