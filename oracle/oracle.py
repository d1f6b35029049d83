"""ctypes front-end for the CPU parity oracle (TEST INFRASTRUCTURE ONLY).

Two libraries, both built by ``oracle/Makefile``:

* ``oracle/liboracle.so`` -- the plain-C restatement ``oracle/sgw_oracle.c``
  (always available; travels to the GPU box).
* ``oracle/_ref/libsgwref.so`` -- the unmodified reference headers
  (``/root/reference/proj/include/sgweno``) driven in place by
  ``oracle/ref_driver.cpp``; built only where the reference exists, then
  travels with the snapshot (git-ignored).

Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU-baseline /
``--impl reference`` leg may import this module.  The product path
(``paper_2007_10196_b200``) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libsgwref.so")

PERIODIC, ZERO = 0, 1
ADVECTION, BURGERS, VLASOV_BOLTZMANN, VLASOV_POISSON, VLASOV_MAXWELL = 0, 1, 2, 3, 4
NONLINEAR, LINEAR = 0, 1
LAGRANGE, WENO = 0, 1
DT_CFL, DT_ACCURACY = 0, 1


class Domain(C.Structure):
    _fields_ = [("d", C.c_int), ("nl", C.c_int), ("lower", C.c_double * 4),
                ("upper", C.c_double * 4), ("root_cells", C.c_int * 4), ("bc", C.c_int * 4)]


class Model(C.Structure):
    _fields_ = [("kind", C.c_int), ("weno_mode", C.c_int), ("epsilon", C.c_double),
                ("speeds", C.c_double * 4), ("space_dim", C.c_int), ("theta", C.c_double),
                ("tau", C.c_double)]


class Policy(C.Structure):
    _fields_ = [("mode", C.c_int), ("cfl", C.c_double), ("reference_spacing", C.c_double),
                ("dt_scale", C.c_double)]


def make_domain(d, nl, lower, upper, root, bc):
    dom = Domain()
    dom.d, dom.nl = d, nl
    for k in range(d):
        dom.lower[k], dom.upper[k] = lower[k], upper[k]
        dom.root_cells[k], dom.bc[k] = root[k], bc[k]
    return dom


def make_model(kind, weno_mode=NONLINEAR, epsilon=1e-6, speeds=(0, 0, 0, 0), space_dim=0,
               theta=1.0, tau=1.0):
    m = Model()
    m.kind, m.weno_mode, m.epsilon = kind, weno_mode, epsilon
    for k, s in enumerate(speeds):
        m.speeds[k] = s
    m.space_dim, m.theta, m.tau = space_dim, theta, tau
    return m


def make_policy(mode, cfl=0.4, reference_spacing=0.0, dt_scale=1.0):
    p = Policy()
    p.mode, p.cfl, p.reference_spacing, p.dt_scale = mode, cfl, reference_spacing, dt_scale
    return p


_DP = C.POINTER(C.c_double)
_IP = C.POINTER(C.c_int)
STOP_CB = C.CFUNCTYPE(None, C.c_double, C.c_void_p)
REF_STOP_CB = C.CFUNCTYPE(None, C.c_double, _DP, C.c_void_p)


def _dp(a):
    return a.ctypes.data_as(_DP)


def _ip(a):
    return a.ctypes.data_as(_IP)


def build():
    """Compile the oracle (and, where /root/reference exists, oracle/_ref)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def _load(path):
    if not os.path.exists(path) and path == ORACLE_SO:
        build()
    return C.CDLL(path)


class _Lib:
    """Common wrappers; `prefix` selects the C restatement or the reference driver."""

    def __init__(self, path, prefix):
        self.lib = _load(path)
        self.prefix = prefix
        L = self.lib
        f = getattr(L, prefix + "enumerate_levels")
        f.argtypes = [C.c_int, C.c_int, _IP, C.c_int]
        f.restype = C.c_int
        self._enum = f
        f = getattr(L, prefix + "weno5_flux_positive")
        f.argtypes = [_DP, C.c_double, C.c_int]
        f.restype = C.c_double
        self._fpos = f
        f = getattr(L, prefix + "weno_derivative_line")
        f.argtypes = [_DP, C.c_int, C.c_int, C.c_double, C.c_double, C.c_double, C.c_int,
                      C.c_double, C.c_int, _DP]
        f.restype = C.c_int
        self._wline = f
        f = getattr(L, prefix + "rhs")
        f.argtypes = [C.POINTER(Domain), _IP, C.POINTER(Model), _DP, _DP]
        f.restype = C.c_int
        self._rhs = f
        f = getattr(L, prefix + "upsample_line")
        f.argtypes = [_DP, C.c_int, _DP, C.c_int, C.c_int, C.c_int, C.c_int, C.c_double]
        f.restype = C.c_int
        self._ups = f
        f = getattr(L, prefix + "prolong")
        f.argtypes = [C.POINTER(Domain), _IP, _DP, C.c_int, C.c_double, _DP]
        f.restype = C.c_int
        self._prolong = f

    # -- geometry -------------------------------------------------------------
    def levels(self, d, nl):
        n = self._enum(d, nl, None, 0)
        if n < 0:
            raise ValueError("enumerate_levels: invalid arguments")
        out = np.zeros(n * d, dtype=np.int32)
        self._enum(d, nl, _ip(out), n)
        return out.reshape(n, d)

    # -- kernels --------------------------------------------------------------
    def weno5_flux_positive(self, s, eps=1e-6, mode=NONLINEAR):
        s = np.ascontiguousarray(s, dtype=np.float64)
        return self._fpos(_dp(s), eps, mode)

    def weno_derivative_line(self, u, flux_kind, c=0.0, alpha=0.0, dx=1.0, bc=PERIODIC,
                             eps=1e-6, mode=NONLINEAR):
        u = np.ascontiguousarray(u, dtype=np.float64)
        out = np.zeros_like(u)
        st = self._wline(_dp(u), len(u), flux_kind, c, alpha, dx, bc, eps, mode, _dp(out))
        if st:
            raise ValueError("weno_derivative_line: invalid arguments")
        return out

    def rhs(self, dom, level, model, state):
        level = np.ascontiguousarray(level, dtype=np.int32)
        state = np.ascontiguousarray(state, dtype=np.float64)
        out = np.zeros_like(state)
        st = self._rhs(C.byref(dom), _ip(level), C.byref(model), _dp(state), _dp(out))
        if st:
            raise ValueError("rhs: invalid arguments")
        return out

    def upsample_line(self, src, n_dst, m, bc, mode, eps=1e-6):
        src = np.ascontiguousarray(src, dtype=np.float64)
        dst = np.zeros(n_dst)
        st = self._ups(_dp(src), len(src), _dp(dst), n_dst, m, bc, mode, eps)
        if st:
            raise ValueError("upsample_line failed")
        return dst

    def prolong(self, dom, level, src, mode, eps, n_out):
        level = np.ascontiguousarray(level, dtype=np.int32)
        src = np.ascontiguousarray(src, dtype=np.float64)
        dst = np.zeros(n_out)
        st = self._prolong(C.byref(dom), _ip(level), _dp(src), mode, eps, _dp(dst))
        if st:
            raise ValueError("prolong failed")
        return dst


class Oracle(_Lib):
    """The C restatement (oracle/sgw_oracle.c)."""

    def __init__(self):
        super().__init__(ORACLE_SO, "sgwo_")
        L = self.lib
        L.sgwo_evolve.argtypes = [C.POINTER(Domain), C.POINTER(Model), C.POINTER(Policy), _DP,
                                  C.c_double, _DP, C.c_int, STOP_CB, C.c_void_p, _DP, C.c_long,
                                  C.POINTER(C.c_long), _IP, C.POINTER(C.c_long), _IP]
        L.sgwo_evolve.restype = C.c_int
        L.sgwo_combine.argtypes = [C.POINTER(Domain), _DP, C.c_int, C.c_double, _DP]
        L.sgwo_combine.restype = C.c_int
        L.sgwo_init_family.argtypes = [C.c_int, C.POINTER(Domain), _DP]
        L.sgwo_init_family.restype = C.c_int
        L.sgwo_family_total_points.argtypes = [C.POINTER(Domain)]
        L.sgwo_family_total_points.restype = C.c_size_t
        L.sgwo_finest_points.argtypes = [C.POINTER(Domain)]
        L.sgwo_finest_points.restype = C.c_size_t
        L.sgwo_vp_field.argtypes = [C.POINTER(Domain), _IP, C.c_int, _DP, _DP, _DP]
        L.sgwo_vp_field.restype = C.c_int
        L.sgwo_rk3_step.argtypes = [C.POINTER(Domain), _IP, C.POINTER(Model), _DP, C.c_double]
        L.sgwo_rk3_step.restype = C.c_int
        L.sgwo_family_wave_speeds.argtypes = [C.POINTER(Domain), C.POINTER(Model), _DP, _DP]
        L.sgwo_family_wave_speeds.restype = C.c_int
        L.sgwo_restrict_preset.argtypes = [C.c_int, C.POINTER(Domain), _IP, _DP]
        L.sgwo_restrict_preset.restype = C.c_int
        L.sgwo_set_threads.argtypes = [C.c_int]
        L.sgwo_set_threads.restype = None
        L.sgwo_combine_box.argtypes = [C.POINTER(Domain), _DP, C.c_int, C.c_double, _IP, _IP, _DP]
        L.sgwo_combine_box.restype = C.c_int
        L.sgwo_field_energy.argtypes = [C.POINTER(Domain), C.c_int, _DP]
        L.sgwo_field_energy.restype = C.c_double
        L.sgwo_set_energy_record.argtypes = [_DP, C.c_long]
        L.sgwo_set_energy_record.restype = None
        L.sgwo_set_max_steps.argtypes = [C.c_long]
        L.sgwo_set_max_steps.restype = None
        self._energy_buf = None

    def combine_box(self, dom, states, lo, hi, mode=WENO, eps=1e-6):
        """the combined solution on the finest-grid box [lo, hi) (bitwise = combine)"""
        states = np.ascontiguousarray(states, dtype=np.float64)
        lo = np.ascontiguousarray(lo, dtype=np.int32)
        hi = np.ascontiguousarray(hi, dtype=np.int32)
        out = np.zeros(int(np.prod(hi - lo)))
        if self.lib.sgwo_combine_box(C.byref(dom), _dp(states), mode, eps, _ip(lo), _ip(hi),
                                     _dp(out)):
            raise ValueError("combine_box failed")
        return out.reshape(tuple(int(h - l) for l, h in zip(lo, hi)))

    def field_energy(self, dom, space_dim, states):
        states = np.ascontiguousarray(states, dtype=np.float64)
        return float(self.lib.sgwo_field_energy(C.byref(dom), space_dim, _dp(states)))

    def record_energy(self, cap):
        """start a per-step field-energy record in evolve (None: stop); returns the buffer"""
        if cap is None:
            self.lib.sgwo_set_energy_record(None, 0)
            self._energy_buf = None
            return None
        self._energy_buf = np.zeros(int(cap))
        self.lib.sgwo_set_energy_record(_dp(self._energy_buf), int(cap))
        return self._energy_buf

    def set_max_steps(self, n):
        """stop evolve after n steps (0: no limit)"""
        self.lib.sgwo_set_max_steps(int(n))
        return self

    def set_threads(self, n):
        """member-level OpenMP threads (bitwise-identical results for any n)"""
        self.lib.sgwo_set_threads(int(n))
        return self

    def total_points(self, dom):
        return int(self.lib.sgwo_family_total_points(C.byref(dom)))

    def finest_points(self, dom):
        return int(self.lib.sgwo_finest_points(C.byref(dom)))

    def init_family(self, preset, dom):
        s = np.zeros(self.total_points(dom))
        if self.lib.sgwo_init_family(preset, C.byref(dom), _dp(s)):
            raise ValueError("init_family failed")
        return s

    def restrict(self, preset, dom, level, n):
        level = np.ascontiguousarray(level, dtype=np.int32)
        out = np.zeros(n)
        self.lib.sgwo_restrict_preset(preset, C.byref(dom), _ip(level), _dp(out))
        return out

    def rk3_step(self, dom, level, model, state, dt):
        level = np.ascontiguousarray(level, dtype=np.int32)
        s = np.array(state, dtype=np.float64)
        f = self.lib.sgwo_rk3_step(C.byref(dom), _ip(level), C.byref(model), _dp(s), dt)
        return s, f

    def evolve(self, dom, model, policy, states, tfinal, stops=(), on_stop=None, cap=1 << 20):
        """Returns (states, dts, status, (member, step, stage)). on_stop(t, states)."""
        states = np.array(states, dtype=np.float64)
        stops = np.ascontiguousarray(stops, dtype=np.float64)
        dts = np.zeros(cap)
        ns = C.c_long(0)
        fm, fst, fsg = C.c_int(-1), C.c_long(-1), C.c_int(0)

        def _cb(t, user):
            if on_stop is not None:
                on_stop(t, states.copy())

        cb = STOP_CB(_cb)
        st = self.lib.sgwo_evolve(C.byref(dom), C.byref(model), C.byref(policy), _dp(states),
                                  tfinal, _dp(stops) if len(stops) else None, len(stops), cb,
                                  None, _dp(dts), cap, C.byref(ns), C.byref(fm), C.byref(fst),
                                  C.byref(fsg))
        return states, dts[:ns.value].copy(), st, (fm.value, fst.value, fsg.value)

    def combine(self, dom, states, mode=WENO, eps=1e-6):
        states = np.ascontiguousarray(states, dtype=np.float64)
        out = np.zeros(self.finest_points(dom))
        if self.lib.sgwo_combine(C.byref(dom), _dp(states), mode, eps, _dp(out)):
            raise ValueError("combine failed")
        return out

    def vp_field(self, dom, level, space_dim, f, nx):
        level = np.ascontiguousarray(level, dtype=np.int32)
        f = np.ascontiguousarray(f, dtype=np.float64)
        rho = np.zeros(nx)
        E = np.zeros(nx * space_dim)
        if self.lib.sgwo_vp_field(C.byref(dom), _ip(level), space_dim, _dp(f), _dp(rho), _dp(E)):
            raise ValueError("vp_field failed")
        return rho, E.reshape(space_dim, nx)

    def wave_speeds(self, dom, model, states):
        states = np.ascontiguousarray(states, dtype=np.float64)
        sp = np.zeros(4)
        self.lib.sgwo_family_wave_speeds(C.byref(dom), C.byref(model), _dp(states), _dp(sp))
        return sp[:dom.d]


def ref_available():
    return os.path.exists(REF_SO)


class Reference(_Lib):
    """The reference headers themselves (oracle/_ref/libsgwref.so)."""

    def __init__(self):
        if not os.path.exists(REF_SO):
            raise FileNotFoundError(REF_SO)
        super().__init__(REF_SO, "sgwref_")
        L = self.lib
        L.sgwref_evolve.argtypes = [C.POINTER(Domain), C.POINTER(Model), C.POINTER(Policy), _DP,
                                    C.c_double, _DP, C.c_int, REF_STOP_CB, C.c_void_p, C.c_int,
                                    _DP, C.c_long, C.POINTER(C.c_long), _IP, C.POINTER(C.c_long),
                                    _IP, _DP]
        L.sgwref_evolve.restype = C.c_int
        L.sgwref_evolve_replay.argtypes = [C.POINTER(Domain), C.POINTER(Model), C.POINTER(Policy),
                                           _DP, C.c_double, _DP, C.c_int, _DP, C.c_long,
                                           C.POINTER(C.c_long)]
        L.sgwref_evolve_replay.restype = C.c_int
        L.sgwref_combine.argtypes = [C.POINTER(Domain), _DP, C.c_int, C.c_double, _DP, C.c_int]
        L.sgwref_combine.restype = C.c_int
        L.sgwref_rhs.argtypes = [C.POINTER(Domain), _IP, C.POINTER(Model), _DP, _DP]
        L.sgwref_rhs.restype = C.c_int
        L.sgwref_init_family.argtypes = [C.c_int, C.POINTER(Domain), C.POINTER(Model), _DP]
        L.sgwref_init_family.restype = C.c_int
        L.sgwref_time_prefix.argtypes = [C.POINTER(Domain), C.POINTER(Model), C.POINTER(Policy),
                                         C.c_int, C.c_double, C.c_int, _DP, C.POINTER(C.c_long),
                                         _DP, C.c_int]
        L.sgwref_time_prefix.restype = C.c_int
        self._o = Oracle()

    def init_family(self, preset, dom, model, state_points=None):
        """state_points: member-state doubles when they exceed the grid points
        (Vlasov-Maxwell: + 3 field lines per member)."""
        s = np.zeros(state_points or self._o.total_points(dom))
        if self.lib.sgwref_init_family(preset, C.byref(dom), C.byref(model), _dp(s)):
            raise ValueError("init_family failed")
        return s

    def evolve(self, dom, model, policy, states, tfinal, stops=(), on_stop=None, threads=1,
               cap=1 << 20):
        states = np.array(states, dtype=np.float64)
        stops = np.ascontiguousarray(stops, dtype=np.float64)
        dts = np.zeros(cap)
        ns = C.c_long(0)
        fm, fst, fsg = C.c_int(-1), C.c_long(-1), C.c_int(0)
        secs = C.c_double(0)
        n = len(states)

        def _cb(t, ptr, user):
            if on_stop is not None:
                on_stop(t, np.ctypeslib.as_array(ptr, shape=(n,)).copy())

        cb = REF_STOP_CB(_cb)
        st = self.lib.sgwref_evolve(C.byref(dom), C.byref(model), C.byref(policy), _dp(states),
                                    tfinal, _dp(stops) if len(stops) else None, len(stops), cb,
                                    None, threads, _dp(dts), cap, C.byref(ns), C.byref(fm),
                                    C.byref(fst), C.byref(fsg), C.byref(secs))
        return states, dts[:ns.value].copy(), st, (fm.value, fst.value, fsg.value)

    def evolve_replay(self, dom, model, policy, states, tfinal, stops=(), cap=1 << 20):
        states = np.array(states, dtype=np.float64)
        stops = np.ascontiguousarray(stops, dtype=np.float64)
        dts = np.zeros(cap)
        ns = C.c_long(0)
        self.lib.sgwref_evolve_replay(C.byref(dom), C.byref(model), C.byref(policy), _dp(states),
                                      tfinal, _dp(stops) if len(stops) else None, len(stops),
                                      _dp(dts), cap, C.byref(ns))
        return states, dts[:ns.value].copy()

    def rhs(self, dom, level, model, state):
        """FamilyModel::rhs of one member (state incl. any field lines)"""
        level = np.ascontiguousarray(level, dtype=np.int32)
        state = np.ascontiguousarray(state, dtype=np.float64)
        out = np.zeros_like(state)
        if self.lib.sgwref_rhs(C.byref(dom), _ip(level), C.byref(model), _dp(state), _dp(out)):
            raise ValueError("rhs failed")
        return out

    def combine(self, dom, states, mode=WENO, eps=1e-6, threads=1):
        states = np.ascontiguousarray(states, dtype=np.float64)
        out = np.zeros(self._o.finest_points(dom))
        if self.lib.sgwref_combine(C.byref(dom), _dp(states), mode, eps, _dp(out), threads):
            raise ValueError("combine failed")
        return out

    def time_prefix(self, dom, model, policy, preset, tfinal, threads=1, interp_mode=WENO,
                    with_combine=False):
        """(evolve seconds, steps, combine seconds or 0).  The reference's combine
        materialises the whole finest grid on the host: off unless asked for."""
        secs, csecs = C.c_double(0), C.c_double(0)
        ns = C.c_long(0)
        st = self.lib.sgwref_time_prefix(C.byref(dom), C.byref(model), C.byref(policy), preset,
                                         tfinal, threads, C.byref(secs), C.byref(ns),
                                         C.byref(csecs) if with_combine else None, interp_mode)
        if st:
            raise ValueError("time_prefix failed")
        return secs.value, ns.value, csecs.value
