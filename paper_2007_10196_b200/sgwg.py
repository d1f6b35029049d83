"""Python mirror of the reference ``sgweno`` solver interface over the C ABI.

The reference is a header-only C++ library; its public entry points for this
path are ``make_family`` (combine.hpp:69-83), ``initialize_family``
(models.hpp:855-871), ``FamilyModel`` (models.hpp:754-851), ``evolve_family``
(timestep.hpp:126-174), ``prolong`` (interp.hpp:197-250) and ``combine``
(combine.hpp:95-122).  :class:`Family` exposes the same operations, with the
same argument meaning and error behaviour (``ValueError`` for the reference's
``std::invalid_argument``, :class:`FamilyIntegratorFailure` for
``FamilyIntegratorFailure{level, step, stage}``), on top of ``libsgwg.so``
(include/sgwg.h).  There is no CPU fallback: if the extension or a Blackwell
GPU is missing every call raises.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Callable, Optional, Sequence

import numpy as np

from . import configs as _cfg

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SGWG_LIB") or os.path.join(HERE, "libsgwg.so")

OK, EINVAL, ENONFINITE, ECUDA, ENCCL, EUNSUPPORTED = range(6)
ARITH_EXACT, ARITH_FAST = 0, 1

_lib = None


class SgwgError(RuntimeError):
    """CUDA / NCCL / unsupported-feature failure of the B200 path."""


class FamilyIntegratorFailure(RuntimeError):
    """timestep.hpp:31-40: non-finite tendency of member `level` at (step, stage)."""

    def __init__(self, msg, member, level, step, stage):
        super().__init__(msg)
        self.member, self.level, self.step, self.stage = member, level, step, stage


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


class Failure(C.Structure):
    _fields_ = [("member", C.c_int), ("step", C.c_longlong), ("stage", C.c_int)]


class FieldStats(C.Structure):
    _fields_ = [("mass", C.c_double), ("min", C.c_double), ("max", C.c_double),
                ("l1", C.c_double), ("linf", C.c_double), ("points", C.c_double)]


class Stats(C.Structure):
    _fields_ = [("evolve_ms", C.c_double), ("combine_ms", C.c_double), ("steps", C.c_longlong),
                ("kernel_launches", C.c_longlong), ("combine_launches", C.c_longlong),
                ("pass_ms_sum", C.c_double), ("pass_launches", C.c_longlong),
                ("pass_flops", C.c_double), ("pass_bytes", C.c_double)]


class KernelTiming(C.Structure):
    _fields_ = [("name", C.c_char * 48), ("ms_sum", C.c_double), ("launches", C.c_longlong),
                ("flops_per_launch", C.c_double), ("bytes_per_launch", C.c_double)]


STOP_CB = C.CFUNCTYPE(None, C.c_double, C.c_void_p)
IC_CB = C.CFUNCTYPE(C.c_double, C.POINTER(C.c_double), C.c_int, C.c_void_p)
_DP = C.POINTER(C.c_double)
_IP = C.POINTER(C.c_int)
_VP = C.c_void_p

# name -> (restype, argtypes); must list every function of include/sgwg.h
SIGNATURES = {
    "sgwg_last_error": (C.c_char_p, []),
    "sgwg_version": (C.c_int, []),
    "sgwg_init": (C.c_int, [C.c_int, C.POINTER(_VP)]),
    "sgwg_shutdown": (C.c_int, [_VP]),
    "sgwg_set_arith": (C.c_int, [_VP, C.c_int]),
    "sgwg_set_profile": (C.c_int, [_VP, C.c_int]),
    "sgwg_stream": (_VP, [_VP]),
    "sgwg_family_create": (C.c_int, [_VP, C.POINTER(Domain), C.POINTER(_VP)]),
    "sgwg_family_create_shard": (C.c_int, [_VP, C.POINTER(Domain), _IP, C.c_int,
                                           C.POINTER(_VP)]),
    "sgwg_family_destroy": (C.c_int, [_VP]),
    "sgwg_family_create_single": (C.c_int, [_VP, C.POINTER(Domain), C.POINTER(_VP)]),
    "sgwg_enumerate_levels": (C.c_int, [C.c_int, C.c_int, _IP, C.c_int, _IP]),
    "sgwg_family_num_members": (C.c_int, [_VP, _IP]),
    "sgwg_family_member": (C.c_int, [_VP, C.c_int, _IP, _IP, _IP]),
    "sgwg_family_sizes": (C.c_int, [_VP, C.POINTER(C.c_size_t), C.POINTER(C.c_size_t)]),
    "sgwg_family_upload": (C.c_int, [_VP, _DP, C.c_size_t]),
    "sgwg_family_download": (C.c_int, [_VP, _DP, C.c_size_t]),
    "sgwg_family_upload_device": (C.c_int, [_VP, _VP, C.c_size_t]),
    "sgwg_family_download_device": (C.c_int, [_VP, _VP, C.c_size_t]),
    "sgwg_set_model": (C.c_int, [_VP, C.POINTER(Model)]),
    "sgwg_nccl_unique_id": (C.c_int, [_VP]),
    "sgwg_family_set_comm": (C.c_int, [_VP, _VP, C.c_int, C.c_int]),
    "sgwg_evolve": (C.c_int, [_VP, C.POINTER(Policy), C.c_double, _DP, C.c_int, STOP_CB, _VP,
                              _DP, C.c_size_t, C.POINTER(C.c_size_t), C.POINTER(Failure)]),
    "sgwg_combine": (C.c_int, [_VP, C.c_int, C.c_double, _VP, C.c_size_t, C.c_int]),
    "sgwg_prolong": (C.c_int, [_VP, C.c_int, C.c_int, C.c_double, _VP, C.c_size_t, C.c_int]),
    "sgwg_rhs": (C.c_int, [_VP, _VP, C.c_size_t, C.c_int]),
    "sgwg_rk3_step": (C.c_int, [_VP, C.c_double, C.POINTER(Failure)]),
    "sgwg_get_stats": (C.c_int, [_VP, C.POINTER(Stats)]),
    "sgwg_family_init_preset": (C.c_int, [_VP, C.c_int]),
    "sgwg_family_init_fn": (C.c_int, [_VP, IC_CB, _VP, C.c_int]),
    "sgwg_fp64_peak": (C.c_int, [_VP, _DP]),
    "sgwg_time_stage": (C.c_int, [_VP, C.c_int, _DP, _DP, _DP]),
    "sgwg_combine_rows": (C.c_int, [_VP, C.c_int, C.c_double, C.c_longlong, C.c_longlong, _VP,
                                    C.c_size_t, C.c_int]),
    "sgwg_combine_local": (C.c_int, [_VP, C.c_int, C.c_double, _VP, C.c_size_t, C.c_int,
                                     C.POINTER(C.c_longlong), C.POINTER(C.c_longlong)]),
    "sgwg_vp_field": (C.c_int, [_VP, _DP, C.c_size_t, _DP, C.c_size_t]),
    "sgwg_field_energy": (C.c_int, [_VP, _DP, C.c_size_t, C.POINTER(C.c_size_t)]),
    "sgwg_combined_stats": (C.c_int, [_VP, C.c_int, C.c_double, C.c_int, C.c_double,
                                      C.POINTER(FieldStats)]),
    "sgwg_eval_points": (C.c_int, [_VP, C.c_int, C.c_double, C.POINTER(C.c_int), C.c_size_t,
                                   _DP]),
    "sgwg_write_snapshot": (C.c_int, [_VP, C.c_int, C.c_double, C.c_char_p]),
    "sgwg_kernel_profile": (C.c_int, [_VP, _VP, C.c_int, _IP]),
    "sgwg_kernel_profile_reset": (C.c_int, [_VP]),
    "sgwg_stage_kernels": (C.c_char_p, [_VP]),
}


def load():
    """Load the in-tree extension; raise (no fallback) when it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise SgwgError(f"{LIB_PATH} missing: run __graft_entry__.build() (no CPU fallback)")
    lib = C.CDLL(LIB_PATH, mode=C.RTLD_GLOBAL)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def _check(status, failure=None, family=None):
    if status == OK:
        return
    msg = load().sgwg_last_error().decode()
    if status == EINVAL:
        raise ValueError(msg)
    if status == ENONFINITE:
        level = None
        if failure is not None and family is not None and failure.member >= 0:
            level = tuple(family.all_levels[failure.member])
        raise FamilyIntegratorFailure(msg, failure.member if failure else -1, level,
                                      failure.step if failure else -1,
                                      failure.stage if failure else 0)
    raise SgwgError(f"[{status}] {msg}")


def enumerate_combination_levels(d: int, nl: int) -> np.ndarray:
    """grid.hpp:57-79 (sorted lexicographically)."""
    lib = load()
    cnt = C.c_int(0)
    _check(lib.sgwg_enumerate_levels(d, nl, None, 0, C.byref(cnt)))
    out = np.zeros(cnt.value * d, dtype=np.int32)
    _check(lib.sgwg_enumerate_levels(d, nl, out.ctypes.data_as(_IP), cnt.value, C.byref(cnt)))
    return out.reshape(cnt.value, d)


class Context:
    """One CUDA device (one process per GPU)."""

    def __init__(self, device: int = 0, arith: str = "exact", profile: bool = False):
        lib = load()
        h = _VP()
        _check(lib.sgwg_init(device, C.byref(h)))
        self.h = h
        self.device = device
        self.set_arith(arith)
        self.set_profile(profile)

    def set_arith(self, arith: str):
        self.arith = arith
        _check(load().sgwg_set_arith(self.h, ARITH_FAST if arith == "fast" else ARITH_EXACT))

    def set_profile(self, on: bool):
        _check(load().sgwg_set_profile(self.h, 1 if on else 0))

    @property
    def stream(self) -> int:
        return load().sgwg_stream(self.h) or 0

    def fp64_peak_tflops(self) -> float:
        v = C.c_double(0)
        _check(load().sgwg_fp64_peak(self.h, C.byref(v)))
        return v.value

    def close(self):
        if self.h:
            load().sgwg_shutdown(self.h)
            self.h = None


def make_domain(d, nl, lower, upper, root, bc) -> Domain:
    dom = Domain()
    dom.d, dom.nl = d, nl
    for k in range(d):
        dom.lower[k], dom.upper[k] = lower[k], upper[k]
        dom.root_cells[k], dom.bc[k] = root[k], bc[k]
    return dom


class Family:
    """CombinationSet + FamilyModel on the device (make_family, combine.hpp:69-83)."""

    def __init__(self, ctx: Context, d, nl, lower, upper, root_cells, bc,
                 members: Optional[Sequence[int]] = None, single: bool = False):
        lib = load()
        self.ctx = ctx
        self.dom = make_domain(d, nl, lower, upper, root_cells, bc)
        self.d, self.nl = d, nl
        self.single = single
        h = _VP()
        if single:  # make_single_grid (runner.hpp:106-115)
            _check(lib.sgwg_family_create_single(ctx.h, C.byref(self.dom), C.byref(h)))
        elif members is None:
            _check(lib.sgwg_family_create(ctx.h, C.byref(self.dom), C.byref(h)))
        else:
            m = np.ascontiguousarray(members, dtype=np.int32)
            _check(lib.sgwg_family_create_shard(ctx.h, C.byref(self.dom),
                                                m.ctypes.data_as(_IP), len(m), C.byref(h)))
        self.h = h
        self.all_levels = (np.full((1, d), nl, dtype=np.int32) if single
                           else enumerate_combination_levels(d, nl))
        n = C.c_int(0)
        _check(lib.sgwg_family_num_members(h, C.byref(n)))
        self.num_members = n.value
        self.global_index, self.levels, self.points = [], [], []
        for mi in range(n.value):
            g = C.c_int(0)
            lv = (C.c_int * 4)()
            pt = (C.c_int * 4)()
            _check(lib.sgwg_family_member(h, mi, C.byref(g), lv, pt))
            self.global_index.append(g.value)
            self.levels.append(tuple(lv[:d]))
            self.points.append(tuple(pt[:d]))
        mp, fp = C.c_size_t(0), C.c_size_t(0)
        _check(lib.sgwg_family_sizes(h, C.byref(mp), C.byref(fp)))
        self.total_points, self.finest_points = mp.value, fp.value
        self._keep = []

    @classmethod
    def from_config(cls, ctx: Context, cfg: dict, members=None, single=False) -> "Family":
        f = cls(ctx, cfg["d"], cfg["nl"], cfg["lower"], cfg["upper"], cfg["root"], cfg["bc"],
                members, single)
        f.set_model(cfg["kind"], speeds=cfg["speeds"], epsilon=cfg["epsilon"],
                    weno_mode=cfg["weno_mode"], space_dim=cfg["space_dim"],
                    theta=cfg["theta"], tau=cfg["tau"])
        return f

    def member_offsets(self):
        off, out = 0, []
        for p in self.points:
            out.append(off)
            off += int(np.prod(p))
        return out

    # -- state -----------------------------------------------------------------
    def initialize(self, preset: int):
        """initialize_family (models.hpp:855-871) for a built-in preset."""
        _check(load().sgwg_family_init_preset(self.h, preset))

    def initialize_fn(self, fn: Callable[[np.ndarray], float], normalize_mass=False):
        cb = IC_CB(lambda x, d, u: float(fn(np.ctypeslib.as_array(x, shape=(d,)))))
        _check(load().sgwg_family_init_fn(self.h, cb, None, 1 if normalize_mass else 0))

    def upload(self, states: np.ndarray):
        s = np.ascontiguousarray(states, dtype=np.float64)
        _check(load().sgwg_family_upload(self.h, s.ctypes.data_as(_DP), s.size))

    def download(self) -> np.ndarray:
        out = np.empty(self.total_points)
        _check(load().sgwg_family_download(self.h, out.ctypes.data_as(_DP), out.size))
        return out

    def download_into(self, out: np.ndarray):
        assert out.dtype == np.float64 and out.size == self.total_points and out.flags.c_contiguous
        _check(load().sgwg_family_download(self.h, out.ctypes.data_as(_DP), out.size))
        return out

    def upload_device(self, ptr: int, n: int):
        _check(load().sgwg_family_upload_device(self.h, _VP(ptr), n))

    def download_device(self, ptr: int, n: int):
        _check(load().sgwg_family_download_device(self.h, _VP(ptr), n))

    # -- physics ---------------------------------------------------------------
    def set_model(self, kind, speeds=(0, 0, 0, 0), epsilon=1e-6, weno_mode=0, space_dim=0,
                  theta=1.0, tau=1.0):
        m = Model()
        m.kind, m.weno_mode, m.epsilon = kind, weno_mode, epsilon
        for k, s in enumerate(list(speeds)[:4]):
            m.speeds[k] = s
        m.space_dim, m.theta, m.tau = space_dim, theta, tau
        _check(load().sgwg_set_model(self.h, C.byref(m)))
        self.model = m
        # member states may carry model state (Vlasov-Maxwell field lines)
        mp, fp = C.c_size_t(0), C.c_size_t(0)
        _check(load().sgwg_family_sizes(self.h, C.byref(mp), C.byref(fp)))
        self.total_points = mp.value

    def set_comm(self, unique_id: bytes, nranks: int, rank: int):
        buf = C.create_string_buffer(bytes(unique_id), 128)
        _check(load().sgwg_family_set_comm(self.h, buf, nranks, rank))

    # -- evolve_family ------------------------------------------------------------
    def evolve(self, mode, tfinal, stops=(), on_stop=None, cfl=0.4, reference_spacing=0.0,
               dt_scale=1.0, cap=1 << 20) -> np.ndarray:
        pol = Policy()
        pol.mode, pol.cfl, pol.reference_spacing, pol.dt_scale = (mode, cfl, reference_spacing,
                                                                  dt_scale)
        st = np.ascontiguousarray(stops, dtype=np.float64)
        dts = np.zeros(cap)
        ns = C.c_size_t(0)
        fail = Failure()

        def _cb(t, user):
            if on_stop is not None:
                on_stop(t)

        cb = STOP_CB(_cb)
        status = load().sgwg_evolve(self.h, C.byref(pol), tfinal,
                                    st.ctypes.data_as(_DP) if st.size else None, st.size, cb,
                                    None, dts.ctypes.data_as(_DP), cap, C.byref(ns),
                                    C.byref(fail))
        _check(status, fail, self)
        return dts[:min(ns.value, cap)].copy()

    def evolve_config(self, cfg, tfinal=None, stops=None, on_stop=None):
        return self.evolve(cfg["dt_mode"], cfg["tfinal"] if tfinal is None else tfinal,
                           cfg["stops"] if stops is None else stops, on_stop, cfl=cfg["cfl"],
                           reference_spacing=cfg["reference_spacing"], dt_scale=cfg["dt_scale"])

    def rk3_step(self, dt):
        fail = Failure()
        _check(load().sgwg_rk3_step(self.h, dt, C.byref(fail)), fail, self)

    def rhs(self) -> np.ndarray:
        out = np.empty(self.total_points)
        _check(load().sgwg_rhs(self.h, out.ctypes.data, out.size, 0))
        return out

    # -- combine / prolong -------------------------------------------------------
    def combine(self, mode=1, eps=1e-6, out_device_ptr: Optional[int] = None,
                out: Optional[np.ndarray] = None) -> np.ndarray:
        if out_device_ptr is not None:
            _check(load().sgwg_combine(self.h, mode, eps, _VP(out_device_ptr),
                                       self.finest_points, 1))
            return None
        if out is None:
            out = np.empty(self.finest_points)
        assert out.dtype == np.float64 and out.size == self.finest_points and out.flags.c_contiguous
        _check(load().sgwg_combine(self.h, mode, eps, out.ctypes.data, out.size, 0))
        return out

    def combine_rows(self, row_begin, row_end, mode=1, eps=1e-6,
                     out_device_ptr: Optional[int] = None) -> np.ndarray:
        """combination restricted to dimension-0 rows [row_begin, row_end) of the finest grid"""
        per_row = self.finest_points // self.fine_extent0
        n = (row_end - row_begin) * per_row
        if out_device_ptr is not None:
            _check(load().sgwg_combine_rows(self.h, mode, eps, row_begin, row_end,
                                            _VP(out_device_ptr), n, 1))
            return None
        out = np.empty(n)
        _check(load().sgwg_combine_rows(self.h, mode, eps, row_begin, row_end, out.ctypes.data,
                                        n, 0))
        return out

    def combine_local(self, mode=1, eps=1e-6):
        """this rank's dimension-0 rows of the combination (option B for a sharded
        family: every member's state gathered, the result left sharded; bitwise the
        one-GPU rows).  Returns (row_begin, row_end, values)."""
        a, b = C.c_longlong(0), C.c_longlong(0)
        _check(load().sgwg_combine_local(self.h, mode, eps, None, 0, 0, C.byref(a), C.byref(b)))
        per_row = self.finest_points // self.fine_extent0
        out = np.empty((b.value - a.value) * per_row)
        _check(load().sgwg_combine_local(self.h, mode, eps, out.ctypes.data, out.size, 0,
                                         C.byref(a), C.byref(b)))
        return a.value, b.value, out

    @property
    def fine_extent0(self) -> int:
        return (self.dom.root_cells[0] << self.nl) + (1 if self.dom.bc[0] == 1 else 0)

    @property
    def fine_extents(self) -> tuple:
        """finest-grid points per dimension (GridGeometry::make at level nl)"""
        return tuple((self.dom.root_cells[k] << self.nl) + (1 if self.dom.bc[k] == 1 else 0)
                     for k in range(self.d))

    def prolong(self, mi, mode=1, eps=1e-6) -> np.ndarray:
        out = np.empty(self.finest_points)
        _check(load().sgwg_prolong(self.h, mi, mode, eps, out.ctypes.data, out.size, 0))
        return out

    def vp_field(self):
        """(rho, E) of the current states, per member: lists of arrays (E: [space_dim, nx])."""
        dx = self.model.space_dim
        nxs = [int(np.prod(p[:dx])) for p in self.points]
        ntot = sum(nxs)
        rho = np.empty(ntot)
        E = np.empty(ntot * dx)
        _check(load().sgwg_vp_field(self.h, rho.ctypes.data_as(_DP), rho.size,
                                    E.ctypes.data_as(_DP), E.size))
        out_r, out_e, o = [], [], 0
        for nx in nxs:
            out_r.append(rho[o:o + nx])
            out_e.append(E[o * dx:(o + nx) * dx].reshape(dx, nx))
            o += nx
        return out_r, out_e

    # -- combined-field diagnostics and output ----------------------
    def combined_stats(self, mode=1, eps=1e-6, exact_preset=-1, t=0.0) -> dict:
        """mass / min / max of the combined field and, for linear advection of a
        periodic preset, error_norms (l1 average, linf) against u0(x - a t)."""
        st = FieldStats()
        _check(load().sgwg_combined_stats(self.h, mode, eps, exact_preset, t, C.byref(st)))
        return {n: getattr(st, n) for n, _ in FieldStats._fields_}

    def eval_points(self, idx, mode=1, eps=1e-6) -> np.ndarray:
        """combined field at finest-grid multi-indices idx (npoints x d)"""
        idx = np.ascontiguousarray(idx, dtype=np.int32).reshape(-1, self.d)
        out = np.empty(idx.shape[0])
        _check(load().sgwg_eval_points(self.h, mode, eps,
                                       idx.ctypes.data_as(C.POINTER(C.c_int)), idx.shape[0],
                                       out.ctypes.data_as(_DP)))
        return out

    def cut_plane(self, dim_a, dim_b, fixed, mode=1, eps=1e-6) -> np.ndarray:
        """combined field on the plane (dim_a, dim_b) through the finest-grid
        indices `fixed` of the other dimensions (write_plane_csv, runner.hpp:126-141)"""
        na, nb = self.fine_extents[dim_a], self.fine_extents[dim_b]
        ia, ib = np.meshgrid(np.arange(na), np.arange(nb), indexing="ij")
        idx = np.tile(np.asarray(fixed, dtype=np.int32), (na * nb, 1))
        idx[:, dim_a] = ia.ravel()
        idx[:, dim_b] = ib.ravel()
        return self.eval_points(idx, mode, eps).reshape(na, nb)

    def write_snapshot(self, path, mode=1, eps=1e-6):
        """SGW5 dump of the combined field (write_field_dump, io.hpp:17-54)"""
        _check(load().sgwg_write_snapshot(self.h, mode, eps, os.fsencode(path)))

    def field_energy(self, cap=1 << 20) -> np.ndarray:
        """||E||_2 of the combined field at the start of every step of the last evolve."""
        out = np.empty(cap)
        n = C.c_size_t(0)
        _check(load().sgwg_field_energy(self.h, out.ctypes.data_as(_DP), cap, C.byref(n)))
        return out[:n.value].copy()

    def time_stage(self, reps=50):
        """(avg ms per stage-kernel launch, algorithmic flops, bytes per launch)."""
        ms, fl, by = C.c_double(0), C.c_double(0), C.c_double(0)
        _check(load().sgwg_time_stage(self.h, reps, C.byref(ms), C.byref(fl), C.byref(by)))
        return ms.value, fl.value, by.value

    def kernel_profile(self) -> list:
        """profile mode: [{name, ms_sum, launches, flops_per_launch, bytes_per_launch}]"""
        n = C.c_int(0)
        _check(load().sgwg_kernel_profile(self.h, None, 0, C.byref(n)))
        arr = (KernelTiming * max(1, n.value))()
        _check(load().sgwg_kernel_profile(self.h, arr, n.value, C.byref(n)))
        return [{"name": k.name.decode(), "ms_sum": k.ms_sum, "launches": k.launches,
                 "flops_per_launch": k.flops_per_launch, "bytes_per_launch": k.bytes_per_launch}
                for k in arr[:n.value]]

    def kernel_profile_reset(self):
        _check(load().sgwg_kernel_profile_reset(self.h))

    @property
    def stage_kernels(self) -> str:
        return (load().sgwg_stage_kernels(self.h) or b"").decode()

    def stats(self) -> dict:
        s = Stats()
        _check(load().sgwg_get_stats(self.h, C.byref(s)))
        return {n: getattr(s, n) for n, _ in Stats._fields_}

    def close(self):
        if self.h:
            load().sgwg_family_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _check(load().sgwg_nccl_unique_id(buf))
    return buf.raw


config = _cfg.config


def read_snapshot(path):
    """read_field_dump (io.hpp:56-75): (extents, spacings, values)."""
    with open(path, "rb") as fh:
        hdr = fh.read(64)
        if len(hdr) != 64 or hdr[:4] != b"SGW5":
            raise ValueError(f"read_snapshot: bad header in {path}")
        version, dim = np.frombuffer(hdr[4:12], dtype="<u4")
        if version != 1 or not 1 <= dim <= 4:
            raise ValueError(f"read_snapshot: bad header in {path}")
        ext = [int(e) for e in np.frombuffer(hdr[12:28], dtype="<u4")[:dim]]
        h = [float(x) for x in np.frombuffer(hdr[32:64], dtype="<f8")[:dim]]
        vals = np.frombuffer(fh.read(), dtype="<f8")
    if vals.size != int(np.prod(ext)):
        raise ValueError(f"read_snapshot: truncated payload in {path}")
    return ext, h, vals
