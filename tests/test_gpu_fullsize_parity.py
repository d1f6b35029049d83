"""Parity at the BASELINE sizes and horizons: the product path (through the C
ABI, the kernels the bench runs) against the CPU oracle on identical inputs.

* C2 (the 2D Burgers family, root 32, N_L = 5): the whole run to T = 0.5 with
  the stop at 0.1 (the shock forms at t ~ 0.159), combined at both stops --
  fast build on its default single-GPU path (the persistent cooperative
  kernel) within 1e-10, exact build bitwise (reference arithmetic).
* C3 (3D advection, root 16, N_L = 4, 31 members): the whole run to T = 0.5
  (1,626 steps) plus the combination -- fast within 1e-10, exact bitwise.
* C4 (1D1V Vlasov-Poisson, root 32, N_L = 5): 2,000 steps with the per-step
  field-energy record, the member states and the combination.
* C5 (2D2V Vlasov-Poisson, 121 members, 12M points): member states after 20
  steps; the reference's cut planes (x1-v1 at x2 = v2 = 0, x1-x2 at
  v1 = v2 = 0, runner.hpp:187-196) through sgwg_eval_points against the
  oracle's sub-block combination (sgwo_combine_box, bitwise equal to the full
  combine); the full combination at reduced level (root 8, N_L = 3) at T = 1.

The oracle steps members in parallel (OpenMP, bitwise independent of the
thread count) so the whole module fits the GPU suite's time budget.  Every
test prints its max |gpu - oracle|.  Vlasov-Poisson has no reference (SURVEY
F4): its oracle is the C restatement with a direct DFT Poisson solve, so the
VP comparisons carry a tolerance in both builds.
"""
import os
import time

import numpy as np
import pytest

from helpers import bitwise_equal, gpu_family, maxabs, oracle_objs
from paper_2007_10196_b200 import configs

pytestmark = pytest.mark.gpu

TOL = 1e-10  # north_star: max-abs difference on the combined fine-grid solution


@pytest.fixture(scope="module")
def orc():
    from oracle.oracle import Oracle
    return Oracle().set_threads(os.cpu_count() or 1)


def _oracle_run(orc, cfg, tfinal, stops=(), energy_cap=None, combine=True):
    dom, model, pol = oracle_objs(cfg)
    s0 = orc.init_family(cfg["ic"], dom)
    combined = []
    rec = orc.record_energy(energy_cap) if energy_cap else None
    t0 = time.perf_counter()

    def on_stop(t, s):
        if combine:
            combined.append(orc.combine(dom, s, cfg["interp"], cfg["epsilon"]))

    try:
        s, dts, st, _ = orc.evolve(dom, model, pol, s0, tfinal, stops, on_stop=on_stop)
    finally:
        if rec is not None:
            rec = rec.copy()
            orc.record_energy(None)
    assert st == 0
    print(f"\n[oracle] {cfg['name']} T={tfinal}: {len(dts)} steps, "
          f"{time.perf_counter() - t0:.1f} s on {os.cpu_count()} threads")
    return {"s0": s0, "s": s, "dts": dts, "combined": combined, "energy": rec}


def _gpu_run(ctx, cfg, tfinal, stops=(), combine=True):
    fam = gpu_family(ctx, cfg)
    fam.initialize(cfg["ic"])
    combined = []

    def on_stop(t):
        if combine:
            combined.append(fam.combine(cfg["interp"], cfg["epsilon"]))

    dts = fam.evolve_config(cfg, tfinal=tfinal, stops=list(stops), on_stop=on_stop)
    return fam, dts, combined


# ---------------------------------------------------------------- C2 ------
@pytest.fixture(scope="module")
def c2_ref(orc):
    cfg = configs.config("C2")
    return cfg, _oracle_run(orc, cfg, cfg["tfinal"], cfg["stops"])


def test_c2_full_fast_persistent(ctx_fast, c2_ref):
    """The benched C2 path: fast build, persistent kernel, stops {0.1, 0.5}."""
    cfg, ref = c2_ref
    fam, dts, comb = _gpu_run(ctx_fast, cfg, cfg["tfinal"], cfg["stops"])
    assert len(dts) == len(ref["dts"]) > 1400
    ddt = maxabs(dts, ref["dts"])
    errs = [maxabs(a, b) for a, b in zip(comb, ref["combined"])]
    es = maxabs(fam.download(), ref["s"])
    print(f"[C2 fast] steps {len(dts)}, max|ddt| {ddt:.2e}, member states {es:.2e}, "
          f"combined at t=0.1 {errs[0]:.2e}, t=0.5 {errs[1]:.2e}")
    assert len(comb) == 2
    # post-shock max|u| (the CFL speed) carries the states' 1e-13 differences, and
    # the landing steps absorb the accumulated t: dt agrees to ~1e-11 relative
    assert ddt <= 1e-14
    assert max(errs) <= TOL
    fam.close()


def test_c2_full_exact_bitwise(ctx, c2_ref):
    cfg, ref = c2_ref
    fam, dts, comb = _gpu_run(ctx, cfg, cfg["tfinal"], cfg["stops"])
    print(f"[C2 exact] steps {len(dts)}, combined max diff "
          f"{max(maxabs(a, b) for a, b in zip(comb, ref['combined'])):.2e}")
    assert bitwise_equal(dts, ref["dts"])
    assert bitwise_equal(fam.download(), ref["s"])
    for a, b in zip(comb, ref["combined"]):
        assert bitwise_equal(a, b), maxabs(a, b)
    fam.close()


# ---------------------------------------------------------------- C3 ------
@pytest.fixture(scope="module")
def c3_ref(orc):
    cfg = configs.config("C3")
    return cfg, _oracle_run(orc, cfg, cfg["tfinal"])


def test_c3_full_fast(ctx_fast, c3_ref):
    cfg, ref = c3_ref
    fam, dts, comb = _gpu_run(ctx_fast, cfg, cfg["tfinal"])
    assert len(dts) == len(ref["dts"]) == 1626
    es = maxabs(fam.download(), ref["s"])
    ec = maxabs(comb[-1], ref["combined"][-1])
    print(f"[C3 fast] member states {es:.2e}, combined {ec:.2e}")
    assert bitwise_equal(dts, ref["dts"])  # accuracy-mode dt: no state dependence
    assert ec <= TOL
    fam.close()


def test_c3_full_exact_bitwise(ctx, c3_ref):
    cfg, ref = c3_ref
    fam, dts, comb = _gpu_run(ctx, cfg, cfg["tfinal"])
    print(f"[C3 exact] combined max diff {maxabs(comb[-1], ref['combined'][-1]):.2e}")
    assert bitwise_equal(dts, ref["dts"])
    assert bitwise_equal(fam.download(), ref["s"])
    assert bitwise_equal(comb[-1], ref["combined"][-1])
    fam.close()


# ---------------------------------------------------------------- C4 ------
C4_T = 1.95  # ~2,000 RK steps of the full family (CFL dt ~ 9.7e-4)


@pytest.fixture(scope="module")
def c4_ref(orc):
    cfg = configs.config("C4")
    return cfg, C4_T, _oracle_run(orc, cfg, C4_T, energy_cap=4096)


@pytest.mark.parametrize("arith", ["fast", "exact"])
def test_c4_2000_steps_with_energy(ctx, ctx_fast, c4_ref, arith):
    cfg, T, ref = c4_ref
    fam, dts, comb = _gpu_run(ctx_fast if arith == "fast" else ctx, cfg, T)
    n = len(ref["dts"])
    assert len(dts) == n >= 2000
    fe = fam.field_energy()
    want = ref["energy"][:n]
    rel_e = float(np.max(np.abs(fe[:n] - want) / want))
    es = maxabs(fam.download(), ref["s"])
    ec = maxabs(comb[-1], ref["combined"][-1])
    ddt = float(np.max(np.abs(dts - ref["dts"]) / ref["dts"]))
    print(f"[C4 {arith}] {n} steps to T={T:.6f}: rel|ddt| {ddt:.2e}, log|E| record rel "
          f"{rel_e:.2e}, member states {es:.2e}, combined {ec:.2e}")
    assert ddt <= 1e-12
    assert rel_e <= 1e-10
    assert es <= TOL and ec <= TOL
    fam.close()


# ---------------------------------------------------------------- C5 ------
C5_STEPS_T = 0.04  # ~20 RK steps of the full family (dt ~ 2e-3)


@pytest.fixture(scope="module")
def c5_ref(orc):
    cfg = configs.config("C5")  # (no full combine: the finest grid is 34.6 GB)
    return cfg, _oracle_run(orc, cfg, C5_STEPS_T, combine=False)


def _c5_cuts(cfg, fam):
    from paper_2007_10196_b200 import runner
    return runner.cut_planes(cfg, fam)


def test_c5_member_states_and_cut_planes(ctx, ctx_fast, orc, c5_ref):
    """Full C5 family: member states after >= 20 steps (fast plane kernels),
    then the two cut planes of the combined field through sgwg_eval_points
    against the oracle's sub-block combination of the same states (fast within
    1e-10; exact build bitwise: it is the reference's arithmetic)."""
    cfg, ref = c5_ref
    fam, dts, _ = _gpu_run(ctx_fast, cfg, C5_STEPS_T, combine=False)
    assert len(dts) == len(ref["dts"]) >= 20
    ddt = float(np.max(np.abs(dts - ref["dts"]) / ref["dts"]))
    got = fam.download()
    es = maxabs(got, ref["s"])
    print(f"[C5 fast] {len(dts)} steps: rel|ddt| {ddt:.2e}, member states {es:.2e}")
    assert ddt <= 1e-12
    assert es <= TOL
    dom, _, _ = oracle_objs(cfg)
    ex = gpu_family(ctx, cfg)
    ex.upload(ref["s"])
    for name, da, db, fixed in _c5_cuts(cfg, fam):
        lo = list(fixed)
        hi = [f + 1 for f in fixed]
        lo[da], hi[da] = 0, fam.fine_extents[da]
        lo[db], hi[db] = 0, fam.fine_extents[db]
        want = orc.combine_box(dom, ref["s"], lo, hi, cfg["interp"], cfg["epsilon"])
        want = want.reshape(hi[da] - lo[da], hi[db] - lo[db])
        plane_fast = fam.cut_plane(da, db, fixed, cfg["interp"], cfg["epsilon"])
        plane_exact = ex.cut_plane(da, db, fixed, cfg["interp"], cfg["epsilon"])
        e = maxabs(plane_fast, want)
        print(f"[C5 {name}] {want.shape}: fast |gpu-oracle| {e:.2e}, exact bitwise "
              f"{bitwise_equal(plane_exact, want)}")
        assert e <= TOL
        assert bitwise_equal(plane_exact, want), maxabs(plane_exact, want)
    ex.close()
    fam.close()


def test_c5_reduced_level_full_combine(ctx_fast, orc):
    """Root 8, N_L = 3 (finest 64^2 x 65^2 = 17.3M points) to T = 1: the full
    combined field, fast build against the oracle."""
    cfg = configs.config("C5", nl=3)
    ref = _oracle_run(orc, cfg, 1.0)
    fam, dts, comb = _gpu_run(ctx_fast, cfg, 1.0)
    assert len(dts) == len(ref["dts"])
    ec = maxabs(comb[-1], ref["combined"][-1])
    print(f"[C5 N_L=3 fast] {len(dts)} steps to T=1, combined {ec:.2e} over "
          f"{comb[-1].size} points")
    assert ec <= TOL
    fam.close()
