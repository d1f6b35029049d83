"""Observed convergence orders (north star: "the same observed convergence
orders" as the CPU reference).  Smooth 2D advection (BASELINE C1 physics)
and 3D advection (C3 physics) on a sequence of sparse-grid levels: the L1
error of the combined solution against the exact solution on each level's
finest grid, from the B200 path (both builds) and from the oracle; the errors
agree to 1e-10 relative and the observed orders to 1e-6; in 2D they are high
order once the combination is resolved."""
import numpy as np
import pytest

from helpers import gpu_family, oracle_objs
from paper_2007_10196_b200 import configs

pytestmark = pytest.mark.gpu


def _errors(run, name, levels, T, root):
    errs = []
    for nl in levels:
        cfg = configs.config(name, nl=nl, root=[root] * configs.config(name)["d"])
        d = cfg["d"]
        nf = root << nl
        h = (cfg["upper"][0] - cfg["lower"][0]) / nf
        cfg["reference_spacing"] = h
        u = run(cfg, T)
        x = cfg["lower"][0] + h * np.arange(nf)
        grids = np.meshgrid(*([x] * d), indexing="ij")
        shift = sum(cfg["speeds"][k] for k in range(d)) * T
        exact = np.sin(np.pi * (sum(grids) - shift)).ravel()
        errs.append(float(np.sum(np.abs(u - exact)) * h ** d))
    return np.array(errs)


def _orders(e):
    return np.log2(e[:-1] / e[1:])


def _gpu_run(ctx):
    def run(cfg, T):
        fam = gpu_family(ctx, cfg)
        fam.initialize(cfg["ic"])
        fam.evolve_config(cfg, tfinal=T, stops=[])
        return fam.combine(cfg["interp"], cfg["epsilon"])
    return run


def _oracle_run(oracle):
    def run(cfg, T):
        dom, model, pol = oracle_objs(cfg)
        s0 = oracle.init_family(cfg["ic"], dom)
        s, _, st, _ = oracle.evolve(dom, model, pol, s0, T, [])
        assert st == 0
        return oracle.combine(dom, s, cfg["interp"], cfg["epsilon"])
    return run


@pytest.mark.parametrize("arith", ["exact", "fast"])
def test_convergence_orders_2d(ctx, ctx_fast, oracle, arith):
    levels, T = [2, 3, 4, 5], 0.05
    g = _errors(_gpu_run(ctx if arith == "exact" else ctx_fast), "C1", levels, T, 8)
    o = _errors(_oracle_run(oracle), "C1", levels, T, 8)
    assert np.all(np.abs(g - o) <= 1e-10 * o), (g, o)
    og, oo = _orders(g), _orders(o)
    assert np.all(np.abs(og - oo) < 1e-6), (og, oo)
    assert og[-1] > 3.0, og  # high order once the combination is resolved


def test_convergence_orders_3d_fast(ctx_fast, oracle):
    # coarse 3D sparse grids are pre-asymptotic (members down to 8 points per
    # wavelength-2 period): the orders are not yet 5, but must be the oracle's
    levels, T = [2, 3, 4], 0.02
    g = _errors(_gpu_run(ctx_fast), "C3", levels, T, 8)
    o = _errors(_oracle_run(oracle), "C3", levels, T, 8)
    assert np.all(np.abs(g - o) <= 1e-10 * o), (g, o)
    assert np.all(np.abs(_orders(g) - _orders(o)) < 1e-6)
    assert np.all(np.diff(g) < 0), g
