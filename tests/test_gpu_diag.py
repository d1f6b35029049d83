"""Combined-field diagnostics and output on the device:
sgwg_combined_stats against numpy on the downloaded combination, point
evaluation (cut planes) against the full combination -- bitwise in the exact
build --, the row-slab path against the single-plan path, and the SGW5
snapshot against the combination."""
import os

import numpy as np
import pytest

from helpers import bitwise_equal, gpu_family, maxabs
from paper_2007_10196_b200 import configs, sgwg

pytestmark = pytest.mark.gpu


def _trap_weights(cfg, fam):
    ws = []
    for k in range(cfg["d"]):
        n = fam.fine_extents[k]
        h = (cfg["upper"][k] - cfg["lower"][k]) / (cfg["root"][k] << cfg["nl"])
        w = np.full(n, h)
        if cfg["bc"][k] == 1:
            w[0] *= 0.5
            w[-1] *= 0.5
        ws.append(w)
    W = ws[0]
    for w in ws[1:]:
        W = np.multiply.outer(W, w)
    return W.ravel()


def _evolved(ctx, name, T, **over):
    cfg = configs.config(name, **over)
    fam = gpu_family(ctx, cfg)
    fam.initialize(cfg["ic"])
    if T > 0:
        fam.evolve_config(cfg, tfinal=T, stops=[])
    return cfg, fam


@pytest.mark.parametrize("name,over,T", [
    ("C1", {}, 0.05),
    ("C4", {"nl": 3, "root": [16, 16]}, 0.05),
    ("C5", {"nl": 3}, 0.02),
])
def test_stats_match_numpy(ctx, name, over, T):
    cfg, fam = _evolved(ctx, name, T, **over)
    u = fam.combine(cfg["interp"], cfg["epsilon"])
    st = fam.combined_stats(cfg["interp"], cfg["epsilon"])
    W = _trap_weights(cfg, fam)
    assert st["points"] == u.size
    assert abs(st["mass"] - np.sum(W * u)) <= 1e-13 * np.sum(np.abs(W * u))
    assert st["min"] == u.min() and st["max"] == u.max()
    assert np.isnan(st["l1"]) and np.isnan(st["linf"])


def test_error_norms_linear_advection(ctx, ctx_fast):
    T = 0.05
    for c in (ctx, ctx_fast):
        cfg, fam = _evolved(c, "C1", T)
        u = fam.combine(cfg["interp"], cfg["epsilon"])
        n = fam.fine_extents[0]
        x = cfg["lower"][0] + (cfg["upper"][0] - cfg["lower"][0]) / n * np.arange(n)
        X, Y = np.meshgrid(x, x, indexing="ij")
        ex = np.sin(np.pi * (X + Y - 2.0 * T)).ravel()
        st = fam.combined_stats(cfg["interp"], cfg["epsilon"], exact_preset=0, t=T)
        e = np.abs(u - ex)
        # device vs numpy sin of the exact solution differ by ~1 ulp per point
        assert abs(st["l1"] - e.mean()) <= 1e-15
        assert abs(st["linf"] - e.max()) <= 1e-15
        assert st["l1"] < 1e-3


def test_stats_exact_requires_a_known_solution(ctx):
    cfg, fam = _evolved(ctx, "C2", 0.0, nl=3, root=[16, 16])  # Burgers
    with pytest.raises(ValueError):
        fam.combined_stats(exact_preset=0)  # the advection preset
    cfg, fam = _evolved(ctx, "C4", 0.0, nl=3, root=[16, 16])  # Vlasov-Poisson
    with pytest.raises(ValueError):
        fam.combined_stats(exact_preset=3)


def test_stats_slabs_match_single_plan(ctx, monkeypatch):
    cfg, fam = _evolved(ctx, "C5", 0.01, nl=3)
    a = fam.combined_stats(cfg["interp"], cfg["epsilon"])
    monkeypatch.setenv("SGWG_COMBINE_BUDGET_GB", "0.002")  # force row slabs
    b = fam.combined_stats(cfg["interp"], cfg["epsilon"])
    assert a["min"] == b["min"] and a["max"] == b["max"]
    assert abs(a["mass"] - b["mass"]) <= 1e-14 * abs(a["mass"])


@pytest.mark.parametrize("name,over,T", [
    ("C2", {"nl": 4, "root": [16, 16]}, 0.02),    # 2D periodic, Burgers
    ("C4", {"nl": 3, "root": [16, 16]}, 0.02),    # 2D periodic x zero
    ("C3", {"nl": 3, "root": [8, 8, 8]}, 0.02),   # 3D
    ("C5", {"nl": 3}, 0.01),                       # 4D, zero v-boundaries
])
@pytest.mark.parametrize("mode", [1, 0])
def test_eval_points_equal_combination(ctx, name, over, T, mode):
    cfg, fam = _evolved(ctx, name, T, **over)
    full = fam.combine(mode, cfg["epsilon"]).reshape(fam.fine_extents)
    rng = np.random.default_rng(11)
    idx = np.stack([rng.integers(0, n, 400) for n in fam.fine_extents], axis=1)
    got = fam.eval_points(idx, mode, cfg["epsilon"])
    want = full[tuple(idx.T)]
    assert bitwise_equal(got, want), maxabs(got, want)
    # a cut plane through the middle (write_cuts, runner.hpp:159-200)
    fixed = [n // 2 for n in fam.fine_extents]
    plane = fam.cut_plane(0, cfg["d"] - 1, fixed, mode, cfg["epsilon"])
    sl = [n // 2 for n in fam.fine_extents]
    sl[0] = slice(None)
    sl[cfg["d"] - 1] = slice(None)
    assert bitwise_equal(plane, full[tuple(sl)])


def test_eval_points_fast_build(ctx_fast):
    cfg, fam = _evolved(ctx_fast, "C5", 0.01, nl=3)
    full = fam.combine(cfg["interp"], cfg["epsilon"]).reshape(fam.fine_extents)
    rng = np.random.default_rng(5)
    idx = np.stack([rng.integers(0, n, 300) for n in fam.fine_extents], axis=1)
    got = fam.eval_points(idx, cfg["interp"], cfg["epsilon"])
    assert maxabs(got, full[tuple(idx.T)]) < 1e-14


def test_eval_points_rejects_out_of_range(ctx):
    cfg, fam = _evolved(ctx, "C1", 0.0)
    with pytest.raises(ValueError):
        fam.eval_points([[0, fam.fine_extents[1]]])


def test_single_grid_diagnostics(ctx):
    cfg = configs.config("C1", nl=2)
    fam = sgwg.Family.from_config(ctx, cfg, single=True)
    fam.initialize(cfg["ic"])
    u = fam.download()
    st = fam.combined_stats()
    assert st["min"] == u.min() and st["max"] == u.max()
    idx = np.array([[1, 2], [5, 7]])
    assert bitwise_equal(fam.eval_points(idx), u.reshape(fam.fine_extents)[tuple(idx.T)])


def test_snapshot_round_trip(ctx, tmp_path, monkeypatch):
    cfg, fam = _evolved(ctx, "C4", 0.02, nl=3, root=[16, 16])
    u = fam.combine(cfg["interp"], cfg["epsilon"])
    p = os.path.join(tmp_path, "snapshot_t0.020000.sgw5")
    fam.write_snapshot(p, cfg["interp"], cfg["epsilon"])
    ext, h, vals = sgwg.read_snapshot(p)
    assert tuple(ext) == fam.fine_extents
    assert np.allclose(h, [(cfg["upper"][k] - cfg["lower"][k]) / (cfg["root"][k] << cfg["nl"])
                           for k in range(cfg["d"])], rtol=0, atol=0)
    assert bitwise_equal(vals, u)
    monkeypatch.setenv("SGWG_COMBINE_BUDGET_GB", "0.0005")  # streamed in row slabs
    fam.write_snapshot(p, cfg["interp"], cfg["epsilon"])
    assert bitwise_equal(sgwg.read_snapshot(p)[2], u)
