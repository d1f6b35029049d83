"""Vlasov-Poisson (BASELINE C4 1D1V / C5 2D2V; no reference):
the GPU field solve and evolution against the oracle restatement."""
import numpy as np
import pytest

from helpers import gpu_family, maxabs, oracle_objs
from paper_2007_10196_b200 import configs
from test_gpu_parity import _evolve_both

pytestmark = pytest.mark.gpu

C5_SMALL = {"nl": 3}  # root 8: x-grids 8..64 (2D), v 9..65; 35 members


@pytest.mark.parametrize("name,over", [("C4", {"nl": 3, "root": [16, 16]}), ("C5", C5_SMALL)])
def test_vp_field_matches_oracle(ctx, oracle, name, over):
    cfg = configs.config(name, **over)
    dom, model, _ = oracle_objs(cfg)
    s = oracle.init_family(cfg["ic"], dom)
    rng = np.random.default_rng(3)
    s = s * (1.0 + 0.05 * rng.standard_normal(s.size))  # break the symmetry a little
    fam = gpu_family(ctx, cfg)
    fam.upload(s)
    rho_g, E_g = fam.vp_field()
    dxs = cfg["space_dim"]
    off = 0
    for mi, lv in enumerate(oracle.levels(cfg["d"], cfg["nl"])):
        n = int(np.prod(fam.points[mi]))
        nx = int(np.prod(fam.points[mi][:dxs]))
        rho_o, E_o = oracle.vp_field(dom, lv, dxs, s[off:off + n], nx)
        assert maxabs(rho_g[mi], rho_o) < 1e-13, mi
        assert maxabs(E_g[mi], E_o) < 1e-12 * (1 + np.max(np.abs(E_o))), mi
        off += n


def test_vp_c5_small_evolve(ctx, oracle):
    cfg = configs.config("C5", **C5_SMALL)
    got, want, gd, wd, gc, wc = _evolve_both(ctx, oracle, cfg, 0.02)
    assert len(gd) == len(wd) > 0
    assert maxabs(gd, wd) < 1e-14
    assert maxabs(got, want) < 1e-10
    assert maxabs(gc[-1], wc[-1]) < 1e-10


@pytest.mark.parametrize("cap,plane4", [(None, "1"), (None, "0"), ("256", "0")])
def test_vp_c5_small_evolve_fast(ctx_fast, oracle, monkeypatch, cap, plane4):
    """Fast build, 2D2V: the two plane launches per stage (dims (x1,x2) ->
    tendency, dims (v1,v2) + RK stage + charge density).  plane4 = 1: the
    whole-plane kernels (plane4d.cuh, the default for C5-shaped families);
    plane4 = 0: the windowed plane kernels, cap 256 splitting velocity planes
    into several windows (several partials per x)."""
    monkeypatch.setenv("SGWG_PLANE4", plane4)
    if cap is not None:
        monkeypatch.setenv("SGWG_PLANE_CAP", cap)
    cfg = configs.config("C5", **C5_SMALL)
    got, want, gd, wd, gc, wc = _evolve_both(ctx_fast, oracle, cfg, 0.02)
    assert len(gd) == len(wd) > 0
    assert maxabs(gd, wd) < 1e-14
    assert maxabs(got, want) < 1e-10
    assert maxabs(gc[-1], wc[-1]) < 1e-10


@pytest.mark.parametrize("plane4", ["1", "0"])
def test_vp_c5_partials_track_state(ctx_fast, oracle, monkeypatch, plane4):
    """The charge density the field solve uses after an evolve comes from the
    plane kernel's partial sums; after an upload it must be recomputed."""
    monkeypatch.setenv("SGWG_PLANE_CAP", "512")
    monkeypatch.setenv("SGWG_PLANE4", plane4)
    cfg = configs.config("C5", **C5_SMALL)
    dom, model, pol = oracle_objs(cfg)
    fam = gpu_family(ctx_fast, cfg)
    fam.initialize(cfg["ic"])
    fam.evolve_config(cfg, tfinal=0.01)
    s = fam.download()
    dxs = cfg["space_dim"]

    def check(fam, s):
        rho_g, E_g = fam.vp_field()
        off = 0
        for mi, lv in enumerate(oracle.levels(cfg["d"], cfg["nl"])):
            n = int(np.prod(fam.points[mi]))
            nx = int(np.prod(fam.points[mi][:dxs]))
            rho_o, E_o = oracle.vp_field(dom, lv, dxs, s[off:off + n], nx)
            assert maxabs(rho_g[mi], rho_o) < 1e-13, mi
            assert maxabs(E_g[mi], E_o) < 1e-12 * (1 + np.max(np.abs(E_o))), mi
            off += n

    check(fam, s)                      # partials left by the last stage-3 launch
    s2 = s * (1.0 + 0.01 * np.random.default_rng(5).standard_normal(s.size))
    fam.upload(s2)                     # invalidates them
    check(fam, s2)
    # evolve again from the uploaded state: graphs captured earlier assume fresh
    # partials at entry, which the runtime must re-establish
    fam.evolve_config(cfg, tfinal=0.01)
    fam2 = gpu_family(ctx_fast, cfg)
    fam2.upload(s2)
    fam2.evolve_config(cfg, tfinal=0.01)
    assert maxabs(fam.download(), fam2.download()) == 0.0


@pytest.mark.parametrize("plane4", ["1", "0"])
def test_advection_4d_evolve_fast(ctx_fast, oracle, monkeypatch, plane4):
    """4D constant-speed advection through the plane launches (fused dt),
    both directions of every sweep (whole-plane and windowed kernels)."""
    monkeypatch.setenv("SGWG_PLANE4", plane4)
    cfg = configs.config("C3", d=4, nl=3, lower=[0.0] * 4, upper=[2.0] * 4, root=[8] * 4,
                         bc=[0, 0, 1, 1], speeds=[1.0, -1.0, 0.5, -0.25])
    T = 4 * cfg["reference_spacing"] ** (5.0 / 3.0)
    got, want, gd, wd, gc, wc = _evolve_both(ctx_fast, oracle, cfg, T)
    assert len(gd) == len(wd) == 4
    assert maxabs(got, want) < 1e-10
    assert maxabs(gc[-1], wc[-1]) < 1e-10
