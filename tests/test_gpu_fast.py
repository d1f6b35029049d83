"""Fast build (FMA, shared-term reconstructions, persistent 2D kernel) against
the CPU oracle: tendencies to 1e-12 relative, combined solutions to the
north-star bar of 1e-10 max-abs, identical dt sequences / failure reports."""
import numpy as np
import pytest

from helpers import gpu_family, maxabs, oracle_objs, random_states
from oracle import oracle as O
from paper_2007_10196_b200 import configs
from test_gpu_parity import RHS_CASES, _evolve_both, _rhs_oracle

pytestmark = pytest.mark.gpu

TOL = 1e-10


@pytest.mark.parametrize("name,over", RHS_CASES + [
    ("C3", {"d": 4, "nl": 3, "lower": [0.0] * 4, "upper": [2.0] * 4, "root": [8] * 4,
            "bc": [0, 0, 1, 1], "speeds": [1.0, -1.0, 0.5, -0.25]}),    # 8/9-point lines
    ("C2", {"d": 3, "nl": 2, "lower": [0.0] * 3, "upper": [2.0] * 3, "root": [8, 8, 8],
            "bc": [0, 1, 0], "speeds": [0.0] * 3}),                        # 3D Burgers
])
def test_rhs_fast(ctx_fast, oracle, name, over):
    cfg = configs.config(name, **over)
    s = random_states(oracle, cfg, seed=7)
    fam = gpu_family(ctx_fast, cfg)
    fam.upload(s)
    got = fam.rhs()
    want = _rhs_oracle(oracle, cfg, s)
    assert maxabs(got, want) <= 1e-12 * (1.0 + np.max(np.abs(want)))


def test_evolve_c1_full_fast(ctx_fast, oracle):
    """BASELINE C1 end to end in the fast build (persistent 2D kernel)."""
    cfg = configs.config("C1")
    got, want, gd, wd, gc, wc = _evolve_both(ctx_fast, oracle, cfg, cfg["tfinal"])
    assert len(gd) == len(wd) == 2048
    assert maxabs(gd, wd) == 0.0
    assert maxabs(gc[-1], wc[-1]) < TOL


def test_evolve_c3_fast(ctx_fast, oracle):
    cfg = configs.config("C3")
    T = 6 * cfg["reference_spacing"] ** (5.0 / 3.0)
    got, want, gd, wd, gc, wc = _evolve_both(ctx_fast, oracle, cfg, T)
    assert len(gd) == len(wd) == 6
    assert maxabs(gc[-1], wc[-1]) < TOL


def test_evolve_c2_stops_fast(ctx_fast, oracle):
    cfg = configs.config("C2", nl=4, root=[16, 16])
    got, want, gd, wd, gc, wc = _evolve_both(ctx_fast, oracle, cfg, 0.05, stops=[0.02])
    assert len(gd) == len(wd)
    assert maxabs(gd, wd) < 1e-15
    for a, b in zip(gc, wc):
        assert maxabs(a, b) < TOL


def test_vp_c4_fast(ctx_fast, oracle):
    cfg = configs.config("C4", nl=3, root=[16, 16])
    got, want, gd, wd, gc, wc = _evolve_both(ctx_fast, oracle, cfg, 0.5)
    assert len(gd) == len(wd)
    assert maxabs(gc[-1], wc[-1]) < TOL


def test_failure_injection_fast(ctx_fast, oracle):
    from paper_2007_10196_b200 import sgwg
    cfg = configs.config("C2", nl=3, root=[8, 8])
    dom, model, pol = oracle_objs(cfg)
    s0 = oracle.init_family(cfg["ic"], dom) * 1e150
    _, _, st, (fm, fst, fsg) = oracle.evolve(dom, model, pol, s0, 0.01)
    assert st == 2
    fam = gpu_family(ctx_fast, cfg)
    fam.upload(s0)
    with pytest.raises(sgwg.FamilyIntegratorFailure) as ei:
        fam.evolve_config(cfg, tfinal=0.01)
    assert (ei.value.member, ei.value.step, ei.value.stage) == (fm, fst, fsg)


def test_combine_fast(ctx_fast, oracle):
    cfg = configs.config("C3", nl=3, root=[8, 8, 8])
    s = random_states(oracle, cfg, seed=5)
    dom, _, _ = oracle_objs(cfg)
    fam = gpu_family(ctx_fast, cfg)
    fam.upload(s)
    for mode in (O.WENO, O.LAGRANGE):
        assert maxabs(fam.combine(mode, 1e-6), oracle.combine(dom, s, mode, 1e-6)) < 1e-12


# Every tile-size variant of the fast 2D / 3D stage kernels and of the
# persistent 2D evolve against the oracle (the defaults pick one per family
# size: 512-point stage tiles, 1024- or 512-point persistent tiles, 512-point
# 3D tiles; the others stay selectable and must stay correct).
@pytest.mark.parametrize("env,name,over,T", [
    ({"SGWG_NO_PERSIST": "1", "SGWG_TILE2D": "2048"}, "C2", {"nl": 3, "root": [16, 16]}, 0.02),
    ({"SGWG_NO_PERSIST": "1", "SGWG_TILE2D": "1024"}, "C2", {"nl": 3, "root": [16, 16]}, 0.02),
    ({"SGWG_NO_PERSIST": "1", "SGWG_TILE2D": "512"}, "C2", {"nl": 3, "root": [16, 16]}, 0.02),
    ({"SGWG_TILE2D": "2048"}, "C4", {"nl": 3, "root": [16, 16]}, 0.2),
    ({"SGWG_TILE2D": "1024"}, "C4", {"nl": 3, "root": [16, 16]}, 0.2),
    ({"SGWG_PERSIST_TILE": "2048"}, "C2", {"nl": 4, "root": [16, 16]}, 0.02),
    ({"SGWG_PERSIST_TILE": "1024"}, "C2", {"nl": 4, "root": [16, 16]}, 0.02),
    ({"SGWG_PERSIST_TILE": "512"}, "C2", {"nl": 4, "root": [16, 16]}, 0.02),
    ({"SGWG_3D_TILE": "2048"}, "C3", {"nl": 3, "root": [16, 16, 16]}, 0.004),
    ({"SGWG_3D_TILE": "1024"}, "C3", {"nl": 3, "root": [16, 16, 16]}, 0.004),
    ({"SGWG_3D_TILE": "512"}, "C3", {"nl": 3, "root": [16, 16, 16]}, 0.004),
])
def test_tile_variants_fast(ctx_fast, oracle, monkeypatch, env, name, over, T):
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    cfg = configs.config(name, **over)
    got, want, gd, wd, gc, wc = _evolve_both(ctx_fast, oracle, cfg, T)
    assert len(gd) == len(wd) > 2
    assert maxabs(gd, wd) < 1e-14
    assert maxabs(got, want) < TOL
    assert maxabs(gc[-1], wc[-1]) < TOL
