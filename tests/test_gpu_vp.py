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
