"""BASELINE configurations at their full sizes, checked through properties that
do not need the (much slower) oracle at that size:

* conservation: the WENO operator is in flux-difference form, so on periodic
  lines every RK stage preserves each member's sum of u up to rounding
  (C2 Burgers, C3 advection, full families);
* C5 (121 members, 12M points): the sum of f over every member changes only
  through the fluxes across its zero-ghost velocity boundaries (~1e-7 relative
  in three steps, the same in the oracle at reduced size, tools/mass_check.py);
  the fast build's changes equal the exact build's;
* the charge density the field solve uses after a C5 step (partial sums of the
  plane kernel) equals a fresh velocity integration of the same state.
"""
import numpy as np
import pytest

from helpers import gpu_family
from paper_2007_10196_b200 import configs

pytestmark = pytest.mark.gpu


def _member_sums(fam, s, weights=None):
    out, off = [], 0
    for mi, pts in enumerate(fam.points):
        n = int(np.prod(pts))
        seg = s[off:off + n]
        out.append(np.sum(seg * weights[mi]) if weights is not None else np.sum(seg))
        off += n
    return np.array(out)


@pytest.mark.parametrize("name,T", [("C2", 0.01), ("C3", 0.003)])
def test_periodic_conservation_full_family(ctx_fast, name, T):
    cfg = configs.config(name)
    fam = gpu_family(ctx_fast, cfg)
    fam.initialize(cfg["ic"])
    s0 = fam.download()
    dts = fam.evolve_config(cfg, tfinal=T, stops=[])
    s1 = fam.download()
    assert len(dts) >= 3
    a, b = _member_sums(fam, s0), _member_sums(fam, s1)
    scale = _member_sums(fam, np.abs(s0))
    assert np.all(np.abs(a - b) <= 1e-11 * scale), np.max(np.abs(a - b) / scale)


def test_c5_full_family_mass_and_charge_density(ctx, ctx_fast):
    cfg = configs.config("C5")
    fam = gpu_family(ctx_fast, cfg)
    assert fam.num_members == 121 and fam.total_points == 12057728
    fam.initialize(cfg["ic"])
    s0 = fam.download()
    dts = fam.evolve_config(cfg, tfinal=0.006, stops=[])
    assert len(dts) >= 3
    s1 = fam.download()
    assert np.all(np.isfinite(s1))
    ref = gpu_family(ctx, cfg)  # exact build, same start
    ref.upload(s0)
    # the dt comes from max|E|, whose last bits depend on the build's f
    np.testing.assert_allclose(ref.evolve_config(cfg, tfinal=0.006, stops=[]), dts, rtol=1e-13)
    m0, m1, me = _member_sums(fam, s0), _member_sums(fam, s1), _member_sums(fam, ref.download())
    assert np.all(np.abs(m1 - m0) <= 1e-6 * np.abs(m0))
    assert np.all(np.abs(m1 - me) <= 1e-12 * np.abs(m0)), np.max(np.abs(m1 - me) / np.abs(m0))
    rho_a, E_a = fam.vp_field()        # from the plane kernel's partial sums
    fam.upload(s1)
    rho_b, E_b = fam.vp_field()        # re-integrated by the moment kernel
    for ra, rb, ea, eb in zip(rho_a, rho_b, E_a, E_b):
        assert np.max(np.abs(ra - rb)) <= 1e-13
        assert np.max(np.abs(ea - eb)) <= 1e-12 * (1.0 + np.max(np.abs(eb)))
