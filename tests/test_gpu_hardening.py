"""Fast-build kernels against their reference forms and the oracle:

* the chunked combination passes (kernels.cuh upsample_fast_kernel and
  final_fast_kernel: 8-point chunks, per-centre smoothness indicators,
  common-denominator weights, tabulated per-offset coefficients) against the
  generic per-point kernels (SGWG_UPSAMPLE_GENERIC=1, SGWG_FINAL_GENERIC=1) and the oracle,
  both interpolation modes, periodic and zero-ghost last dimensions;
* overflow guard: states of magnitude ~1e40, where the fast build's
  common-denominator WENO weights overflow but the reference's separate
  divides do not (weno.hpp:60-72) -- advection tendencies, a few RK steps and
  the combination must still match the oracle.
"""
import numpy as np
import pytest

from helpers import gpu_family, maxabs, oracle_objs
from paper_2007_10196_b200 import configs
from test_gpu_parity import _rhs_oracle

pytestmark = pytest.mark.gpu

COMBINE_CASES = [
    ("C1", {}),
    ("C2", {"nl": 4, "root": [16, 16]}),
    ("C3", {"nl": 3, "root": [8, 8, 8]}),
    ("C4", {"nl": 3, "root": [16, 16]}),
    ("C5", {"nl": 3}),
    ("ex1", {}),  # Lagrange prolongation
]


def _noisy_states(oracle, cfg, seed=11, scale=1.0):
    dom, _, _ = oracle_objs(cfg)
    s = oracle.init_family(cfg["ic"], dom)
    rng = np.random.default_rng(seed)
    return scale * (s + 0.1 * rng.standard_normal(s.size))


@pytest.mark.parametrize("name,over", COMBINE_CASES)
def test_final_chunked_matches_generic_and_oracle(ctx_fast, oracle, monkeypatch, name, over):
    cfg = configs.config(name, **over)
    s = _noisy_states(oracle, cfg)
    fam = gpu_family(ctx_fast, cfg)
    fam.upload(s)
    got = fam.combine(cfg["interp"], cfg["epsilon"])
    monkeypatch.setenv("SGWG_FINAL_GENERIC", "1")
    monkeypatch.setenv("SGWG_UPSAMPLE_GENERIC", "1")
    gen = fam.combine(cfg["interp"], cfg["epsilon"])
    monkeypatch.delenv("SGWG_FINAL_GENERIC")
    monkeypatch.delenv("SGWG_UPSAMPLE_GENERIC")
    dom, _, _ = oracle_objs(cfg)
    want = oracle.combine(dom, s, cfg["interp"], cfg["epsilon"])
    scale = max(1.0, float(np.max(np.abs(want))))
    print(f"\n[{name}] chunked vs generic {maxabs(got, gen):.2e}, vs oracle {maxabs(got, want):.2e}")
    assert maxabs(got, gen) <= 1e-12 * scale
    assert maxabs(got, want) <= 1e-10 * scale
    fam.close()


OVERFLOW_CASES = [
    ("C1", {}),                                   # 2D stage / persistent kernels
    ("C3", {"nl": 2, "root": [8, 8, 8]}),          # 3D stage kernel
    ("C3", {"d": 4, "nl": 3, "lower": [0.0] * 4, "upper": [2.0] * 4, "root": [8] * 4,
            "bc": [0, 0, 1, 1], "speeds": [1.0, -1.0, 0.5, -0.25]}),  # 4D whole-plane kernels
]


@pytest.mark.parametrize("name,over", OVERFLOW_CASES)
def test_overflow_guard_huge_states(ctx_fast, oracle, name, over):
    cfg = configs.config(name, **over)
    s = _noisy_states(oracle, cfg, seed=5, scale=1e40)
    fam = gpu_family(ctx_fast, cfg)
    fam.upload(s)
    got = fam.rhs()
    want = _rhs_oracle(oracle, cfg, s)
    assert np.all(np.isfinite(want))
    rel = maxabs(got, want) / float(np.max(np.abs(want)))
    # a few RK steps (the reference stays finite, so must the fast build)
    dom, model, pol = oracle_objs(cfg)
    T = 3 * cfg["reference_spacing"] ** (5.0 / 3.0)
    ws, wd, st, _ = oracle.evolve(dom, model, pol, s, T)
    assert st == 0
    fam.upload(s)
    gd = fam.evolve_config(cfg, tfinal=T, stops=[])
    gs = fam.download()
    srel = maxabs(gs, ws) / float(np.max(np.abs(ws)))
    comb = fam.combine(cfg["interp"], cfg["epsilon"])
    wc = oracle.combine(dom, ws, cfg["interp"], cfg["epsilon"])
    crel = maxabs(comb, wc) / float(np.max(np.abs(wc)))
    print(f"\n[{name} d={cfg['d']} |u|~1e40] rhs rel {rel:.2e}, states rel {srel:.2e}, "
          f"combined rel {crel:.2e}")
    assert len(gd) == len(wd)
    assert rel <= 1e-10 and srel <= 1e-10 and crel <= 1e-10
    # back to ordinary magnitudes: the fast kernels again (and still correct)
    s1 = _noisy_states(oracle, cfg, seed=6)
    fam.upload(s1)
    assert maxabs(fam.rhs(), _rhs_oracle(oracle, cfg, s1)) <= 1e-10
    fam.close()
