"""Pin the CPU oracle (oracle/sgw_oracle.c) to the reference.

1. Against the committed golden fixtures made by tests/golden/make_golden.py
   from the unmodified reference headers: BITWISE.
2. Against the reference headers live (oracle/_ref/libsgwref.so, where built):
   BITWISE, on more configurations.
3. The reference's own known-answer tests (proj/tests/test_weno.cpp,
   test_interp.cpp, test_combine.cpp, test_grid.cpp), restated.
"""
import os

import numpy as np
import pytest

from helpers import bitwise_equal, oracle_objs
from oracle import oracle as O
from paper_2007_10196_b200 import configs

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def gold(name):
    return np.load(os.path.join(GOLD, name))


# ---- 1. golden fixtures ------------------------------------------------------
def test_golden_flux(oracle):
    g = gold("weno_flux.npz")
    nl = np.array([oracle.weno5_flux_positive(s, 1e-6, O.NONLINEAR) for s in g["flux_stencils"]])
    li = np.array([oracle.weno5_flux_positive(s, 1e-6, O.LINEAR) for s in g["flux_stencils"]])
    assert bitwise_equal(nl, g["flux_nonlinear"])
    assert bitwise_equal(li, g["flux_linear"])


def test_golden_lines(oracle):
    g = gold("weno_lines.npz")
    ci = 0
    while f"u{ci}" in g:
        n, fk, c, alpha, dx, bc = g[f"case{ci}"]
        du = oracle.weno_derivative_line(g[f"u{ci}"], int(fk), c, alpha, dx, int(bc))
        assert bitwise_equal(du, g[f"du{ci}"]), ci
        ci += 1
    assert ci == 6


def test_golden_upsample(oracle):
    g = gold("upsample.npz")
    ci = 0
    while f"src{ci}" in g:
        m, bc, mode, n_dst = g[f"case{ci}"]
        dst = oracle.upsample_line(g[f"src{ci}"], int(n_dst), int(m), int(bc), int(mode), 1e-6)
        assert bitwise_equal(dst, g[f"dst{ci}"]), ci
        ci += 1
    assert ci == 12


def test_golden_c1_full(oracle):
    cfg = configs.config("C1")
    dom, m, p = oracle_objs(cfg)
    g = gold("c1_full.npz")
    s0 = oracle.init_family(cfg["ic"], dom)
    s, dts, st, _ = oracle.evolve(dom, m, p, s0, cfg["tfinal"])
    assert st == 0 and len(dts) == 2048
    assert bitwise_equal(dts, g["dts"])
    assert bitwise_equal(s, g["states"])
    assert bitwise_equal(oracle.combine(dom, s, cfg["interp"], cfg["epsilon"]), g["combined"])


def test_golden_c2_small(oracle):
    cfg = configs.config("C2", nl=3, root=[16, 16])
    dom, m, p = oracle_objs(cfg)
    g = gold("c2_small.npz")
    s0 = oracle.init_family(cfg["ic"], dom)
    comb = []
    s, dts, st, _ = oracle.evolve(dom, m, p, s0, 0.2, [0.1], on_stop=lambda t, x: comb.append(
        oracle.combine(dom, x, cfg["interp"], cfg["epsilon"])))
    assert st == 0
    assert bitwise_equal(dts, g["dts"])
    assert bitwise_equal(s, g["states"])
    assert bitwise_equal(comb[0], g["combined_t01"])
    assert bitwise_equal(comb[1], g["combined_t02"])


def test_golden_c3_small(oracle):
    cfg = configs.config("C3", nl=2, root=[8, 8, 8])
    dom, m, _ = oracle_objs(cfg)
    g = gold("c3_small.npz")
    s = g["states"]
    rhs, off = [], 0
    for l in oracle.levels(3, 2):
        n = int(np.prod([8 << int(q) for q in l]))
        rhs.append(oracle.rhs(dom, l, m, s[off:off + n]))
        off += n
    assert bitwise_equal(np.concatenate(rhs), g["rhs"])
    assert bitwise_equal(oracle.combine(dom, s, O.WENO, 1e-6), g["combined"])
    assert bitwise_equal(oracle.combine(dom, s, O.LAGRANGE, 1e-6), g["combined_lagrange"])


# ---- 2. live reference (built here from /root/reference; travels as a .so) --
ref_only = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")


@ref_only
@pytest.mark.parametrize("name,over,T,stops", [
    ("C1", {}, 0.05, []),
    ("C2", {"nl": 3, "root": [16, 16]}, 0.05, [0.01]),
    ("C3", {"nl": 2, "root": [8, 8, 8]}, 0.02, []),
    ("ex1", {}, 0.05, []),
    ("ex3a", {}, 0.05, []),
    ("ex5a", {}, 0.05, [0.02]),
    ("C2", {"nl": 2, "root": [8, 8], "bc": [1, 0]}, 0.05, []),
])
def test_oracle_equals_reference(oracle, name, over, T, stops):
    ref = O.Reference()
    cfg = configs.config(name, **over)
    dom, m, p = oracle_objs(cfg)
    s0 = oracle.init_family(cfg["ic"], dom)
    assert bitwise_equal(s0, ref.init_family(cfg["ic"], dom, m))
    a, da, sa, _ = oracle.evolve(dom, m, p, s0, T, stops)
    b, db, sb, _ = ref.evolve(dom, m, p, s0, T, stops)
    assert sa == sb == 0
    assert bitwise_equal(da, db)
    assert bitwise_equal(a, b)
    for mode in (O.WENO, O.LAGRANGE):
        assert bitwise_equal(oracle.combine(dom, a, mode, cfg["epsilon"]),
                             ref.combine(dom, b, mode, cfg["epsilon"]))


@ref_only
def test_oracle_failure_matches_reference(oracle):
    ref = O.Reference()
    cfg = configs.config("C2", nl=3, root=[8, 8])
    dom, m, p = oracle_objs(cfg)
    s0 = oracle.init_family(cfg["ic"], dom) * 1e150
    _, _, sa, fa = oracle.evolve(dom, m, p, s0, 0.01)
    _, _, sb, fb = ref.evolve(dom, m, p, s0, 0.01)
    assert sa == sb == 2 and fa == fb


# ---- 3. reference known-answer tests, restated --------------------------------
def test_kat_smoothness_and_flux(oracle):
    # test_weno.cpp:101-117, 143-151
    assert oracle.weno5_flux_positive([3, 3, 3, 3, 3]) == pytest.approx(3.0, abs=1e-14)
    assert oracle.weno5_flux_positive([0, 1, 2, 3, 4]) == pytest.approx(2.5, rel=1e-14)
    assert oracle.weno5_flux_positive([0, 1, 2, 3, 4], mode=O.LINEAR) == pytest.approx(2.5)
    assert abs(oracle.weno5_flux_positive([0, 0, 0, 1, 1])) < 1e-4
    for c in (0.0, 1.0, -4.5, 1e6):
        assert oracle.weno5_flux_positive([c] * 5) == pytest.approx(c, abs=1e-14 * abs(c) + 1e-16)


def test_kat_combination_coefficients():
    # test_combine.cpp:76-104: (1), (1,-1), (1,-2,1), (1,-3,3,-1)
    from math import comb
    for d, want in [(1, [1]), (2, [1, -1]), (3, [1, -2, 1]), (4, [1, -3, 3, -1])]:
        assert [(-1) ** j * comb(d - 1, j) for j in range(d)] == want


def test_kat_level_enumeration(oracle):
    # test_grid.cpp:16-29 brute force: all l >= 0 with max(0, nl-d+1) <= |l| <= nl, sorted
    import itertools
    for d in (1, 2, 3, 4):
        for nl in range(d - 1, d + 3):
            lo = max(0, nl - d + 1)
            want = sorted(t for t in itertools.product(range(nl + 1), repeat=d)
                          if lo <= sum(t) <= nl)
            got = [tuple(r) for r in oracle.levels(d, nl)]
            assert got == want


def test_kat_constant_preserved_by_combine(oracle):
    # test_combine.cpp:110-141: constants preserved to 1e-13 in 2D/3D
    for d, nl in ((2, 3), (3, 2)):
        cfg = configs.config("C3" if d == 3 else "C1", nl=nl, root=[8] * d)
        dom, _, _ = oracle_objs(cfg)
        s = np.full(oracle.total_points(dom), 2.5)
        out = oracle.combine(dom, s, O.WENO, 1e-6)
        assert np.max(np.abs(out - 2.5)) < 1e-13


def test_kat_interp_nodal_passthrough(oracle):
    # test_interp.cpp:218-239: nodal values pass through bitwise
    rng = np.random.default_rng(3)
    src = rng.uniform(-1, 1, 16)
    for m in (1, 2, 3):
        dst = oracle.upsample_line(src, 16 << m, m, O.PERIODIC, O.WENO, 1e-6)
        assert bitwise_equal(dst[:: 1 << m], src)
