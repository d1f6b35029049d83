"""GPU parity: the B200 path (through the C ABI) against the CPU oracle on
identical seeded inputs.

Bars (BASELINE.json north_star): the exact-arithmetic build (``arith="exact"``,
reference expression order, no FMA contraction) is BITWISE equal to the
oracle, which is itself bitwise equal to the reference headers
(tests/test_oracle_pin.py).  The fast build is within a max-abs difference of
1e-10 on the combined fine-grid solution.  Vlasov-Poisson has no reference
(SURVEY F4): GPU vs the oracle restatement within 1e-10.
"""
import numpy as np
import pytest

from helpers import bitwise_equal, gpu_family, maxabs, oracle_objs, random_states
from oracle import oracle as O
from paper_2007_10196_b200 import configs

pytestmark = pytest.mark.gpu

TOL = 1e-10  # north_star: max-abs difference on the combined fine-grid solution


def _rhs_oracle(orc, cfg, states):
    dom, model, _ = oracle_objs(cfg)
    lv = orc.levels(cfg["d"], cfg["nl"])
    out, off = [], 0
    for l in lv:
        n = int(np.prod([p for p in _points(cfg, l)]))
        out.append(orc.rhs(dom, l, model, states[off:off + n]))
        off += n
    return np.concatenate(out)


def _points(cfg, l):
    return [(cfg["root"][k] << int(l[k])) + (1 if cfg["bc"][k] == 1 else 0)
            for k in range(cfg["d"])]


RHS_CASES = [
    ("C1", {}),
    ("C2", {"nl": 3, "root": [16, 16]}),
    ("C3", {"nl": 2, "root": [8, 8, 8]}),
    ("C1", {"speeds": [-1.0, 0.5], "bc": [1, 1]}),        # downwind + zero ghosts
    ("C2", {"nl": 2, "root": [8, 8], "bc": [1, 0]}),     # Burgers, mixed bc
    ("C1", {"d": 1, "nl": 3, "lower": [0.0], "upper": [2.0], "root": [8], "bc": [0],
            "speeds": [1.0]}),
    ("C3", {"d": 4, "nl": 3, "lower": [0.0] * 4, "upper": [2.0] * 4, "root": [6] * 4,
            "bc": [0, 0, 1, 1], "speeds": [1.0, -1.0, 0.5, -0.25]}),
    ("C1", {"weno_mode": 1}),                            # linear weights
]


@pytest.mark.parametrize("name,over", RHS_CASES)
def test_rhs_bitwise(ctx, oracle, name, over):
    cfg = configs.config(name, **over)
    s = random_states(oracle, cfg, seed=7)
    fam = gpu_family(ctx, cfg)
    fam.upload(s)
    got = fam.rhs()
    want = _rhs_oracle(oracle, cfg, s)
    assert bitwise_equal(got, want), maxabs(got, want)


@pytest.mark.parametrize("name,over", RHS_CASES[:5])
def test_rk3_step_bitwise(ctx, oracle, name, over):
    cfg = configs.config(name, **over)
    s = random_states(oracle, cfg, seed=11)
    dom, model, _ = oracle_objs(cfg)
    dt = 1e-3
    fam = gpu_family(ctx, cfg)
    fam.upload(s)
    fam.rk3_step(dt)
    got = fam.download()
    want, off = [], 0
    for l in oracle.levels(cfg["d"], cfg["nl"]):
        n = int(np.prod(_points(cfg, l)))
        w, f = oracle.rk3_step(dom, l, model, s[off:off + n], dt)
        assert f == 0
        want.append(w)
        off += n
    want = np.concatenate(want)
    assert bitwise_equal(got, want), maxabs(got, want)


@pytest.mark.parametrize("name,over,mode", [
    ("C1", {}, O.WENO), ("C1", {}, O.LAGRANGE), ("C2", {"nl": 4, "root": [16, 16]}, O.WENO),
    ("C3", {"nl": 3, "root": [8, 8, 8]}, O.WENO),
    ("C2", {"nl": 3, "root": [8, 8], "bc": [1, 0]}, O.WENO),
    ("C2", {"nl": 3, "root": [8, 8], "bc": [0, 1]}, O.LAGRANGE),
])
def test_combine_bitwise(ctx, oracle, name, over, mode):
    cfg = configs.config(name, **over)
    s = random_states(oracle, cfg, seed=23)
    dom, _, _ = oracle_objs(cfg)
    fam = gpu_family(ctx, cfg)
    fam.upload(s)
    got = fam.combine(mode, 1e-6)
    want = oracle.combine(dom, s, mode, 1e-6)
    assert bitwise_equal(got, want), maxabs(got, want)


@pytest.mark.parametrize("name,over", [
    ("C3", {"nl": 3, "root": [8, 8, 8]}),
    ("C2", {"nl": 3, "root": [8, 8], "bc": [1, 0]}),
    ("C3", {"d": 4, "nl": 3, "lower": [0.0] * 4, "upper": [2.0] * 4, "root": [6] * 4,
            "bc": [0, 0, 1, 1], "speeds": [1.0] * 4}),
])
def test_combine_row_slabs_bitwise(ctx, oracle, monkeypatch, name, over):
    """Row-slab combination (how C5's 4.3e9-point finest grid is produced):
    forced by a tiny memory budget, and sgwg_combine_rows on a sub-range."""
    cfg = configs.config(name, **over)
    s = random_states(oracle, cfg, seed=29)
    dom, _, _ = oracle_objs(cfg)
    want = oracle.combine(dom, s, O.WENO, 1e-6)
    fam = gpu_family(ctx, cfg)
    fam.upload(s)
    monkeypatch.setenv("SGWG_COMBINE_BUDGET_GB", "0.00002")  # 20 kB: many slabs
    got = fam.combine(O.WENO, 1e-6)
    assert bitwise_equal(got, want), maxabs(got, want)
    monkeypatch.delenv("SGWG_COMBINE_BUDGET_GB")
    rows = fam.fine_extent0
    per_row = fam.finest_points // rows
    a, b = rows // 3, rows // 3 + 5
    part = fam.combine_rows(a, b, O.WENO, 1e-6)
    assert bitwise_equal(part, want[a * per_row:b * per_row])


def test_prolong_bitwise(ctx, oracle):
    cfg = configs.config("C3", nl=3, root=[8, 8, 8])
    s = random_states(oracle, cfg, seed=31)
    dom, _, _ = oracle_objs(cfg)
    fam = gpu_family(ctx, cfg)
    fam.upload(s)
    offs = fam.member_offsets()
    for mi in (0, 3, len(offs) - 1):
        n = int(np.prod(fam.points[mi]))
        got = fam.prolong(mi, O.WENO, 1e-6)
        want = oracle.prolong(dom, np.array(fam.levels[mi]), s[offs[mi]:offs[mi] + n], O.WENO,
                              1e-6, fam.finest_points)
        assert bitwise_equal(got, want), (mi, maxabs(got, want))


def _evolve_both(ctx, oracle, cfg, tfinal, stops=()):
    dom, model, pol = oracle_objs(cfg)
    s0 = oracle.init_family(cfg["ic"], dom)
    want_combined = []
    want, want_dts, st, _ = oracle.evolve(
        dom, model, pol, s0, tfinal, stops,
        on_stop=lambda t, s: want_combined.append(oracle.combine(dom, s, cfg["interp"],
                                                                 cfg["epsilon"])))
    assert st == 0
    fam = gpu_family(ctx, cfg)
    fam.initialize(cfg["ic"])
    assert bitwise_equal(fam.download(), s0)  # initialize_family on the host is exact
    got_combined = []
    got_dts = fam.evolve_config(
        cfg, tfinal=tfinal, stops=stops,
        on_stop=lambda t: got_combined.append(fam.combine(cfg["interp"], cfg["epsilon"])))
    return fam.download(), want, got_dts, want_dts, got_combined, want_combined


def test_evolve_c1_full_bitwise(ctx, oracle):
    """BASELINE C1 end to end (T=1, 2048 steps): bitwise."""
    cfg = configs.config("C1")
    got, want, gd, wd, gc, wc = _evolve_both(ctx, oracle, cfg, cfg["tfinal"])
    assert len(gd) == len(wd) == 2048
    assert bitwise_equal(gd, wd)
    assert bitwise_equal(got, want), maxabs(got, want)
    assert bitwise_equal(gc[-1], wc[-1]), maxabs(gc[-1], wc[-1])


def test_evolve_c2_stops_bitwise(ctx, oracle):
    """BASELINE C2 family, CFL dt from the family max|u|, stop landing."""
    cfg = configs.config("C2", nl=4, root=[16, 16])
    got, want, gd, wd, gc, wc = _evolve_both(ctx, oracle, cfg, 0.05, stops=[0.02, 0.02 + 1e-14])
    assert bitwise_equal(gd, wd), (len(gd), len(wd))
    assert len(gc) == len(wc) == 2
    assert bitwise_equal(got, want), maxabs(got, want)
    for a, b in zip(gc, wc):
        assert bitwise_equal(a, b), maxabs(a, b)


def test_evolve_c2_per_dimension_passes_bitwise(ctx, oracle, monkeypatch):
    """The per-dimension pass kernels (used for d != 2) on the 2D family too."""
    monkeypatch.setenv("SGWG_NO_FUSED2D", "1")
    cfg = configs.config("C2", nl=3, root=[16, 16])
    got, want, gd, wd, gc, wc = _evolve_both(ctx, oracle, cfg, 0.03, stops=[0.01])
    assert bitwise_equal(gd, wd)
    assert bitwise_equal(got, want), maxabs(got, want)


def test_evolve_c3_short_bitwise(ctx, oracle):
    """BASELINE C3 family (3D, 31 members, dt = h^{5/3}) for a few steps."""
    cfg = configs.config("C3")
    T = 4 * cfg["reference_spacing"] ** (5.0 / 3.0)
    got, want, gd, wd, gc, wc = _evolve_both(ctx, oracle, cfg, T)
    assert len(gd) == len(wd) == 4
    assert bitwise_equal(got, want), maxabs(got, want)
    assert bitwise_equal(gc[-1], wc[-1]), maxabs(gc[-1], wc[-1])


def test_sharded_family_with_nccl_comm_bitwise(ctx, oracle):
    """The multi-GPU step (local speeds -> NCCL all-reduce(max) -> dt, captured
    in the step graph) and the combine all-reduce, on a one-rank communicator:
    identical to the single-device path and to the oracle."""
    from paper_2007_10196_b200 import sgwg
    cfg = configs.config("C2", nl=3, root=[16, 16])
    dom, model, pol = oracle_objs(cfg)
    s0 = oracle.init_family(cfg["ic"], dom)
    want, wd, st, _ = oracle.evolve(dom, model, pol, s0, 0.03)
    fam = gpu_family(ctx, cfg, members=list(range(len(oracle.levels(2, 3)))))
    fam.set_comm(sgwg.nccl_unique_id(), 1, 0)
    fam.upload(s0)
    gd = fam.evolve_config(cfg, tfinal=0.03, stops=[])
    assert bitwise_equal(gd, wd)
    assert bitwise_equal(fam.download(), want)
    assert bitwise_equal(fam.combine(O.WENO, 1e-6), oracle.combine(dom, want, O.WENO, 1e-6))


def test_shard_subset_matches_members(ctx, oracle):
    """A shard holds only its members; its partial combination is the sum over them."""
    cfg = configs.config("C2", nl=3, root=[16, 16])
    dom, model, pol = oracle_objs(cfg)
    s0 = oracle.init_family(cfg["ic"], dom)
    lv = oracle.levels(2, 3)
    pts = [int(np.prod(_points(cfg, l))) for l in lv]
    offs = np.concatenate([[0], np.cumsum(pts)])
    mine = [1, 4, 5]
    fam = gpu_family(ctx, cfg, members=mine)
    fam.upload(np.concatenate([s0[offs[m]:offs[m + 1]] for m in mine]))
    fam.rk3_step(1e-3)
    got = fam.download()
    o = 0
    for m in mine:
        w, f = oracle.rk3_step(dom, lv[m], model, s0[offs[m]:offs[m + 1]], 1e-3)
        assert bitwise_equal(got[o:o + pts[m]], w)
        o += pts[m]


def test_evolve_fast_within_tol(ctx_fast, oracle):
    cfg = configs.config("C2", nl=4, root=[16, 16])
    got, want, gd, wd, gc, wc = _evolve_both(ctx_fast, oracle, cfg, 0.05)
    assert len(gd) == len(wd)
    assert maxabs(gd, wd) < 1e-15
    assert maxabs(gc[-1], wc[-1]) < TOL


@pytest.mark.parametrize("T,stops", [
    (0.0, []),                                   # tfinal == 0: one stop at 0, no steps
    (0.02, [-1.0, 0.0, 0.01, 0.01 + 1e-14, 0.5]),  # out-of-range and duplicate stops
    (0.02, [0.02, 0.005]),                         # unsorted, stop == T
])
def test_evolve_stop_list_semantics(ctx, oracle, T, stops):
    """timestep.hpp:133-172 stop handling, bitwise (dts, stop count, combined fields)."""
    cfg = configs.config("C2", nl=3, root=[16, 16])
    got, want, gd, wd, gc, wc = _evolve_both(ctx, oracle, cfg, T, stops=stops)
    assert len(gc) == len(wc)
    assert bitwise_equal(gd, wd), (gd, wd)
    assert bitwise_equal(got, want)
    for a, b in zip(gc, wc):
        assert bitwise_equal(a, b)


def test_failure_injection(ctx, oracle):
    """test_timestep.cpp:145-155: state x 1e150 -> FamilyIntegratorFailure."""
    from paper_2007_10196_b200 import sgwg
    cfg = configs.config("C2", nl=3, root=[8, 8])
    dom, model, pol = oracle_objs(cfg)
    s0 = oracle.init_family(cfg["ic"], dom) * 1e150
    _, _, st, (fm, fst, fsg) = oracle.evolve(dom, model, pol, s0, 0.01)
    assert st == 2  # SGWO_ENONFINITE
    fam = gpu_family(ctx, cfg)
    fam.upload(s0)
    with pytest.raises(sgwg.FamilyIntegratorFailure) as ei:
        fam.evolve_config(cfg, tfinal=0.01)
    assert (ei.value.member, ei.value.step, ei.value.stage) == (fm, fst, fsg)


def test_invalid_arguments(ctx):
    from paper_2007_10196_b200 import sgwg
    with pytest.raises(ValueError):
        sgwg.Family(ctx, 2, 0, [0, 0], [1, 1], [8, 8], [0, 0])   # N_L < d-1
    with pytest.raises(ValueError):
        sgwg.Family(ctx, 2, 2, [0, 0], [0, 1], [8, 8], [0, 0])   # upper <= lower
    cfg = configs.config("C1", root=[4, 4], nl=1)
    fam = sgwg.Family(ctx, 2, 1, [0, 0], [2, 2], [4, 4], [0, 0])
    with pytest.raises(ValueError):  # periodic line of 4 < 6 points (weno.hpp:122)
        fam.set_model(0, speeds=[1, 1])
    fam2 = gpu_family(ctx, configs.config("C1"))
    with pytest.raises(ValueError):
        fam2.evolve_config(configs.config("C1"), tfinal=-1.0)
    assert cfg


def test_vp_c4_short_within_tol(ctx, oracle):
    """BASELINE C4 physics (no reference: oracle restatement), short horizon."""
    cfg = configs.config("C4", nl=3, root=[16, 16])
    got, want, gd, wd, gc, wc = _evolve_both(ctx, oracle, cfg, 0.5)
    assert len(gd) == len(wd)
    assert maxabs(gd, wd) < 1e-14
    assert maxabs(got, want) < TOL
    assert maxabs(gc[-1], wc[-1]) < TOL
