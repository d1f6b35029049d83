"""Single-grid mode (make_single_grid, runner.hpp:106-115): the full grid at
level (N_L, ..., N_L) stepped through the same B200 path, bitwise against the
oracle's SspRk3 steps with evolve_family's dt / landing rules (restated here in
Python float arithmetic, which is IEEE double like the reference)."""
import numpy as np
import pytest

from helpers import bitwise_equal, oracle_objs
from paper_2007_10196_b200 import configs, sgwg

pytestmark = pytest.mark.gpu


def _dt_sequence_and_states(oracle, cfg, T):
    dom, model, pol = oracle_objs(cfg)
    lv = np.full(cfg["d"], cfg["nl"], dtype=np.int32)
    n = int(np.prod([(cfg["root"][k] << cfg["nl"]) + (1 if cfg["bc"][k] else 0)
                     for k in range(cfg["d"])]))
    u = oracle.restrict(cfg["ic"], dom, lv, n)
    h = [(cfg["upper"][k] - cfg["lower"][k]) / cfg["root"][k] / (1 << cfg["nl"])
         for k in range(cfg["d"])]
    eps_t = 1e-12 * max(1.0, T)
    t, dts = 0.0, []
    while T - t > eps_t:  # timestep.hpp:152-168
        rem = T - t
        if cfg["dt_mode"] == 0:
            sp = float(np.max(np.abs(u))) if cfg["kind"] == 1 else None
            inv = 0.0
            for k in range(cfg["d"]):
                inv += (sp if sp is not None else abs(cfg["speeds"][k])) / h[k]
            dt = rem if inv == 0.0 else min(cfg["cfl"] / inv, rem)
        else:
            dt = cfg["reference_spacing"] ** (5.0 / 3.0)
            if cfg["dt_scale"] != 1.0:
                dt = cfg["dt_scale"] * dt
            dt = min(dt, rem)
        if T - (t + dt) <= eps_t:
            dt = T - t
        u, f = oracle.rk3_step(dom, lv, model, u, dt)
        assert f == 0
        t += dt
        dts.append(dt)
    return u, np.array(dts), n


@pytest.mark.parametrize("name,over,T", [("C1", {}, 0.01), ("C2", {"nl": 3, "root": [16, 16]}, 0.02)])
def test_single_grid_bitwise(ctx, oracle, name, over, T):
    cfg = configs.config(name, **over)
    want, wd, n = _dt_sequence_and_states(oracle, cfg, T)
    fam = sgwg.Family.from_config(ctx, cfg, single=True)
    assert fam.num_members == 1 and fam.total_points == n == fam.finest_points
    fam.initialize(cfg["ic"])
    gd = fam.evolve_config(cfg, tfinal=T, stops=[])
    assert bitwise_equal(gd, wd)
    got = fam.combine(cfg["interp"], cfg["epsilon"])  # the grid's own field
    assert bitwise_equal(got, want)
