"""N>1 host logic on CPU with gloo, world_size 2.

The B200 path shards the family by member (paper_2007_10196_b200/shard.py):
each rank evolves its members, the family wave speed is an all-reduce(max)
per step and the combination an all-reduce(sum) of per-rank partial sums.
Here the per-rank work is done by the CPU oracle (test infrastructure) and
the collectives by gloo, checking that the sharded pipeline reproduces the
single-process reference result: identical dt sequence and member states
(members are independent given the shared dt), combination within 1e-13
(summation order differs only across ranks).

Option B (libsgwg's sgwg_combine_local / combined_stats / eval_points for a
sharded family): every rank gathers all member states and combines its own
dimension-0 rows [rows*r/N, rows*(r+1)/N) for every member -- the rows must be
BITWISE those of the single-process combination (dimension-sequential
prolongation, interp.hpp:217-244, makes row slabs independent).
"""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2007_10196_b200 import configs, shard


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_lpt_shards_deterministic_and_balanced():
    cfg = configs.config("C3")
    from oracle.oracle import Oracle
    lv = Oracle().levels(3, cfg["nl"])
    pts = shard.member_points(lv, cfg["root"], cfg["bc"])
    for n in (1, 2, 4, 8):
        sh = shard.lpt_shards(pts, n)
        assert sorted(i for s in sh for i in s) == list(range(len(pts)))
        assert all(s == sorted(s) for s in sh)
        assert sh == shard.lpt_shards(pts, n)
    assert shard.shard_balance(pts, shard.lpt_shards(pts, 2)) < 1.01
    assert shard.shard_balance(pts, shard.lpt_shards(pts, 8)) < 1.05
    with pytest.raises(ValueError):
        shard.lpt_shards(pts, 0)


def _worker(rank, world, port, cfg_name, over, T, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import torch
    from oracle import oracle as O
    from helpers import oracle_objs
    orc = O.Oracle()
    cfg = configs.config(cfg_name, **over)
    dom, model, pol = oracle_objs(cfg)
    lv = orc.levels(cfg["d"], cfg["nl"])
    pts = shard.member_points(lv, cfg["root"], cfg["bc"])
    mine = shard.lpt_shards(pts, world)[rank]
    offs = np.concatenate([[0], np.cumsum(pts)])
    s_all = orc.init_family(cfg["ic"], dom)
    states = {m: s_all[offs[m]:offs[m + 1]].copy() for m in mine}
    fine_h = [(cfg["upper"][k] - cfg["lower"][k]) / cfg["root"][k] / (1 << cfg["nl"])
              for k in range(cfg["d"])]
    t, dts = 0.0, []
    eps_t = 1e-12 * max(1.0, T)
    while T - t > eps_t:
        # family wave speed: local max|u| -> all-reduce(max) (models.hpp:798-802)
        local = max((float(np.max(np.abs(states[m]))) for m in mine), default=0.0)
        g = torch.tensor([local], dtype=torch.float64)
        dist.all_reduce(g, op=dist.ReduceOp.MAX)
        sp = np.full(cfg["d"], g.item())
        remaining = T - t
        inv = 0.0
        for k in range(cfg["d"]):
            inv += sp[k] / fine_h[k]
        dt = min(cfg["cfl"] / inv, remaining)
        if T - (t + dt) <= eps_t:
            dt = T - t
        for m in mine:
            states[m], f = orc.rk3_step(dom, lv[m], model, states[m], dt)
            assert f == 0
        t += dt
        dts.append(dt)
    # partial combination sum in member order, all-reduce(sum)
    fine = orc.finest_points(dom)
    part = np.zeros(fine)
    coef = {0: 1.0, 1: -1.0, 2: 1.0}
    for m in mine:
        c = [1, -1, 1, -1][cfg["nl"] - int(sum(lv[m]))] * (1 if cfg["d"] < 3 else 1)
        if cfg["d"] == 3:
            c = [1, -2, 1][cfg["nl"] - int(sum(lv[m]))]
        p = orc.prolong(dom, lv[m], states[m], cfg["interp"], cfg["epsilon"], fine)
        part = part + c * p
    del coef
    tp = torch.from_numpy(part)
    dist.all_reduce(tp, op=dist.ReduceOp.SUM)
    # option B: gather every shard's states, combine this rank's dimension-0 rows
    shards = [None] * world
    dist.all_gather_object(shards, {int(m): states[m] for m in mine})
    full = np.concatenate([next(sh[m] for sh in shards if m in sh) for m in range(len(pts))])
    fine_ext = [(cfg["root"][k] << cfg["nl"]) + (1 if cfg["bc"][k] == 1 else 0)
                for k in range(cfg["d"])]
    a, b = fine_ext[0] * rank // world, fine_ext[0] * (rank + 1) // world
    rows = orc.combine_box(dom, full, [a] + [0] * (cfg["d"] - 1), [b] + fine_ext[1:],
                           cfg["interp"], cfg["epsilon"])
    if rank == 0:
        q.put((np.array(dts), {int(m): states[m] for m in mine}, tp.numpy().copy(), (a, b, rows)))
    else:
        q.put((None, {int(m): states[m] for m in mine}, None, (a, b, rows)))
    dist.destroy_process_group()


@pytest.mark.parametrize("cfg_name,over,T", [
    ("C2", {"nl": 3, "root": [16, 16]}, 0.02),
    ("C3", {"nl": 2, "root": [8, 8, 8], "kind": 1, "dt_mode": 0, "cfl": 0.5}, 0.01),
])
def test_two_rank_sharded_pipeline_matches_single(cfg_name, over, T):
    from helpers import oracle_objs
    from oracle import oracle as O
    world = 2
    ctxm = mp.get_context("spawn")
    q = ctxm.Queue()
    port = _free_port()
    procs = [ctxm.Process(target=_worker, args=(r, world, port, cfg_name, over, T, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    dts = next(r[0] for r in res if r[0] is not None)
    combined = next(r[2] for r in res if r[2] is not None)
    states = {}
    for r in res:
        states.update(r[1])
    orc = O.Oracle()
    cfg = configs.config(cfg_name, **over)
    dom, model, pol = oracle_objs(cfg)
    s0 = orc.init_family(cfg["ic"], dom)
    s, wdts, st, _ = orc.evolve(dom, model, pol, s0, T)
    assert st == 0
    assert np.array_equal(dts, wdts)
    lv = orc.levels(cfg["d"], cfg["nl"])
    pts = shard.member_points(lv, cfg["root"], cfg["bc"])
    offs = np.concatenate([[0], np.cumsum(pts)])
    for m in range(len(pts)):
        assert np.array_equal(states[m], s[offs[m]:offs[m + 1]])
    want = orc.combine(dom, s, cfg["interp"], cfg["epsilon"])
    assert np.max(np.abs(combined - want)) < 1e-13
    # option B: the ranks' row slabs tile the finest grid and are bitwise the combination
    slabs = sorted(r[3][:2] + (r[3][2],) for r in res)
    assert slabs[0][0] == 0 and all(slabs[i][1] == slabs[i + 1][0] for i in range(world - 1))
    rows = np.concatenate([sl[2].ravel() for sl in slabs])
    assert np.array_equal(rows, want.ravel())
