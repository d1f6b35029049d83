"""Sharded families through libsgwg (the product's NCCL path).

* option B on a one-rank communicator (SGWG_OPTION_B=1 forces the gathered view):
  sgwg_combine_local, combined_stats and eval_points equal the unsharded family's
  bitwise (the exact build: the reference's arithmetic);
* two ranks (tools/multirank_check.py under torchrun, one process per GPU): shards,
  per-step all-reduce, option-B rows / stats / cut plane against the unsharded family,
  failure propagation -- skipped when fewer than 2 GPUs are visible.
"""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

from helpers import gpu_family
from paper_2007_10196_b200 import configs

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("name,over,arith,T", [
    ("C3", {"nl": 2, "root": [8, 8, 8]}, "exact", 0.004),
    ("C5", {"nl": 3}, "fast", 0.02),
    ("C2", {"nl": 3, "root": [16, 16]}, "fast", 0.02),
])
def test_option_b_one_rank_matches_unsharded(monkeypatch, name, over, arith, T):
    from paper_2007_10196_b200 import sgwg
    cfg = configs.config(name, **over)
    ctx = sgwg.Context(0, arith=arith)
    ref = gpu_family(ctx, cfg)
    ref.initialize(cfg["ic"])
    ref.evolve_config(cfg, tfinal=T, stops=[])
    full = ref.combine(cfg["interp"], cfg["epsilon"])
    rst = ref.combined_stats(cfg["interp"], cfg["epsilon"])
    rplane = ref.cut_plane(0, cfg["d"] - 1, [0] * cfg["d"], cfg["interp"], cfg["epsilon"])
    fam = gpu_family(ctx, cfg, members=list(range(ref.num_members)))
    fam.set_comm(sgwg.nccl_unique_id(), 1, 0)
    fam.initialize(cfg["ic"])
    fam.evolve_config(cfg, tfinal=T, stops=[])
    monkeypatch.setenv("SGWG_OPTION_B", "1")
    a, b, rows = fam.combine_local(cfg["interp"], cfg["epsilon"])
    st = fam.combined_stats(cfg["interp"], cfg["epsilon"])
    plane = fam.cut_plane(0, cfg["d"] - 1, [0] * cfg["d"], cfg["interp"], cfg["epsilon"])
    print(f"\n[{name} {arith}] option-B rows [{a}, {b}), |rows - full| "
          f"{float(np.max(np.abs(rows - full))):.1e}")
    assert (a, b) == (0, ref.fine_extent0)
    assert np.array_equal(rows, full)
    assert np.array_equal(plane, rplane)
    for k in ("mass", "min", "max"):
        assert st[k] == pytest.approx(rst[k], rel=1e-14, abs=1e-14)
    fam.close()
    ref.close()
    ctx.close()


def _gpus():
    try:
        import torch
        return torch.cuda.device_count()
    except Exception:  # pragma: no cover
        return 0


@pytest.mark.skipif(_gpus() < 2, reason="needs 2 GPUs (one process per GPU)")
@pytest.mark.parametrize("name", ["C2", "C5"])
def test_two_ranks_through_libsgwg(name):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", "29517",
           os.path.join(ROOT, "tools", "multirank_check.py"), name]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    print(r.stdout[-2000:], r.stderr[-2000:])
    assert r.returncode == 0 and len(lines) == 2 and all(x["ok"] for x in lines)
