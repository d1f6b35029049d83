"""The reference's acceptance experiments through the B200 path: run() of
runner.hpp:270-416 (paper_2007_10196_b200.runner) reproduces the error tables
the reference itself printed (proj/test_output.txt, criteria 1-4 of
proj/tests/acceptance.cpp) to the printed digits -- refinement studies of the
paper's Tables 1, 2 and 4 on sparse and single grids, with the error norms and
orders computed on the device (sgwg_combined_stats)."""
import os

import numpy as np
import pytest

from paper_2007_10196_b200 import configs, runner, sgwg

pytestmark = pytest.mark.gpu


def _fmt(v):
    return "%.4e" % v


def test_table1_ex1_sparse(ctx):
    """criterion 1: ex1 sparse, linear scheme, Lagrange prolongation, N_L = 3."""
    r = runner.run(configs.config("ex1"), roots=[10, 20, 40], ctx=ctx)
    assert [_fmt(x["l1"]) for x in r["rows"]] == ["3.1760e-07", "9.9140e-09", "3.0987e-10"]
    assert _fmt(r["rows"][-1]["order_l1"]) == "4.9997e+00"


def test_table1_ex1_single(ctx):
    """criterion 2: the 80^2 single-grid anchor and the L1/Linf ratio."""
    r = runner.run(configs.config("ex1"), roots=[10], grid_mode="single", ctx=ctx)
    row = r["rows"][0]
    assert _fmt(row["l1"]) == "3.1557e-07"
    assert _fmt(row["l1"] / row["linf"]) == "6.3658e-01"


def test_table4_ex3a_burgers(ctx):
    """criterion 3: 2D Burgers, WENO scheme and prolongation, epsilon 1e-3."""
    r = runner.run(configs.config("ex3a"), roots=[10, 20], ctx=ctx)
    assert [_fmt(x["l1"]) for x in r["rows"]] == ["7.1354e-05", "2.7404e-07"]
    assert _fmt(r["rows"][-1]["order_l1"]) == "8.0244e+00"


def test_table2_ex3b_and_ex2(ctx):
    """criterion 4: 3D Burgers with the linear scheme / Lagrange prolongation
    (the published Table 2 values) and genuine 3D advection (ex2)."""
    cfg = configs.config("ex3b", weno_mode=configs.LINEAR, interp=configs.LAGRANGE)
    r = runner.run(cfg, roots=[10, 20], ctx=ctx)
    assert [_fmt(x["l1"]) for x in r["rows"]] == ["7.6908e-06", "6.8082e-08"]
    assert _fmt(r["rows"][-1]["order_l1"]) == "6.8197e+00"
    ra = runner.run(configs.config("ex2"), roots=[10, 20], ctx=ctx)
    assert [_fmt(x["l1"]) for x in ra["rows"]] == ["1.6096e-06", "5.0811e-08"]
    assert _fmt(ra["rows"][-1]["order_l1"]) == "4.9854e+00"


def test_table4_fast_build(ctx_fast):
    r = runner.run(configs.config("ex3a"), roots=[10, 20], ctx=ctx_fast)
    want = [7.1354e-05, 2.7404e-07]
    assert all(abs(x["l1"] / w - 1.0) < 1e-4 for x, w in zip(r["rows"], want))


def test_series_outputs(ctx, tmp_path):
    """time-series path: stops, mass/min/max on the device, SGW5 snapshots and
    cut planes, run_meta; compare_runs of a run with itself is zero."""
    cfg = configs.config("C4", nl=3, root=[16, 16], tfinal=0.1)
    out = os.path.join(tmp_path, "a")
    r = runner.run(cfg, out_dir=out, stops=[0.0, 0.05], ctx=ctx)
    assert [round(x["t"], 6) for x in r["series"]] == [0.0, 0.05, 0.1]
    files = sorted(os.listdir(out))
    assert "timeseries.csv" in files and "run_meta.csv" in files
    snaps = [f for f in files if f.endswith(".sgw5")]
    assert snaps == ["snapshot_t0.000000.sgw5", "snapshot_t0.050000.sgw5",
                     "snapshot_t0.100000.sgw5"]
    assert "cut_xv_t0.100000.csv" in files
    ext, h, vals = sgwg.read_snapshot(os.path.join(out, snaps[-1]))
    # mass of the last snapshot equals the series row (trapezoid weights)
    w0 = np.full(ext[0], h[0])
    w1 = np.full(ext[1], h[1])
    w1[0] *= 0.5
    w1[-1] *= 0.5
    m = np.sum(np.multiply.outer(w0, w1).ravel() * vals)
    assert abs(m - r["series"][-1]["mass"]) <= 1e-13 * abs(m)
    with open(os.path.join(out, "timeseries.csv")) as fh:
        lines = fh.read().splitlines()
    assert lines[0] == "t,mass,min,max,h2,hlog" and len(lines) == 4
    cmp = runner.compare_runs(out, out)
    assert all(row["l1"] == 0.0 and row["linf"] == 0.0 for row in cmp["rows"])
    assert runner.compare_csv(cmp).startswith("snapshot,l1_diff,linf_diff\n")
