"""Experiment runner on the B200 path: run() of the reference's runner
(/root/reference/proj/include/sgweno/runner.hpp:270-416) over the C ABI.

Refinement study (table path, runner.hpp:330-349): for each root size, build
the family (sparse, make_family; or single, make_single_grid runner.hpp:106-115),
initialise, evolve to T with dt from the finest spacing, and compute the error
norms of the combined field against the exact solution on the device
(sgwg_combined_stats) -- L1 grid-point average and max (error_norms,
diag.hpp:30-43) with observed orders log2(e_prev / e).  Time-series path
(runner.hpp:350-366): at every stop, mass / min / max of the combined field on
the device, the SGW5 snapshot and the example's cut planes (write_cuts,
runner.hpp:159-200) when an output directory is given.  The files written
(errors.csv, timeseries.csv, run_meta.csv, snapshot_t*.sgw5, cut_*.csv) use the
reference's pinned formats.
"""
from __future__ import annotations

import os
import time
from typing import Optional, Sequence

import numpy as np

from . import configs, sgwg

# exact solutions known to the device diagnostics (sgwg_combined_stats)
_EXACT = {configs.IC_C1, configs.IC_C3, configs.IC_EX1, configs.IC_EX2, configs.IC_EX3}


def has_error_table(cfg) -> bool:
    """has_error_table (runner.hpp:87-91): smooth examples with an exact solution."""
    return cfg["ic"] in _EXACT or (cfg["ic"] == configs.IC_C2 and cfg["d"] == 2
                                   and cfg["tfinal"] < 1.0 / (2.0 * np.pi))


def emit_table(rows) -> str:
    """CSV convergence table, pinned format (runner.hpp:228-247)."""
    out = "grid,l1,l1_order,linf,linf_order,wall_seconds\n"
    for r in rows:
        o1 = "" if r.get("order_l1") is None else "%.3f" % r["order_l1"]
        o2 = "" if r.get("order_linf") is None else "%.3f" % r["order_linf"]
        out += "%d,%.4e,%s,%.4e,%s,%.5e\n" % (r["grid"], r["l1"], o1, r["linf"], o2,
                                               r["wall_seconds"])
    return out


def emit_series(rows) -> str:
    """timeseries.csv (runner.hpp:380-396); h2/hlog columns empty (no M state)."""
    out = "t,mass,min,max,h2,hlog\n"
    for r in rows:
        out += "%.6f,%.10e,%.10e,%.10e,,\n" % (r["t"], r["mass"], r["min"], r["max"])
    return out


def _coord(cfg, fam, k, i):
    h = (cfg["upper"][k] - cfg["lower"][k]) / (cfg["root"][k] << cfg["nl"])
    return cfg["lower"][k] + i * h  # grid_point_coordinate_1d


def _nearest(cfg, fam, k, x):
    h = (cfg["upper"][k] - cfg["lower"][k]) / (cfg["root"][k] << cfg["nl"])
    return int(np.clip(np.rint((x - cfg["lower"][k]) / h), 0, fam.fine_extents[k] - 1))


def cut_planes(cfg, fam):
    """The example's standard cut planes (write_cuts, runner.hpp:159-200):
    2D: the whole x-v plane; 3D: the y-z plane at x index 0; 4D (ex5b / C5):
    x1-v1 at x2 = v2 = 0 and x1-x2 at v1 = v2 = 0 (nearest indices)."""
    d = cfg["d"]
    if d == 2:
        return [("cut_xv", 0, 1, [0, 0])]
    if d == 3:
        return [("cut_yz_x0", 1, 2, [0, 0, 0])]
    if d == 4:
        f1 = [0, _nearest(cfg, fam, 1, 0.0), 0, _nearest(cfg, fam, 3, 0.0)]
        f2 = [0, 0, _nearest(cfg, fam, 2, 0.0), _nearest(cfg, fam, 3, 0.0)]
        return [("cut_x1v1", 0, 2, f1), ("cut_x1x2", 0, 1, f2)]
    return []


def write_plane_csv(path, cfg, fam, da, db, plane):
    """write_plane_csv (runner.hpp:126-141): c1,c2,value with %.10e"""
    with open(path, "w") as fh:
        fh.write("c1,c2,value\n")
        for ia in range(plane.shape[0]):
            ca = _coord(cfg, fam, da, ia)
            for ib in range(plane.shape[1]):
                fh.write("%.10e,%.10e,%.10e\n" % (ca, _coord(cfg, fam, db, ib), plane[ia, ib]))


def run(cfg: dict, roots: Optional[Sequence[int]] = None, grid_mode: str = "sparse",
        out_dir: Optional[str] = None, stops: Optional[Sequence[float]] = None,
        ctx: Optional[sgwg.Context] = None, arith: str = "exact") -> dict:
    """run(cfg) of runner.hpp:270-416 on the GPU path; returns
    {"rows": [...], "series": [...], "wall_seconds": s, "finest_nh": n}."""
    own = ctx is None
    if own:
        ctx = sgwg.Context(0, arith=arith)
    d = cfg["d"]
    roots = list(roots) if roots else [cfg["root"][0]]
    if any(nr < 6 for nr in roots):
        raise ValueError("invalid config (nr): root grid must have at least 6 cells per direction")
    if grid_mode == "sparse" and cfg["nl"] < d - 1:
        raise ValueError("invalid config (nl): sparse mode needs N_L >= d-1")
    table = has_error_table(cfg)
    if not table and len(roots) > 1:
        raise ValueError("invalid config (nr): refinement lists apply to the smooth examples only")
    stops = list(cfg["stops"] if stops is None else stops)
    if out_dir:
        os.makedirs(out_dir, exist_ok=True)
    result = {"rows": [], "series": [], "wall_seconds": 0.0, "finest_nh": 0}
    try:
        for nr in roots:
            c = dict(cfg, root=[nr] * d)
            c["reference_spacing"] = min((c["upper"][k] - c["lower"][k]) / nr / (1 << c["nl"])
                                         for k in range(d))
            fam = sgwg.Family.from_config(ctx, c, single=(grid_mode == "single"))
            try:
                _run_one(fam, c, nr, table, stops, out_dir, result)
            finally:
                fam.close()  # before ctx.close(): the family's stream lives in the context
    finally:
        if own:
            ctx.close()
    if out_dir:
        with open(os.path.join(out_dir, "errors.csv" if table else "timeseries.csv"), "w") as fh:
            fh.write(emit_table(result["rows"]) if table else emit_series(result["series"]))
        with open(os.path.join(out_dir, "run_meta.csv"), "w") as fh:
            fh.write("key,value\n")
            fh.write(f"example,{cfg.get('name', '?')}\n")
            fh.write(f"grid_mode,{grid_mode}\n")
            fh.write(f"nr,{roots[-1]}\n")
            fh.write(f"nl,{cfg['nl']}\n")
            fh.write(f"nh,{result['finest_nh']}\n")
            fh.write("tfinal,%.10e\n" % cfg["tfinal"])
            fh.write("scheme,%s\n" % ("linear" if cfg["weno_mode"] == configs.LINEAR else "weno"))
            fh.write("prolongation,%s\n" % ("lagrange" if cfg["interp"] == configs.LAGRANGE
                                            else "weno"))
            fh.write("wall_seconds,%.5e\n" % result["wall_seconds"])
    return result


def _run_one(fam, c, nr, table, stops, out_dir, result):
    """One root of run()'s refinement loop (runner.hpp:293-365) on an open family."""
    fam.initialize(c["ic"])
    result["finest_nh"] = nr << c["nl"]
    series = []

    def record(t, fam=fam, c=c, series=series):
        st = fam.combined_stats(c["interp"], c["epsilon"])
        series.append({"t": t, "mass": st["mass"], "min": st["min"], "max": st["max"]})
        if out_dir:
            tag = "%.6f" % t
            fam.write_snapshot(os.path.join(out_dir, f"snapshot_t{tag}.sgw5"),
                               c["interp"], c["epsilon"])
            for name, da, db, fixed in cut_planes(c, fam):
                plane = fam.cut_plane(da, db, fixed, c["interp"], c["epsilon"])
                write_plane_csv(os.path.join(out_dir, f"{name}_t{tag}.csv"), c, fam,
                                da, db, plane)

    if not table and (0.0 in stops or c["tfinal"] == 0.0):
        record(0.0)
    t0 = time.perf_counter()
    if c["tfinal"] > 0.0:
        fam.evolve_config(c, tfinal=c["tfinal"], stops=[] if table else stops,
                          on_stop=None if table else record)
    if table:
        st = fam.combined_stats(c["interp"], c["epsilon"], exact_preset=c["ic"],
                                t=c["tfinal"])
    t1 = time.perf_counter()
    result["wall_seconds"] = t1 - t0
    if table:
        row = {"grid": nr << c["nl"], "l1": st["l1"], "linf": st["linf"],
               "wall_seconds": t1 - t0, "order_l1": None, "order_linf": None}
        if result["rows"]:
            prev = result["rows"][-1]
            row["order_l1"] = float(np.log2(prev["l1"] / row["l1"]))
            row["order_linf"] = float(np.log2(prev["linf"] / row["linf"]))
        result["rows"].append(row)
    else:
        result["series"] = series


def compare_runs(dir_a: str, dir_b: str) -> dict:
    """compare_runs (runner.hpp:420-470): L1 / max differences of the common
    snapshots of two runs and their wall-time ratio."""
    def meta(d):
        kv = {}
        with open(os.path.join(d, "run_meta.csv")) as fh:
            next(fh)
            for line in fh:
                k, _, v = line.rstrip("\n").partition(",")
                kv[k] = v
        return kv
    ma, mb = meta(dir_a), meta(dir_b)
    if ma["example"] != mb["example"] or ma["nh"] != mb["nh"]:
        raise RuntimeError("compare: incompatible runs (example or finest grid differ)")
    names = sorted(n for n in os.listdir(dir_a) if n.startswith("snapshot_t")
                   and n.endswith(".sgw5") and os.path.exists(os.path.join(dir_b, n)))
    if not names:
        raise RuntimeError("compare: no common snapshots")
    rows = []
    for n in names:
        ea, _, a = sgwg.read_snapshot(os.path.join(dir_a, n))
        eb, _, b = sgwg.read_snapshot(os.path.join(dir_b, n))
        if ea != eb:
            raise RuntimeError("compare: snapshot extents differ")
        e = np.abs(a - b)
        rows.append({"name": n, "l1": float(e.mean()), "linf": float(e.max())})
    return {"rows": rows,
            "wall_ratio": float(ma["wall_seconds"]) / float(mb["wall_seconds"])}


def compare_csv(r: dict) -> str:
    out = "snapshot,l1_diff,linf_diff\n"
    for row in r["rows"]:
        out += "%s,%.4e,%.4e\n" % (row["name"], row["l1"], row["linf"])
    out += "wall_ratio,%.5e,\n" % r["wall_ratio"]
    return out
