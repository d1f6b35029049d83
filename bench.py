#!/usr/bin/env python
"""Benchmark of the sparse-grid WENO5 hot path on B200 (BASELINE.json metric:
component-grid WENO5 point-updates/sec per RK stage; wall time to T; % of
roofline).

Default workload: BASELINE C5, the largest configuration that fits one GPU --
2D2V Vlasov-Poisson Landau damping, root 8, N_L = 5: 121 component grids,
12,057,728 points per RK stage, finest grid 256^2 x 257^2 = 4.33e9 points
(34.6 GB), CFL 0.5, T = 20 (9,855 SSP-RK3 steps).

One bench "step" = the reference's timed region (runner.hpp:318-330) once:
initial states -> evolve to T (every member, per-stage charge density and
Poisson field, CFL dt per step) -> at T the combination of all 121 members
onto the finest grid (WENO prolongation + signed sum, computed on the device
in dimension-0 row slabs and reduced to mass / min / max: every one of the
4.33e9 finest points is formed) plus the reference's two cut planes
(x1-v1 at x2 = v2 = 0, x1-x2 at v1 = v2 = 0, runner.hpp:187-196).

  value  point-updates (sum of member points x 3 stages x RK steps) / device
         time of the step (CUDA events on the library's stream), initial
         states resident in HBM (device-to-device reset inside the step), L2
         flushed between steps.
  e2e    the same through the public C ABI with HOST buffers: pinned H2D of
         the initial member states, D2H of the step's results (diagnostics +
         cut planes) inside the timed region.

Other configurations (--config C1..C4, S2, S3): one step = the whole run to T
with the full combination at every stop (finest grid to a device buffer;
D2H in e2e).

N>1 (torchrun): members sharded by LPT over ranks (strong scaling of the
fixed family), NCCL all-reduce(max) of the wave speeds per step and
all-reduce(sum) of the combination inside libsgwg; time = max over ranks.
--impl reference: the reference's own CPU implementation of the path on this
host -- the reference headers compiled in place (oracle/_ref) for C1-C3, the
oracle's C restatement (oracle/liboracle.so, all host threads) for the
Vlasov-Poisson configs the reference lacks -- rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOAD = "C5"
WORKLOADS = {
    "C1": "C1: 2D advection [0,2]^2 periodic, root 16, N_L=3 (7 grids, 11264 pts/stage), "
          "dt=0.5h^(5/3), T=1, WENO prolongation",
    "C2": "C2: 2D Burgers [0,2]^2 periodic, root 32x32, N_L=5, 11 component grids "
          "(278528 pts/stage), finest 1024^2, CFL 0.5, stops {0.1,0.5}, WENO5-JS+LF, SSP-RK3, "
          "WENO prolongation",
    "C3": "C3: 3D advection [0,2]^3 periodic, root 16, N_L=4 (31 grids, 1409024 pts/stage), "
          "finest 256^3, dt=h^(5/3), T=0.5",
    "C4": "C4: 1D1V Vlasov-Poisson Landau damping, root 32, N_L=5 (11 grids), CFL 0.5, T=40",
    "C5": "C5: 2D2V Vlasov-Poisson Landau damping [0,4pi]^2 x [-6,6]^2, root 8, N_L=5 (121 "
          "grids, 12057728 pts/stage), finest 256^2 x 257^2, CFL 0.5, T=20, WENO5-JS upwind, "
          "SSP-RK3, per-stage Poisson field, WENO prolongation + combination at T",
}
METRIC = "component-grid WENO5 point-updates/sec per RK stage"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--arith", default="fast", choices=["fast", "exact"])
    ap.add_argument("--config", default=WORKLOAD)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--tfinal", type=float, default=None,
                    help="override T (prefix runs of the long configs)")
    ap.add_argument("--no-combine", action="store_true",
                    help="skip the combination at the stops")
    ap.add_argument("--e2e-steps", type=int, default=None,
                    help="steps of the host-buffer (e2e) measurement (default: all for short "
                         "configs, min(steps, 3) for C5)")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def _levels(cfg):
    # enumerate_combination_levels (grid.hpp:57-79), pure python (no GPU needed)
    d, nl = cfg["d"], cfg["nl"]
    lo = max(0, nl - d + 1)
    out = []

    def rec(k, used, cur):
        if k == d - 1:
            for last in range(max(0, lo - used), nl - used + 1):
                if used + last >= lo:
                    out.append(cur + [last])
            return
        for l in range(0, nl - used + 1):
            rec(k + 1, used + l, cur + [l])

    rec(0, 0, [])
    return sorted(out)


def member_extents(cfg, lv):
    return [(cfg["root"][k] << lv[k]) + (1 if cfg["bc"][k] == 1 else 0) for k in range(cfg["d"])]


def family_pts_stage(cfg):
    tot = 0
    for lv in _levels(cfg):
        n = 1
        for e in member_extents(cfg, lv):
            n *= e
        tot += n
    return tot


def combine_flops(cfg):
    """Algorithmic flops of one full combination:
    prolong every member dimension by dimension (59 flops per interpolated
    fine point + 33 per source interval for the WENO smoothness indicators,
    copies free), then acc += c * p (2 flops) per finest point and member."""
    d, nl = cfg["d"], cfg["nl"]
    fine = [(cfg["root"][k] << nl) + (1 if cfg["bc"][k] == 1 else 0) for k in range(d)]
    nfine = 1
    for e in fine:
        nfine *= e
    tot = 0.0
    for lv in _levels(cfg):
        ext = member_extents(cfg, lv)
        for k in range(d):
            m = nl - lv[k]
            if m == 0:
                continue
            lines = 1
            for q in range(d):
                if q != k:
                    lines *= ext[q]
            n_dst = fine[k]
            interp = n_dst - (n_dst + (1 << m) - 1) // (1 << m)  # r != 0 points
            tot += lines * (59.0 * interp + 33.0 * ext[k])
            ext[k] = n_dst
        tot += 2.0 * nfine
    return tot, nfine


def cpu_info():
    model = ""
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return os.cpu_count() or 1, model


def _oracle_objs(O, cfg):
    dom = O.make_domain(cfg["d"], cfg["nl"], cfg["lower"], cfg["upper"], cfg["root"], cfg["bc"])
    m = O.make_model(cfg["kind"], cfg["weno_mode"], cfg["epsilon"], cfg["speeds"],
                     cfg["space_dim"], cfg["theta"], cfg["tau"])
    pol = O.make_policy(cfg["dt_mode"], cfg["cfl"], cfg["reference_spacing"], cfg["dt_scale"])
    return dom, m, pol


def _sample_steps(cfg, budget_pt_stages):
    return max(1, int(budget_pt_stages / (3 * family_pts_stage(cfg))))


# --------------------------------------------------------------------------
# reference arm
# --------------------------------------------------------------------------
def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    from oracle import oracle as O
    from paper_2007_10196_b200 import configs
    cfg = configs.config(args.config)
    ncores, model = cpu_info()
    pts = family_pts_stage(cfg)
    dom, m, pol = _oracle_objs(O, cfg)
    vp = cfg["kind"] == configs.VLASOV_POISSON
    if vp or not O.ref_available():
        # no Vlasov-Poisson in the reference: its C restatement
        # (vb_rhs_into transport + the Poisson field), members on all threads
        orc = O.Oracle().set_threads(ncores)
        s0 = orc.init_family(cfg["ic"], dom)
        nsteps = 2 if cfg["d"] == 4 else _sample_steps(cfg, 2e7 * ncores)

        def sample():  # the first nsteps RK steps of the run
            orc.set_max_steps(nsteps)
            t0 = time.perf_counter()
            _, dts, st, _ = orc.evolve(dom, m, pol, s0, cfg["tfinal"])
            secs = time.perf_counter() - t0
            orc.set_max_steps(0)
            return secs, len(dts)

        kind = "port"
        desc = (f"C restatement of the reference path (oracle/liboracle.so, evolve_family over the "
                f"packed family, members on {ncores} OpenMP threads)")
    else:
        ref = O.Reference()
        nsteps = _sample_steps(cfg, 2e7 * 2)
        probe = O.Oracle().set_max_steps(nsteps)
        _, dts, _, _ = probe.evolve(dom, m, pol, probe.init_family(cfg["ic"], dom), cfg["tfinal"])
        probe.set_max_steps(0)
        t_sample = float(sum(dts)) * (1 - 1e-12)

        def sample():
            s, n, _ = ref.time_prefix(dom, m, pol, cfg["ic"], t_sample, ncores, cfg["interp"])
            return s, n

        kind = "reference"
        desc = (f"the reference headers (oracle/_ref/libsgwref.so): make_family, initialize_family, "
                f"evolve_family with threads={ncores}")
    for _ in range(args.warmup):
        sample()
    secs, steps = [], 0
    for _ in range(args.steps):
        s, n = sample()
        secs.append(s)
        steps = n
    tot = sum(secs)
    value = pts * 3 * steps * len(secs) / tot
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "pt-stage/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * tot / len(secs), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (analytic initial condition)",
        "config": {"workload": WORKLOADS.get(args.config, args.config),
                   "sample": f"each step: the first {steps} RK steps of the run (evolve only; the "
                             f"combination is not timed on the CPU)"},
        "cpu_baseline": {"value": value, "unit": "pt-stage/s", "cores": ncores, "kind": kind,
                         "sample": f"{desc}; {steps} RK steps of the {args.config} family per "
                                   f"step, cpu={model}"},
        "e2e": {"value": value, "unit": "pt-stage/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


# --------------------------------------------------------------------------
# clocks during the timed region
# --------------------------------------------------------------------------
class Clocks:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.p = None

    def __enter__(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "100"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except OSError:
            self.p = None
        time.sleep(0.15)
        return self

    def __exit__(self, *a):
        if self.p is not None:
            self.p.terminate()
            try:
                self.p.wait(2)
            except subprocess.TimeoutExpired:
                self.p.kill()

    def summary(self):
        try:
            rows = [r.split(",") for r in open(self.f.name).read().strip().splitlines() if r]
        except OSError:
            rows = []
        sm, mx, reasons = [], 0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            try:
                sm.append(float(r[1]))
                mx = max(mx, float(r[2]))
                for nm, v in zip(names, r[5:9]):
                    if v.strip().lower() == "active":
                        reasons.add(nm)
            except (ValueError, IndexError):
                continue
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


# --------------------------------------------------------------------------
# B200 arm
# --------------------------------------------------------------------------
def run_b200(args):
    import numpy as np
    import torch

    from paper_2007_10196_b200 import configs, runner, sgwg, shard

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg = configs.config(args.config)
    if args.tfinal is not None:
        cfg["tfinal"] = args.tfinal
        cfg["stops"] = [s for s in cfg["stops"] if s < args.tfinal]
    levels = _levels(cfg)
    pts_all = shard.member_points(levels, cfg["root"], cfg["bc"])
    total_pts = sum(pts_all)
    shards = shard.lpt_shards(pts_all, world)
    mine = shards[rank]

    ctx = sgwg.Context(local, arith=args.arith)
    fam = sgwg.Family.from_config(ctx, cfg, members=mine if world > 1 else None)
    if world > 1:
        import torch.distributed as dist
        uid = sgwg.nccl_unique_id() if rank == 0 else bytes(128)
        obj = [uid]
        dist.broadcast_object_list(obj, src=0)
        fam.set_comm(obj[0], world, rank)
    fam.initialize(cfg["ic"])  # initialize_family on the host, uploaded once
    init_host = fam.download()
    pinned_init = torch.from_numpy(init_host).pin_memory()
    n_local = fam.total_points
    dev_init = torch.empty(n_local, dtype=torch.float64, device=f"cuda:{local}")
    fam.download_device(dev_init.data_ptr(), n_local)
    # output at the stops: the full combined field (device buffer; D2H in e2e),
    # or -- when the finest grid is too large to keep (C5: 34.6 GB) -- the
    # combination reduced on the device slab by slab (mass / min / max) plus
    # the reference's cut planes
    big = fam.finest_points * 8 > 8e9
    output = "none" if args.no_combine else ("stats+cuts" if big else "combine")
    cuts = runner.cut_planes(cfg, fam) if output == "stats+cuts" else []
    combined = pinned_out = None
    if output == "combine":
        combined = torch.empty(fam.finest_points, dtype=torch.float64, device=f"cuda:{local}")
        pinned_out = torch.empty(fam.finest_points, dtype=torch.float64).pin_memory()
    pinned_states = torch.empty(n_local, dtype=torch.float64).pin_memory() \
        if output == "none" else None
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=f"cuda:{local}")  # 256 MB > L2
    stream = torch.cuda.ExternalStream(ctx.stream, device=f"cuda:{local}")

    box = {"d2h": 0}

    def one_sim(host_io=False):
        """one bench step: reset states, evolve to T with the output at every stop."""
        outs = []
        d2h = 0
        if host_io:
            fam.upload(pinned_init.numpy())  # pinned H2D through the public API
        else:
            fam.upload_device(dev_init.data_ptr(), n_local)

        def on_stop(t):
            nonlocal d2h
            if output == "stats+cuts":
                st = fam.combined_stats(cfg["interp"], cfg["epsilon"])
                planes = [fam.cut_plane(da, db, fx, cfg["interp"], cfg["epsilon"])
                          for _, da, db, fx in cuts]
                outs.append((st, planes))
                d2h += 5 * 8 + sum(p.size * 8 for p in planes)
            elif host_io:  # D2H of the combined field into pinned host memory
                outs.append(fam.combine(cfg["interp"], cfg["epsilon"], out=pinned_out.numpy()))
                d2h += fam.finest_points * 8
            else:
                fam.combine(cfg["interp"], cfg["epsilon"], out_device_ptr=combined.data_ptr())

        dts = fam.evolve_config(cfg, on_stop=None if output == "none" else on_stop)
        box["n"] = len(dts)
        box["dts"] = dts
        if host_io and output == "none":  # the result is the member states
            fam.download_into(pinned_states.numpy())
            d2h += n_local * 8
        box["d2h"] = d2h
        return outs

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x):
        if world == 1:
            return x
        import torch.distributed as dist
        t = torch.tensor([x], dtype=torch.float64, device=f"cuda:{local}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    warmup = max(3, args.warmup)
    for _ in range(warmup):
        one_sim()
    # ---- device-timed region (value) ----
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * args.steps)]
    barrier()
    with Clocks(local) as clk:
        for i in range(args.steps):
            flush.zero_()
            torch.cuda.synchronize()
            ev[2 * i].record(stream)
            one_sim()
            ev[2 * i + 1].record(stream)
        barrier()
    step_ms = [ev[2 * i].elapsed_time(ev[2 * i + 1]) for i in range(args.steps)]
    ms_total = max_over_ranks(sum(step_ms))
    nsteps = box["n"]
    pu = total_pts * 3 * nsteps  # point-updates of the whole family per simulation
    value = pu * args.steps / (ms_total * 1e-3)
    st = fam.stats()
    evolve_ms = max_over_ranks(st["evolve_ms"])
    combine_ms = max_over_ranks(st["combine_ms"])
    launches = int(st["kernel_launches"] + st["combine_launches"]) + len(cuts)

    # ---- end to end through the public API with host buffers (e2e) ----
    e2e_steps = args.e2e_steps or (min(args.steps, 3) if big else args.steps)
    one_sim(host_io=True)  # untimed warm-up of the host-buffer path
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record(stream)
    for _ in range(e2e_steps):
        one_sim(host_io=True)
    e1.record(stream)
    barrier()
    wall_e2e = time.perf_counter() - t0
    e2e_ms = max_over_ranks(max(e0.elapsed_time(e1), wall_e2e * 1e3))
    e2e_value = pu * e2e_steps / (e2e_ms * 1e-3)
    h2d = n_local * 8

    # ---- roofline of the dominant stage kernel: event times of every stage
    # launch inside a short evolve in profile mode (no graphs), algorithmic
    # flops per launch from the library (SURVEY 8(a)/(d) counting) ----
    peak = ctx.fp64_peak_tflops()
    stage_kernels = fam.stage_kernels
    pctx = sgwg.Context(local, arith=args.arith, profile=True)
    pfam = sgwg.Family.from_config(pctx, cfg, members=mine if world > 1 else None)
    pfam.upload_device(dev_init.data_ptr(), n_local)
    pT = sum(box["dts"][:min(len(box["dts"]), 12)]) * (1 - 1e-12)
    pfam.evolve_config(cfg, tfinal=pT, stops=[])
    kprof = pfam.kernel_profile()
    pfam.close()
    pctx.close()
    kernels = []
    for k in kprof:
        avg = k["ms_sum"] / max(1, k["launches"])
        kernels.append({"kernel": k["name"], "launches": k["launches"], "avg_launch_us": avg * 1e3,
                        "flops_per_launch": k["flops_per_launch"],
                        "achieved_tflops": k["flops_per_launch"] / (avg * 1e-3) / 1e12,
                        "bytes_per_launch": k["bytes_per_launch"],
                        "achieved_gbs": k["bytes_per_launch"] / (avg * 1e-3) / 1e9,
                        "share_ms": k["ms_sum"]})
    per_pt_step = 3 * (142.0 if cfg["kind"] == 1 else 70.0) * cfg["d"] + 2 + 5 + 5
    evolve_flops = total_pts * per_pt_step * nsteps
    # the persistent cooperative kernel ran iff the evolve needed fewer launches than RK
    # steps (families that are not co-resident -- S2 -- fall back to one launch per stage)
    persistent = (args.arith == "fast" and cfg["d"] == 2 and cfg["kind"] in (0, 1)
                  and world == 1 and not os.environ.get("SGWG_NO_PERSIST")
                  and st["kernel_launches"] < nsteps)
    if kernels:
        dom_k = max(kernels, key=lambda k: k["share_ms"])
        achieved = dom_k["achieved_tflops"]
        kname = dom_k["kernel"]
        avg_us, fpl, bpl = dom_k["avg_launch_us"], dom_k["flops_per_launch"], dom_k["bytes_per_launch"]
        per_launch = (f"{kname}: algorithmic flops per launch = {fpl / total_pts:.0f} per point x "
                      f"{total_pts} points (SURVEY 8(a)/(d): 70 per point and direction, + RK "
                      "stage / accumulate / charge density), / its average event time over "
                      "every launch of a profile-mode evolve")
    elif persistent and evolve_ms:
        achieved = evolve_flops / (evolve_ms * 1e-3) / 1e12
        kname, avg_us = "evolve2d_persistent_kernel", evolve_ms * 1e3
        fpl, bpl = evolve_flops, total_pts * (16 + 24 + 24) * nsteps
        per_launch = (f"algorithmic flops of the whole evolve: {total_pts} pts x "
                      f"{per_pt_step:.0f} flops/pt-step x {nsteps} steps, time = evolve device time")
    else:
        fam.upload_device(dev_init.data_ptr(), n_local)
        avg_ms, fpl, bpl = fam.time_stage(reps=50)
        achieved = fpl / (avg_ms * 1e-3) / 1e12
        kname, avg_us = stage_kernels, avg_ms * 1e3
        per_launch = "algorithmic flops of RK stage 1 divided by the stage's launches"
    stage_ms = sum(k["avg_launch_us"] for k in kernels) * 1e-3 if kernels else None
    stage_tf = (sum(k["flops_per_launch"] for k in kernels) / (stage_ms * 1e-3) / 1e12
                if kernels else None)
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        try:
            traffic = json.load(open(tpath)).get(args.config, {}).get(args.arith)
        except (OSError, ValueError):
            traffic = None
    hbm_peak = None
    ppath = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(ppath):
        hbm_peak = json.load(open(ppath)).get("hbm_gbs")
    cflops, nfine = combine_flops(cfg)

    # ---- CPU baseline: the same path on this host, bounded sample (rank 0, N=1) ----
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(cfg, box.get("dts"))

    if rank == 0:
        clocks = clk.summary()
        line = {
            "metric": METRIC,
            "value": value, "unit": "pt-stage/s", "n_gpus": world, "steps": args.steps,
            "warmup": warmup, "ms_per_step": ms_total / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": f"synthetic (analytic initial condition of BASELINE {args.config}, no dataset)",
            "config": {"workload": WORKLOADS.get(args.config, args.config),
                       "members": len(levels), "pts_per_stage": total_pts,
                       "step": f"one full simulation to T={cfg['tfinal']} "
                               + ("(no output)" if output == "none" else
                                  f"with {output} at t={cfg['stops'] + [cfg['tfinal']]}"),
                       "rk_steps_per_sim": nsteps, "arith": args.arith,
                       "l2": "flushed (256 MB write) between timed steps",
                       "parallelism": f"members sharded over {world} GPU(s) (LPT)",
                       "members_per_rank": [len(s) for s in shards]},
            "wall_time_to_T_ms": ms_total / args.steps,
            "evolve_ms_per_sim": evolve_ms,
            "evolve_only_value": pu / (evolve_ms * 1e-3) if evolve_ms else None,
            "evolve_roofline_frac": (evolve_flops / (evolve_ms * 1e-3) / 1e12 / peak
                                     if evolve_ms and peak else None),
            "combine": {"ms": combine_ms, "finest_points": nfine,
                        "finest_points_per_s": nfine / (combine_ms * 1e-3) if combine_ms else None,
                        "algorithmic_tflops": cflops / (combine_ms * 1e-3) / 1e12
                        if combine_ms else None,
                        "frac_fp64_peak": cflops / (combine_ms * 1e-3) / 1e12 / peak
                        if combine_ms and peak else None,
                        "flops": cflops, "output": output},
            "e2e": {"value": e2e_value, "unit": "pt-stage/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": box["d2h"], "ms_per_step": e2e_ms / e2e_steps,
                    "steps": e2e_steps},
            "gpu_launches": launches * args.steps,
            "roofline": {"bound": "fp64", "achieved": achieved, "peak": peak,
                         "unit": "TFLOP/s", "frac": achieved / peak if peak else None,
                         "traffic": traffic, "kernel": kname, "stage_kernels": stage_kernels,
                         "per_launch": per_launch, "avg_launch_us": avg_us,
                         "flops_per_launch": fpl,
                         "stage": ({"ms": stage_ms, "achieved_tflops": stage_tf,
                                    "frac": stage_tf / peak if peak else None}
                                   if kernels else None),
                         "kernels": kernels,
                         "peak_source": "measured live: DFMA microbenchmark (sgwg_fp64_peak)",
                         "hbm": {"achieved_gbs": bpl / (avg_us * 1e-6) / 1e9,
                                 "peak_gbs": hbm_peak,
                                 "peak_source": "MEASURED_PEAKS.json hbm_gbs"}},
            "clocks": clocks,
        }
        if cpu is not None:
            line["cpu_baseline"] = cpu
        print(json.dumps(line))
    fam.close()
    ctx.close()
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()
    return 0


def cpu_baseline(cfg, dts=None):
    """The same path on this host, bounded sample (~10-30 s of one core): the
    first RK steps of the run -- the reference itself where it has the model,
    its C restatement (the oracle port) for Vlasov-Poisson."""
    from oracle import oracle as O
    ncores, model = cpu_info()
    dom, m, pol = _oracle_objs(O, cfg)
    pts = family_pts_stage(cfg)
    vp = cfg["kind"] == 3
    nsteps = 3 if vp else _sample_steps(cfg, 1.0e8)
    if O.ref_available() and not vp:
        if dts is not None and len(dts) > 0:
            t_sample = float(sum(dts[:nsteps])) * (1 - 1e-9)
        else:
            t_sample = 0.02
        ref = O.Reference()
        secs, n, _ = ref.time_prefix(dom, m, pol, cfg["ic"], t_sample, 1, cfg["interp"])
        kind, desc = "reference", "reference headers (oracle/_ref/libsgwref.so), threads=1"
    else:
        orc = O.Oracle().set_threads(1).set_max_steps(nsteps)
        s0 = orc.init_family(cfg["ic"], dom)
        t0 = time.perf_counter()
        _, dts2, _, _ = orc.evolve(dom, m, pol, s0, cfg["tfinal"])
        secs, n = time.perf_counter() - t0, len(dts2)
        orc.set_max_steps(0)
        kind, desc = "port", "C restatement (oracle/liboracle.so), 1 thread"
    return {"value": pts * 3 * n / secs, "unit": "pt-stage/s", "cores": 1, "kind": kind,
            "sample": f"{desc}: evolve_family of the {cfg['name']} family, the first {n} RK "
                      f"steps of the run ({secs:.1f} s) on {model} ({ncores} host cores)"}


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_b200(args)


if __name__ == "__main__":
    sys.exit(main())
