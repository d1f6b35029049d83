#!/usr/bin/env python
"""Benchmark of the sparse-grid WENO5 hot path on B200 (BASELINE.json metric).

Workload (BASELINE configs[1], C2): 2D Burgers on [0,2]^2 periodic,
u0 = 0.5 + sin(pi(x+y)), sparse-grid family root 32x32, N_L = 5 (11 component
grids, 278,528 points per RK stage, finest grid 1024^2), WENO5-JS + LF
splitting, SSP-RK3, CFL 0.5 with the family max|u|, stops {0.1, 0.5}, WENO
interpolation prolongation + signed combination at both stops.

One bench "step" = one complete simulation to T = 0.5 (evolve through both
stops, combining at each), i.e. the whole hot path once.  metric = component-
grid WENO5 point-updates per second per RK stage (sum of member points x 3
stages x RK steps / time), plus wall time to T and % of roofline.

  value  device-timed (CUDA events on the library's stream), initial states
         already resident in HBM (device-to-device reset inside the step), L2
         flushed between steps.
  e2e    the same through the public C ABI with HOST buffers: pinned H2D of
         the initial member states and D2H of both combined fields per step.

N>1 (torchrun): members sharded by LPT over ranks (strong scaling of the
fixed family), per-step all-reduce(max) of the family wave speed and
all-reduce(sum) of the combination inside libsgwg (NCCL), time = max over
ranks.  --impl reference times the reference's own CPU implementation
(oracle/_ref/libsgwref.so: the unmodified reference headers) on the same
config, rank 0 only.
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

WORKLOAD = "C2"
WORKLOADS = {
    "C1": "C1: 2D advection [0,2]^2 periodic, root 16, N_L=3 (7 grids, 11264 pts/stage), "
          "dt=0.5h^(5/3), T=1, WENO prolongation",
    "C2": "C2: 2D Burgers [0,2]^2 periodic, root 32x32, N_L=5, 11 component grids "
          "(278528 pts/stage), finest 1024^2, CFL 0.5, stops {0.1,0.5}, WENO5-JS+LF, SSP-RK3, "
          "WENO prolongation",
    "C3": "C3: 3D advection [0,2]^3 periodic, root 16, N_L=4 (31 grids, 1409024 pts/stage), "
          "finest 256^3, dt=h^(5/3), T=0.5",
    "C4": "C4: 1D1V Vlasov-Poisson Landau damping, root 32, N_L=5 (11 grids), CFL 0.5, T=40",
    "C5": "C5: 2D2V Vlasov-Poisson Landau damping, root 8, N_L=5 (121 grids, 12057728 "
          "pts/stage), CFL 0.5",
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--arith", default="fast", choices=["fast", "exact"])
    ap.add_argument("--config", default=WORKLOAD)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--tfinal", type=float, default=None,
                    help="override T (prefix runs of the long configs, e.g. C5)")
    ap.add_argument("--no-combine", action="store_true",
                    help="skip the combination at the stops (C5's finest grid is 34.6 GB)")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def family_pts_stage(cfg):
    from paper_2007_10196_b200 import shard
    from oracle import oracle as O  # noqa: F401  (levels only)
    import numpy as np  # noqa: F401
    lv = _levels(cfg)
    return sum(shard.member_points(lv, cfg["root"], cfg["bc"]))


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


def kernel_name(cfg, arith):
    phys = {0: "Advect", 1: "Burgers", 3: "VlasovPoisson"}.get(cfg["kind"], "?")
    if cfg["d"] == 2:
        k = "stage2d_fast_kernel" if arith == "fast" else "stage2d_kernel"
        return f"{k}<{phys}> (both WENO5 sweeps + RK3 stage, all members, 1 launch)"
    if arith == "fast" and cfg["d"] == 3 and cfg["kind"] == 0:
        return ("stage3d_pipe_kernel<Advect> (persistent, cp.async-pipelined; all three WENO5 "
                "sweeps + RK3 stage of all members, 1 launch)")
    if arith == "fast" and cfg["d"] == 4 and cfg["kind"] in (0, 3):
        return (f"plane_fast_kernel<{phys}> (fast; 2 launches per stage: dims (0,1) -> K, "
                "dims (2,3) + RK3 stage + charge-density partials)")
    return (f"pass_kernel<{phys}> ({arith}; one WENO5 direction of all members per launch, "
            "RK3 stage fused into the last direction)")


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
    if not O.ref_available():
        print(json.dumps({"impl": "reference",
                          "unavailable": "oracle/_ref/libsgwref.so not built (needs /root/reference "
                                         "at build time)"}))
        return 0
    ref = O.Reference()
    dom = O.make_domain(cfg["d"], cfg["nl"], cfg["lower"], cfg["upper"], cfg["root"], cfg["bc"])
    m = O.make_model(cfg["kind"], cfg["weno_mode"], cfg["epsilon"], cfg["speeds"],
                     cfg["space_dim"], cfg["theta"], cfg["tau"])
    pol = O.make_policy(cfg["dt_mode"], cfg["cfl"], cfg["reference_spacing"], cfg["dt_scale"])
    pts = family_pts_stage(cfg)
    t_sample = 0.01  # bounded sample: the first ~31 RK steps of the C2 run
    threads = ncores
    for _ in range(args.warmup):
        ref.time_prefix(dom, m, pol, cfg["ic"], t_sample, threads, cfg["interp"])
    secs, steps = [], 0
    for _ in range(args.steps):
        s, n, _c = ref.time_prefix(dom, m, pol, cfg["ic"], t_sample, threads, cfg["interp"])
        secs.append(s)
        steps = n
    tot = sum(secs)
    value = pts * 3 * steps * len(secs) / tot
    line = {
        "impl": "reference", "metric": "component-grid WENO5 point-updates/sec per RK stage",
        "value": value, "unit": "pt-stage/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * tot / len(secs), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{args.config}: 2D Burgers root 32 N_L=5 (11 grids, 278528 pts/stage)",
                   "sample": f"evolve prefix to t={t_sample} ({steps} RK steps) per step"},
        "cpu_baseline": {"value": value, "unit": "pt-stage/s", "cores": threads,
                         "kind": "reference",
                         "sample": f"reference headers (oracle/_ref), evolve_family to t={t_sample}, "
                                   f"threads={threads}, cpu={model}"},
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

    from paper_2007_10196_b200 import configs, sgwg, shard

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
    if args.no_combine:
        combined = pinned_out = None
        pinned_states = torch.empty(n_local, dtype=torch.float64).pin_memory()
    else:
        combined = torch.empty(fam.finest_points, dtype=torch.float64, device=f"cuda:{local}")
        pinned_out = torch.empty(fam.finest_points, dtype=torch.float64).pin_memory()
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=f"cuda:{local}")  # 256 MB > L2
    stream = torch.cuda.ExternalStream(ctx.stream, device=f"cuda:{local}")

    nsteps_box = {}

    def one_sim(host_io=False):
        """one bench step: reset states, evolve to T with a combine at each stop."""
        outs = []
        if host_io:
            fam.upload(pinned_init.numpy())  # pinned H2D through the public API
        else:
            fam.upload_device(dev_init.data_ptr(), n_local)

        def on_stop(t):
            if host_io:  # D2H of the combined field into pinned host memory
                outs.append(fam.combine(cfg["interp"], cfg["epsilon"], out=pinned_out.numpy()))
            else:
                fam.combine(cfg["interp"], cfg["epsilon"], out_device_ptr=combined.data_ptr())

        dts = fam.evolve_config(cfg, on_stop=None if args.no_combine else on_stop)
        nsteps_box["n"] = len(dts)
        nsteps_box["dts"] = dts
        if host_io and args.no_combine:  # the result is the member states
            fam.download_into(pinned_states.numpy())
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

    for _ in range(max(3, args.warmup)):
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
    ms_local = sum(step_ms)
    ms_total = max_over_ranks(ms_local)
    nsteps = nsteps_box["n"]
    pu = total_pts * 3 * nsteps  # point-updates of the whole family per simulation
    value = pu * args.steps / (ms_total * 1e-3)
    st = fam.stats()
    evolve_ms = max_over_ranks(st["evolve_ms"])
    combine_ms = max_over_ranks(st["combine_ms"])

    # ---- end to end through the public API with host buffers (e2e) ----
    one_sim(host_io=True)  # untimed warm-up of the host-buffer path
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record(stream)
    for i in range(args.steps):
        outs = one_sim(host_io=True)
    e1.record(stream)
    barrier()
    wall_e2e = time.perf_counter() - t0
    e2e_ms = max_over_ranks(max(e0.elapsed_time(e1), wall_e2e * 1e3))
    e2e_value = pu * args.steps / (e2e_ms * 1e-3)
    h2d = n_local * 8
    n_out = 1 + len(cfg["stops"])
    d2h = n_local * 8 if args.no_combine else n_out * fam.finest_points * 8

    # ---- roofline of the dominant kernel: the fused WENO5 + RK3 stage kernel,
    # launched back to back between CUDA events on the library's stream ----
    fam.upload_device(dev_init.data_ptr(), n_local)
    avg_ms, flops_per_launch, bytes_per_launch = fam.time_stage(reps=200)
    peak = ctx.fp64_peak_tflops()
    achieved = flops_per_launch / (avg_ms * 1e-3) / 1e12
    # the kernel the evolve actually runs: for small 2D families (fast build,
    # one rank) the persistent multi-step kernel, timed over the whole evolve
    persistent = (args.arith == "fast" and cfg["d"] == 2 and cfg["kind"] in (0, 1)
                  and world == 1 and not os.environ.get("SGWG_NO_PERSIST"))
    per_pt_step = 3 * (142.0 if cfg["kind"] == 1 else 70.0) * cfg["d"] + 2 + 5 + 5
    evolve_flops = total_pts * per_pt_step * nsteps
    single_stage = {"avg_launch_us": avg_ms * 1e3, "flops_per_launch": flops_per_launch,
                    "achieved_tflops": achieved, "frac": achieved / peak if peak else None}
    if persistent and evolve_ms:
        achieved = evolve_flops / (evolve_ms * 1e-3) / 1e12
        bytes_per_launch = total_pts * (16 + 24 + 24) * nsteps
        avg_ms = evolve_ms
        flops_per_launch = evolve_flops
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

    # ---- CPU baseline: the reference on this host, bounded sample (rank 0, N=1) ----
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(cfg, nsteps_box.get("dts"))

    if rank == 0:
        clocks = clk.summary()
        line = {
            "metric": "component-grid WENO5 point-updates/sec per RK stage",
            "value": value, "unit": "pt-stage/s", "n_gpus": world, "steps": args.steps,
            "warmup": max(3, args.warmup), "ms_per_step": ms_total / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": f"synthetic (analytic initial condition of BASELINE {args.config}, no dataset)",
            "config": {"workload": WORKLOADS.get(args.config, args.config),
                       "members": len(levels), "pts_per_stage": total_pts,
                       "step": f"one full simulation to T={cfg['tfinal']} "
                               + ("(no combine)" if args.no_combine else
                                  f"incl. combine at t={cfg['stops'] + [cfg['tfinal']]}"),
                       "rk_steps_per_sim": nsteps, "arith": args.arith,
                       "l2": "flushed (256 MB write) between timed steps",
                       "parallelism": f"members sharded over {world} GPU(s) (LPT)",
                       "members_per_rank": [len(s) for s in shards]},
            "wall_time_to_T_ms": ms_total / args.steps,
            "evolve_ms_per_sim": evolve_ms, "combine_ms_last": combine_ms,
            "evolve_only_value": pu / (evolve_ms * 1e-3) if evolve_ms else None,
            "e2e": {"value": e2e_value, "unit": "pt-stage/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "ms_per_step": e2e_ms / args.steps},
            "gpu_launches": int(st["kernel_launches"] + st["combine_launches"] * 2) * args.steps,
            "roofline": {"bound": "fp64", "achieved": achieved, "peak": peak,
                         "unit": "TFLOP/s", "frac": achieved / peak if peak else None,
                         "traffic": traffic,
                         "kernel": ("evolve2d_persistent_kernel (all RK steps of the evolve, "
                                    "both WENO5 sweeps + RK3 stages, grid barrier per stage)"
                                    if persistent else kernel_name(cfg, args.arith)),
                         "per_launch": (f"algorithmic flops of the whole evolve: {total_pts} pts "
                                        f"x {per_pt_step:.0f} flops/pt-step x {nsteps} steps "
                                        "(SURVEY 8(a)/(d) counting), time = evolve device time"
                                        if persistent else
                                        f"algorithmic flops of RK stage 1 over all "
                                        f"{len(levels)} members ({total_pts} pts; SURVEY "
                                        "8(a)/(d) counting: 142/70 flops per point and "
                                        "direction, +2 RK) divided by the stage's launches"),
                         "avg_launch_us": avg_ms * 1e3,
                         "flops_per_launch": flops_per_launch,
                         "single_stage_launch": single_stage,
                         "peak_source": "measured live: DFMA microbenchmark (sgwg_fp64_peak)",
                         "hbm": {"achieved_gbs": bytes_per_launch / (avg_ms * 1e-3) / 1e9,
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
    """The reference on this host, bounded sample: the first RK steps of the
    same run (~10 s of single-thread work at ~1e7 pt-stage/s)."""
    from oracle import oracle as O
    ncores, model = cpu_info()
    dom = O.make_domain(cfg["d"], cfg["nl"], cfg["lower"], cfg["upper"], cfg["root"], cfg["bc"])
    m = O.make_model(cfg["kind"], cfg["weno_mode"], cfg["epsilon"], cfg["speeds"],
                     cfg["space_dim"], cfg["theta"], cfg["tau"])
    pol = O.make_policy(cfg["dt_mode"], cfg["cfl"], cfg["reference_spacing"], cfg["dt_scale"])
    pts = family_pts_stage(cfg)
    nsteps = max(1, int(1.0e8 / (3 * pts)))
    if dts is not None and len(dts) > 0:
        t_sample = float(sum(dts[:nsteps])) * (1 - 1e-9)
    else:
        t_sample = 0.02
    vp = cfg["kind"] == 3
    if vp:  # no Vlasov-Poisson in the reference: time the transport only
        nsteps = 1
        t_sample = float(dts[0]) if dts is not None and len(dts) else 1e-3
    if O.ref_available() and not vp:
        ref = O.Reference()
        secs, n, _ = ref.time_prefix(dom, m, pol, cfg["ic"], t_sample, 1, cfg["interp"])
        kind, desc = "reference", "reference headers (oracle/_ref/libsgwref.so), threads=1"
    else:
        orc = O.Oracle()
        s0 = orc.init_family(cfg["ic"], dom)
        t0 = time.perf_counter()
        _, dts, _, _ = orc.evolve(dom, m, pol, s0, t_sample)
        secs, n = time.perf_counter() - t0, len(dts)
        kind, desc = "port", "C restatement (oracle/liboracle.so), 1 thread"
    return {"value": pts * 3 * n / secs, "unit": "pt-stage/s", "cores": 1, "kind": kind,
            "sample": f"{desc}: evolve_family of the {cfg['name']} family to t={t_sample:.4g} "
                      f"({n} RK steps, {secs:.1f} s) on {model} ({ncores} host cores)"}


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_b200(args)


if __name__ == "__main__":
    sys.exit(main())
