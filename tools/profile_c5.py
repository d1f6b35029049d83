"""Per-kernel event times of the C5 stage kernels inside a real evolve
(profile mode: every stage launch bracketed by CUDA events, no graphs)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2007_10196_b200 import configs, sgwg  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C5"
T = float(sys.argv[2]) if len(sys.argv) > 2 else 0.02
cfg = configs.config(name)
ctx = sgwg.Context(0, arith="fast", profile=True)
fam = sgwg.Family.from_config(ctx, cfg)
fam.initialize(cfg["ic"])
fam.evolve_config(cfg, tfinal=T / 4, stops=[])  # warm-up
fam.kernel_profile_reset()
dts = fam.evolve_config(cfg, tfinal=T, stops=[])
peak = ctx.fp64_peak_tflops()
out = {"config": name, "steps": len(dts), "stage_kernels": fam.stage_kernels, "peak_tflops": peak,
       "kernels": []}
for k in fam.kernel_profile():
    avg = k["ms_sum"] / max(1, k["launches"])
    k["avg_us"] = avg * 1e3
    k["tflops"] = k["flops_per_launch"] / (avg * 1e-3) / 1e12
    k["frac"] = k["tflops"] / peak
    k["gbs"] = k["bytes_per_launch"] / (avg * 1e-3) / 1e9
    out["kernels"].append(k)
print(json.dumps(out, indent=1))
