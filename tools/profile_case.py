"""Small fixed workload for ncu: a few RK steps of a BASELINE family plus one
combine through the C ABI (no CUDA graphs: --profile mode launches every
kernel individually so ncu sees each one)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2007_10196_b200 import configs, sgwg  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C2")
ap.add_argument("--arith", default="fast")
ap.add_argument("--steps", type=int, default=3)
ap.add_argument("--nl", type=int, default=None)
ap.add_argument("--no-combine", action="store_true")
args = ap.parse_args()

over = {} if args.nl is None else {"nl": args.nl}
cfg = configs.config(args.config, **over)
ctx = sgwg.Context(0, arith=args.arith, profile=True)
fam = sgwg.Family.from_config(ctx, cfg)
fam.initialize(cfg["ic"])
h = cfg["reference_spacing"]
dt = 0.5 * h if cfg["dt_mode"] == 0 else cfg["dt_scale"] * h ** (5.0 / 3.0)
for _ in range(args.steps):
    fam.rk3_step(dt * 0.5)
out = fam.download() if args.no_combine else fam.combine(cfg["interp"], cfg["epsilon"])
st = fam.stats()
print(f"{args.config} members={fam.num_members} pts={fam.total_points} finest={fam.finest_points} "
      f"sum={out.sum():.6e}")
