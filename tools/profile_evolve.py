"""Short evolve of a BASELINE family through sgwg_evolve (the production step
loop: persistent kernel for small 2D families) for ncu."""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2007_10196_b200 import configs, sgwg  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C2")
ap.add_argument("--arith", default="fast")
ap.add_argument("--tfinal", type=float, default=0.005)
args = ap.parse_args()
cfg = configs.config(args.config)
ctx = sgwg.Context(0, arith=args.arith)
fam = sgwg.Family.from_config(ctx, cfg)
fam.initialize(cfg["ic"])
dts = fam.evolve_config(cfg, tfinal=args.tfinal, stops=[])
print(args.config, "steps", len(dts), fam.stats())
