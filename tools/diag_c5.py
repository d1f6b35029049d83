"""Step-by-step probe of the full BASELINE C5 family (diagnostics)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2007_10196_b200 import configs, sgwg

arith = sys.argv[1] if len(sys.argv) > 1 else "fast"
nl = int(sys.argv[2]) if len(sys.argv) > 2 else 5
cfg = configs.config("C5", nl=nl)
ctx = sgwg.Context(0, arith=arith)
t = time.time(); fam = sgwg.Family.from_config(ctx, cfg); print("create", time.time() - t, fam.num_members, fam.total_points, flush=True)
t = time.time(); fam.initialize(cfg["ic"]); print("init", time.time() - t, flush=True)
t = time.time(); rho, E = fam.vp_field(); print("field", time.time() - t, "max|E|", max(np.abs(e).max() for e in E), "rho range", min(r.min() for r in rho), max(r.max() for r in rho), flush=True)
t = time.time(); fam.rk3_step(1e-3); print("rk3_step", time.time() - t, flush=True)
s = fam.download(); print("state finite", np.isfinite(s).all(), np.abs(s).max(), flush=True)
fam.initialize(cfg["ic"])
t = time.time(); dts = fam.evolve(cfg["dt_mode"], 0.01, cfl=cfg["cfl"]); print("evolve 0.01", time.time() - t, len(dts), dts[:4], flush=True)
st = fam.stats(); print(st, flush=True)
