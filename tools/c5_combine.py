"""Full-size BASELINE C5 combination (finest grid 256^2 x 257^2 = 4.33e9 points,
34.6 GB) into a device buffer through sgwg_combine's row-slab path; prints the
device time and a checksum of a few rows against sgwg_combine_rows."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2007_10196_b200 import configs, sgwg

cfg = configs.config("C5")
ctx = sgwg.Context(0, arith=sys.argv[1] if len(sys.argv) > 1 else "fast")
fam = sgwg.Family.from_config(ctx, cfg)
fam.initialize(cfg["ic"])
fam.evolve_config(cfg, tfinal=0.01)
out = torch.empty(fam.finest_points, dtype=torch.float64, device="cuda:0")
torch.cuda.synchronize()
t0 = time.perf_counter()
fam.combine(cfg["interp"], cfg["epsilon"], out_device_ptr=out.data_ptr())
torch.cuda.synchronize()
t1 = time.perf_counter()
st = fam.stats()
rows = fam.fine_extent0
per_row = fam.finest_points // rows
part = fam.combine_rows(100, 103, cfg["interp"], cfg["epsilon"])
same = np.array_equal(part, out[100 * per_row:103 * per_row].cpu().numpy())
print(f"C5 combine: {fam.finest_points} finest points, wall {t1 - t0:.2f} s, device {st['combine_ms']:.1f} ms, "
      f"finest-points/s {fam.finest_points / (st['combine_ms'] * 1e-3):.3e}, rows check {same}, "
      f"mean {out.mean().item():.6e}")
