"""Phase trace of the persistent 2D kernel (experiment build with -DSGWG_TRACE,
loaded via SGWG_LIB): per stage, cycles in staging / sweeps / epilogue /
grid barrier for four CTAs."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2007_10196_b200 import configs, sgwg  # noqa: E402

cfg = configs.config(sys.argv[1] if len(sys.argv) > 1 else "C2")
ctx = sgwg.Context(0, arith="fast")
fam = sgwg.Family.from_config(ctx, cfg)
fam.initialize(cfg["ic"])
fam.evolve_config(cfg, tfinal=0.05, stops=[])
lib = sgwg.load()
buf = np.zeros((4, 600, 5), dtype=np.int64)
assert lib.sgwg_trace_dump(buf.ctypes.data_as(C.POINTER(C.c_longlong))) == 0
for w in range(4):
    t = buf[w, 30:570].astype(np.float64)  # skip the launch's first steps
    ok = np.all(t > 0, axis=1)
    t = t[ok]
    d = np.diff(t, axis=1)
    per = t[1:, 0] - t[:-1, 0]
    wait = t[1:, 0] - t[:-1, 4]
    print(f"cta{w}: stage {np.median(per):8.0f} cyc | staging {np.median(d[:,0]):6.0f} "
          f"sweep {np.median(d[:,1]):6.0f} epilogue {np.median(d[:,2]):6.0f} "
          f"barrier {np.median(d[:,3]):6.0f} wait-next {np.median(wait):6.0f} | n={len(t)}")
