"""Per-CTA phase sums of the persistent x pass (trace build, SGWG_LIB, SGWG_P4_XPERSIST=1)."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2007_10196_b200 import configs, sgwg  # noqa: E402

cfg = configs.config("C5")
ctx = sgwg.Context(0, arith="fast")
fam = sgwg.Family.from_config(ctx, cfg)
fam.initialize(cfg["ic"])
fam.evolve_config(cfg, tfinal=0.01, stops=[])
lib = sgwg.load()
buf = np.zeros((2, 8192, 10), dtype=np.int64)
assert lib.sgwg_p4trace_dump(buf.ctypes.data_as(C.POINTER(C.c_longlong))) == 0
t = buf[0][:296].astype(np.float64)
names = ["gather wait", "bar A", "issue next", "x1 sweep", "bar B", "x2 sweep+K"]
tot = t[:, :6].sum(axis=1)
print(f"CTAs {len(t)}, cycles per CTA median {np.median(tot):.0f} (max {tot.max():.0f})")
for k, nm in enumerate(names):
    print(f"  {nm:12s} median {np.median(t[:, k]):9.0f}  share {np.median(t[:, k]) / np.median(tot):.3f}")
