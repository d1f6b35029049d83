"""Phase trace of the C5 plane kernels (experiment build with -DSGWG_TRACE,
loaded via SGWG_LIB): per pass, median cycles of each CTA phase, and the
number of CTAs resident per SM over time (from globaltimer stamps)."""
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
names = {0: ["setup+issue", "load wait+bar", "sweeps", "bar", "K store", "-"],
         1: ["setup+bar", "U wait", "sweeps", "K/un wait+bar", "epilogue", "moment"]}
for ps in (0, 1):
    t = buf[ps]
    ok = t[:, 0] > 0
    t = t[ok]
    cyc = t[:, 1:8].astype(np.float64)
    d = np.diff(cyc, axis=1)
    tot = cyc[:, 5] - cyc[:, 0]
    print(f"pass {ps}: {len(t)} CTAs, median total {np.median(tot):.0f} cyc")
    for k, nm in enumerate(names[ps]):
        if nm == "-":
            continue
        col = d[:, k] if not (ps == 1 and k == 4) else cyc[:, 6] - cyc[:, 4]
        if ps == 1 and k == 5:
            col = cyc[:, 5] - cyc[:, 6]
        print(f"   {nm:14s} median {np.median(col):8.0f}  mean {np.mean(col):8.0f}")
    g0, g1, sm = t[:, 0], t[:, 9], t[:, 8]
    span = g1.max() - g0.min()
    print(f"   span {span / 1e3:.1f} us; CTAs per SM {len(t) / max(1, len(set(sm.tolist()))):.1f}")
