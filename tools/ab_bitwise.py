"""Dump member states, dt sequence and VP fields of a few short runs with the
library named by SGWG_LIB (A/B bitwise check of two builds):
    SGWG_LIB=a.so python tools/ab_bitwise.py out_a.npz; ... ; python tools/ab_bitwise.py --cmp a.npz b.npz
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

if sys.argv[1] == "--cmp":
    a, b = np.load(sys.argv[2]), np.load(sys.argv[3])
    bad = 0
    for k in a.files:
        same = np.array_equal(a[k].view(np.uint64), b[k].view(np.uint64))
        print(f"{k:24s} bitwise={same} maxabs={np.max(np.abs(a[k] - b[k])) if a[k].size else 0:.3e}")
        bad += not same
    sys.exit(1 if bad else 0)

from paper_2007_10196_b200 import configs, sgwg  # noqa: E402

out = {}
ctx = sgwg.Context(0, arith="fast")
for name, over, T in [("C4", {}, 0.3), ("C5", {"nl": 3}, 0.05), ("C2", {}, 0.02),
                      ("C3", {"nl": 3, "root": [16, 16, 16]}, 0.004)]:
    cfg = configs.config(name, **over)
    fam = sgwg.Family.from_config(ctx, cfg)
    fam.initialize(cfg["ic"])
    if cfg["kind"] == 3:
        rho, E = fam.vp_field()
        out[name + "_rho0"] = np.concatenate([np.ravel(r) for r in rho])
        out[name + "_E0"] = np.concatenate([np.ravel(e) for e in E])
    dts = fam.evolve_config(cfg, tfinal=T, stops=[])
    out[name + "_dts"] = np.array(dts)
    out[name + "_state"] = fam.download()
    fam.close()
np.savez(sys.argv[1], **out)
print("saved", sys.argv[1], {k: v.shape for k, v in out.items()})
