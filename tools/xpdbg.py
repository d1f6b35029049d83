import os, sys
sys.path.insert(0, '/root/repo')
import numpy as np
from paper_2007_10196_b200 import configs, sgwg
cfg = configs.config("C5", nl=3)
res = {}
for xp in ("0", "1"):
    os.environ["SGWG_P4_XPERSIST"] = xp
    ctx = sgwg.Context(0, arith="fast")
    fam = sgwg.Family.from_config(ctx, cfg)
    fam.initialize(cfg["ic"])
    s = fam.download()
    rng = np.random.default_rng(3)
    s = s + 0.01 * rng.standard_normal(s.size)
    fam.upload(s)
    try:
        res[xp] = fam.rhs()
    except Exception as e:
        print("xp", xp, "error", e)
        res[xp] = None
    print("xp", xp, "stage kernels", fam.stage_kernels, flush=True)
    fam.close(); ctx.close()
if res["0"] is not None and res["1"] is not None:
    d = np.abs(res["0"] - res["1"])
    print("max diff", d.max(), "count", int((d > 1e-12).sum()), "of", d.size)
    idx = np.nonzero(d > 1e-12)[0]
    print("first bad indices", idx[:20])
    # member layout
    import bench
    lv = bench._levels(cfg)
    off = 0
    for mi, l in enumerate(lv):
        n = bench.member_extents(cfg, l)
        npts = int(np.prod(n))
        bad = ((idx >= off) & (idx < off + npts)).sum()
        if bad:
            loc = idx[(idx >= off) & (idx < off + npts)][:5] - off
            V = n[2] * n[3]
            print("member", mi, l, n, "bad", bad, "of", npts, "first (x, v):", [(int(q // V), int(q % V)) for q in loc])
        off += npts
