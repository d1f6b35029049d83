import sys; sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import numpy as np
from helpers import gpu_family, oracle_objs
from oracle import oracle as O
from paper_2007_10196_b200 import configs, sgwg
for over in ({"nl": 3}, {}):
    cfg = configs.config("C5", **over)
    orc = O.Oracle()
    dom, model, pol = oracle_objs(cfg)
    s0 = orc.init_family(cfg["ic"], dom)
    T = 0.006
    for arith in ("fast", "exact"):
        ctx = sgwg.Context(0, arith=arith)
        fam = gpu_family(ctx, cfg)
        fam.upload(s0)
        dts = fam.evolve_config(cfg, tfinal=T, stops=[])
        g = fam.download()
        off = 0; rel = []
        for pts in fam.points:
            n = int(np.prod(pts)); rel.append(abs(g[off:off+n].sum() - s0[off:off+n].sum()) / abs(s0[off:off+n].sum())); off += n
        print(over, arith, len(dts), 'max rel mass change gpu', max(rel))
        fam.close(); ctx.close()
    if over:
        s, wd, st, _ = orc.evolve(dom, model, pol, s0, T)
        off = 0; rel = []
        for pts in fam.points:
            n = int(np.prod(pts)); rel.append(abs(s[off:off+n].sum() - s0[off:off+n].sum()) / abs(s0[off:off+n].sum())); off += n
        print(over, 'oracle', len(wd), 'max rel mass change', max(rel))
