"""Small invocations of every kernel family for compute-sanitizer
(memcheck / racecheck / synccheck):

    compute-sanitizer --tool memcheck python tools/sanitize_cases.py

C2-like 2D Burgers family (fast build: persistent cooperative evolve), C3-like
3D advection (3D stage kernel), C5-like 2D2V Vlasov-Poisson (x pass, persistent
v pass, field kernels, energy record), each followed by the combination (chunked
upsample + final kernels) and a cut-plane evaluation; the exact build on C1."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2007_10196_b200 import configs, sgwg  # noqa: E402

CASES = [
    ("C2", {"nl": 3, "root": [16, 16]}, "fast", 0.01),
    ("C3", {"nl": 2, "root": [8, 8, 8]}, "fast", 0.004),
    ("C5", {"nl": 3}, "fast", 0.02),
    ("C1", {}, "exact", 0.002),
]
only = sys.argv[1:] or None
for name, over, arith, T in CASES:
    if only and name not in only:
        continue
    cfg = configs.config(name, **over)
    ctx = sgwg.Context(0, arith=arith)
    fam = sgwg.Family.from_config(ctx, cfg)
    fam.initialize(cfg["ic"])
    dts = fam.evolve_config(cfg, tfinal=T, stops=[])
    out = fam.combine(cfg["interp"], cfg["epsilon"])
    st = fam.combined_stats(cfg["interp"], cfg["epsilon"])
    plane = fam.cut_plane(0, cfg["d"] - 1, [0] * cfg["d"], cfg["interp"], cfg["epsilon"])
    print(f"{name} {arith}: {len(dts)} steps, combined {out.size} pts, finite {np.all(np.isfinite(out))}, "
          f"mass {st['mass']:.6e}, cut plane {plane.shape}", flush=True)
    fam.close()
    ctx.close()
