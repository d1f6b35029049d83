"""The batched energy record (default) against the per-step kernel (SGWG_ENERGY_BATCH=0):
the records must be bitwise equal; evolve time of both."""
import os, subprocess, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if len(sys.argv) > 1 and sys.argv[1] == "child":
    import numpy as np
    from paper_2007_10196_b200 import configs, sgwg
    cfg = configs.config("C5")
    ctx = sgwg.Context(0, arith="fast")
    fam = sgwg.Family.from_config(ctx, cfg)
    fam.initialize(cfg["ic"])
    fam.evolve_config(cfg, tfinal=0.1, stops=[])  # warm-up (graph capture)
    fam.initialize(cfg["ic"])
    dts = fam.evolve_config(cfg, tfinal=0.55, stops=[0.21, 0.55])
    fe = np.asarray(fam.field_energy())
    s = fam.stats()
    np.save(sys.argv[2], fe)
    print(json.dumps({"steps": len(dts), "evolve_ms": s["evolve_ms"], "n_fe": int(fe.size),
                      "fe0": float(fe[0]), "feN": float(fe[-1]), "zeros": int((fe == 0).sum())}))
else:
    import numpy as np
    out = "gpurun_out/energy_ab"
    os.makedirs(out, exist_ok=True)
    for mode in ("1", "0"):
        env = dict(os.environ, SGWG_ENERGY_BATCH=mode)
        r = subprocess.run([sys.executable, __file__, "child", f"{out}/fe{mode}.npy"], env=env,
                           capture_output=True, text=True)
        print("batch=" + mode, r.stdout.strip(), r.stderr.strip()[-400:])
    a, b = np.load(f"{out}/fe1.npy"), np.load(f"{out}/fe0.npy")
    print("equal:", a.shape == b.shape and bool((a == b).all()), "max rel diff",
          float((np.abs(a - b) / np.abs(b)).max()) if a.shape == b.shape else None)
