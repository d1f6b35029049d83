"""Generate the golden fixtures under tests/golden/ FROM THE REFERENCE ITSELF.

Runs the unmodified reference headers (oracle/_ref/libsgwref.so, built by
oracle/Makefile from /root/reference/proj/include/sgweno, in place) on seeded
inputs and stores inputs + outputs as small .npz files.  The fixtures pin the
CPU oracle (tests/test_oracle_pin.py) and the GPU path (tests/test_gpu_golden.py)
to the reference on machines where /root/reference does not exist.

    python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402
from paper_2007_10196_b200 import configs  # noqa: E402


def objs(cfg):
    dom = O.make_domain(cfg["d"], cfg["nl"], cfg["lower"], cfg["upper"], cfg["root"], cfg["bc"])
    m = O.make_model(cfg["kind"], cfg["weno_mode"], cfg["epsilon"], cfg["speeds"],
                     cfg["space_dim"], cfg["theta"], cfg["tau"])
    p = O.make_policy(cfg["dt_mode"], cfg["cfl"], cfg["reference_spacing"], cfg["dt_scale"])
    return dom, m, p


def main():
    ref = O.Reference()
    orc = O.Oracle()
    out = {}

    # 1. WENO5 flux reconstruction on random stencils (weno.hpp:60-72)
    rng = np.random.default_rng(7)
    st = rng.uniform(-2, 2, (300, 5))
    st = np.vstack([st, [[0, 1, 2, 3, 4], [0, 0, 0, 1, 1], [3, 3, 3, 3, 3], [1, 2, 4, 0, 0]]])
    out["flux_stencils"] = st
    out["flux_nonlinear"] = np.array([ref.weno5_flux_positive(s, 1e-6, O.NONLINEAR) for s in st])
    out["flux_linear"] = np.array([ref.weno5_flux_positive(s, 1e-6, O.LINEAR) for s in st])
    np.savez_compressed(os.path.join(HERE, "weno_flux.npz"), **out)

    # 2. derivative lines (weno.hpp:118-192): periodic/zero, Burgers/advect, +/- c
    rng = np.random.default_rng(11)
    lines = {}
    cases = [(16, 1, 0.0, 1.7, 0.1, O.PERIODIC), (16, 1, 0.0, 1.7, 0.1, O.ZERO),
             (9, 0, 1.0, 0.0, 0.25, O.ZERO), (12, 0, -0.5, 0.0, 0.25, O.PERIODIC),
             (6, 0, 2.0, 0.0, 0.5, O.PERIODIC), (1, 0, 1.0, 0.0, 0.5, O.ZERO)]
    for ci, (n, fk, c, alpha, dx, bc) in enumerate(cases):
        u = rng.uniform(-1, 1, n)
        lines[f"u{ci}"] = u
        lines[f"du{ci}"] = ref.weno_derivative_line(u, fk, c, alpha, dx, bc, 1e-6, O.NONLINEAR)
        lines[f"case{ci}"] = np.array([n, fk, c, alpha, dx, bc], dtype=np.float64)
    np.savez_compressed(os.path.join(HERE, "weno_lines.npz"), **lines)

    # 3. upsample lines (interp.hpp:151-189)
    rng = np.random.default_rng(13)
    ups = {}
    ci = 0
    for m in (1, 2, 3):
        for bc in (O.PERIODIC, O.ZERO):
            for mode in (O.WENO, O.LAGRANGE):
                n_src = 8 + (1 if bc == O.ZERO else 0)
                n_dst = (8 << m) + (1 if bc == O.ZERO else 0)
                src = rng.uniform(-1, 1, n_src)
                ups[f"src{ci}"] = src
                ups[f"dst{ci}"] = ref.upsample_line(src, n_dst, m, bc, mode, 1e-6)
                ups[f"case{ci}"] = np.array([m, bc, mode, n_dst])
                ci += 1
    np.savez_compressed(os.path.join(HERE, "upsample.npz"), **ups)

    # 4. BASELINE C1 end to end through evolve_family + combine (dt = 0.5 h^{5/3})
    cfg = configs.config("C1")
    dom, m, p = objs(cfg)
    s0 = ref.init_family(cfg["ic"], dom, m)
    s, dts, stat, _ = ref.evolve(dom, m, p, s0, cfg["tfinal"])
    assert stat == 0
    np.savez_compressed(os.path.join(HERE, "c1_full.npz"), dts=dts, states=s,
                        combined=ref.combine(dom, s, cfg["interp"], cfg["epsilon"]))

    # 5. C2 family at reduced level with a stop (CFL dt, family max|u|, landing)
    cfg = configs.config("C2", nl=3, root=[16, 16])
    dom, m, p = objs(cfg)
    s0 = ref.init_family(cfg["ic"], dom, m)
    comb = []
    s, dts, stat, _ = ref.evolve(dom, m, p, s0, 0.2, [0.1],
                                 on_stop=lambda t, st_: comb.append(
                                     ref.combine(dom, st_, cfg["interp"], cfg["epsilon"])))
    assert stat == 0
    np.savez_compressed(os.path.join(HERE, "c2_small.npz"), dts=dts, states=s,
                        combined_t01=comb[0], combined_t02=comb[1])

    # 6. C3 family at reduced level: random states -> combine (WENO) and rhs
    cfg = configs.config("C3", nl=2, root=[8, 8, 8])
    dom, m, p = objs(cfg)
    rng = np.random.default_rng(23)
    s = rng.uniform(-1, 1, orc.total_points(dom))
    lv = ref.levels(3, 2)
    rhs, off = [], 0
    for l in lv:
        n = int(np.prod([8 << int(q) for q in l]))
        rhs.append(ref.rhs(dom, l, m, s[off:off + n]))
        off += n
    np.savez_compressed(os.path.join(HERE, "c3_small.npz"), states=s, rhs=np.concatenate(rhs),
                        combined=ref.combine(dom, s, O.WENO, 1e-6),
                        combined_lagrange=ref.combine(dom, s, O.LAGRANGE, 1e-6))
    for f in sorted(os.listdir(HERE)):
        if f.endswith(".npz"):
            print(f, os.path.getsize(os.path.join(HERE, f)))


if __name__ == "__main__":
    main()
