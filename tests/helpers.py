"""Test helpers: run a BASELINE config through the CPU oracle (the checker) and
through the B200 path (the product) on identical inputs."""
import numpy as np

from oracle import oracle as O
from paper_2007_10196_b200 import configs


def oracle_objs(cfg):
    dom = O.make_domain(cfg["d"], cfg["nl"], cfg["lower"], cfg["upper"], cfg["root"], cfg["bc"])
    model = O.make_model(cfg["kind"], cfg["weno_mode"], cfg["epsilon"], cfg["speeds"],
                         cfg["space_dim"], cfg["theta"], cfg["tau"])
    pol = O.make_policy(cfg["dt_mode"], cfg["cfl"], cfg["reference_spacing"], cfg["dt_scale"])
    return dom, model, pol


def small(name, **over):
    """A config shrunk so the oracle finishes in seconds."""
    return configs.config(name, **over)


def random_states(orc, cfg, seed, lo=-1.0, hi=1.0):
    dom, _, _ = oracle_objs(cfg)
    n = orc.total_points(dom)
    rng = np.random.default_rng(seed)
    return rng.uniform(lo, hi, n)


def gpu_family(ctx, cfg, members=None):
    from paper_2007_10196_b200 import sgwg
    return sgwg.Family.from_config(ctx, cfg, members)


def maxabs(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    assert a.shape == b.shape, (a.shape, b.shape)
    if a.size == 0:
        return 0.0
    return float(np.max(np.abs(a - b)))


def bitwise_equal(a, b):
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    return a.shape == b.shape and np.array_equal(a.view(np.uint64), b.view(np.uint64))
