"""Reduced Vlasov-Maxwell system (x2, xi1, xi2) of the reference
(models.hpp:376-527, paper example ex6) on the GPU path:
per-line coefficients xi2 / E1 + xi2 B3 / E2 - xi1 B3, currents, the
characteristic field lines w+- = E1 +- B3 and family wave speeds.  The parity
oracle is the reference itself (oracle/_ref, no C restatement): bitwise in the
exact build, within 1e-10 in the fast build."""
import numpy as np
import pytest

from helpers import bitwise_equal, gpu_family, maxabs, oracle_objs
from oracle import oracle as O
from paper_2007_10196_b200 import configs

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ref():
    if not O.ref_available():
        pytest.skip("oracle/_ref not built")
    return O.Reference()


def _cfg(**over):
    return configs.config("ex6", nl=2, root=[8, 8, 8], **over)


def _member_slices(fam):
    out, off = [], 0
    for pts in fam.points:
        n = int(np.prod(pts)) + 3 * pts[0]
        out.append(slice(off, off + n))
        off += n
    return out


def test_init_family_bitwise(ctx, ref):
    cfg = _cfg()
    dom, model, _ = oracle_objs(cfg)
    fam = gpu_family(ctx, cfg)
    fam.initialize(cfg["ic"])
    want = ref.init_family(cfg["ic"], dom, model, state_points=fam.total_points)
    assert bitwise_equal(fam.download(), want)


def _perturbed(ref, cfg, fam, seed):
    dom, model, _ = oracle_objs(cfg)
    s = ref.init_family(cfg["ic"], dom, model, state_points=fam.total_points)
    rng = np.random.default_rng(seed)
    for sl, pts in zip(_member_slices(fam), fam.points):
        npts = int(np.prod(pts))
        s[sl][:npts] *= 1.0 + 0.1 * rng.standard_normal(npts)
        s[sl][npts:] += 0.05 * rng.standard_normal(3 * pts[0])  # nonzero E1, E2, B3
    return s


@pytest.mark.parametrize("arith", ["exact", "fast"])
def test_rhs_matches_reference(ctx, ctx_fast, ref, arith):
    cfg = _cfg()
    dom, model, _ = oracle_objs(cfg)
    fam = gpu_family(ctx if arith == "exact" else ctx_fast, cfg)
    s = _perturbed(ref, cfg, fam, 3)
    fam.upload(s)
    got = fam.rhs()
    for mi, sl in enumerate(_member_slices(fam)):
        want = ref.rhs(dom, fam.levels[mi], model, s[sl])
        if arith == "exact":
            assert bitwise_equal(got[sl], want), (mi, maxabs(got[sl], want))
        else:
            assert maxabs(got[sl], want) <= 1e-12 * (1.0 + np.max(np.abs(want))), mi


@pytest.mark.parametrize("arith", ["exact", "fast"])
def test_evolve_matches_reference(ctx, ctx_fast, ref, arith):
    cfg = _cfg()
    dom, model, pol = oracle_objs(cfg)
    fam = gpu_family(ctx if arith == "exact" else ctx_fast, cfg)
    s = _perturbed(ref, cfg, fam, 5)
    fam.upload(s)
    T = 0.3
    got_dts = fam.evolve_config(cfg, tfinal=T, stops=[0.1])
    want, want_dts, st, _ = ref.evolve(dom, model, pol, s, T, [0.1])
    assert st == 0 and len(got_dts) == len(want_dts) > 3
    got = fam.download()
    if arith == "exact":
        assert bitwise_equal(got_dts, want_dts)
        assert bitwise_equal(got, want), maxabs(got, want)
    else:
        assert maxabs(got_dts, want_dts) < 1e-14
        assert maxabs(got, want) < 1e-10
    # the combination uses the distributions only (MemberState::field, combine.hpp:55-59)
    f_only = np.concatenate([want[sl][:int(np.prod(p))]
                             for sl, p in zip(_member_slices(fam), fam.points)])
    comb = fam.combine(cfg["interp"], cfg["epsilon"])
    wc = ref.combine(dom, f_only, cfg["interp"], cfg["epsilon"])
    assert maxabs(comb, wc) < (0.0 if arith == "exact" else 1e-10) or bitwise_equal(comb, wc)


def test_vm_rejects_bad_geometry(ctx):
    cfg = configs.config("C3", nl=2, root=[8, 8, 8], kind=configs.VLASOV_MAXWELL)
    with pytest.raises(ValueError):
        gpu_family(ctx, cfg)
