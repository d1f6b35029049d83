"""Vlasov-Poisson physics check (BASELINE C4 has no reference: SURVEY F4).

Linear Landau damping of the k = 0.5 mode: the electric-field energy
log ||E||_2 decays at the rate gamma ~ -0.1533 (classical result for
f0 = (1 + a cos(kx)) exp(-v^2/2)/sqrt(2 pi), k = 0.5).  The sparse-grid
solution on the GPU (fast build, reduced level) is combined at output times,
rho = 1 - int f dv, E from the periodic Poisson equation, and the decay rate
of the envelope is fitted.
"""
import numpy as np
import pytest

from helpers import gpu_family
from paper_2007_10196_b200 import configs

pytestmark = pytest.mark.gpu


def field_norm(comb, cfg):
    nx = cfg["root"][0] << cfg["nl"]
    nv = (cfg["root"][1] << cfg["nl"]) + 1
    f = comb.reshape(nx, nv)
    hv = (cfg["upper"][1] - cfg["lower"][1]) / (nv - 1)
    w = np.full(nv, hv)
    w[0] *= 0.5
    w[-1] *= 0.5
    rho = 1.0 - f @ w
    L = cfg["upper"][0] - cfg["lower"][0]
    k = 2 * np.pi * np.fft.fftfreq(nx, d=L / nx)
    rh = np.fft.fft(rho)
    Eh = np.zeros_like(rh)
    nz = k != 0
    Eh[nz] = -1j * rh[nz] / k[nz]
    E = np.real(np.fft.ifft(Eh))
    return np.sqrt(L / nx * np.sum(E * E))


def test_field_energy_record(ctx_fast, oracle):
    """sgwg_field_energy: per-step ||E_c||_2, E_c = sum_m c_m Lagrange(E_m) on the
    finest x-grid, checked at step 0 against a host restatement."""
    from oracle import oracle as O
    cfg = configs.config("C4", nl=3)
    fam = gpu_family(ctx_fast, cfg)
    fam.initialize(cfg["ic"])
    rho, E = fam.vp_field()  # field of u^0 (= what step 0 records)
    nfx = cfg["root"][0] << cfg["nl"]
    Ec = np.zeros(nfx)
    for mi, lv in enumerate(fam.levels):
        m = cfg["nl"] - lv[0]
        c = [1, -1][cfg["nl"] - sum(lv)]
        Ec += c * oracle.upsample_line(E[mi][0], nfx, m, O.PERIODIC, O.LAGRANGE) if m else c * E[mi][0]
    want0 = np.sqrt(np.sum(Ec * Ec) * (cfg["upper"][0] - cfg["lower"][0]) / nfx)
    dts = fam.evolve(cfg["dt_mode"], 1.0, cfl=cfg["cfl"])
    fe = fam.field_energy()
    assert len(fe) == len(dts) > 10
    assert abs(fe[0] - want0) <= 1e-12 * want0
    assert np.all(np.isfinite(fe)) and np.all(fe > 0)


def test_landau_damping_rate(ctx_fast):
    cfg = configs.config("C4", nl=3)
    fam = gpu_family(ctx_fast, cfg)
    fam.initialize(cfg["ic"])
    ts = np.arange(0.25, 20.0 + 1e-9, 0.25)
    norms = []
    fam.evolve(cfg["dt_mode"], 20.0, list(ts[:-1]), cfl=cfg["cfl"],
               on_stop=lambda t: norms.append(field_norm(fam.combine(cfg["interp"], 1e-6), cfg)))
    norms = np.array(norms)
    assert len(norms) == len(ts)
    logE = np.log(norms)
    # envelope: local maxima of log|E|, fitted over the linear phase
    peaks = [i for i in range(1, len(logE) - 1) if logE[i] >= logE[i - 1] and logE[i] >= logE[i + 1]]
    peaks = [i for i in peaks if ts[i] <= 18.0]
    assert len(peaks) >= 4
    slope = np.polyfit(ts[peaks], logE[peaks], 1)[0]
    assert -0.18 < slope < -0.13, slope


@pytest.mark.parametrize("groups", ["0", "1", "legacy"])
def test_field_energy_record_2d2v(ctx_fast, oracle, monkeypatch, groups):
    """Same record for 2D2V (member by member, or members grouped by x-grid
    on the device: the one-kernel row form energy_rows_kernel, or the legacy
    group + point kernels): step 0 against separable Lagrange upsampling of
    every member's (E_1, E_2)."""
    from oracle import oracle as O
    monkeypatch.setenv("SGWG_ENERGY_GROUPS", "0" if groups == "0" else "1")
    if groups == "legacy":
        monkeypatch.setenv("SGWG_ENERGY_LEGACY", "1")
    cfg = configs.config("C5", nl=3)
    fam = gpu_family(ctx_fast, cfg)
    fam.initialize(cfg["ic"])
    rho, E = fam.vp_field()
    nf = [cfg["root"][k] << cfg["nl"] for k in range(2)]
    Ec = np.zeros((2, nf[0], nf[1]))
    for mi, lv in enumerate(fam.levels):
        c = [1, -3, 3, -1][cfg["nl"] - sum(lv)]
        n0, n1 = fam.points[mi][0], fam.points[mi][1]
        for comp in range(2):
            g = np.asarray(E[mi][comp]).reshape(n0, n1)
            m1 = cfg["nl"] - lv[1]
            rows = np.array([oracle.upsample_line(g[i], nf[1], m1, O.PERIODIC, O.LAGRANGE)
                             if m1 else g[i] for i in range(n0)])
            m0 = cfg["nl"] - lv[0]
            full = np.array([oracle.upsample_line(rows[:, j], nf[0], m0, O.PERIODIC, O.LAGRANGE)
                             if m0 else rows[:, j] for j in range(nf[1])]).T
            Ec[comp] += c * full
    hvol = (cfg["upper"][0] - cfg["lower"][0]) / nf[0] * (cfg["upper"][1] - cfg["lower"][1]) / nf[1]
    want0 = np.sqrt(np.sum(Ec * Ec) * hvol)
    fam.evolve(cfg["dt_mode"], 0.05, cfl=cfg["cfl"])
    fe = fam.field_energy()
    assert len(fe) > 3
    assert abs(fe[0] - want0) <= 1e-12 * want0
    assert np.all(np.isfinite(fe)) and np.all(fe > 0)


def test_field_energy_batched_matches_per_step(ctx_fast, monkeypatch):
    """The batched record of captured step chunks (step-start fields in a ring, one
    group + one row launch per chunk: energy_rows_batch_kernel) against the per-step
    kernel (SGWG_ENERGY_BATCH=0) on the same run, with stops that cut chunks short:
    the same steps recorded, equal to rounding (the batched rows sum the groups of an
    x2 class before interpolating)."""
    monkeypatch.setenv("SGWG_ENERGY_GROUPS", "1")
    cfg = configs.config("C5", nl=3)
    rec = {}
    for mode in ("1", "0"):
        monkeypatch.setenv("SGWG_ENERGY_BATCH", mode)
        fam = gpu_family(ctx_fast, cfg)
        fam.initialize(cfg["ic"])
        dts = fam.evolve(cfg["dt_mode"], 0.9, cfl=cfg["cfl"], stops=[0.13, 0.5, 0.9])
        fe = np.asarray(fam.field_energy())
        assert len(fe) == len(dts) > 70  # more than one 64-step chunk
        rec[mode] = fe
    assert np.all(rec["1"] > 0)
    assert np.max(np.abs(rec["1"] - rec["0"]) / rec["0"]) < 1e-13
