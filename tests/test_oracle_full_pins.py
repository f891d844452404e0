"""Pins of O19, the full Eq. (10) objective with per-frame probe shifts s^p_kj and the reference
term (Eq. (12)), in both oracles:
* s^p = 0 reduces to O8-O12 (+ O14 with reference frames), which are pinned on their own;
* central finite differences of F in psi and in q with nonzero probe shifts and the reference
  term (16^2 torus, mt != 1);
* P:111's remark that a probe shift can be moved onto psi and the data: for one plane at mt = 1
  and no crop (N = L), an integer probe shift t gives the same F and gradients as s^p = 0 with
  the sample shift s - t and the data rolled by -t;
* the C and numpy implementations agree.
"""
import numpy as np
import pytest

import oracle
import synth
from oracle import np_oracle as npo


def crand(*sh, seed=[0]):
    seed[0] += 1
    g = np.random.default_rng(100 + seed[0])
    return g.standard_normal(sh) + 1j * g.standard_normal(sh)


def case(L=16, N=8, K=2, R=2):
    cfg = synth.CONFIGS["cfg0"]
    g = oracle.Geometry(cfg.wavelength, cfg.Z, cfg.z1, cfg.det_pixel)
    psi, q, s = synth.small_geometry_case(seed=5, L=L, N=N, K=K, nz=g.nz)
    sp = np.random.default_rng(6).uniform(-2, 2, size=(K, g.nz, 2))
    d = np.abs(oracle.fwd(g, 1 + 0.2 * crand(*psi.shape), q * (1 + 0.1 * crand(L, L)), s, N)) + 0.05
    rs = np.random.default_rng(7).uniform(-3, 3, size=(R, 2))
    dr = np.abs(crand(R, N, N)) + 0.5
    return g, psi, q, s, sp, d, rs, dr


def test_zero_probe_shift_reduces_to_o8_o12_and_o14():
    g, psi, q, s, sp, d, rs, dr = case()
    z = np.zeros_like(sp)
    F, gp, gq = oracle.grad(g, psi, q, s, d)
    Fr, gqr = oracle.grad_ref(g, q, rs, dr)
    F1, gp1, gq1 = oracle.grad_full(g, psi, q, s, z, d)
    assert abs(F1 - F) < 1e-12 * F and np.allclose(gp1, gp, rtol=0, atol=1e-12) and np.allclose(gq1, gq, atol=1e-12)
    F2, gp2, gq2 = oracle.grad_full(g, psi, q, s, z, d, rs, dr)
    assert abs(F2 - F - Fr) < 1e-12 * F2 and np.allclose(gq2, gq + gqr, atol=1e-12)
    assert np.allclose(gp2, gp, atol=1e-12)


@pytest.mark.parametrize("block", ["psi", "q"])
def test_full_objective_finite_differences(block):
    g, psi, q, s, sp, d, rs, dr = case()
    F0, gp, gq = oracle.grad_full(g, psi, q, s, sp, d, rs, dr)
    h = 1e-6
    for _ in range(3):
        v = crand(*(psi.shape if block == "psi" else q.shape))
        if block == "psi":
            Fp = oracle.grad_full(g, psi + h * v, q, s, sp, d, rs, dr, False, False)[0]
            Fm = oracle.grad_full(g, psi - h * v, q, s, sp, d, rs, dr, False, False)[0]
            an = np.vdot(gp, v).real
        else:
            Fp = oracle.grad_full(g, psi, q + h * v, s, sp, d, rs, dr, False, False)[0]
            Fm = oracle.grad_full(g, psi, q - h * v, s, sp, d, rs, dr, False, False)[0]
            an = np.vdot(gq, v).real
        assert abs((Fp - Fm) / (2 * h) - an) / abs(an) < 1e-6


def test_probe_shift_commutes_onto_sample_and_data():
    """mt = 1, N = L, integer probe shift t: F(s, t; d) = F(s - t, 0; roll(d, -t)), same gradients."""
    cfg = synth.CONFIGS["cfg0"]
    g = oracle.Geometry(cfg.wavelength, cfg.Z, cfg.z1[:1], cfg.det_pixel)  # one plane: mt = 1, omega = 0
    L = 16
    psi, q, s = synth.small_geometry_case(seed=8, L=L, N=L, K=2, nz=1)
    t = np.array([[[3.0, -2.0]], [[-1.0, 4.0]]])
    d = np.abs(crand(2, 1, L, L)) + 0.3
    F1, gp1, gq1 = oracle.grad_full(g, psi, q, s, t, d)
    d2 = np.stack([np.roll(d[k], (-int(t[k, 0, 1]), -int(t[k, 0, 0])), axis=(-2, -1)) for k in range(2)])
    F2, gp2, gq2 = oracle.grad_full(g, psi, q, s - t, np.zeros_like(t), d2)
    assert abs(F1 - F2) < 1e-12 * F1
    assert np.max(np.abs(gp1 - gp2)) < 1e-11 and np.max(np.abs(gq1 - gq2)) < 1e-11


def test_c_and_numpy_agree():
    g, psi, q, s, sp, d, rs, dr = case(L=32, N=16)
    Fc, gpc, gqc = oracle.grad_full(g, psi, q, s, sp, d, rs, dr)
    Fn, gpn, gqn = npo.Problem(g, 32, 16).grad_full(psi, q, s, sp, d, rs, dr)
    assert abs(Fc - Fn) < 1e-12 * Fc
    assert np.linalg.norm(gpc - gpn) < 1e-12 * np.linalg.norm(gpn)
    assert np.linalg.norm(gqc - gqn) < 1e-12 * np.linalg.norm(gqn)
