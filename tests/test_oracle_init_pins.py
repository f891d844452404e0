"""Pins of the initialiser oracles: O17 init_probe (the reference image
propagated back to sample plane 0, P:147/P:241/P:272) and O18 multi-distance Paganin (P:147,
SPEC's documented stand-in; reading R4).  Both oracles (C naive DFT sums, numpy FFT) are checked
against closed forms and special cases, and against each other.
"""
import numpy as np
import pytest

import oracle
import synth
from oracle import np_oracle as npo


def geom():
    cfg = synth.CONFIGS["cfg1"]
    return oracle.Geometry(cfg.wavelength, cfg.Z, cfg.z1, cfg.det_pixel)


@pytest.mark.parametrize("impl", ["c", "np"])
def test_init_probe_flat_reference_is_constant(impl):
    """SPEC's trivial example: a flat reference sqrt(d~r) = c gives q0 = c (zero phase, R3 ring)."""
    g = geom()
    L, N, R = 32, 16, 3
    a = np.full((R, N, N), 1.7)
    rs = np.random.default_rng(1).uniform(-4, 4, (R, 2))
    q0 = oracle.init_probe(g, rs, a, L) if impl == "c" else npo.init_probe(g.wavelength, g.p0, g.zeta[0], rs, a, L)
    assert np.max(np.abs(q0 - 1.7)) < 1e-12


def test_init_probe_undoes_integer_shifts():
    """Full-torus frames (N = L) that are integer rolls of one amplitude b: every back-propagated,
    back-shifted frame equals P_{-zeta0} b, so q0 = P_{-zeta0} b (O3's own propagator)."""
    g = geom()
    L = 32
    rng = np.random.default_rng(2)
    b = 1 + 0.3 * rng.uniform(size=(L, L))
    rs = np.array([[0, 0], [3, -2], [-5, 7], [1, 1]], float)
    a = np.stack([np.roll(b, (int(s[1]), int(s[0])), axis=(0, 1)) for s in rs])  # (S_s b)(u) = b(u - s)
    ref = oracle.prop(b, g.wavelength, g.p0, -g.zeta[0])
    for q0 in (oracle.init_probe(g, rs, a, L), npo.init_probe(g.wavelength, g.p0, g.zeta[0], rs, a, L)):
        assert np.max(np.abs(q0 - ref)) < 1e-12


def test_init_probe_c_equals_numpy():
    g = geom()
    rng = np.random.default_rng(3)
    a = rng.uniform(0.5, 1.5, (2, 12, 12))
    rs = rng.uniform(-3, 3, (2, 2))
    qc = oracle.init_probe(g, rs, a, 32)
    qn = npo.init_probe(g.wavelength, g.p0, g.zeta[0], rs, a, 32)
    assert np.linalg.norm(qc - qn) < 1e-12 * np.linalg.norm(qn)


def _tie_intensity(T, L, g, zeta, delta_beta):
    """The linear TIE (Paganin) model Paganin's filter inverts exactly: I = IDFT2(DFT2(T)(1 + pi lambda zeta db |f|^2))."""
    fb = npo.fbar(L) / (L * g.p0)
    f2 = fb[:, None] ** 2 + fb[None, :] ** 2
    return np.real(np.fft.ifft2(np.fft.fft2(T) * (1 + np.pi * g.wavelength * zeta * delta_beta * f2)))


def _periodic_phase(L, amp=0.03):
    """A low-order trigonometric phase (f = 1 and (2, 1) cycles per torus): exp(2 phi / db) stays
    positive under the TIE model while the |f|^2 term of the filter (factors ~5 and ~21 here) matters."""
    y, x = np.meshgrid(np.arange(L), np.arange(L), indexing="ij")
    return amp * (np.cos(2 * np.pi * x / L) + np.cos(2 * np.pi * y / L)) + amp / 3 * np.cos(2 * np.pi * (2 * x + y) / L)


def _bump_phase(L, amp=-0.01, sigma=6.0):
    """A small centred bump, ~0 within 5 sigma of the torus edge (so compressing the torus by mt <= 1.53
    only wraps the flat part)."""
    y, x = np.meshgrid(np.arange(L) - L / 2, np.arange(L) - L / 2, indexing="ij")
    return amp * np.exp(-(x ** 2 + (1.3 * y) ** 2) / (2 * sigma ** 2))


@pytest.mark.parametrize("impl", ["c", "np"])
def test_multipaganin_flat_data_gives_unit_object(impl):
    g = geom()
    L, N = 32, 16
    d = np.full((g.nz, N, N), 0.8)
    s = np.random.default_rng(4).uniform(-2, 2, (g.nz, 2))
    f = oracle.multipaganin if impl == "c" else (lambda *a: npo.multipaganin(*a))
    psi0 = f(g, L, s, d, np.full((N, N), 0.8), 100.0)
    assert np.max(np.abs(psi0 - 1.0)) < 1e-12


@pytest.mark.parametrize("impl", ["c", "np"])
def test_multipaganin_inverts_tie_model_single_plane(impl):
    """N_z = 1 (mt = 1), no padding (N = L), no shift: classic Paganin inverts the TIE model exactly,
    so phi and psi0 = exp((i + 1/db) phi) are recovered to fp64 rounding."""
    cfg = synth.CONFIGS["cfg1"]
    g = oracle.Geometry(cfg.wavelength, cfg.Z, cfg.z1[:1], cfg.det_pixel)
    L, db = 32, 1.0
    phi = _periodic_phase(L)
    T = np.exp(2 * phi / db)
    I1 = _tie_intensity(T, L, g, g.zeta[0], db)
    assert I1.min() > 0
    f = oracle.multipaganin if impl == "c" else (lambda *a: npo.multipaganin(*a))
    psi0 = f(g, L, np.zeros((1, 2)), np.sqrt(I1)[None], np.ones((L, L)), db)
    assert np.max(np.abs(psi0 - np.exp((1j + 1 / db) * phi))) < 1e-10


def test_multipaganin_combines_magnified_planes():
    """Four planes of the cfg1 geometry, each datum the plane-j TIE intensity compressed by O5's
    M_{1/mt_j} (the data frame): the oracle's demagnification + multi-distance filter returns phi.
    Approximate only through the compressed torus's seam and the TIE linearisation (measured 1.5e-5): 1e-4."""
    g = geom()
    L, db = 64, 1.0
    phi = _bump_phase(L)
    T = np.exp(2 * phi / db)
    d = np.stack([np.sqrt(np.abs(npo.MagOp(L, g.mt[j]).fwd(_tie_intensity(T, L, g, g.zeta[j], db), 0, 0)))
                  for j in range(g.nz)])
    psi_c = oracle.multipaganin(g, L, np.zeros((g.nz, 2)), d, np.ones((L, L)), db)
    psi_n = npo.multipaganin(g, L, np.zeros((g.nz, 2)), d, np.ones((L, L)), db)
    assert np.linalg.norm(psi_c - psi_n) < 1e-12 * np.linalg.norm(psi_n)
    err = np.max(np.abs(np.angle(psi_n) - phi)) / np.max(np.abs(phi))
    assert err < 1e-4, err  # measured 1.5e-5
