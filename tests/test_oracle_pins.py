"""Pins of the fp64 oracle (oracle/) to what the paper and the mathematics fix.

Every test here checks the oracle against something other than itself: values the
paper prints (tests/golden/, cited), closed forms, invariants stated in the paper,
special cases that reduce to a textbook routine (numpy), brute force on tiny
inputs (explicit matrices, finite differences).  CPU only.
"""
import json
import os

import numpy as np
import pytest

import oracle
from oracle import np_oracle as npo
from oracle import cg as ocg
import synth

GOLD = os.path.join(os.path.dirname(__file__), "golden")
RNG = np.random.default_rng(20240720)


def crand(*shape):
    return RNG.standard_normal(shape) + 1j * RNG.standard_normal(shape)


def rel(a, b):
    return np.linalg.norm(np.ravel(a - b)) / max(np.linalg.norm(np.ravel(b)), 1e-300)


def cfg_geometry(cfg):
    return oracle.Geometry(cfg.wavelength, cfg.Z, cfg.z1, cfg.det_pixel)


# --------------------------------------------------------------------- O1 --
def test_o1_table1_magnifications():
    """m_j = Z/z1_j reproduces Table 1's printed magnifications and pixel sizes."""
    t = json.load(open(os.path.join(GOLD, "table1.json")))
    z1 = np.array(t["z1_mm"]) * 1e-3
    g = oracle.Geometry(t["wavelength_m_printed"], t["focus_to_detector_m"], z1, t["binned_detector_pixel_m"])
    m = g.m0 / g.mt  # m_j = Z / z1_j = m0 / mt_j
    for mj, printed, tol in zip(m, t["magnifications_printed"], t["magnifications_half_ulp"]):
        assert abs(mj - printed) <= tol
    assert abs(g.p0 * 1e9 - t["object_pixel_nm_printed"]) <= 0.5
    gs = oracle.Geometry(t["wavelength_m_printed"], t["focus_to_detector_m"], z1, t["synthetic_detector_pixel_m"])
    assert abs(gs.p0 * 1e9 - t["synthetic_voxel_nm_printed"]) <= 0.5


@pytest.mark.parametrize("cfg", ["cfg0", "cfg1", "table1"])
def test_o1_effective_distance_identity(cfg):
    """zdet_j + omega_j = zeta_0 (algebra of Eq. (8)/Thm 2; the psi=1 consistency check P:101-102)."""
    if cfg == "table1":
        g = oracle.Geometry(7.27183e-11, 1.208, np.array([4.026, 4.199, 4.890, 6.325]) * 1e-3, 3e-6)
    else:
        g = cfg_geometry(synth.CONFIGS[cfg])
    assert np.allclose(g.zdet + g.omega, g.zeta[0], rtol=1e-14, atol=0)
    assert g.mt[0] == 1.0 and g.omega[0] == 0.0
    # zeta_j = z1 z2 / Z directly (Eq. (6))
    z1 = g.z1
    assert np.allclose(g.zeta, z1 * (g.Z - z1) / g.Z, rtol=1e-15)


def test_o1_rejects_bad_geometry():
    with pytest.raises(ValueError):
        oracle.Geometry(1e-10, 1.0, [2e-3, 1e-3], 1e-6)
    with pytest.raises(ValueError):
        oracle.Geometry(1e-10, 1.0, [2e-3, 2.0], 1e-6)


# --------------------------------------------------------------------- O2 --
@pytest.mark.parametrize("L", [16, 128, 6144])
def test_o2_dft_matches_numpy(L):
    x = crand(L)
    assert rel(oracle.dft1(x), np.fft.fft(x)) < 1e-12
    assert rel(oracle.dft1(x, inverse=True), np.fft.ifft(x)) < 1e-12
    X = oracle.dft1(x)
    assert abs(np.vdot(X, X).real / L - np.vdot(x, x).real) / np.vdot(x, x).real < 1e-12  # Parseval


# --------------------------------------------------------------------- O3 --
G1 = cfg_geometry(synth.CONFIGS["cfg1"])


@pytest.mark.parametrize("impl", ["c", "np"])
def test_o3_propagation_invariants(impl):
    P = oracle.prop if impl == "c" else npo.prop
    L = 64
    x, y = crand(L, L), crand(L, L)
    lam, p0 = G1.wavelength, G1.p0
    assert rel(P(x, lam, p0, 0.0), x) < 1e-13                                   # z = 0 -> identity
    assert abs(np.linalg.norm(P(x, lam, p0, 3e-3)) / np.linalg.norm(x) - 1) < 1e-13  # unitarity
    assert rel(P(P(x, lam, p0, 1e-3), lam, p0, 2.5e-3), P(x, lam, p0, 3.5e-3)) < 1e-13  # semigroup
    lhs = np.vdot(y, P(x, lam, p0, 2e-3))
    rhs = np.vdot(P(y, lam, p0, -2e-3), x)                                      # P_z^* = P_{-z}
    assert abs(lhs - rhs) / abs(lhs) < 1e-13


@pytest.mark.parametrize("impl", ["c", "np"])
def test_o3_gaussian_beam_closed_form(impl):
    """x = exp(-|u|^2/(2 s^2)) -> P_z x = (s^2/s_z^2) exp(-|u|^2/(2 s_z^2)), s_z^2 = s^2 + i lambda z/(2 pi p0^2) [px^2]."""
    P = oracle.prop if impl == "c" else npo.prop
    L, s, p0, lam = 256, 8.0, 10e-9, 3.717667e-11
    b = 64.0  # lambda z / (2 pi p0^2) in px^2
    z = b * 2 * np.pi * p0 ** 2 / lam
    u = np.arange(L) - L // 2
    r2 = u[:, None] ** 2 + u[None, :] ** 2
    x = np.exp(-r2 / (2 * s * s)).astype(np.complex128)
    sz2 = s * s + 1j * b
    expect = (s * s / sz2) * np.exp(-r2 / (2 * sz2))
    assert rel(P(x, lam, p0, z), expect) < 1e-12


def test_o3_transfer_at_nyquist():
    """A pure Nyquist plane wave is an eigenvector of P_z with eigenvalue h_z(Nyquist, 0)."""
    t = json.load(open(os.path.join(GOLD, "transfer_nyquist.json")))
    L = t["N"]
    n = np.arange(L)
    x = np.tile(np.exp(1j * np.pi * n)[None, :], (L, 1))  # fbar = -L/2 along x, 0 along y
    y = oracle.prop(x, t["wavelength_m"], t["pixel_m"], t["z_m"])
    h = y[3, 5] / x[3, 5]
    assert abs(h - complex(t["value_re"], t["value_im"])) < 1e-8
    assert abs(np.angle(h) + t["phase_rad"]) < 1e-9
    assert rel(y, h * x) < 1e-13


# --------------------------------------------------------------------- O4 --
@pytest.mark.parametrize("impl", ["c", "np"])
def test_o4_shift(impl):
    S = oracle.shift if impl == "c" else npo.shift
    L = 32
    x = crand(L, L)
    assert rel(S(x, 0, 0), x) < 1e-13
    assert rel(S(x, 3, -5), np.roll(np.roll(x, 3, axis=1), -5, axis=0)) < 1e-13   # (S_s x)(u) = x(u - s)
    assert rel(S(S(x, 1.3, -0.7), -1.3, 0.7), x) < 1e-13
    assert abs(np.linalg.norm(S(x, 0.37, 2.2)) / np.linalg.norm(x) - 1) < 1e-13


# --------------------------------------------------------------------- O5 --
MAGS = {"c": (oracle.mag, oracle.mag_adj),
        "np": (lambda x, m, sx=0, sy=0: npo.MagOp(x.shape[0], m).fwd(x, sx, sy),
               lambda y, m, sx=0, sy=0: npo.MagOp(y.shape[0], m).adj(y, sx, sy))}


@pytest.mark.parametrize("impl", ["c", "np"])
def test_o5_identity_and_constant(impl):
    M, _ = MAGS[impl]
    L = 64
    x = crand(L, L)
    assert rel(M(x, 1.0), x) < 1e-13                       # mt = 1, s = 0 -> identity
    assert rel(M(x, 1.0, 2.0, -3.0), np.roll(np.roll(x, 2, 1), -3, 0)) < 1e-13  # mt = 1 -> pure shift
    c = np.full((L, L), 0.7 - 0.2j)
    assert rel(M(c, 1.5248691, 0.3, 1.1), c) < 1e-13       # M S 1 = 1 (kappa keeps DC)


@pytest.mark.parametrize("impl", ["c", "np"])
@pytest.mark.parametrize("mt,s", [(1.2, 1.7), (1.524869, 1.7), (1.197208, -0.6)])
def test_o5_gaussian_dilation(impl, mt, s):
    """output(u) = x(mt u - s) for a band-limited Gaussian (M_m f(x) = f(x/m))."""
    M, _ = MAGS[impl]
    L, sig = 256, 8.0
    u = np.arange(L) - L // 2
    g = lambda t: np.exp(-t ** 2 / (2 * sig * sig))
    x = (g(u)[:, None] * g(u)[None, :]).astype(np.complex128)
    expect = g(mt * u - (-s))[:, None] * g(mt * u - s)[None, :]  # rows are y: sy = -s; columns x: sx = s
    got = M(x, mt, s, -s)
    assert rel(got, expect) < 1e-12


@pytest.mark.parametrize("impl", ["c", "np"])
def test_o5_mt2_textbook_reduction(impl):
    """mt = 2: y[n] = IFFT(FFT(x) kappa)[(2(n - c) + c) mod L], c = L/2 (numpy)."""
    M, _ = MAGS[impl]
    L = 32
    x = crand(L, L)
    fb = np.fft.fftfreq(L, 1.0 / L)
    kap = ((2 * fb >= -L // 2) & (2 * fb < L // 2)).astype(float)
    X = np.fft.fft2(x) * kap[:, None] * kap[None, :]
    xi = np.fft.ifft2(X)
    c = L // 2
    idx = (2 * (np.arange(L) - c) + c) % L
    assert rel(M(x, 2.0), xi[np.ix_(idx, idx)]) < 1e-13


@pytest.mark.parametrize("impl", ["c", "np"])
def test_o5_adjoint_is_explicit_conjugate_transpose(impl):
    """Explicit matrix of M_{1/mt} S_s on a 16 x 16 torus: adjoint == conjugate transpose."""
    M, MA = MAGS[impl]
    L, mt, sx, sy = 16, 1.31, 0.45, -1.2
    A = np.zeros((L * L, L * L), complex)
    B = np.zeros((L * L, L * L), complex)
    for i in range(L * L):
        e = np.zeros(L * L, complex)
        e[i] = 1
        A[:, i] = M(e.reshape(L, L), mt, sx, sy).ravel()
        B[:, i] = MA(e.reshape(L, L), mt, sx, sy).ravel()
    assert np.abs(B - A.conj().T).max() < 1e-13


def test_o5_c_and_numpy_oracles_agree():
    L = 64
    x = crand(L, L)
    for mt in (1.0, 1.03948517, 1.52486911):
        assert rel(oracle.mag(x, mt, 0.3, -1.7), MAGS["np"][0](x, mt, 0.3, -1.7)) < 1e-13
        assert rel(oracle.mag_adj(x, mt, 0.3, -1.7), MAGS["np"][1](x, mt, 0.3, -1.7)) < 1e-13


# ----------------------------------------------------------------- O6, O7 --
def small_problem(L=32, N=16, K=2, cfgname="cfg1"):
    cfg = synth.CONFIGS[cfgname]
    g = cfg_geometry(cfg)
    psi = 1 + 0.3 * crand(K, L, L)
    q = 1 + 0.3 * crand(L, L)
    s = RNG.uniform(-2, 2, size=(K, g.nz, 2))
    return g, psi, q, s, N


def test_o7_psi_one_gives_reference_form():
    """psi = 1 -> w_kj = C(P_{zeta0} q) for every k, j and shift."""
    g, psi, q, s, N = small_problem()
    w = oracle.fwd(g, np.ones_like(psi), q, s, N)
    ref = oracle.crop(oracle.prop(q, g.wavelength, g.p0, g.zeta[0]), N)
    for k in range(w.shape[0]):
        for j in range(g.nz):
            assert rel(w[k, j], ref) < 1e-12


def test_o7_q_one_gives_conventional_form():
    """q = 1 -> w_kj = C(P_{zdet_j} M_{1/mt_j} S psi_k): the conventional conic form (Eq. (7))."""
    g, psi, q, s, N = small_problem()
    w = oracle.fwd(g, psi, np.ones_like(q), s, N)
    for k in range(psi.shape[0]):
        for j in range(g.nz):
            ref = oracle.crop(oracle.prop(oracle.mag(psi[k], g.mt[j], *s[k, j]), g.wavelength, g.p0, g.zdet[j]), N)
            assert rel(w[k, j], ref) < 1e-12


def test_o7_single_plane_reduces_to_fresnel():
    """N_z = 1, mt = 1, s = 0, q = 1: plain Fresnel holography C P_{zeta0} psi (Eq. (1) with d^r = 1)."""
    g = oracle.Geometry(3.717667e-11, 1.208, [4.584e-3], 3e-6)
    L, N = 32, 16
    psi = 1 + 0.3 * crand(1, L, L)
    w = oracle.fwd(g, psi, np.ones((L, L)), np.zeros((1, 1, 2)), N)
    assert rel(w[0, 0], oracle.crop(oracle.prop(psi[0], g.wavelength, g.p0, g.zeta[0]), N)) < 1e-12


def test_o7_dot_tests_L_and_Q():
    """<L psi, y> = <psi, L^* y> and <Q q, y> = <q, Q^* y> over 20 random trials."""
    g, psi, q, s, N = small_problem()
    K = psi.shape[0]
    for _ in range(20):
        dpsi = crand(*psi.shape)
        dq = crand(*q.shape)
        y = crand(K, g.nz, N, N)
        ap, aq = oracle.adj(g, y, psi, q, s)
        Lpsi = oracle.fwd(g, dpsi, q, s, N)  # linear in psi at fixed q
        Qq = oracle.fwd(g, psi, dq, s, N)    # linear in q at fixed psi
        assert abs(np.vdot(y, Lpsi) - np.vdot(ap, dpsi)) / abs(np.vdot(y, Lpsi)) < 1e-12
        assert abs(np.vdot(y, Qq) - np.vdot(aq, dq)) / abs(np.vdot(y, Qq)) < 1e-12


def test_o7_c_and_numpy_forward_agree():
    g, psi, q, s, N = small_problem(L=64, N=32)
    w = oracle.fwd(g, psi, q, s, N)
    pr = npo.Problem(g, 64, 32)
    out = pr.fwd(psi, q, s)
    for (k, j), wk in out.items():
        assert rel(w[k, j], wk) < 1e-12


# --------------------------------------------------------------- O8 - O12 --
def fd_case():
    cfg = synth.CONFIGS["cfg0"]
    g = cfg_geometry(cfg)  # mt = [1, 1.19869], cfg0 distances
    psi, q, s = synth.small_geometry_case(seed=3, L=16, N=8, K=2, nz=g.nz)
    d = np.abs(oracle.fwd(g, 1 + 0.2 * crand(*psi.shape), q * (1 + 0.1 * crand(16, 16)), s, 8)) + 0.05
    return g, psi, q, s, d


@pytest.mark.parametrize("block", ["psi", "q"])
def test_o8_o12_finite_differences(block):
    """[F(x + h v) - F(x - h v)]/(2h) = Re<v, grad F> on a 16^2 torus, fp64."""
    g, psi, q, s, d = fd_case()
    F0, gp, gq = oracle.grad(g, psi, q, s, d)
    h = 1e-6
    for trial in range(3):
        if block == "psi":
            v = crand(*psi.shape)
            Fp = oracle.grad(g, psi + h * v, q, s, d, False, False)[0]
            Fm = oracle.grad(g, psi - h * v, q, s, d, False, False)[0]
            an = np.vdot(gp, v).real
        else:
            v = crand(*q.shape)
            Fp = oracle.grad(g, psi, q + h * v, s, d, False, False)[0]
            Fm = oracle.grad(g, psi, q - h * v, s, d, False, False)[0]
            an = np.vdot(gq, v).real
        fd = (Fp - Fm) / (2 * h)
        assert abs(fd - an) / abs(an) < 1e-6


def test_o8_o12_zero_at_exact_data():
    """Noise-free data generated by the same forward: F = 0 and grad F = 0."""
    g, psi, q, s, _ = fd_case()
    d = np.abs(oracle.fwd(g, psi, q, s, 8))
    F, gp, gq = oracle.grad(g, psi, q, s, d)
    assert F < 1e-24
    assert np.abs(gp).max() < 1e-12 and np.abs(gq).max() < 1e-12


def test_o8_objective_is_plain_sum():
    """F1 = sum over frames and N x N pixels of (|w| - sqrt d)^2, no 1/2, no weights (Eq. (10))."""
    g, psi, q, s, d = fd_case()
    w = oracle.fwd(g, psi, q, s, 8)
    F = oracle.grad(g, psi, q, s, d, False, False)[0]
    assert abs(F - np.sum((np.abs(w) - d) ** 2)) / F < 1e-13


def test_o12_c_and_numpy_gradients_agree():
    g, psi, q, s, N = small_problem(L=32, N=16)
    d = np.abs(oracle.fwd(g, psi * (1 + 0.2 * crand(*psi.shape)), q, s, N))
    F, gp, gq = oracle.grad(g, psi, q, s, d)
    F2, gp2, gq2 = npo.Problem(g, 32, 16).grad(psi, q, s, d)
    assert abs(F - F2) / F < 1e-12 and rel(gp, gp2) < 1e-12 and rel(gq, gq2) < 1e-12


# -------------------------------------------------------------------- O14 --
def test_o14_reference_arm_matches_main_chain():
    """w^r = C P_{zeta0} S_{s_r} q equals the main chain at psi = 1 with q replaced by S_{s_r} q."""
    g, psi, q, s, N = small_problem()
    rs = RNG.uniform(-3, 3, size=(3, 2))
    d = np.abs(crand(3, N, N)) + 0.1
    Fr, gq = oracle.grad_ref(g, q, rs, d)
    Fm, gqm = 0.0, np.zeros_like(q)
    for r in range(3):
        sq = oracle.shift(q, *rs[r])
        g1 = oracle.Geometry(g.wavelength, g.Z, g.z1[:1], g.detector_pixel)
        F1, _, gq1 = oracle.grad(g1, np.ones((1,) + q.shape), sq, np.zeros((1, 1, 2)), d[r][None, None])
        Fm += F1
        gqm += oracle.shift(gq1, -rs[r][0], -rs[r][1])
    assert abs(Fr - Fm) / Fm < 1e-12 and rel(gq, gqm) < 1e-12


def test_o14_reference_arm_finite_difference():
    g, psi, q, s, N = small_problem(L=16, N=8)
    rs = RNG.uniform(-3, 3, size=(2, 2))
    d = np.abs(crand(2, N, N)) + 0.1
    F0, gq = oracle.grad_ref(g, q, rs, d)
    v, h = crand(*q.shape), 1e-6
    fd = (oracle.grad_ref(g, q + h * v, rs, d, False)[0] - oracle.grad_ref(g, q - h * v, rs, d, False)[0]) / (2 * h)
    assert abs(fd - np.vdot(gq, v).real) / abs(fd) < 1e-6


# -------------------------------------------------------------------- O13 --
def test_o13_first_direction_is_steepest_descent():
    g = [crand(4), crand(3)]
    eta, beta, reset = ocg.dai_yuan_direction(g, None, None, [1.0, 0.5])
    assert reset and np.allclose(eta[0], -g[0]) and np.allclose(eta[1], -0.5 * g[1])


def test_o13_dai_yuan_quadratic_terminates():
    """Exact line search on a convex quadratic in R^n: Dai-Yuan CG terminates in <= n steps (Dai-Yuan '99)."""
    n = 8
    A = RNG.standard_normal((n, n))
    A = A @ A.T + n * np.eye(n)
    b = RNG.standard_normal(n)
    x = np.zeros(n)
    grad = lambda x: A @ x - b
    g_prev = eta_prev = None
    g = grad(x)
    for m in range(n):
        eta, _, _ = ocg.dai_yuan_direction([g.astype(complex)], None if g_prev is None else [g_prev.astype(complex)],
                                           eta_prev, [1.0])
        e = eta[0].real
        gamma = -(g @ e) / (e @ A @ e)
        x = x + gamma * e
        g_prev, g, eta_prev = g, grad(x), [e.astype(complex)]
        if np.linalg.norm(g) < 1e-10 * np.linalg.norm(b):
            break
    assert np.linalg.norm(grad(x)) < 1e-9 * np.linalg.norm(b)
    assert m <= n - 1


def test_o13_equal_gradient_guard_resets():
    """den = Re<g - g_prev, eta_prev> = 0 -> steepest descent."""
    g = [crand(5)]
    eta, beta, reset = ocg.dai_yuan_direction(g, g, [crand(5)], [1.0])
    assert reset and np.allclose(eta[0], -g[0])


def _cfg0_instance():
    cfg = synth.CONFIGS["cfg0"]
    g = cfg_geometry(cfg)
    psi_t = synth.psi_stack(cfg).numpy()
    q_t = synth.probe(cfg).numpy()
    s = synth.shifts(cfg)
    w = oracle.fwd(g, psi_t, q_t, s, cfg.n)
    return cfg, g, psi_t, q_t, s, w


def test_o13_monotone_objective_cfg0():
    """F is non-increasing over CG iterations -- cfg0, 25 iterations."""
    cfg, g, psi_t, q_t, s, w = _cfg0_instance()
    d = synth.poisson_amplitude(np.abs(w) ** 2, cfg.photons, cfg)
    sweep = lambda x: (lambda r: (r[0], [r[1], r[2]]))(oracle.grad(g, x[0], x[1], s, d))
    x0 = [np.ones_like(psi_t), q_t * 0.9]
    _, hist = ocg.run(sweep, x0, [1.0, 1.0 / (cfg.n_angles * cfg.nz)], 25)
    F = [h["F"] for h in hist]
    assert all(b <= a for a, b in zip(F, F[1:]))
    assert F[-1] < 0.5 * F[0]


def test_o13_truth_is_a_fixed_point():
    """Starting at the noise-free truth CG stays there: F stays at the rounding floor."""
    cfg, g, psi_t, q_t, s, w = _cfg0_instance()
    d = np.abs(w)
    sweep = lambda x: (lambda r: (r[0], [r[1], r[2]]))(oracle.grad(g, x[0], x[1], s, d))
    x, hist = ocg.run(sweep, [psi_t, q_t], [1.0, 1.0], 2, max_halvings=3)
    assert all(h["F"] < 1e-20 for h in hist)
    assert rel(x[0], psi_t) < 1e-10 and rel(x[1], q_t) < 1e-10


def test_o14_numpy_reference_arm_equals_c_oracle():
    """np_oracle.grad_ref (numpy.fft DFT) against the naive-DFT C oracle's O14 (R = 3, ragged shifts)."""
    from oracle import np_oracle as npo
    cfg = synth.CONFIGS["cfg4"]
    g = oracle.Geometry(cfg.wavelength, cfg.Z, cfg.z1, cfg.det_pixel)
    L, N, R = 32, 16, 3
    rng = np.random.default_rng(14)
    q = 1 + 0.2 * (rng.standard_normal((L, L)) + 1j * rng.standard_normal((L, L)))
    rs = rng.uniform(-5, 5, size=(R, 2))
    d = np.abs(rng.standard_normal((R, N, N)))
    Fc, gc = oracle.grad_ref(g, q, rs, d)
    Fn, gn = npo.grad_ref(g.wavelength, g.p0, g.zeta[0], q, rs, d)
    assert abs(Fn - Fc) / Fc < 1e-12
    assert rel(gn, gc) < 1e-11


def test_f2_intensity_objective_finite_differences():
    """F_2 (tau = 2, Eq. (9)) in the numpy oracle: central finite differences of F_2
    in psi and q directions equal Re<v, grad F_2> (App. A.3 proposition), and F_2 = 0, grad = 0
    at exact intensity data."""
    cfg = synth.CONFIGS["cfg0"]
    g = oracle.Geometry(cfg.wavelength, cfg.Z, cfg.z1, cfg.det_pixel)
    L, N, K = 16, 8, 2
    rng = np.random.default_rng(22)
    psi = np.exp(1j * 0.3 * rng.standard_normal((K, L, L)))
    q = 1 + 0.2 * (rng.standard_normal((L, L)) + 1j * rng.standard_normal((L, L)))
    s = rng.uniform(-2, 2, size=(K, 2, 2))
    pr = npo.Problem(g, L, N)
    out = pr.fwd(psi, q, s)
    d_exact = np.stack([np.stack([np.abs(out[(k, j)]) for j in range(2)]) for k in range(K)])
    F0, gp0, gq0 = pr.grad(psi, q, s, d_exact, tau=2)
    assert F0 < 1e-20 and np.abs(gp0).max() < 1e-10 and np.abs(gq0).max() < 1e-10
    d = d_exact * (1 + 0.3 * rng.standard_normal(d_exact.shape))
    F, gp, gq = pr.grad(psi, q, s, d, tau=2)
    h = 1e-6
    vp = rng.standard_normal(psi.shape) + 1j * rng.standard_normal(psi.shape)
    fd = (pr.grad(psi + h * vp, q, s, d, tau=2)[0] - pr.grad(psi - h * vp, q, s, d, tau=2)[0]) / (2 * h)
    assert abs(fd - np.vdot(gp, vp).real) / abs(fd) < 1e-6
    vq = rng.standard_normal(q.shape) + 1j * rng.standard_normal(q.shape)
    fd = (pr.grad(psi, q + h * vq, s, d, tau=2)[0] - pr.grad(psi, q - h * vq, s, d, tau=2)[0]) / (2 * h)
    assert abs(fd - np.vdot(gq, vq).real) / abs(fd) < 1e-6


def test_f2_reference_arm_finite_differences():
    """F_2 reference term (Eq. (9)) in np_oracle.grad_ref: central differences vs Re<v, grad>."""
    cfg = synth.CONFIGS["cfg4"]
    g = oracle.Geometry(cfg.wavelength, cfg.Z, cfg.z1, cfg.det_pixel)
    L, N, R = 32, 16, 2
    rng = np.random.default_rng(23)
    q = 1 + 0.2 * (rng.standard_normal((L, L)) + 1j * rng.standard_normal((L, L)))
    rs = rng.uniform(-5, 5, size=(R, 2))
    d = np.abs(rng.standard_normal((R, N, N)))
    F, gq = npo.grad_ref(g.wavelength, g.p0, g.zeta[0], q, rs, d, tau=2)
    h = 1e-6
    v = rng.standard_normal(q.shape) + 1j * rng.standard_normal(q.shape)
    Fp = npo.grad_ref(g.wavelength, g.p0, g.zeta[0], q + h * v, rs, d, False, tau=2)[0]
    Fm = npo.grad_ref(g.wavelength, g.p0, g.zeta[0], q - h * v, rs, d, False, tau=2)[0]
    fd = (Fp - Fm) / (2 * h)
    assert abs(fd - np.vdot(gq, v).real) / abs(fd) < 1e-6


@pytest.mark.parametrize("tau", [0.5, 1.5, 3.0])
def test_g_tau_objective_finite_differences(tau):
    """General penalty G_tau (App. A.3) in the numpy oracle: central finite differences
    of G_tau in psi and q directions equal Re<v, 2 L^*(h'(|Lpsi|^2) Lpsi)> (the proposition), and
    G_tau = 0, grad = 0 at exact data."""
    cfg = synth.CONFIGS["cfg0"]
    g = oracle.Geometry(cfg.wavelength, cfg.Z, cfg.z1, cfg.det_pixel)
    L, N, K = 16, 8, 2
    rng = np.random.default_rng(31)
    psi = np.exp(1j * 0.3 * rng.standard_normal((K, L, L)))
    q = 1 + 0.2 * (rng.standard_normal((L, L)) + 1j * rng.standard_normal((L, L)))
    s = rng.uniform(-2, 2, size=(K, 2, 2))
    pr = npo.Problem(g, L, N)
    out = pr.fwd(psi, q, s)
    d_exact = np.stack([np.stack([np.abs(out[(k, j)]) for j in range(2)]) for k in range(K)])
    F0, gp0, gq0 = pr.grad(psi, q, s, d_exact, tau=tau)
    assert F0 < 1e-20 and np.abs(gp0).max() < 1e-10 and np.abs(gq0).max() < 1e-10
    d = d_exact * np.abs(1 + 0.3 * rng.standard_normal(d_exact.shape))
    F, gp, gq = pr.grad(psi, q, s, d, tau=tau)
    h = 1e-6
    vp = rng.standard_normal(psi.shape) + 1j * rng.standard_normal(psi.shape)
    fd = (pr.grad(psi + h * vp, q, s, d, tau=tau)[0] - pr.grad(psi - h * vp, q, s, d, tau=tau)[0]) / (2 * h)
    assert abs(fd - np.vdot(gp, vp).real) / abs(fd) < 1e-6
    vq = rng.standard_normal(q.shape) + 1j * rng.standard_normal(q.shape)
    fd = (pr.grad(psi, q + h * vq, s, d, tau=tau)[0] - pr.grad(psi, q - h * vq, s, d, tau=tau)[0]) / (2 * h)
    assert abs(fd - np.vdot(gq, vq).real) / abs(fd) < 1e-6


def test_g_tau_reduces_to_f1_f2():
    """G_tau at tau = 1 is F_1 (Eq. (10)) and at tau = 2 is F_2 (Eq. (9)), App. A.3 ("we retrieve the
    main terms ... by setting tau equal to 2 and 1"): the general residual equals the two dedicated
    branches (both pinned by finite differences above), also at w = 0 (reading C7)."""
    rng = np.random.default_rng(32)
    w = rng.standard_normal((8, 8)) + 1j * rng.standard_normal((8, 8))
    w[0, 0] = 0
    a = np.abs(rng.standard_normal((8, 8)))
    F1, r1 = npo.residual_tau(w, a, 1.0)
    m = np.abs(w)
    assert abs(F1 - np.sum((m - a) ** 2)) < 1e-12 * F1
    assert np.abs(r1 - np.where(m > 0, w - a * w / np.where(m > 0, m, 1), 0)).max() < 1e-13
    F2, r2 = npo.residual_tau(w, a, 2.0)
    assert abs(F2 - np.sum((m ** 2 - a ** 2) ** 2)) < 1e-12 * F2
    assert np.abs(r2 - 2 * (m ** 2 - a ** 2) * w).max() < 1e-12


@pytest.mark.parametrize("tau", [0.5, 1.5])
def test_g_tau_reference_arm_finite_differences(tau):
    """G_tau reference term in np_oracle.grad_ref: central differences vs Re<v, grad>."""
    cfg = synth.CONFIGS["cfg4"]
    g = oracle.Geometry(cfg.wavelength, cfg.Z, cfg.z1, cfg.det_pixel)
    L, N, R = 32, 16, 2
    rng = np.random.default_rng(33)
    q = 1 + 0.2 * (rng.standard_normal((L, L)) + 1j * rng.standard_normal((L, L)))
    rs = rng.uniform(-5, 5, size=(R, 2))
    d = np.abs(rng.standard_normal((R, N, N)))
    F, gq = npo.grad_ref(g.wavelength, g.p0, g.zeta[0], q, rs, d, tau=tau)
    h = 1e-6
    v = rng.standard_normal(q.shape) + 1j * rng.standard_normal(q.shape)
    Fp = npo.grad_ref(g.wavelength, g.p0, g.zeta[0], q + h * v, rs, d, False, tau=tau)[0]
    Fm = npo.grad_ref(g.wavelength, g.p0, g.zeta[0], q - h * v, rs, d, False, tau=tau)[0]
    fd = (Fp - Fm) / (2 * h)
    assert abs(fd - np.vdot(gq, v).real) / abs(fd) < 1e-6
