"""Row a-12 on the GPU: the Dai-Yuan CG step (Eqs. (13)-(14)) through the C ABI
(holo_grad -> holo_q_dots -> holo_cg_step, driven by solver.JointCG) against the O13
oracle (oracle.cg.dai_yuan_direction, steps (i)-(v) in the paper's order) over the fp64 C
oracle's sweeps.  SURVEY 8c protocol: cfg0, all frames, gamma forced equal in both
implementations (fp32 / fp64 accept decisions may differ near ties).

Compared per iteration, element by element: eta_psi, eta_q (the new direction),
psi_trial / q_trial (x + gamma eta, accepted), and the scalars F, beta and
Re<g_{m+1}, eta_m> (the DY numerator of the next step; correlated, no cancellation).
Tolerances: 1e-4 relative (north_star gradient tolerance; eta is built from gradients).
"""
import numpy as np
import pytest
import torch

import oracle
import synth
from oracle import cg as ocg

pytestmark = pytest.mark.gpu

TOL = 1e-4


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.linalg.norm((a - b).ravel()) / np.linalg.norm(b.ravel()))


def dev(x, dt=torch.complex64):
    return torch.as_tensor(np.ascontiguousarray(x)).to(dt).cuda().contiguous()


def host(t):
    torch.cuda.synchronize()
    return t.cpu().numpy().astype(np.complex128 if t.is_complex() else np.float64)


@pytest.mark.parametrize("batch,fourier", [(1, False), (4, False), (4, True)])
def test_cg_two_iterations_cfg0_vs_oracle(batch, fourier):
    """fourier: the psi block is held as DFT2 of the object arrays (holo_set_fourier); the oracle's
    eta_psi is compared through numpy.fft.fft2, psi through JointCG.psi (converted back)."""
    import paper_2407_20304_b200 as hb
    from paper_2407_20304_b200.solver import JointCG
    cfg = synth.CONFIGS["cfg0"]
    K = 4
    g = oracle.Geometry(cfg.wavelength, cfg.Z, cfg.z1, cfg.det_pixel)
    psi_t = synth.psi_stack(cfg, K=K).numpy()
    q_t = synth.probe(cfg).numpy()
    s = synth.shifts(cfg, K=K)
    d = synth.poisson_amplitude(np.abs(oracle.fwd(g, psi_t, q_t, s, cfg.n)) ** 2, cfg.photons, cfg)
    rho = [1.0, 1.0 / K]
    x0 = [np.ones_like(psi_t), 0.9 * q_t]
    gam = [0.5, 0.35]

    def sweep(x):
        F, gp, gq = oracle.grad(g, x[0], x[1], s, d)
        return F, [gp, gq]

    # ---- oracle, step by step (O13 (i)-(v))
    F0, g0 = sweep(x0)
    eta0, beta0, _ = ocg.dai_yuan_direction(g0, None, None, rho)
    x1 = [a + gam[0] * e for a, e in zip(x0, eta0)]
    F1, g1 = sweep(x1)
    eta1, beta1, reset1 = ocg.dai_yuan_direction(g1, g0, eta0, rho)
    assert not reset1 and beta1 != 0.0  # the second step really is a DY step
    x2 = [a + gam[1] * e for a, e in zip(x1, eta1)]
    F2, g2 = sweep(x2)
    assert np.linalg.norm(np.abs(oracle.fwd(g, *x2, s, cfg.n)) - d) / np.linalg.norm(d) > 0.05  # not converged

    # ---- GPU
    plan = hb.Plan(cfg.n, cfg.npad, cfg.z1, K, cfg.wavelength, cfg.Z, cfg.det_pixel, device=0, angle_batch=batch)
    plan.set_shifts(s)
    cg = JointCG(plan, dev(d, torch.float32), dev(x0[0]), dev(x0[1]), rho_psi=rho[0], rho_q=rho[1],
                 distributed=False, fourier=fourier)
    assert cg.fourier == fourier
    Fd = (lambda a: np.fft.fft2(a, axes=(-2, -1))) if fourier else (lambda a: a)
    assert abs(cg.start() - F0) / F0 < TOL
    h1 = cg.iterate(forced_gamma=gam[0])
    assert abs(h1["F"] - F1) / F1 < TOL and h1["beta"] == 0.0 and h1["reset"]
    assert rel(host(cg.eta_psi), Fd(eta0[0])) < TOL and rel(host(cg.eta_q), eta0[1]) < TOL
    assert rel(host(cg.psi), x1[0]) < TOL and rel(host(cg.q), x1[1]) < TOL
    ge = ocg.rdot(g1, eta0)  # Re<g_1, eta_0> (psi + q blocks), from the fused sweep scalars
    assert abs(cg.g_eta - ge) / abs(ge) < TOL
    h2 = cg.iterate(forced_gamma=gam[1])
    assert abs(h2["beta"] - beta1) / abs(beta1) < TOL and not h2["reset"]
    assert abs(h2["F"] - F2) / F2 < TOL
    assert rel(host(cg.eta_psi), Fd(eta1[0])) < TOL and rel(host(cg.eta_q), eta1[1]) < TOL
    assert rel(host(cg.psi), x2[0]) < TOL and rel(host(cg.q), x2[1]) < TOL
    assert abs(cg.g_eta - ocg.rdot(g2, eta1)) / abs(ocg.rdot(g2, eta1)) < TOL


def test_cg_step_guards_and_retry():
    """holo_cg_step scalar rule (O13 (i)-(ii)) and the line-search retry (reuse_eta) on the GPU."""
    import paper_2407_20304_b200 as hb
    cfg = synth.CONFIGS["cfg0"]
    plan = hb.Plan(cfg.n, cfg.npad, cfg.z1, 2, cfg.wavelength, cfg.Z, cfg.det_pixel, device=0)
    L = cfg.npad
    rng = np.random.default_rng(3)
    c = lambda *sh: rng.standard_normal(sh) + 1j * rng.standard_normal(sh)
    psi, ep, gp = c(2, L, L), c(2, L, L), c(2, L, L)
    q, eq, gq = c(L, L), c(L, L), c(L, L)
    T = [dev(a) for a in (psi, ep, gp, q, eq, gq)]
    pt, qt = torch.empty_like(T[0]), torch.empty_like(T[3])
    rp, rq = 1.0, 0.25
    gPg = rp * np.vdot(gp, gp).real + rq * np.vdot(gq, gq).real
    # (i) DY step: den = Re<g, eta> - Re<g_prev, eta_prev>
    g_eta, gprev_eta = -0.3 * gPg, -0.9 * gPg
    out = plan.cg_step(hb.HoloCgIn(gPg, g_eta, gprev_eta, 0.7, rp, rq, 0, 0), T[0], T[1], T[2], pt, T[3], T[4],
                       T[5], qt)
    beta = gPg / (g_eta - gprev_eta)
    assert abs(out.beta - beta) <= 1e-15 * beta and not out.reset
    assert abs(out.g_eta_new - (-gPg + beta * g_eta)) <= 1e-12 * gPg
    assert rel(host(T[1]), -rp * gp + beta * ep) < 1e-6 and rel(host(T[4]), -rq * gq + beta * eq) < 1e-6
    assert rel(host(pt), psi + 0.7 * (-rp * gp + beta * ep)) < 1e-6
    assert rel(host(qt), q + 0.7 * (-rq * gq + beta * eq)) < 1e-6
    # retry with the same direction (reuse_eta): only x_trial changes
    e_before = host(T[1])
    plan.cg_step(hb.HoloCgIn(0, 0, 0, 0.35, rp, rq, 0, 1), T[0], T[1], None, pt, T[3], T[4], None, qt)
    assert np.array_equal(host(T[1]), e_before)
    assert rel(host(pt), psi + 0.35 * e_before) < 1e-6
    # (ii) ascent guard: beta = 1/0.3, Re<g, eta_new> = (-1 + 0.5/0.3) gPg >= 0 -> steepest descent, reset
    out = plan.cg_step(hb.HoloCgIn(gPg, 0.5 * gPg, 0.2 * gPg, 1.0, rp, rq, 0, 0), T[0], T[1], T[2], pt, T[3],
                       T[4], T[5], qt)
    assert out.reset and out.beta == 0.0 and out.g_eta_new == -gPg
    assert rel(host(T[1]), -rp * gp) < 1e-6 and rel(host(T[4]), -rq * gq) < 1e-6
    # (i) equal-gradient guard: |den| < 1e-30 gPg -> steepest descent
    out = plan.cg_step(hb.HoloCgIn(gPg, 0.2 * gPg, 0.2 * gPg, 1.0, rp, rq, 0, 0), T[0], T[1], T[2], pt, T[3],
                       T[4], T[5], qt)
    assert out.reset and out.beta == 0.0


def test_q_dots_full_size_vs_numpy():
    """holo_q_dots at L = 4096 (the cfg3 probe block) vs fp64 numpy: ||g||^2 and Re<g, eta>."""
    import paper_2407_20304_b200 as hb
    cfg = synth.CONFIGS["cfg3"]
    L = cfg.npad
    plan = hb.Plan(cfg.n, L, cfg.z1, 0, cfg.wavelength, cfg.Z, cfg.det_pixel, device=0)
    gen = torch.Generator(device="cuda").manual_seed(11)
    gq = torch.randn(L, L, dtype=torch.complex64, device="cuda", generator=gen)
    eq = (-0.5 * gq + 0.1 * torch.randn(L, L, dtype=torch.complex64, device="cuda", generator=gen)).contiguous()
    out = torch.zeros(2, dtype=torch.float64, device="cuda")
    plan.q_dots(gq, eq, out)
    a = host(gq).astype(np.complex128)
    b = host(eq).astype(np.complex128)
    ref = [np.vdot(a, a).real, np.vdot(b, a).real]
    o = host(out).real
    assert abs(o[0] - ref[0]) / ref[0] < 1e-6
    assert abs(o[1] - ref[1]) / abs(ref[1]) < 1e-6
    plan.q_dots(gq, None, out)
    assert host(out).real[1] == 0.0


@pytest.mark.parametrize("fourier", [False, True])
def test_fused_cg_step_bit_identical(fourier):
    """holo_set_cg_fuse: the psi-block CG update run inside the next sweep's X1 gives the same
    iterates, bit for bit, as the separate pointwise pass (4 iterations with the line search, cfg0)."""
    import paper_2407_20304_b200 as hb
    from paper_2407_20304_b200.solver import JointCG
    cfg = synth.CONFIGS["cfg0"]
    K = 4
    g = oracle.Geometry(cfg.wavelength, cfg.Z, cfg.z1, cfg.det_pixel)
    psi_t = synth.psi_stack(cfg, K=K).numpy()
    q_t = synth.probe(cfg).numpy()
    s = synth.shifts(cfg, K=K)
    d = synth.poisson_amplitude(np.abs(oracle.fwd(g, psi_t, q_t, s, cfg.n)) ** 2, cfg.photons, cfg)
    out = []
    for fuse in (False, True):
        plan = hb.Plan(cfg.n, cfg.npad, cfg.z1, K, cfg.wavelength, cfg.Z, cfg.det_pixel, device=0, angle_batch=2)
        plan.set_shifts(s)
        cg = JointCG(plan, dev(d, torch.float32), dev(np.ones_like(psi_t)), dev(0.9 * q_t), rho_psi=1.0,
                     rho_q=1.0 / K, distributed=False, fourier=fourier, fuse_cg=fuse)
        cg.start()
        hist = [cg.iterate() for _ in range(4)]
        out.append(([(h["F"], h["gamma"], h["beta"]) for h in hist], host(cg.psi), host(cg.q), host(cg.eta_psi)))
    assert out[0][0] == out[1][0]
    for a, b in zip(out[0][1:], out[1][1:]):
        assert np.array_equal(a, b)
