"""GPU (sm_100a, libholo.so through the C ABI) vs the fp64 oracle, element by element.

Tolerances (BASELINE.json north_star): relative L2 error <= 2e-5 on the forward data,
<= 1e-4 on the gradients; F and the DY scalars <= 1e-4 relative (SURVEY 8c protocol).
Parity states are non-converged (|| |w| - sqrt d || / || sqrt d || >= 0.05).
"""
import numpy as np
import pytest
import torch

import oracle
import synth
from oracle import np_oracle as npo

pytestmark = pytest.mark.gpu

TOL_W, TOL_G, TOL_S = 2e-5, 1e-4, 1e-4


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.linalg.norm((a - b).ravel()) / np.linalg.norm(b.ravel()))


def geom(cfg, z1=None):
    return oracle.Geometry(cfg.wavelength, cfg.Z, cfg.z1 if z1 is None else z1, cfg.det_pixel)


def make_plan(cfg, K, L=None, N=None, z1=None, batch=None):
    import paper_2407_20304_b200 as hb
    z1 = cfg.z1 if z1 is None else z1
    return hb.Plan(cfg.n if N is None else N, cfg.npad if L is None else L, z1, K, cfg.wavelength, cfg.Z,
                   cfg.det_pixel, device=0, angle_batch=batch)


def dev(x, dt=torch.complex64):
    return torch.as_tensor(np.ascontiguousarray(x)).to(dt).cuda().contiguous()


def host(t):
    torch.cuda.synchronize()
    return t.cpu().numpy().astype(np.complex128 if t.is_complex() else np.float64)


class Case:
    """Truth from synth, data from the ORACLE forward (never from the GPU), and a
    non-converged evaluation state (psi = 1, q = 0.9 q_truth)."""

    def __init__(self, name, K, oracle_kind="c", noise=True):
        cfg = synth.CONFIGS[name]
        self.cfg, self.K = cfg, K
        self.g = geom(cfg)
        self.psi_t = synth.psi_stack(cfg, K=K).numpy()
        self.q_t = synth.probe(cfg).numpy()
        self.s = synth.shifts(cfg, K=K)
        L, N = cfg.npad, cfg.n
        if oracle_kind == "c":
            w = oracle.fwd(self.g, self.psi_t, self.q_t, self.s, N)
        else:
            pr = npo.Problem(self.g, L, N)
            out = pr.fwd(self.psi_t, self.q_t, self.s)
            w = np.stack([np.stack([out[(k, j)] for j in range(cfg.nz)]) for k in range(K)])
        self.w = w
        self.d = synth.poisson_amplitude(np.abs(w) ** 2, cfg.photons, cfg) if noise else np.abs(w)
        self.psi = np.ones_like(self.psi_t)
        self.q = 0.9 * self.q_t
        self.kind = oracle_kind

    def oracle_grad(self):
        if self.kind == "c":
            return oracle.grad(self.g, self.psi, self.q, self.s, self.d)
        return npo.Problem(self.g, self.cfg.npad, self.cfg.n).grad(self.psi, self.q, self.s, self.d)


def correlated_eta(g, seed=1):
    """eta = -g e^{i phi} (1 + 0.2 n), phi a smooth random phase field in [-0.6, 0.6] rad: a
    descent-like direction near -g (no cancellation in Re<g, eta>), as fp32."""
    rng = np.random.default_rng(seed)
    L = g.shape[-1]
    yy, xx = np.meshgrid(np.arange(L), np.arange(L), indexing="ij")
    phi = 0.6 * np.sin(2 * np.pi * (xx * rng.uniform(1, 3) + yy * rng.uniform(1, 3)) / L + rng.uniform(0, 6.3))
    amp = 1 + 0.2 * rng.standard_normal(g.shape)
    return (-g * np.exp(1j * phi) * amp).astype(np.complex64)


@pytest.fixture(scope="module")
def cfg0():
    return Case("cfg0", 4)


def test_library_loads_and_plan(cfg0):
    p = make_plan(cfg0.cfg, cfg0.K)
    d = p.derived()
    assert np.allclose(d["mt"], cfg0.g.mt, rtol=1e-15) and np.allclose(d["zdet"], cfg0.g.zdet, rtol=1e-15)
    assert np.allclose(d["omega"], cfg0.g.omega, rtol=1e-15) and abs(d["p0"] - cfg0.g.p0) < 1e-22
    assert p.workspace_bytes > 0


def test_cfg0_forward_parity(cfg0):
    c = cfg0
    p = make_plan(c.cfg, c.K)
    p.set_shifts(c.s)
    w = torch.empty(c.K, c.cfg.nz, c.cfg.n, c.cfg.n, dtype=torch.complex64, device="cuda")
    p.fwd(dev(c.psi_t), dev(c.q_t), w)
    wo = oracle.fwd(c.g, c.psi_t, c.q_t, c.s, c.cfg.n)
    assert rel(host(w), wo) < TOL_W


def test_cfg0_gradient_parity(cfg0):
    c = cfg0
    p = make_plan(c.cfg, c.K)
    p.set_shifts(c.s)
    F, gp, gq = c.oracle_grad()
    assert np.linalg.norm(np.abs(oracle.fwd(c.g, c.psi, c.q, c.s, c.cfg.n)) - c.d) / np.linalg.norm(c.d) > 0.05
    # a direction correlated with the gradient (eta = -g with a smooth phase error), as a CG
    # direction is: Re<g, eta> is then a well-conditioned sum and is held to the DY tolerance
    eta = correlated_eta(gp)
    sc = torch.zeros(3, dtype=torch.float64, device="cuda")
    gpsi = torch.empty(c.psi.shape, dtype=torch.complex64, device="cuda")
    gqd = torch.empty(c.q.shape, dtype=torch.complex64, device="cuda")
    p.grad(dev(c.psi), dev(c.q), dev(c.d, torch.float32), sc, dev(eta), gpsi, gqd)
    s = host(sc).real
    assert abs(s[0] - F) / F < TOL_S
    assert rel(host(gpsi), gp) < TOL_G
    assert rel(host(gqd), gq) < TOL_G
    assert abs(s[1] - np.vdot(gp, gp).real) / np.vdot(gp, gp).real < TOL_S
    ge = np.vdot(eta.astype(np.complex128), gp).real
    assert abs(s[2] - ge) / abs(ge) < TOL_S


def test_cfg0_objective_only_matches(cfg0):
    c = cfg0
    p = make_plan(c.cfg, c.K)
    p.set_shifts(c.s)
    import paper_2407_20304_b200 as hb
    sc = torch.zeros(3, dtype=torch.float64, device="cuda")
    p.grad(dev(c.psi), dev(c.q), dev(c.d, torch.float32), sc, flags=hb.HOLO_OBJECTIVE_ONLY)
    F = oracle.grad(c.g, c.psi, c.q, c.s, c.d, False, False)[0]
    assert abs(host(sc).real[0] - F) / F < TOL_S


def test_cfg0_adjoint_parity(cfg0):
    c = cfg0
    p = make_plan(c.cfg, c.K)
    p.set_shifts(c.s)
    rng = np.random.default_rng(5)
    y = rng.standard_normal((c.K, c.cfg.nz, c.cfg.n, c.cfg.n)) + 1j * rng.standard_normal((c.K, c.cfg.nz, c.cfg.n, c.cfg.n))
    ap, aq = oracle.adj(c.g, y, c.psi_t, c.q_t, c.s)
    gap = torch.empty(c.psi.shape, dtype=torch.complex64, device="cuda")
    gaq = torch.empty(c.q.shape, dtype=torch.complex64, device="cuda")
    p.adj(dev(y), dev(c.psi_t), dev(c.q_t), gap, gaq)
    assert rel(host(gap), ap) < TOL_G and rel(host(gaq), aq) < TOL_G


@pytest.mark.parametrize("K", [2, 8])
def test_cfg1_parity_two_angles(K):
    """cfg1 (512^2 torus, 4 planes); K = 8 is SURVEY 8(c)'s "8 angles x 4 distances" (one batch of 8)."""
    c = Case("cfg1", K, oracle_kind="np")
    p = make_plan(c.cfg, c.K)
    p.set_shifts(c.s)
    w = torch.empty(c.K, c.cfg.nz, c.cfg.n, c.cfg.n, dtype=torch.complex64, device="cuda")
    p.fwd(dev(c.psi_t), dev(c.q_t), w)
    pr = npo.Problem(c.g, c.cfg.npad, c.cfg.n)
    out = pr.fwd(c.psi_t, c.q_t, c.s)
    wn = host(w)
    for (k, j), wo in out.items():
        assert rel(wn[k, j], wo) < TOL_W, (k, j)
    F, gp, gq = c.oracle_grad()
    sc = torch.zeros(3, dtype=torch.float64, device="cuda")
    gpsi = torch.empty(c.psi.shape, dtype=torch.complex64, device="cuda")
    gqd = torch.empty(c.q.shape, dtype=torch.complex64, device="cuda")
    p.grad(dev(c.psi), dev(c.q), dev(c.d, torch.float32), sc, None, gpsi, gqd)
    assert abs(host(sc).real[0] - F) / F < TOL_S
    assert rel(host(gpsi), gp) < TOL_G and rel(host(gqd), gq) < TOL_G


@pytest.mark.parametrize("L", [256, 1024])
def test_other_torus_sizes_forward(L):
    """FFT shapes F = 16 (L = 256) and F = 4 (L = 1024), random psi/q, ragged shifts."""
    cfg = synth.CONFIGS["cfg1"]
    N = L // 2
    rng = np.random.default_rng(L)
    K = 1
    psi = 1 + 0.3 * (rng.standard_normal((K, L, L)) + 1j * rng.standard_normal((K, L, L)))
    q = 1 + 0.3 * (rng.standard_normal((L, L)) + 1j * rng.standard_normal((L, L)))
    s = rng.uniform(-3, 3, size=(K, cfg.nz, 2))
    g = geom(cfg)
    p = make_plan(cfg, K, L=L, N=N)
    p.set_shifts(s)
    w = torch.empty(K, cfg.nz, N, N, dtype=torch.complex64, device="cuda")
    p.fwd(dev(psi), dev(q), w)
    out = npo.Problem(g, L, N).fwd(psi, q, s)
    wn = host(w)
    for (k, j), wo in out.items():
        assert rel(wn[k, j], wo) < TOL_W, (k, j)


@pytest.mark.parametrize("name", ["cfg2", "cfg3"])
def test_full_size_one_angle_parity(name):
    """Full torus sizes (2048^2, 4096^2) in the bench's launch configuration, one angle x 4 planes."""
    c = Case(name, 1, oracle_kind="np", noise=False)
    p = make_plan(c.cfg, 1)
    p.set_shifts(c.s)
    w = torch.empty(1, c.cfg.nz, c.cfg.n, c.cfg.n, dtype=torch.complex64, device="cuda")
    p.fwd(dev(c.psi_t), dev(c.q_t), w)
    wn = host(w)
    for j in range(c.cfg.nz):
        assert rel(wn[0, j], c.w[0, j]) < TOL_W, j
    F, gp, gq = c.oracle_grad()
    sc = torch.zeros(3, dtype=torch.float64, device="cuda")
    gpsi = torch.empty(c.psi.shape, dtype=torch.complex64, device="cuda")
    gqd = torch.empty(c.q.shape, dtype=torch.complex64, device="cuda")
    eta = correlated_eta(gp, seed=3)
    p.grad(dev(c.psi), dev(c.q), dev(c.d, torch.float32), sc, dev(eta), gpsi, gqd)
    s = host(sc).real
    assert abs(s[0] - F) / F < TOL_S
    assert rel(host(gpsi), gp) < TOL_G and rel(host(gqd), gq) < TOL_G
    assert abs(s[1] - np.vdot(gp, gp).real) / np.vdot(gp, gp).real < TOL_S
    ge = np.vdot(eta.astype(np.complex128), gp).real
    assert abs(s[2] - ge) / abs(ge) < TOL_S


@pytest.mark.parametrize("batch", [1, 4, 8])
def test_angle_batch_ragged_parity(batch):
    """angle_batch B in {1, 4, 8} on K = 6 angles of cfg1 (4 + 2 ragged for B = 4; B = 8 > K):
    F, grad_psi, grad_q and the fused scalars vs the numpy oracle; also through holo_fwd."""
    c = Case("cfg1", 6, oracle_kind="np")
    p = make_plan(c.cfg, c.K, batch=batch)
    p.set_shifts(c.s)
    w = torch.empty(c.K, c.cfg.nz, c.cfg.n, c.cfg.n, dtype=torch.complex64, device="cuda")
    p.fwd(dev(c.psi_t), dev(c.q_t), w)
    assert rel(host(w), c.w) < TOL_W
    F, gp, gq = c.oracle_grad()
    eta = correlated_eta(gp, seed=batch)
    sc = torch.zeros(3, dtype=torch.float64, device="cuda")
    gpsi = torch.empty(c.psi.shape, dtype=torch.complex64, device="cuda")
    gqd = torch.empty(c.q.shape, dtype=torch.complex64, device="cuda")
    p.grad(dev(c.psi), dev(c.q), dev(c.d, torch.float32), sc, dev(eta), gpsi, gqd)
    s = host(sc).real
    assert abs(s[0] - F) / F < TOL_S
    assert rel(host(gpsi), gp) < TOL_G and rel(host(gqd), gq) < TOL_G
    ge = np.vdot(eta.astype(np.complex128), gp).real
    assert abs(s[2] - ge) / abs(ge) < TOL_S


@pytest.mark.parametrize("K,batch,fourier", [(17, 16, False), (17, 16, True), (7, 3, True), (5, 2, False)])
def test_angle_batch_extremes_parity(K, batch, fourier):
    """The largest angle batch the ABI accepts (16) with a one-angle tail (K = 17), and odd batches with
    ragged tails (7 = 3 + 3 + 1, 5 = 2 + 2 + 1), at cfg1 (512^2 torus, 4 planes): the batched X1 / X3 launches stage the next
    (angle, plane) pair's rows across angle boundaries, so every boundary position is exercised.  F,
    grad_psi, grad_q, the fused scalars vs the numpy oracle, in the object and the Fourier-domain state."""
    c = Case("cfg1", K, oracle_kind="np")
    p = make_plan(c.cfg, c.K, batch=batch)
    p.set_shifts(c.s)
    F, gp, gq = c.oracle_grad()
    eta = correlated_eta(gp, seed=K + batch)
    f2 = (lambda a: np.fft.fft2(a, axes=(-2, -1))) if fourier else (lambda a: a)
    if fourier:
        p.set_fourier(True)
    sc = torch.zeros(3, dtype=torch.float64, device="cuda")
    gpsi = torch.empty(c.psi.shape, dtype=torch.complex64, device="cuda")
    gqd = torch.empty(c.q.shape, dtype=torch.complex64, device="cuda")
    p.grad(dev(f2(c.psi)), dev(c.q), dev(c.d, torch.float32), sc, dev(f2(eta.astype(np.complex128))), gpsi, gqd)
    s = host(sc).real
    assert abs(s[0] - F) / F < TOL_S
    assert rel(host(gpsi), f2(gp)) < TOL_G and rel(host(gqd), gq) < TOL_G
    assert abs(s[1] - np.vdot(gp, gp).real) / np.vdot(gp, gp).real < TOL_S
    ge = np.vdot(eta.astype(np.complex128), gp).real
    assert abs(s[2] - ge) / abs(ge) < TOL_S


def test_accumulate_q_flag(cfg0):
    """HOLO_ACCUMULATE_Q adds the probe-gradient partial into grad_q_part (SURVEY 8b flag)."""
    import paper_2407_20304_b200 as hb
    c = cfg0
    p = make_plan(c.cfg, c.K)
    p.set_shifts(c.s)
    F, gp, gq = c.oracle_grad()
    sc = torch.zeros(3, dtype=torch.float64, device="cuda")
    base = (np.random.default_rng(4).standard_normal(c.q.shape) * (1 + 1j)).astype(np.complex64) * 1e-3
    gqd = dev(base)
    p.grad(dev(c.psi), dev(c.q), dev(c.d, torch.float32), sc, None, None, gqd, flags=hb.HOLO_ACCUMULATE_Q)
    assert rel(host(gqd), gq + base) < TOL_G


@pytest.mark.parametrize("name,K", [("cfg0", 4), ("cfg1", 2)])
def test_intensity_objective_f2_parity(name, K):
    """HOLO_INTENSITY: F_2 (tau = 2, Eq. (9)) and its gradients vs the numpy oracle (tau = 2)."""
    import paper_2407_20304_b200 as hb
    c = Case(name, K, oracle_kind="np")
    p = make_plan(c.cfg, c.K)
    p.set_shifts(c.s)
    F, gp, gq = npo.Problem(c.g, c.cfg.npad, c.cfg.n).grad(c.psi, c.q, c.s, c.d, tau=2)
    sc = torch.zeros(3, dtype=torch.float64, device="cuda")
    gpsi = torch.empty(c.psi.shape, dtype=torch.complex64, device="cuda")
    gqd = torch.empty(c.q.shape, dtype=torch.complex64, device="cuda")
    p.grad(dev(c.psi), dev(c.q), dev(c.d, torch.float32), sc, None, gpsi, gqd, flags=hb.HOLO_INTENSITY)
    assert abs(host(sc).real[0] - F) / F < TOL_S
    assert rel(host(gpsi), gp) < TOL_G and rel(host(gqd), gq) < TOL_G


@pytest.mark.parametrize("name,K,tau", [("cfg0", 4, 1.5), ("cfg0", 4, 0.5), ("cfg1", 2, 3.0)])
def test_g_tau_objective_parity(name, K, tau):
    """holo_set_tau: the general penalty G_tau (App. A.3) and its gradients vs the numpy
    oracle's residual_tau; setting tau back to 1 restores F_1 exactly as before."""
    c = Case(name, K, oracle_kind="np")
    p = make_plan(c.cfg, c.K)
    p.set_shifts(c.s)
    pr = npo.Problem(c.g, c.cfg.npad, c.cfg.n)
    F, gp, gq = pr.grad(c.psi, c.q, c.s, c.d, tau=tau)
    sc = torch.zeros(3, dtype=torch.float64, device="cuda")
    gpsi = torch.empty(c.psi.shape, dtype=torch.complex64, device="cuda")
    gqd = torch.empty(c.q.shape, dtype=torch.complex64, device="cuda")
    p.set_tau(tau)
    p.grad(dev(c.psi), dev(c.q), dev(c.d, torch.float32), sc, None, gpsi, gqd)
    assert abs(host(sc).real[0] - F) / F < TOL_S
    assert rel(host(gpsi), gp) < TOL_G and rel(host(gqd), gq) < TOL_G
    p.set_tau(1.0)
    F1, gp1, gq1 = pr.grad(c.psi, c.q, c.s, c.d)
    p.grad(dev(c.psi), dev(c.q), dev(c.d, torch.float32), sc, None, gpsi, gqd)
    assert abs(host(sc).real[0] - F1) / F1 < TOL_S
    assert rel(host(gpsi), gp1) < TOL_G and rel(host(gqd), gq1) < TOL_G


def test_set_tau_rejects_out_of_range():
    import paper_2407_20304_b200 as hb
    c = synth.CONFIGS["cfg0"]
    p = make_plan(c, 1)
    for bad in (0.0, -1.0, 5.0, float("nan")):
        with pytest.raises(hb.HoloError):
            p.set_tau(bad)
    p.set_tau(2.0)


def test_staged_data_stream_matches_resident():
    """holo_stage_sqrt_d: the data streamed from pinned host memory per angle batch (copy stream,
    per-batch events) gives the same sweep as data already on the device, bit for bit; the stage is
    consumed by one call and later calls read the resident data."""
    c = Case("cfg0", 4, oracle_kind="c")
    p = make_plan(c.cfg, c.K, batch=2)
    p.set_shifts(c.s)
    F, gp, gq = c.oracle_grad()
    outs = []
    for staged in (False, True, False):
        dd = dev(c.d, torch.float32) if not staged else torch.zeros(c.d.shape, dtype=torch.float32, device="cuda")
        if staged:
            host_d = torch.from_numpy(np.ascontiguousarray(c.d, dtype=np.float32)).pin_memory()
            p.stage_sqrt_d(host_d, dd)
        sc = torch.zeros(3, dtype=torch.float64, device="cuda")
        gpsi = torch.empty(c.psi.shape, dtype=torch.complex64, device="cuda")
        gqd = torch.empty(c.q.shape, dtype=torch.complex64, device="cuda")
        p.grad(dev(c.psi), dev(c.q), dd, sc, None, gpsi, gqd)
        outs.append((host(sc).real.copy(), host(gpsi), host(gqd), host(dd)))
    assert abs(outs[1][0][0] - F) / F < TOL_S and rel(outs[1][1], gp) < TOL_G and rel(outs[1][2], gq) < TOL_G
    for a, b in zip(outs[0], outs[1]):
        assert np.array_equal(a, b)
    assert np.array_equal(outs[1][3], c.d.astype(np.float32))
