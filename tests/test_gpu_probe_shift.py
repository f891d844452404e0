"""f-1 on the GPU: per-frame probe shifts s^p_kj and the reference term fused into the sweep
(Eq. (10)/(12) in full; O19) through the C ABI against the oracle, element by element.
Tolerances as the object chain: forward 2e-5, F and gradients 1e-4 (relative L2)."""
import numpy as np
import pytest
import torch

import oracle
import synth
from oracle import cg as ocg
from oracle import np_oracle as npo

pytestmark = pytest.mark.gpu
TOL_W, TOL = 2e-5, 1e-4


def rel(a, b):
    return float(np.linalg.norm((np.asarray(a) - np.asarray(b)).ravel()) / np.linalg.norm(np.asarray(b).ravel()))


def dev(x, dt=torch.complex64):
    return torch.as_tensor(np.ascontiguousarray(x)).to(dt).cuda().contiguous()


def host(t):
    torch.cuda.synchronize()
    return t.cpu().numpy().astype(np.complex128 if t.is_complex() else np.float64)


class Case:
    def __init__(self, name, K, R=0, kind="c"):
        cfg = synth.CONFIGS[name]
        self.cfg, self.K, self.R, self.kind = cfg, K, R, kind
        self.g = oracle.Geometry(cfg.wavelength, cfg.Z, cfg.z1, cfg.det_pixel)
        L, N = cfg.npad, cfg.n
        self.psi_t = synth.psi_stack(cfg, K=K).numpy()
        self.q_t = synth.probe(cfg).numpy()
        self.s = synth.shifts(cfg, K=K)
        self.sp = np.random.default_rng(11).uniform(-3, 3, size=(K, cfg.nz, 2))
        self.pr = npo.Problem(self.g, L, N)
        out = self.pr.fwd_full(self.psi_t, self.q_t, self.s, self.sp)
        self.w = np.stack([np.stack([out[(k, j)] for j in range(cfg.nz)]) for k in range(K)])
        self.d = synth.poisson_amplitude(np.abs(self.w) ** 2, cfg.photons, cfg)
        self.rs = synth.ref_shifts(synth.CONFIGS["cfg4"])[:R] if R else None
        self.dref = (np.stack([np.abs(oracle.crop(npo.prop(npo.shift(self.q_t, *self.rs[r]), self.g.wavelength,
                                                                   self.g.p0, self.g.zeta[0]), N)) for r in range(R)])
                     if R else None)
        self.psi, self.q = np.ones_like(self.psi_t), 0.9 * self.q_t

    def oracle_grad(self, psi=None, q=None):
        psi = self.psi if psi is None else psi
        q = self.q if q is None else q
        if self.kind == "c":
            return oracle.grad_full(self.g, psi, q, self.s, self.sp, self.d, self.rs, self.dref)
        return self.pr.grad_full(psi, q, self.s, self.sp, self.d, self.rs, self.dref)

    def plan(self, batch=None):
        import paper_2407_20304_b200 as hb
        c = self.cfg
        p = hb.Plan(c.n, c.npad, c.z1, self.K, c.wavelength, c.Z, c.det_pixel, device=0, angle_batch=batch)
        p.set_shifts(self.s)
        p.set_probe_shifts(self.sp)
        if self.R:
            p.set_ref_shifts(self.rs)
        return p


@pytest.mark.parametrize("name,K,R,kind,batch", [("cfg0", 4, 0, "c", 1), ("cfg0", 4, 3, "c", 3),
                                                  ("cfg1", 2, 2, "np", 2), ("cfg3", 1, 1, "np", 1)])
def test_probe_shift_forward_and_gradient_parity(name, K, R, kind, batch):
    c = Case(name, K, R, kind)
    p = c.plan(batch)
    cfg = c.cfg
    w = torch.empty(K, cfg.nz, cfg.n, cfg.n, dtype=torch.complex64, device="cuda")
    p.fwd(dev(c.psi_t), dev(c.q_t), w)
    assert rel(host(w), c.w) < TOL_W
    F, gp, gq = c.oracle_grad()
    sc = torch.zeros(3, dtype=torch.float64, device="cuda")
    gpsi = torch.empty(c.psi.shape, dtype=torch.complex64, device="cuda")
    gqd = torch.empty(c.q.shape, dtype=torch.complex64, device="cuda")
    if R:
        p.grad_full(dev(c.psi), dev(c.q), dev(c.d, torch.float32), dev(c.dref, torch.float32), sc, None, gpsi, gqd)
    else:
        p.grad(dev(c.psi), dev(c.q), dev(c.d, torch.float32), sc, None, gpsi, gqd)
    assert abs(host(sc).real[0] - F) / F < TOL
    assert rel(host(gpsi), gp) < TOL and rel(host(gqd), gq) < TOL


def test_zero_probe_shift_path_equals_plain_path():
    import paper_2407_20304_b200 as hb
    c = Case("cfg0", 4)
    cfg = c.cfg
    outs = []
    for ps in (False, True):
        p = hb.Plan(cfg.n, cfg.npad, cfg.z1, 4, cfg.wavelength, cfg.Z, cfg.det_pixel, device=0)
        p.set_shifts(c.s)
        if ps:
            p.set_probe_shifts(np.zeros_like(c.sp))
        sc = torch.zeros(3, dtype=torch.float64, device="cuda")
        gpsi = torch.empty(c.psi.shape, dtype=torch.complex64, device="cuda")
        gqd = torch.empty(c.q.shape, dtype=torch.complex64, device="cuda")
        p.grad(dev(c.psi), dev(c.q), dev(c.d, torch.float32), sc, None, gpsi, gqd)
        outs.append((host(sc).real[0], host(gpsi), host(gqd)))
    assert abs(outs[0][0] - outs[1][0]) / outs[0][0] < 1e-5
    assert rel(outs[1][1], outs[0][1]) < 1e-5 and rel(outs[1][2], outs[0][2]) < 1e-5


def test_probe_shift_adjoint_identity():
    """holo_adj's probe adjoint on the PS path: Re<Q x, y> = Re<x, Q^* y>, Q x = holo_fwd(psi, x)."""
    c = Case("cfg0", 4)
    p = c.plan()
    cfg = c.cfg
    rng = np.random.default_rng(3)
    x = rng.standard_normal(c.q.shape) + 1j * rng.standard_normal(c.q.shape)
    y = rng.standard_normal((4, cfg.nz, cfg.n, cfg.n)) + 1j * rng.standard_normal((4, cfg.nz, cfg.n, cfg.n))
    w = torch.empty(4, cfg.nz, cfg.n, cfg.n, dtype=torch.complex64, device="cuda")
    p.fwd(dev(c.psi_t), dev(x), w)
    aq = torch.empty(c.q.shape, dtype=torch.complex64, device="cuda")
    ap = torch.empty(c.psi.shape, dtype=torch.complex64, device="cuda")
    p.adj(dev(y), dev(c.psi_t), dev(c.q_t), ap, aq)
    lhs = np.vdot(y, host(w)).real
    rhs = np.vdot(host(aq), x).real
    assert abs(lhs - rhs) / abs(lhs) < 1e-5


def test_fused_cg_iteration_vs_oracle():
    """JointCG over holo_grad_full (probe shifts + 3 reference frames), gamma forced, vs O13 over O19."""
    from paper_2407_20304_b200.solver import JointCG
    c = Case("cfg0", 4, R=3)
    rho = [1.0, 0.25]
    gam = [0.5, 0.3]

    def sweep(x):
        F, gp, gq = c.oracle_grad(x[0], x[1])
        return F, [gp, gq]

    x_or, hist = ocg.run(sweep, [c.psi, c.q], rho, 2, forced_gammas=gam)
    cg = JointCG(c.plan(), dev(c.d, torch.float32), dev(c.psi), dev(c.q), rho_psi=rho[0], rho_q=rho[1],
                 sqrt_dref=dev(c.dref, torch.float32), distributed=False)
    assert cg.fused
    out = [cg.iterate(forced_gamma=g) for g in gam]
    for a, b in zip(out, hist):
        assert abs(a["F"] - b["F"]) / b["F"] < TOL
    assert abs(out[1]["beta"] - hist[1]["beta"]) / abs(hist[1]["beta"]) < TOL
    assert rel(host(cg.psi), x_or[0]) < TOL and rel(host(cg.q), x_or[1]) < TOL
