"""Reference arm (O14, holo_grad_ref) on the GPU vs the fp64 oracles, element by element.

Reference constraint P:102; reference terms of Eq. (10) and Eq. (12).
Tolerances as the main chain (north_star): F <= 1e-4 relative, grad_q <= 1e-4 relative L2.
Data come from the ORACLE forward (|w| with a multiplicative perturbation so that the
evaluation state is not converged), never from the GPU.
"""
import numpy as np
import pytest
import torch

import oracle
import synth
from oracle import np_oracle as npo

pytestmark = pytest.mark.gpu

TOL_S, TOL_G = 1e-4, 1e-4


def rel(a, b):
    return float(np.linalg.norm((np.asarray(a) - np.asarray(b)).ravel()) / np.linalg.norm(np.asarray(b).ravel()))


def dev(x, dt=torch.complex64):
    return torch.as_tensor(np.ascontiguousarray(x)).to(dt).cuda().contiguous()


def plan(cfg, L, N):
    import paper_2407_20304_b200 as hb
    return hb.Plan(N, L, cfg.z1, 0, cfg.wavelength, cfg.Z, cfg.det_pixel, device=0)


def ref_data(g, q, rs, N, seed):
    rng = np.random.default_rng(seed)
    L = q.shape[-1]
    d = []
    for r in range(rs.shape[0]):
        w = npo.crop(npo.prop(npo.shift(q, rs[r, 0], rs[r, 1]), g.wavelength, g.p0, g.zeta[0]), N)
        d.append(np.abs(w) * (1 + 0.05 * rng.standard_normal(w.shape)))
    return np.maximum(np.stack(d), 0.0)


def run_gpu(p, q, d, acc_into=None, flags=0):
    sc = torch.zeros(1, dtype=torch.float64, device="cuda")
    gq = dev(acc_into) if acc_into is not None else torch.empty(q.shape, dtype=torch.complex64, device="cuda")
    p.grad_ref(dev(q), dev(d, torch.float32), sc, gq, flags=flags)
    torch.cuda.synchronize()
    return float(sc.cpu()[0]), gq.cpu().numpy().astype(np.complex128)


@pytest.mark.parametrize("L,N,R", [(128, 64, 3), (256, 128, 5), (512, 256, 2)])
def test_ref_arm_pow2_parity_vs_c_oracle(L, N, R):
    """Power-of-two tori, random shifts in [-8, 8] (cfg4 recipe), naive-DFT C oracle."""
    cfg = synth.CONFIGS["cfg4"]
    g = oracle.Geometry(cfg.wavelength, cfg.Z, cfg.z1, cfg.det_pixel)
    q_t = synth.probe(cfg, L=L).numpy()
    rs = np.random.default_rng(L).uniform(-8, 8, size=(R, 2))
    d = ref_data(g, q_t, rs, N, L)
    q = 0.9 * q_t
    F, gq = oracle.grad_ref(g, q, rs, d)
    p = plan(cfg, L, N)
    p.set_ref_shifts(rs)
    Fg, gg = run_gpu(p, q, d)
    assert abs(Fg - F) / F < TOL_S
    assert rel(gg, gq) < TOL_G


def test_ref_arm_accumulate_and_objective_only():
    import paper_2407_20304_b200 as hb
    cfg = synth.CONFIGS["cfg4"]
    g = oracle.Geometry(cfg.wavelength, cfg.Z, cfg.z1, cfg.det_pixel)
    L, N, R = 256, 128, 3
    q_t = synth.probe(cfg, L=L).numpy()
    rs = np.random.default_rng(3).uniform(-8, 8, size=(R, 2))
    d = ref_data(g, q_t, rs, N, 3)
    q = 0.9 * q_t
    F, gq = oracle.grad_ref(g, q, rs, d)
    p = plan(cfg, L, N)
    p.set_ref_shifts(rs)
    base = np.random.default_rng(4).standard_normal((L, L)) * (1 + 1j)
    _, ga = run_gpu(p, q, d, acc_into=base, flags=hb.HOLO_ACCUMULATE_Q)
    assert rel(ga - base, gq) < TOL_G
    Fo, go = run_gpu(p, q, d, acc_into=base, flags=hb.HOLO_OBJECTIVE_ONLY)
    assert abs(Fo - F) / F < TOL_S
    assert np.array_equal(go, base.astype(np.complex64).astype(np.complex128))  # untouched


def test_ref_arm_cfg4_full_size_parity():
    """configs[4] geometry at full size: 3072^2 frames on the 6144^2 torus (radix-3 engine,
    reading C16), two reference frames, numpy.fft oracle."""
    cfg = synth.CONFIGS["cfg4"]
    g = oracle.Geometry(cfg.wavelength, cfg.Z, cfg.z1, cfg.det_pixel)
    L, N, R = cfg.npad, cfg.n, 2
    q_t = synth.probe(cfg).numpy()
    rs = synth.ref_shifts(cfg)[:R]
    d = ref_data(g, q_t, rs, N, 6144)
    q = 0.9 * q_t
    F, gq = npo.grad_ref(g.wavelength, g.p0, g.zeta[0], q, rs, d)
    p = plan(cfg, L, N)
    p.set_ref_shifts(rs)
    Fg, gg = run_gpu(p, q, d)
    assert abs(Fg - F) / F < TOL_S
    assert rel(gg, gq) < TOL_G


def test_radix3_plan_rejects_object_chain():
    import paper_2407_20304_b200 as hb
    cfg = synth.CONFIGS["cfg4"]
    with pytest.raises(hb.HoloError):
        hb.Plan(cfg.n, cfg.npad, cfg.z1, 4, cfg.wavelength, cfg.Z, cfg.det_pixel, device=0)


def test_fwd_ref_matches_oracle_forward():
    """holo_fwd_ref: w_r = C(P_{zeta0} S_{s_r} q) vs the numpy oracle, forward tolerance 2e-5."""
    cfg = synth.CONFIGS["cfg4"]
    g = oracle.Geometry(cfg.wavelength, cfg.Z, cfg.z1, cfg.det_pixel)
    for L, N, R in [(256, 128, 3), (6144, 3072, 1)]:
        q = synth.probe(cfg, L=L).numpy()
        rs = np.random.default_rng(L).uniform(-8, 8, size=(R, 2))
        p = plan(cfg, L, N)
        p.set_ref_shifts(rs)
        w = torch.empty(R, N, N, dtype=torch.complex64, device="cuda")
        p.fwd_ref(dev(q), w)
        wn = w.cpu().numpy()
        for r in range(R):
            wo = npo.crop(npo.prop(npo.shift(q, rs[r, 0], rs[r, 1]), g.wavelength, g.p0, g.zeta[0]), N)
            assert rel(wn[r], wo) < 2e-5, (L, r)


def test_ref_arm_f2_parity():
    """HOLO_INTENSITY on the reference arm: F_2 reference term and its q-gradient."""
    import paper_2407_20304_b200 as hb
    cfg = synth.CONFIGS["cfg4"]
    g = oracle.Geometry(cfg.wavelength, cfg.Z, cfg.z1, cfg.det_pixel)
    L, N, R = 256, 128, 3
    q_t = synth.probe(cfg, L=L).numpy()
    rs = np.random.default_rng(9).uniform(-8, 8, size=(R, 2))
    d = ref_data(g, q_t, rs, N, 9)
    q = 0.9 * q_t
    F, gq = npo.grad_ref(g.wavelength, g.p0, g.zeta[0], q, rs, d, tau=2)
    p = plan(cfg, L, N)
    p.set_ref_shifts(rs)
    Fg, gg = run_gpu(p, q, d, flags=hb.HOLO_INTENSITY)
    assert abs(Fg - F) / F < TOL_S
    assert rel(gg, gq) < TOL_G


@pytest.mark.parametrize("tau", [0.5, 1.5])
def test_ref_arm_g_tau_parity(tau):
    """holo_set_tau on the reference arm: G_tau reference term and its q-gradient (App. A.3)."""
    cfg = synth.CONFIGS["cfg4"]
    g = oracle.Geometry(cfg.wavelength, cfg.Z, cfg.z1, cfg.det_pixel)
    L, N, R = 256, 128, 3
    q_t = synth.probe(cfg, L=L).numpy()
    rs = np.random.default_rng(19).uniform(-8, 8, size=(R, 2))
    d = ref_data(g, q_t, rs, N, 19)
    q = 0.9 * q_t
    F, gq = npo.grad_ref(g.wavelength, g.p0, g.zeta[0], q, rs, d, tau=tau)
    p = plan(cfg, L, N)
    p.set_ref_shifts(rs)
    p.set_tau(tau)
    Fg, gg = run_gpu(p, q, d)
    assert abs(Fg - F) / F < TOL_S
    assert rel(gg, gq) < TOL_G


def test_ref_arm_staged_data_matches_resident():
    """holo_stage_sqrt_dref: reference frames streamed from pinned host memory per frame batch give
    the same F and grad_q as device-resident frames, bit for bit (12 frames: batches of 8 + 4)."""
    cfg = synth.CONFIGS["cfg4"]
    g = oracle.Geometry(cfg.wavelength, cfg.Z, cfg.z1, cfg.det_pixel)
    L, N, R = 256, 128, 12
    q_t = synth.probe(cfg, L=L).numpy()
    rs = np.random.default_rng(29).uniform(-8, 8, size=(R, 2))
    d = ref_data(g, q_t, rs, N, 29).astype(np.float32)
    p = plan(cfg, L, N)
    p.set_ref_shifts(rs)
    res = []
    for staged in (False, True):
        dd = dev(d, torch.float32) if not staged else torch.zeros(d.shape, dtype=torch.float32, device="cuda")
        if staged:
            p.stage_sqrt_dref(torch.from_numpy(np.ascontiguousarray(d)).pin_memory(), dd)
        sc = torch.zeros(1, dtype=torch.float64, device="cuda")
        gq = torch.empty(L, L, dtype=torch.complex64, device="cuda")
        p.grad_ref(dev(0.9 * q_t), dd, sc, gq)
        torch.cuda.synchronize()
        res.append((sc.cpu().numpy(), gq.cpu().numpy(), dd.cpu().numpy()))
    assert np.array_equal(res[0][0], res[1][0]) and np.array_equal(res[0][1], res[1][1])
    assert np.array_equal(res[1][2], d)
