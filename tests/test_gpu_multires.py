"""Multiresolution schedule on the GPU: holo_upsample2 (O15) and
holo_bin2 (O16) through the C ABI against the oracle, element by element, and the level
driver (multires.run_schedule) handing the state from one level to the next exactly as the
oracle's upsample2 of the previous level's state.
Tolerances: 2e-5 relative L2 for the transforms (forward-data tolerance; two length-2L
transforms per axis in fp32), 1e-6 for the binning (one rounding per pixel)."""
import numpy as np
import pytest
import torch

import oracle
import synth
from oracle import np_oracle as npo

pytestmark = pytest.mark.gpu


def rel(a, b):
    return float(np.linalg.norm((np.asarray(a) - np.asarray(b)).ravel()) / np.linalg.norm(np.asarray(b).ravel()))


def dev(x, dt=torch.complex64):
    return torch.as_tensor(np.ascontiguousarray(x)).to(dt).cuda().contiguous()


def plan(n, L, K=1, px=3e-6):
    import paper_2407_20304_b200 as hb
    cfg = synth.CONFIGS["cfg1"]
    return hb.Plan(n, L, cfg.z1, K, cfg.wavelength, cfg.Z, px, device=0)


@pytest.mark.parametrize("L", [128, 512, 1024, 4096])
def test_upsample2_parity(L):
    rng = np.random.default_rng(L)
    M = 2 if L <= 1024 else 1
    x = rng.standard_normal((M, L // 2, L // 2)) + 1j * rng.standard_normal((M, L // 2, L // 2))
    p = plan(L // 2, L)
    y = torch.empty(M, L, L, dtype=torch.complex64, device="cuda")
    p.upsample2(dev(x), y)
    yh = y.cpu().numpy()
    for m in range(M):
        ref = oracle.upsample2(x[m]) if L <= 128 else npo.upsample2(x[m])
        assert rel(yh[m], ref) < 2e-5, m


def test_bin2_parity():
    rng = np.random.default_rng(9)
    a = rng.uniform(0.2, 2.0, size=(3, 2, 256, 256))
    p = plan(128, 256)
    c = torch.empty(3, 2, 128, 128, dtype=torch.float32, device="cuda")
    p.bin2(dev(a, torch.float32), c)
    ref = oracle.bin2(a.astype(np.float32).astype(np.float64).reshape(6, 256, 256)).reshape(3, 2, 128, 128)
    assert rel(c.cpu().numpy(), ref) < 1e-6


def test_schedule_two_levels():
    """Two levels (2x2-binned on a 128^2 torus, then full on 256^2; cfg1 geometry and probe recipe,
    4 angles): each level's CG lowers F, and the state handed to the fine level equals the oracle's
    O15 upsampling of the coarse result."""
    import paper_2407_20304_b200 as hb
    from paper_2407_20304_b200 import multires
    cfg = synth.CONFIGS["cfg1"]
    K, L, N = 4, 256, 128
    g = oracle.Geometry(cfg.wavelength, cfg.Z, cfg.z1, cfg.det_pixel)
    psi_t = synth.psi_stack(cfg, K=K, L=L).numpy()
    q_t = synth.probe(cfg, L=L).numpy()
    s = np.round(synth.shifts(cfg, K=K) / 2) * 2  # even shifts: whole pixels at both levels
    pr = npo.Problem(g, L, N)
    out = pr.fwd(psi_t, q_t, s)
    d = np.stack([np.stack([np.abs(out[(k, j)]) for j in range(cfg.nz)]) for k in range(K)])
    sqrt_d = dev(d, torch.float32)
    qc = 0.9 * 0.25 * (q_t[0::2, 0::2] + q_t[1::2, 0::2] + q_t[0::2, 1::2] + q_t[1::2, 1::2])
    psi0 = torch.ones(K, L // 2, L // 2, dtype=torch.complex64, device="cuda")
    psi_c, q_c, hist_c = multires.run_schedule([(2, 6)], sqrt_d, s, N, L, cfg.z1, cfg.wavelength, cfg.Z,
                                               cfg.det_pixel, psi0, dev(qc), rho_q=1.0 / K)
    assert hist_c[0]["F_end"] < hist_c[0]["F_start"]
    pf = hb.Plan(N, L, cfg.z1, K, cfg.wavelength, cfg.Z, cfg.det_pixel, device=0)
    up_psi = torch.empty(K, L, L, dtype=torch.complex64, device="cuda")
    pf.upsample2(psi_c.contiguous(), up_psi)
    ref = np.stack([npo.upsample2(x) for x in psi_c.cpu().numpy().astype(np.complex128)])
    assert rel(up_psi.cpu().numpy(), ref) < 2e-5
    psi_f, q_f, hist = multires.run_schedule([(2, 6), (1, 4)], sqrt_d, s, N, L, cfg.z1, cfg.wavelength, cfg.Z,
                                             cfg.det_pixel, psi0, dev(qc), rho_q=1.0 / K)
    assert [h["factor"] for h in hist] == [2, 1]
    assert abs(hist[0]["F_end"] - hist_c[0]["F_end"]) <= 1e-6 * hist_c[0]["F_end"]  # deterministic
    assert hist[1]["F_end"] < hist[1]["F_start"]
    # the fine level starts from the upsampled coarse fit, better than psi = 1 with the upsampled q0
    F_naive = pr.grad(np.ones_like(psi_t), npo.upsample2(qc), s, d)[0]
    assert hist[1]["F_start"] < F_naive


def test_object_only_sweep_parity():
    """rho_q = 0 path (probe frozen): holo_grad with grad_q_part = NULL gives the oracle's F and
    grad_psi (cfg0, 4 angles) -- the probe-gradient work is skipped, nothing else changes."""
    cfg = synth.CONFIGS["cfg0"]
    K = 4
    g = oracle.Geometry(cfg.wavelength, cfg.Z, cfg.z1, cfg.det_pixel)
    psi_t, q_t, s = synth.psi_stack(cfg, K=K).numpy(), synth.probe(cfg).numpy(), synth.shifts(cfg, K=K)
    d = synth.poisson_amplitude(np.abs(oracle.fwd(g, psi_t, q_t, s, cfg.n)) ** 2, cfg.photons, cfg)
    psi, q = np.ones_like(psi_t), 0.9 * q_t
    F, gp, _ = oracle.grad(g, psi, q, s, d)
    import paper_2407_20304_b200 as hb
    p = hb.Plan(cfg.n, cfg.npad, cfg.z1, K, cfg.wavelength, cfg.Z, cfg.det_pixel, device=0)
    p.set_shifts(s)
    sc = torch.zeros(3, dtype=torch.float64, device="cuda")
    gpsi = torch.empty(K, cfg.npad, cfg.npad, dtype=torch.complex64, device="cuda")
    p.grad(dev(psi), dev(q), dev(d, torch.float32), sc, None, gpsi, None)
    torch.cuda.synchronize()
    assert abs(float(sc[0]) - F) / F < 1e-4
    assert rel(gpsi.cpu().numpy(), gp) < 1e-4


def test_probe_subset_schedule():
    """Probe-subset schedule (reading R6) on the GPU, cfg1 geometry at 256^2 (8 angles,
    subset of 3): stage 1 (joint CG on the subset) and stage 2 (object-only CG on all angles) each
    lower F, the plans hold the evenly spread subset and then all angles, and the final state's
    F is the oracle's F there (the CPU test pins the driver to O13 step by step)."""
    import paper_2407_20304_b200 as hb
    from paper_2407_20304_b200.multires import run_probe_subset
    cfg = synth.CONFIGS["cfg1"]
    K, L, N = 8, 256, 128
    g = oracle.Geometry(cfg.wavelength, cfg.Z, cfg.z1, cfg.det_pixel)
    psi_t = synth.psi_stack(cfg, K=K, L=L).numpy()
    q_t = synth.probe(cfg, L=L).numpy()
    s = np.random.default_rng(5).uniform(-2, 2, size=(K, cfg.nz, 2))
    pr = npo.Problem(g, L, N)
    out = pr.fwd(psi_t, q_t, s)
    d = np.stack([np.stack([np.abs(out[(k, j)]) for j in range(cfg.nz)]) for k in range(K)])
    psi0, q0 = np.ones_like(psi_t), 0.9 * q_t
    seen = {}

    def make_plan(idx):
        p = hb.Plan(N, L, cfg.z1, len(idx), cfg.wavelength, cfg.Z, cfg.det_pixel, device=0, angle_batch=4)
        p.set_shifts(s[np.asarray(idx)])
        seen.setdefault("idx", []).append(np.asarray(idx).copy())
        return p

    psi, q, hist = run_probe_subset(dev(d, torch.float32), s, dev(psi0), dev(q0), 3, 4, 4, make_plan)
    assert [list(i) for i in seen["idx"]] == [[0, 3, 5], list(range(K))]
    for h in hist:
        assert h["F_end"] < h["F_start"], h
    # the final state's F (stage 2 never moved q) is the oracle's F there
    q1 = q.cpu().numpy().astype(np.complex128)
    F_end = pr.grad(psi.cpu().numpy().astype(np.complex128), q1, s, d)[0]
    assert abs(F_end - hist[1]["F_end"]) / F_end < 1e-4
