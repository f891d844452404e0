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
