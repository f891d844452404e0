"""Initialisers on the GPU: holo_init_probe (O17) and holo_init_psi (O18,
multi-distance Paganin) through the C ABI against the oracle, element by element, on synthetic
data of the configs' recipe (the data come from the oracle's forward, never from the GPU).

Tolerances: init_probe 2e-5 relative L2 (a sum of back-propagations, like the forward data);
init_psi 2e-4 relative L2: phi = (db/2) ln T amplifies the relative error of the filtered
intensity T by db/2 = 50 (db = 100), on top of ~12 fp32 transforms per plane."""
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


@pytest.mark.parametrize("L,N,R", [(128, 64, 3), (512, 256, 2), (6144, 3072, 1)])
def test_init_probe_parity(L, N, R):
    import paper_2407_20304_b200 as hb
    cfg = synth.CONFIGS["cfg4"]
    g = oracle.Geometry(cfg.wavelength, cfg.Z, cfg.z1, cfg.det_pixel)
    q = synth.probe(cfg, L=L).numpy()
    rs = synth.ref_shifts(cfg)[:R]
    w = [oracle.crop(npo.prop(npo.shift(q, *rs[r]), g.wavelength, g.p0, g.zeta[0]), N) for r in range(R)]
    a = np.abs(np.stack(w))
    ref = oracle.init_probe(g, rs, a, L) if L <= 128 else npo.init_probe(g.wavelength, g.p0, g.zeta[0], rs, a, L)
    p = hb.Plan(N, L, cfg.z1, 0, cfg.wavelength, cfg.Z, cfg.det_pixel, device=0)
    p.set_ref_shifts(rs)
    q0 = torch.empty(L, L, dtype=torch.complex64, device="cuda")
    p.init_probe(dev(a, torch.float32), q0)
    assert rel(q0.cpu().numpy(), ref) < 2e-5


@pytest.mark.parametrize("name,K,L,kind", [("cfg0", 2, None, "c"), ("cfg1", 1, None, "np"), ("cfg3", 1, None, "np")])
def test_init_psi_parity(name, K, L, kind):
    import paper_2407_20304_b200 as hb
    cfg = synth.CONFIGS[name]
    L = cfg.npad
    N = cfg.n
    g = oracle.Geometry(cfg.wavelength, cfg.Z, cfg.z1, cfg.det_pixel)
    psi_t = synth.psi_stack(cfg, K=K).numpy()
    q_t = synth.probe(cfg).numpy()
    s = synth.shifts(cfg, K=K)
    pr = npo.Problem(g, L, N)
    out = pr.fwd(psi_t, q_t, s)
    d = np.stack([np.stack([np.abs(out[(k, j)]) for j in range(cfg.nz)]) for k in range(K)])
    dref = np.abs(oracle.crop(npo.prop(q_t, g.wavelength, g.p0, g.zeta[0]), N))  # flat field
    db = 100.0
    p = hb.Plan(N, L, cfg.z1, K, cfg.wavelength, cfg.Z, cfg.det_pixel, device=0)
    p.set_shifts(s)
    psi0 = torch.empty(K, L, L, dtype=torch.complex64, device="cuda")
    p.init_psi(dev(d, torch.float32), dev(dref, torch.float32), db, psi0)
    got = psi0.cpu().numpy()
    for k in range(K):
        ref = (oracle.multipaganin(g, L, s[k], d[k], dref, db) if kind == "c"
               else npo.multipaganin(g, L, s[k], d[k], dref, db))
        assert rel(got[k], ref) < 2e-4, k
    # usefulness: the Paganin start fits the data better than psi = 1 (with the true probe)
    F_one = pr.grad(np.ones_like(psi_t), q_t, s, d)[0]
    F_pag = pr.grad(got.astype(np.complex128), q_t, s, d)[0]
    assert F_pag < F_one
