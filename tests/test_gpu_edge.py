"""Edge cases and full-size properties of the object chain on the GPU (through the C ABI).

* single plane (nz = 1, mt = 1: no magnification), ragged row tiles (N not a multiple of
  the rows per CTA), the smallest frame (N = 8), an empty angle shard (K = 0);
* at the full cfg3 size (4096^2 torus): the paper's consistency statement psi == 1 ->
  w_kj = C(P_{zeta0} q) for every plane, and the adjoint identities
  Re<L x, y> = Re<x, L* y>, Re<Q x, y> = Re<x, Q* y> (the operators of Eq. (11)-(12)).
Oracle: numpy fp64 (oracle/np_oracle.py); tolerances as test_gpu_parity.
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
    return float(np.linalg.norm((np.asarray(a) - np.asarray(b)).ravel()) / np.linalg.norm(np.asarray(b).ravel()))


def dev(x, dt=torch.complex64):
    return torch.as_tensor(np.ascontiguousarray(x)).to(dt).cuda().contiguous()


def mkplan(cfg, K, L, N, z1):
    import paper_2407_20304_b200 as hb
    return hb.Plan(N, L, z1, K, cfg.wavelength, cfg.Z, cfg.det_pixel, device=0)


def rand_state(L, K, seed):
    rng = np.random.default_rng(seed)
    psi = np.exp(1j * 0.3 * rng.standard_normal((K, L, L)) - 0.01)
    q = 1 + 0.2 * (rng.standard_normal((L, L)) + 1j * rng.standard_normal((L, L)))
    return psi, q


@pytest.mark.parametrize("L,N,z1,K", [(512, 256, [4.584e-3], 2),        # single plane, no magnification
                                      (256, 104, None, 1),                # ragged: 104 rows over 32-row tiles
                                      (128, 8, None, 1)])                 # smallest frame
def test_edge_shapes_forward_and_gradient(L, N, z1, K):
    cfg = synth.CONFIGS["cfg1"]
    z1 = cfg.z1 if z1 is None else z1
    g = oracle.Geometry(cfg.wavelength, cfg.Z, z1, cfg.det_pixel)
    psi_t, q_t = rand_state(L, K, L + N)
    s = np.random.default_rng(N).uniform(-3, 3, size=(K, len(z1), 2))
    pr = npo.Problem(g, L, N)
    out = pr.fwd(psi_t, q_t, s)
    p = mkplan(cfg, K, L, N, z1)
    p.set_shifts(s)
    w = torch.empty(K, len(z1), N, N, dtype=torch.complex64, device="cuda")
    p.fwd(dev(psi_t), dev(q_t), w)
    wn = w.cpu().numpy()
    for (k, j), wo in out.items():
        assert rel(wn[k, j], wo) < TOL_W, (k, j)
    d = np.stack([np.stack([np.abs(out[(k, j)]) * 1.1 for j in range(len(z1))]) for k in range(K)])
    psi, q = np.ones_like(psi_t), 0.9 * q_t
    F, gp, gq = pr.grad(psi, q, s, d)
    sc = torch.zeros(3, dtype=torch.float64, device="cuda")
    gpsi = torch.empty(psi.shape, dtype=torch.complex64, device="cuda")
    gqd = torch.empty(q.shape, dtype=torch.complex64, device="cuda")
    p.grad(dev(psi), dev(q), dev(d, torch.float32), sc, None, gpsi, gqd)
    assert abs(float(sc.cpu()[0]) - F) / F < TOL_S
    assert rel(gpsi.cpu().numpy(), gp) < TOL_G and rel(gqd.cpu().numpy(), gq) < TOL_G


def test_empty_angle_shard():
    """K = 0 (a rank without angles): F = 0 and a zero probe-gradient partial."""
    cfg = synth.CONFIGS["cfg1"]
    L, N = 256, 128
    p = mkplan(cfg, 0, L, N, cfg.z1)
    sc = torch.full((3,), 7.0, dtype=torch.float64, device="cuda")
    gq = torch.full((L, L), 3.0 + 1j, dtype=torch.complex64, device="cuda")
    e = torch.empty(0, L, L, dtype=torch.complex64, device="cuda")
    p.grad(e, torch.ones(L, L, dtype=torch.complex64, device="cuda"), torch.empty(0, device="cuda"), sc, None, e, gq)
    torch.cuda.synchronize()
    assert torch.count_nonzero(sc).item() == 0 and torch.count_nonzero(gq).item() == 0


def test_psi_one_invariant_full_size():
    """with psi == 1 every plane sees the reference form C(P_{zeta0} q)
    (M S 1 = 1 and P_{zdet_j} P_{omega_j} = P_{zeta0}), cfg3 size, random shifts."""
    cfg = synth.CONFIGS["cfg3"]
    L, N = cfg.npad, cfg.n
    g = oracle.Geometry(cfg.wavelength, cfg.Z, cfg.z1, cfg.det_pixel)
    q = synth.probe(cfg).numpy()
    s = synth.shifts(cfg, K=1)
    p = mkplan(cfg, 1, L, N, cfg.z1)
    p.set_shifts(s)
    w = torch.empty(1, cfg.nz, N, N, dtype=torch.complex64, device="cuda")
    p.fwd(torch.ones(1, L, L, dtype=torch.complex64, device="cuda"), dev(q), w)
    ref = npo.crop(npo.prop(q, g.wavelength, g.p0, g.zeta[0]), N)
    wn = w.cpu().numpy()
    for j in range(cfg.nz):
        assert rel(wn[0, j], ref) < TOL_W, j


def test_adjoint_identities_full_size():
    """Re<L x, y> = Re<x, L* y> and Re<Q x, y> = Re<x, Q* y> at the cfg3 size (4096^2 torus,
    4 planes, 1 angle) through holo_fwd / holo_adj, in the bench's launch configuration."""
    cfg = synth.CONFIGS["cfg3"]
    L, N = cfg.npad, cfg.n
    rng = np.random.default_rng(33)
    p = mkplan(cfg, 1, L, N, cfg.z1)
    s = synth.shifts(cfg, K=1)
    p.set_shifts(s)
    psi = dev(np.exp(0.2j * rng.standard_normal((1, L, L))))
    q = dev(synth.probe(cfg).numpy())
    y = dev(rng.standard_normal((1, cfg.nz, N, N)) + 1j * rng.standard_normal((1, cfg.nz, N, N)))
    x_psi = dev(rng.standard_normal((1, L, L)) + 1j * rng.standard_normal((1, L, L)))
    x_q = dev(rng.standard_normal((L, L)) + 1j * rng.standard_normal((L, L)))
    w = torch.empty(1, cfg.nz, N, N, dtype=torch.complex64, device="cuda")
    a_psi = torch.empty(1, L, L, dtype=torch.complex64, device="cuda")
    a_q = torch.empty(L, L, dtype=torch.complex64, device="cuda")
    p.adj(y, psi, q, a_psi, a_q)
    d = lambda a, b: torch.vdot(b.flatten().to(torch.complex128), a.flatten().to(torch.complex128)).real.item()
    p.fwd(x_psi, q, w)                      # L x: linear in psi at fixed q
    lhs, rhs = d(w, y), d(x_psi, a_psi)
    assert abs(lhs - rhs) / abs(lhs) < 1e-4
    p.fwd(psi, x_q, w)                      # Q x: linear in q at fixed psi
    lhs, rhs = d(w, y), d(x_q, a_q)
    assert abs(lhs - rhs) / abs(lhs) < 1e-4


def test_gq_event_marks_complete_probe_gradient():
    """holo_set_gq_event (SURVEY 8e overlap): a side stream that waits ONLY on the event sees the
    finished probe-gradient partial, although the last batch's X3 passes are still queued after it;
    the event sits before X3 (it completes before the sweep's last kernel)."""
    import paper_2407_20304_b200 as hb
    cfg = synth.CONFIGS["cfg1"]
    K = 12
    rng = np.random.default_rng(21)
    psi = np.exp(0.2j * rng.standard_normal((K, cfg.npad, cfg.npad)))
    q = 1 + 0.2 * (rng.standard_normal((cfg.npad, cfg.npad)) + 1j * rng.standard_normal((cfg.npad, cfg.npad)))
    d = 1 + 0.1 * rng.uniform(size=(K, cfg.nz, cfg.n, cfg.n))
    p = hb.Plan(cfg.n, cfg.npad, cfg.z1, K, cfg.wavelength, cfg.Z, cfg.det_pixel, device=0, angle_batch=4)
    ev = torch.cuda.Event()
    p.set_gq_event(ev)
    side = torch.cuda.Stream()
    sc = torch.zeros(3, dtype=torch.float64, device="cuda")
    gpsi = torch.empty(K, cfg.npad, cfg.npad, dtype=torch.complex64, device="cuda")
    gq = torch.zeros(cfg.npad, cfg.npad, dtype=torch.complex64, device="cuda")
    snap = torch.empty_like(gq)
    P, Q, D = dev(psi), dev(q), dev(d, torch.float32)
    torch.cuda.synchronize()
    p.grad(P, Q, D, sc, None, gpsi, gq)
    side.wait_event(ev)
    with torch.cuda.stream(side):
        snap.copy_(gq)
    done_at_event = torch.cuda.Event()
    done_at_event.record(side)
    torch.cuda.synchronize()
    assert torch.equal(snap, gq)
    assert float(gq.abs().max()) > 0
    p.set_gq_event(None)
