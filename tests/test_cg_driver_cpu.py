"""CPU pin of the CG driver (paper_2407_20304_b200.solver.JointCG) to the O13 oracle.

JointCG runs Eqs. (13)-(14) over a plan; here the plan is the fp64 test
double of tests/dist_worker.py (array work = the C oracle, holo_cg_step's scalar rule
restated).  The oracle side is oracle.cg.run, which follows O13 step by step in the
paper's notation.  Over >= 6 iterations with the line search active (readings C9-C11),
the F history, the accepted step lengths gamma and the DY betas must agree to fp64
rounding, and the final (psi, q) too.  The GPU half of row a-12 (the real holo_cg_step,
holo_q_dots and k_cg against the same oracle) is tests/test_gpu_cg.py.
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tests"))

import oracle  # noqa: E402
import synth  # noqa: E402
from oracle import cg as ocg  # noqa: E402
from dist_worker import FakePlan  # noqa: E402


def _problem(K=4):
    cfg = synth.CONFIGS["cfg0"]
    g = oracle.Geometry(cfg.wavelength, cfg.Z, cfg.z1, cfg.det_pixel)
    psi_t = synth.psi_stack(cfg, K=K).numpy()
    q_t = synth.probe(cfg).numpy()
    s = synth.shifts(cfg, K=K)
    d = synth.poisson_amplitude(np.abs(oracle.fwd(g, psi_t, q_t, s, cfg.n)) ** 2, cfg.photons, cfg)
    return cfg, g, psi_t, q_t, s, d


def test_joint_cg_driver_reproduces_oracle_cg():
    from paper_2407_20304_b200.solver import JointCG
    cfg, g, psi_t, q_t, s, d = _problem()
    K = psi_t.shape[0]
    rho = (1.0, 1.0 / K)
    psi0, q0 = np.ones_like(psi_t), 0.9 * q_t
    n_iter = 7

    def sweep(x):
        F, gp, gq = oracle.grad(g, x[0], x[1], s, d)
        return F, [gp, gq]

    x_or, hist = ocg.run(sweep, [psi0, q0], rho, n_iter)

    plan = FakePlan(g, s)
    cg = JointCG(plan, torch.from_numpy(d.copy()), torch.from_numpy(psi0.copy()), torch.from_numpy(q0.copy()),
                 rho_psi=rho[0], rho_q=rho[1], distributed=False)
    F0 = cg.start()
    assert abs(F0 - sweep([psi0, q0])[0]) <= 1e-13 * F0
    out = [cg.iterate() for _ in range(n_iter)]
    for m, (a, b) in enumerate(zip(out, hist)):
        assert abs(a["F"] - b["F"]) <= 1e-12 * abs(b["F"]), m
        assert abs(a["gamma"] - b["gamma"]) <= 1e-12 * max(abs(b["gamma"]), 1e-300), m
        assert abs(a["beta"] - b["beta"]) <= 1e-12 * max(abs(b["beta"]), 1e-12), m
        assert a["reset"] == b["reset"], m
        assert a["sweeps"] == b["sweeps"], m
    # the run really exercised the DY recursion and the line search
    assert any(h["beta"] != 0.0 for h in hist) and any(h["sweeps"] > 1 for h in hist)
    assert hist[-1]["F"] < 0.5 * F0
    for got, ref in ((cg.psi.numpy(), x_or[0]), (cg.q.numpy(), x_or[1])):
        assert np.linalg.norm(got - ref) <= 1e-12 * np.linalg.norm(ref)


def test_joint_cg_driver_forced_gamma_matches_oracle():
    """forced_gamma (the GPU parity protocol) follows oracle.cg.run(forced_gammas=...)."""
    from paper_2407_20304_b200.solver import JointCG
    cfg, g, psi_t, q_t, s, d = _problem()
    K = psi_t.shape[0]
    rho = (1.0, 1.0 / K)
    gam = [0.5, 0.25, 0.4]

    def sweep(x):
        F, gp, gq = oracle.grad(g, x[0], x[1], s, d)
        return F, [gp, gq]

    x_or, hist = ocg.run(sweep, [np.ones_like(psi_t), 0.9 * q_t], rho, len(gam), forced_gammas=gam)
    cg = JointCG(FakePlan(g, s), torch.from_numpy(d.copy()), torch.from_numpy(np.ones_like(psi_t)),
                 torch.from_numpy(0.9 * q_t), rho_psi=rho[0], rho_q=rho[1], distributed=False)
    out = [cg.iterate(forced_gamma=gm) for gm in gam]
    for a, b in zip(out, hist):
        assert abs(a["F"] - b["F"]) <= 1e-12 * b["F"]
        assert abs(a["beta"] - b["beta"]) <= 1e-12 * max(abs(b["beta"]), 1e-12)
    assert np.linalg.norm(cg.q.numpy() - x_or[1]) <= 1e-12 * np.linalg.norm(x_or[1])


def test_probe_subset_schedule_reproduces_oracle():
    """Probe-subset schedule (reading R6): multires.run_probe_subset over the fp64 test
    double equals O13 run twice -- joint CG on the subset angles, then CG with P = diag(1, 0)
    (probe frozen) over all angles -- F histories, final psi and q (q bitwise unchanged in stage 2)."""
    from paper_2407_20304_b200.multires import probe_subset_indices, run_probe_subset
    cfg, g, psi_t, q_t, s, d = _problem(K=4)
    K = psi_t.shape[0]
    idx = probe_subset_indices(K, 2)
    assert list(idx) == [0, 2]
    assert list(probe_subset_indices(180, 20)) == [int(np.floor(i * 9 + 0.5)) for i in range(20)]
    assert list(probe_subset_indices(3, 50)) == [0, 1, 2]
    psi0, q0 = np.ones_like(psi_t), 0.9 * q_t
    n1, n2 = 3, 3

    def sweep_sub(x):
        F, gp, gq = oracle.grad(g, x[0], x[1], s[idx], d[idx])
        return F, [gp, gq]

    x1, h1 = ocg.run(sweep_sub, [psi0[idx], q0], (1.0, 1.0 / len(idx)), n1)
    psi_mid = psi0.copy()
    psi_mid[idx] = x1[0]

    def sweep_all(x):
        F, gp, gq = oracle.grad(g, x[0], x[1], s, d)
        return F, [gp, gq]

    x2, h2 = ocg.run(sweep_all, [psi_mid, x1[1]], (1.0, 0.0), n2)
    assert np.array_equal(x2[1], x1[1])

    psi, q, hist = run_probe_subset(torch.from_numpy(d.copy()), s, torch.from_numpy(psi0.copy()),
                                    torch.from_numpy(q0.copy()), 2, n1, n2,
                                    make_plan=lambda ii: FakePlan(g, s[np.asarray(ii)]), distributed=False)
    assert abs(hist[0]["F_end"] - h1[-1]["F"]) <= 1e-12 * h1[-1]["F"]
    assert abs(hist[1]["F_end"] - h2[-1]["F"]) <= 1e-12 * h2[-1]["F"]
    assert hist[1]["F_end"] <= hist[1]["F_start"]
    assert np.abs(q.numpy() - x1[1]).max() <= 1e-12 * np.abs(x1[1]).max()
    assert np.abs(psi.numpy() - x2[0]).max() <= 1e-10 * np.abs(x2[0]).max()
