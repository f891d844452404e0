"""Worker of tests/test_dist_cpu.py: one rank of the joint CG driver (solver.JointCG) on CPU.

The plan is a TEST DOUBLE (FakePlan) whose array work is the fp64 C oracle (oracle/):
it exercises the host-side N>1 logic -- angle / reference-frame sharding, the two
allreduce exchanges of a sweep (grad_q partial, scalars), the replicated q-block
update -- over the gloo backend.  Usage (env RANK, WORLD_SIZE, MASTER_ADDR, MASTER_PORT):
    python tests/dist_worker.py <problem> <iterations> <out.npz>
"""
import os
import sys
from types import SimpleNamespace

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import synth  # noqa: E402


class FakePlan:
    """holo_grad / holo_grad_ref / holo_q_dots / holo_cg_step semantics (include/holo.h) in fp64 numpy."""

    def __init__(self, geom, shifts, ref_shifts=None):
        self.g, self.s, self.rs = geom, shifts, ref_shifts
        self.K = shifts.shape[0]

    def grad(self, psi, q, sqrt_d, sc, eta_psi_prev=None, grad_psi=None, grad_q_part=None, flags=0):
        if self.K == 0:  # holo_grad on an empty shard: F = 0, zero probe-gradient partial
            sc.zero_()
            if grad_q_part is not None and not flags & 1:
                grad_q_part.zero_()
            return
        F, gp, gq = oracle.grad(self.g, psi.numpy(), q.numpy(), self.s, sqrt_d.numpy())
        sc[0] = F
        sc[1] = float(np.vdot(gp, gp).real)
        sc[2] = float(np.vdot(eta_psi_prev.numpy(), gp).real) if eta_psi_prev is not None else 0.0
        grad_psi.copy_(torch.from_numpy(gp))
        if grad_q_part is not None:  # NULL: no probe gradient (include/holo.h)
            grad_q_part.copy_(torch.from_numpy(gq))

    def grad_ref(self, q, sqrt_dref, sc, grad_q_part=None, flags=0):
        F, gq = oracle.grad_ref(self.g, q.numpy(), self.rs, sqrt_dref.numpy())
        sc[0] = F
        if flags & 1:
            grad_q_part += torch.from_numpy(gq)
        else:
            grad_q_part.copy_(torch.from_numpy(gq))

    def q_dots(self, grad_q, eta_q_prev, out):
        out[0] = float(torch.vdot(grad_q.flatten(), grad_q.flatten()).real)
        out[1] = float(torch.vdot(eta_q_prev.flatten(), grad_q.flatten()).real) if eta_q_prev is not None else 0.0

    def cg_step(self, cin, psi=None, eta_psi=None, grad_psi=None, psi_trial=None, q=None, eta_q=None, grad_q=None,
                q_trial=None):
        mode, beta, gen, reset = 2, 0.0, cin.g_eta_prev, 0
        if not cin.reuse_eta:
            if cin.first:
                mode, reset, gen = 0, 1, -cin.gPg
            else:
                den = cin.g_eta_prev - cin.gprev_eta_prev
                if not abs(den) >= 1e-30 * cin.gPg:
                    mode, reset, gen = 0, 1, -cin.gPg
                else:
                    beta = cin.gPg / den
                    gen = -cin.gPg + beta * cin.g_eta_prev
                    if not gen < 0.0:
                        mode, reset, beta, gen = 0, 1, 0.0, -cin.gPg
                    else:
                        mode = 1
        for x, eta, g, xt, rho in ((psi, eta_psi, grad_psi, psi_trial, cin.rho_psi),
                                   (q, eta_q, grad_q, q_trial, cin.rho_q)):
            if x is None or x.numel() == 0:
                continue
            if mode == 0:
                eta.copy_(-rho * g)
            elif mode == 1:
                eta.mul_(beta).add_(-rho * g)
            xt.copy_(x + cin.gamma * eta)
        return SimpleNamespace(beta=beta, g_eta_new=gen, reset=reset)


def problem(name, rank, world):
    if name == "joint":  # cfg0 geometry, 4 angles x 2 planes, sharded by angle
        cfg = synth.CONFIGS["cfg0"]
        K = 4
        g = oracle.Geometry(cfg.wavelength, cfg.Z, cfg.z1, cfg.det_pixel)
        psi_t = synth.psi_stack(cfg, K=K).numpy()
        q_t = synth.probe(cfg).numpy()
        s = synth.shifts(cfg, K=K)
        d = np.abs(oracle.fwd(g, psi_t, q_t, s, cfg.n))
        k0, k1 = rank * K // world, (rank + 1) * K // world
        plan = FakePlan(g, s[k0:k1])
        psi0 = torch.ones(k1 - k0, cfg.npad, cfg.npad, dtype=torch.complex128)
        return plan, torch.from_numpy(d[k0:k1].copy()), psi0, torch.from_numpy(0.9 * q_t), None, 1.0 / K
    # "ref": probe-only (configs[4] recipe at a small torus), reference frames sharded
    cfg = synth.CONFIGS["cfg4"]
    L, N, R = 32, 16, 4
    g = oracle.Geometry(cfg.wavelength, cfg.Z, cfg.z1, cfg.det_pixel)
    q_t = synth.probe(cfg, L=L).numpy()
    rs = np.random.default_rng(7).uniform(-8, 8, size=(R, 2))
    d = np.stack([np.abs(oracle.crop(oracle.prop(oracle.shift(q_t, *rs[r]), g.wavelength, g.p0, g.zeta[0]), N))
                  for r in range(R)])
    r0, r1 = rank * R // world, (rank + 1) * R // world
    plan = FakePlan(g, np.zeros((0, cfg.nz, 2)), rs[r0:r1])
    psi0 = torch.ones(0, L, L, dtype=torch.complex128)
    q0 = torch.from_numpy(q_t * (1 + 0.1 * np.cos(np.arange(L) / 3.0))[None, :])
    return plan, torch.zeros(0), psi0, q0, torch.from_numpy(d[r0:r1].copy()), 1.0


def main():
    name, iters, out = sys.argv[1], int(sys.argv[2]), sys.argv[3]
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world > 1:
        dist.init_process_group("gloo")
    from paper_2407_20304_b200.solver import JointCG
    plan, d, psi0, q0, dref, rho_q = problem(name, rank, world)
    cg = JointCG(plan, d, psi0, q0, rho_psi=1.0, rho_q=rho_q, sqrt_dref=dref)
    hist = [cg.start()]
    gam = []
    for _ in range(iters):
        h = cg.iterate()
        hist.append(h["F"])
        gam.append(h["gamma"])
    np.savez(out, F=np.array(hist), gamma=np.array(gam), q=cg.q.numpy(), psi=cg.psi.numpy(), sweeps=cg.sweeps)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
