"""Multiresolution schedule and probe-subset updates.

The paper starts the joint reconstruction on 8x8-binned data, then 4x4, 2x2 and full
resolution, "extrapolat[ing] the recovered object with the probe function to a grid twice
as dense" between levels.  Each level is a full JointCG problem on its own plan:
data side n/f, torus npad/f, detector pixel x f (so the object-plane pixel p0 doubles per
level, reading R2), shifts / f.  Between levels psi and q are Fourier-upsampled by
holo_upsample2 (O15, reading R1) and the data are re-binned by holo_bin2 (O16) from the
next finer level -- all array work in libholo; this module only sequences it.
"""
from __future__ import annotations

import numpy as np
import torch

from . import Plan
from .solver import JointCG


def level_geometry(n, npad, detector_pixel, factor):
    if n % factor or npad % factor:
        raise ValueError(f"binning factor {factor} does not divide n = {n}, npad = {npad}")
    return n // factor, npad // factor, detector_pixel * factor


def bin_pyramid(sqrt_d, n, npad, z1, K, wavelength, Z, detector_pixel, factors, device=0):
    """Binned copies of the amplitude data [K][nz][n][n] for every factor (powers of 2), built
    by repeated holo_bin2 from the finest level.  Returns {factor: tensor}."""
    out = {1: sqrt_d}
    cur, f = sqrt_d, 1
    for target in sorted(factors):
        while f < target:
            f *= 2
            nc, Lc, pc = level_geometry(n, npad, detector_pixel, f)
            plan = Plan(nc, Lc, z1, K, wavelength, Z, pc, device=device, angle_batch=1)
            nxt = torch.empty(K, len(z1), nc, nc, dtype=torch.float32, device=sqrt_d.device)
            plan.bin2(cur.contiguous(), nxt)
            out[f] = nxt
            cur = nxt
    return out


def run_schedule(levels, sqrt_d, shifts, n, npad, z1, wavelength, Z, detector_pixel, psi0, q0,
                 rho_psi=1.0, rho_q=None, device=0, angle_batch=None, on_level=None):
    """levels: [(factor, iterations), ...], factors decreasing powers of two ending anywhere
    (e.g. [(4, 200), (2, 100), (1, 50)]).  psi0 [K][npad/f0][npad/f0] and q0 [npad/f0]^2 are the
    initial guesses at the FIRST (coarsest) level.  Returns (psi, q, history) at the last level;
    history = per level dict(factor, F_start, F_end, iterations, sweeps)."""
    K, nz = sqrt_d.shape[0], sqrt_d.shape[1]
    factors = [f for f, _ in levels]
    if any(b != a // 2 for a, b in zip(factors, factors[1:])):
        raise ValueError("consecutive levels must halve the binning factor")
    pyr = bin_pyramid(sqrt_d, n, npad, z1, K, wavelength, Z, detector_pixel, factors, device)
    psi, q = psi0, q0
    hist = []
    for li, (f, iters) in enumerate(levels):
        nc, Lc, pc = level_geometry(n, npad, detector_pixel, f)
        plan = Plan(nc, Lc, z1, K, wavelength, Z, pc, device=device,
                    angle_batch=angle_batch if angle_batch else max(1, min(8, K)))
        plan.set_shifts(np.asarray(shifts, np.float64) / f)
        if li > 0:  # upsample the previous level's state onto this grid (this plan = fine level)
            psi_f = torch.empty(K, Lc, Lc, dtype=torch.complex64, device=psi.device)
            q_f = torch.empty(Lc, Lc, dtype=torch.complex64, device=psi.device)
            plan.upsample2(psi.contiguous(), psi_f)
            plan.upsample2(q.contiguous(), q_f)
            psi, q = psi_f, q_f
        cg = JointCG(plan, pyr[f].contiguous(), psi, q, rho_psi=rho_psi,
                     rho_q=(1.0 / K if rho_q is None else rho_q))
        F0 = cg.start()
        for _ in range(iters):
            cg.iterate()
        hist.append(dict(factor=f, F_start=F0, F_end=cg.F, iterations=iters, sweeps=cg.sweeps))
        if on_level is not None:
            on_level(hist[-1])
        psi, q = cg.psi, cg.q
        del cg, plan
    return psi, q, hist


# ---------------------------------------------------------------------------------- probe subset
def probe_subset_indices(K, n_sub):
    """n_sub angles spread evenly over [0, K) ("the probe can be approximated by considering
    only a limited set of projections ... 20-50 projections"): round(i K / n_sub), i < n_sub."""
    n_sub = max(1, min(int(n_sub), K))
    return np.unique(np.floor(np.arange(n_sub) * K / n_sub + 0.5).astype(np.int64).clip(0, K - 1))


def run_probe_subset(sqrt_d, shifts, psi0, q0, n_sub, iters_probe, iters_object, make_plan,
                     rho_psi=1.0, rho_q=None, distributed=None):
    """Probe-subset schedule (reading R6 of P:257): stage 1 runs the joint psi/q CG on the n_sub
    angles of probe_subset_indices only (their psi and the shared probe q); stage 2 freezes q
    (rho_q = 0: no probe-gradient work) and runs object-only CG over all K angles, starting from
    psi0 with the subset angles replaced by their stage-1 result.  make_plan(idx) -> a plan whose
    angles are idx (shifts set); stage 1's plan is released before stage 2's is made.
    Returns (psi, q, history) with history = [stage-1 dict, stage-2 dict]."""
    K = sqrt_d.shape[0]
    idx = probe_subset_indices(K, n_sub)
    sel = torch.as_tensor(idx, device=sqrt_d.device)
    plan = make_plan(idx)
    cg = JointCG(plan, sqrt_d.index_select(0, sel).contiguous(), psi0.index_select(0, sel).contiguous(), q0,
                 rho_psi=rho_psi, rho_q=(1.0 / len(idx) if rho_q is None else rho_q), distributed=distributed)
    hist = [dict(stage="probe", angles=[int(i) for i in idx], F_start=cg.start())]
    for _ in range(iters_probe):
        cg.iterate()
    hist[0].update(F_end=cg.F, iterations=iters_probe, sweeps=cg.sweeps)
    q = cg.q.clone()
    psi = psi0.clone()
    psi.index_copy_(0, sel, cg.psi)
    del cg, plan
    plan = make_plan(np.arange(K))
    cg = JointCG(plan, sqrt_d, psi, q, rho_psi=rho_psi, rho_q=0.0, distributed=distributed)
    hist.append(dict(stage="object", angles=K, F_start=cg.start()))
    for _ in range(iters_object):
        cg.iterate()
    hist[1].update(F_end=cg.F, iterations=iters_object, sweeps=cg.sweeps)
    return cg.psi, cg.q, hist
