"""Multiresolution schedule.

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
