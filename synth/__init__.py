"""Seeded synthetic inputs for the holotomography hot path (arXiv 2407.20304).

This module is the ONLY code shared by the oracle side (tests) and the CUDA side
(bench, GPU tests).  It holds none of the method's arithmetic -- no propagation,
shift, magnification, residual or gradient: only the workload recipes of
BASELINE.json's configs (readings C13-C16, C19) and the
seeded generators that evaluate them.

Random parameters come from numpy's counter-based Philox-4x32 keyed by
(seed, stream, item) with seed s_i = 240720304 + i; streams:
1 phantom, 2 probe, 3 shifts, 4 noise.  Grid evaluation uses torch so the same
recipe runs on the host (float64, tests) or on the device (float32, bench).
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np
import torch

SEED0 = 240720304
STREAM_PHANTOM, STREAM_PROBE, STREAM_SHIFTS, STREAM_NOISE = 1, 2, 3, 4
WAVELENGTH_33KEV = 3.717667e-11  # m, 33.35 keV with hc = 1.23984198e-6 eV m (reading C18)
Z_FOCUS_DET = 1.208              # m, Table 1
DET_PIXEL = 3.0e-6               # m, binned detector pixel
Z1_4 = (4.584e-3, 4.765e-3, 5.488e-3, 6.990e-3)


@dataclasses.dataclass(frozen=True)
class Config:
    name: str
    n: int               # detector side N
    npad: int            # torus side N_p (2x padding)
    z1: tuple            # focus-to-sample distances [m]
    n_angles: int        # K (cfg4: number of reference frames R = 64 x 4)
    shift_max: float     # shifts ~ U[-shift_max, shift_max] px (psi grid)
    photons: float       # Poisson photons per pixel (reading C13)
    n_stripes: int       # probe stripes (reading C14)
    probe_phase: float   # probe phase stripe amplitude [rad]
    phantom: str         # phantom family (reading C15)
    phase_min: float     # minimum phase of the phantom [rad]
    seed_index: int
    wavelength: float = WAVELENGTH_33KEV
    Z: float = Z_FOCUS_DET
    det_pixel: float = DET_PIXEL
    curvature: bool = False

    @property
    def nz(self):
        return len(self.z1)


CONFIGS = {
    "cfg0": Config("cfg0", 64, 128, (4.58e-3, 5.49e-3), 4, 2.0, 1e4, 6, 0.5, "ellipses", -1.0, 0),
    "cfg1": Config("cfg1", 256, 512, Z1_4, 180, 2.0, 1e4, 12, 0.5, "layers", -0.3, 1),
    "cfg2": Config("cfg2", 1024, 2048, Z1_4, 720, 2.0, 5e3, 24, 0.5, "ellipsoids", -1.5, 2, curvature=True),
    "cfg3": Config("cfg3", 2048, 4096, Z1_4, 1440, 4.0, 1e4, 24, 0.5, "layers_fine", -2.0, 3),
    "cfg4": Config("cfg4", 3072, 6144, Z1_4, 256, 8.0, 2e4, 48, 1.0, "none", 0.0, 4),
}


def rng(cfg_or_seed, stream, item=0):
    seed = SEED0 + (cfg_or_seed.seed_index if isinstance(cfg_or_seed, Config) else int(cfg_or_seed))
    return np.random.Generator(np.random.Philox(key=[seed, stream * 1000003 + item]))


# ------------------------------------------------------------------ shifts --
def shifts(cfg: Config, K=None, seed=None):
    """s^s_kj ~ U[-s, s] per (k, j, axis), float64 [K][nz][2] = (sx, sy) (reading C4)."""
    K = cfg.n_angles if K is None else K
    g = rng(cfg if seed is None else seed, STREAM_SHIFTS)
    return g.uniform(-cfg.shift_max, cfg.shift_max, size=(cfg.n_angles, cfg.nz, 2))[:K].copy()


def ref_shifts(cfg: Config, R=None):
    """cfg4 reference-frame shifts of q, float64 [R][2] (reading C16)."""
    R = cfg.n_angles if R is None else R
    g = rng(cfg, STREAM_SHIFTS, 1)
    return g.uniform(-cfg.shift_max, cfg.shift_max, size=(cfg.n_angles, 2))[:R].copy()


# ------------------------------------------------------------------- probe --
def probe(cfg: Config, L=None, device="cpu", dtype=torch.complex128):
    """q on the L x L torus: Gaussian envelope (sigma = N) x (1 + 0.2/n_s sum of stripes),
    phase (Phi/n_s) sum of stripes; cfg2 adds c pi (|u|/N)^2 (reading C14)."""
    L = cfg.npad if L is None else L
    N = cfg.n * L // cfg.npad
    g = rng(cfg, STREAM_PROBE)
    ns = cfg.n_stripes
    rdt = torch.float64 if dtype == torch.complex128 else torch.float32
    u = torch.arange(L, device=device, dtype=rdt) - L // 2
    Y, X = u[:, None], u[None, :]
    amp_s = torch.zeros(L, L, device=device, dtype=rdt)
    ph_s = torch.zeros(L, L, device=device, dtype=rdt)
    for acc in (amp_s, ph_s):
        horiz = g.random(ns) < 0.5
        period = g.uniform(3.0, 40.0, ns)
        phase0 = g.uniform(0, 2 * math.pi, ns)
        for i in range(ns):
            t = Y if horiz[i] else X
            acc += torch.sin(2 * math.pi * t / float(period[i]) + float(phase0[i]))
    env = torch.exp(-(X * X + Y * Y) / (2.0 * N * N))
    amp = env * (1.0 + 0.2 / ns * amp_s)
    phase = cfg.probe_phase / ns * ph_s
    if cfg.curvature:
        c = float(g.uniform(-1, 1))
        phase = phase + c * math.pi * (X * X + Y * Y) / (N * N)
    return torch.polar(amp, phase).to(dtype)


# ----------------------------------------------------------------- phantom --
def _shapes(cfg: Config):
    """Random shape parameters of the cfg's phantom (reading C15), in units of N."""
    g = rng(cfg, STREAM_PHANTOM)
    if cfg.phantom == "ellipses":  # 2-D, same for every angle
        return [("ellipse", g.uniform(-0.3, 0.3, 2), g.uniform(0.05, 0.25, 2), g.uniform(0, math.pi),
                 g.uniform(0, 1)) for _ in range(8)]
    if cfg.phantom in ("layers", "layers_fine"):
        # nested cube shells; thickness in px of the N grid
        lo, hi = (2, 20) if cfg.phantom == "layers" else (1, 12)
        shells, half = [], 0.36 * cfg.n
        while half > 0.08 * cfg.n:
            th = float(g.integers(lo, hi + 1))
            shells.append(("box", half, float(g.uniform(0.3, 1.0))))
            half -= th
        return shells
    if cfg.phantom == "ellipsoids":
        sh = [("ellipsoid", g.uniform(-0.25, 0.25, 3) * cfg.n, g.uniform(0.03, 0.15, 3) * cfg.n,
               float(g.uniform(0, 1))) for _ in range(12)]
        half, inset = 0.12 * cfg.n, []
        while half > 0.03 * cfg.n:
            inset.append(("box", half, float(g.uniform(0.3, 1.0))))
            half -= float(g.integers(1, 6))
        return sh + inset
    return []


def _box_chord(X, Yv, half, theta):
    """Length of a ray through the cube [-half, half]^3 rotated by theta about y.
    Rays travel along the beam; X is the detector coordinate normal to the rotation axis."""
    c, s = math.cos(theta), math.sin(theta)
    # slab intersection in the rotated x-z plane: ray p(t) = X e_x' + t e_z'
    big = torch.full_like(X, 1e30)
    tmin = torch.full_like(X, -1e30)
    tmax = big.clone()
    for (ax, az) in ((c, s), (-s, c)):  # the two rotated slab normals projected on (X, t)
        # coordinate along the normal: X*ax + t*az  in [-half, half]
        if abs(az) < 1e-12:
            inside = (X * ax).abs() <= half
            tmin = torch.where(inside, tmin, big)
            continue
        t1 = (-half - X * ax) / az
        t2 = (half - X * ax) / az
        tmin = torch.maximum(tmin, torch.minimum(t1, t2))
        tmax = torch.minimum(tmax, torch.maximum(t1, t2))
    chord = (tmax - tmin).clamp(min=0)
    return torch.where(Yv.abs() <= half, chord, torch.zeros_like(chord))


def phase_map(cfg: Config, k, K, device="cpu", dtype=torch.float64):
    """phi_k on the N x N detector window (unnormalised, <= 0) for angle theta_k = pi k / K."""
    N = cfg.n
    u = torch.arange(N, device=device, dtype=dtype) - N // 2
    Y, X = u[:, None].expand(N, N), u[None, :].expand(N, N)
    S = torch.zeros(N, N, device=device, dtype=dtype)
    theta = math.pi * k / max(K, 1)
    sign = 1.0
    for sh in _shapes(cfg):
        if sh[0] == "ellipse":
            _, cxy, ab, rot, wgt = sh
            c, s = math.cos(rot), math.sin(rot)
            xr = (X - cxy[0] * N) * c + (Y - cxy[1] * N) * s
            yr = -(X - cxy[0] * N) * s + (Y - cxy[1] * N) * c
            S += float(wgt) * ((xr / (ab[0] * N)) ** 2 + (yr / (ab[1] * N)) ** 2 <= 1).to(dtype)
        elif sh[0] == "box":  # alternating-delta nested shells
            _, half, wgt = sh
            S += sign * wgt * _box_chord(X, Y, half, theta) / N
            sign = -sign
        elif sh[0] == "ellipsoid":
            _, cen, ax, wgt = sh
            c, s = math.cos(theta), math.sin(theta)
            # ellipsoid centre rotated about y; axis-aligned semi-axes rotated with it
            xc = cen[0] * c + cen[2] * s
            # chord of a ray along the rotated z through an ellipsoid: 2 * sqrt(1 - r^2) * t_half
            ex = math.sqrt((ax[0] * c) ** 2 + (ax[2] * s) ** 2)
            r2 = ((X - xc) / ex) ** 2 + ((Y - cen[1]) / ax[1]) ** 2
            thick = ax[0] * ax[2] / ex
            S += float(wgt) * 2 * thick * torch.sqrt((1 - r2).clamp(min=0)) / N
    S = S.abs() if cfg.phantom == "ellipses" else S - S.min()
    return S


def psi_stack(cfg: Config, K=None, L=None, device="cpu", dtype=torch.complex128, k0=0):
    """psi_k = exp(i phi - 0.01 |phi|) on the L x L torus, phi supported in the central
    N x N window scaled to [phase_min, 0]; psi = 1 in the padding ring (reading C3, C15)."""
    K = cfg.n_angles if K is None else K
    L = cfg.npad if L is None else L
    N = cfg.n
    rdt = torch.float64 if dtype == torch.complex128 else torch.float32
    out = torch.ones(K, L, L, device=device, dtype=dtype)
    if cfg.phantom == "none":
        return out
    o = (L - N) // 2
    for i in range(K):
        S = phase_map(cfg, k0 + i, cfg.n_angles, device=device, dtype=rdt)
        m = S.abs().max()
        phi = cfg.phase_min * S / (m if m > 0 else 1)
        out[i, o:o + N, o:o + N] = torch.polar(torch.exp(-0.01 * phi.abs()), phi).to(dtype)
    return out


# ------------------------------------------------------------------- noise --
def poisson_amplitude(intensity, photons, cfg: Config, item=0):
    """a = sqrt(Poisson(n |w|^2) / n)  (reading C13: the paper's /20 protocol)."""
    if isinstance(intensity, torch.Tensor) and intensity.is_cuda:
        gen = torch.Generator(device=intensity.device)
        gen.manual_seed(SEED0 + cfg.seed_index * 7919 + item)
        return torch.sqrt(torch.poisson(intensity * photons, generator=gen) / photons)
    g = rng(cfg, STREAM_NOISE, item)
    x = np.asarray(intensity)
    return np.sqrt(g.poisson(x * photons) / photons)


def small_geometry_case(seed=0, L=16, N=8, K=2, nz=2):
    """A 16 x 16 torus instance for finite-difference pins (mt != 1, random shifts):
    random smooth-ish psi and q (complex128 numpy) and shifts."""
    g = rng(seed, 9)
    psi = (1 + 0.3 * (g.standard_normal((K, L, L)) + 1j * g.standard_normal((K, L, L))))
    q = (1 + 0.3 * (g.standard_normal((L, L)) + 1j * g.standard_normal((L, L))))
    s = g.uniform(-2, 2, size=(K, nz, 2))
    return psi, q, s
