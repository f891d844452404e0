"""fp64 CPU oracle for the hot path of arXiv 2407.20304 -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product package
``paper_2407_20304_b200`` never imports it and shares no code with it.

Two independent implementations of the same definitions (O1..O14):

* ``liboracle.so`` (``holo_oracle.c``): plain C, naive O(L^2) DFT per axis, OpenMP
  over lines -- the oracle named by BASELINE.json's north_star.
* ``np_oracle`` (``np_oracle.py``): numpy, ``numpy.fft`` as the DFT primitive and
  the O5 magnification as an explicit dense matrix; used where the naive C
  oracle would take minutes (L >= 2048).  Cross-checked against the C oracle.

The CG reference (O13, Eqs. (13)-(14)) is ``oracle.cg``.

Array conventions: complex128 arrays row-major [y][x]; per-frame arrays [k][j][y][x];
shifts float64 [K][nz][2] = (sx, sy) in psi-grid pixels (reading C4).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "holo_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (plain -O2, OpenMP, no -ffast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + ".tmp%d" % os.getpid()
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=c11",
                               _SRC, "-o", tmp, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        P = ctypes.c_void_p
        D = ctypes.c_double
        Ic = ctypes.c_int
        lib.or_geometry.argtypes = [Ic, D, P, D, P, P, P, P, P, P]
        lib.or_geometry.restype = Ic
        lib.or_dft1.argtypes = [Ic, Ic, P, P]
        lib.or_prop.argtypes = [Ic, D, D, D, P, P]
        lib.or_shift.argtypes = [Ic, D, D, P, P]
        lib.or_mag.argtypes = [Ic, D, D, D, P, P]
        lib.or_mag_adj.argtypes = [Ic, D, D, D, P, P]
        geo = [Ic, Ic, Ic, Ic, D, D, P, P, P, P]
        lib.or_fwd.argtypes = geo + [P, P, P]
        lib.or_adj.argtypes = geo + [P, P, P, P, P]
        lib.or_grad.argtypes = geo + [P, P, P, P, P]
        lib.or_grad.restype = D
        lib.or_grad_ref.argtypes = [Ic, Ic, Ic, D, D, D, P, P, P, P]
        lib.or_grad_ref.restype = D
        lib.or_upsample2.argtypes = [Ic, P, P]
        lib.or_bin2.argtypes = [Ic, Ic, P, P]
        lib.or_init_probe.argtypes = [Ic, Ic, Ic, D, D, D, P, P, P]
        lib.or_grad_full.argtypes = geo + [P, P, P, P, Ic, D, P, P, P, P]
        lib.or_grad_full.restype = D
        lib.or_multipaganin.argtypes = [Ic, Ic, Ic, D, D, P, P, P, P, P, D, P]
        _lib = lib
    return _lib


def _c(a, dtype):
    a = np.ascontiguousarray(a, dtype=dtype)
    return a


def _p(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


class Geometry:
    """O1: derived geometry (Eq. (8); Thm 2; Eq. (6))."""

    def __init__(self, wavelength, Z, z1, detector_pixel):
        lib = _load()
        z1 = _c(z1, np.float64)
        nz = z1.size
        self.nz, self.wavelength, self.Z, self.z1, self.detector_pixel = nz, float(wavelength), float(Z), z1, float(detector_pixel)
        m0, p0 = ctypes.c_double(), ctypes.c_double()
        self.mt, self.zeta, self.zdet, self.omega = (np.zeros(nz) for _ in range(4))
        rc = lib.or_geometry(nz, self.Z, _p(z1), self.detector_pixel, ctypes.byref(m0), _p(self.mt),
                             _p(self.zeta), _p(self.zdet), _p(self.omega), ctypes.byref(p0))
        if rc != 0:
            raise ValueError("invalid geometry")
        self.m0, self.p0 = m0.value, p0.value


def dft1(x, inverse=False):
    """O2: X[f] = sum_n x[n] exp(-2 pi i f n / L); inverse scaled by 1/L."""
    x = _c(x, np.complex128)
    out = np.empty_like(x)
    _load().or_dft1(x.size, int(bool(inverse)), _p(x), _p(out))
    return out


def prop(x, wavelength, p0, z):
    """O3: P_z on an [L][L] torus."""
    x = _c(x, np.complex128)
    out = np.empty_like(x)
    _load().or_prop(x.shape[0], float(wavelength), float(p0), float(z), _p(x), _p(out))
    return out


def shift(x, sx, sy):
    """O4: S_(sx,sy), periodic Fourier shift, (S_s x)(u) = x(u - s)."""
    x = _c(x, np.complex128)
    out = np.empty_like(x)
    _load().or_shift(x.shape[0], float(sx), float(sy), _p(x), _p(out))
    return out


def mag(x, mt, sx=0.0, sy=0.0):
    """O5: M_{1/mt} S_(sx,sy) x  (band-limited Fourier rescale about the grid centre)."""
    x = _c(x, np.complex128)
    out = np.empty_like(x)
    _load().or_mag(x.shape[0], float(mt), float(sx), float(sy), _p(x), _p(out))
    return out


def mag_adj(y, mt, sx=0.0, sy=0.0):
    """O5 adjoint: (M_{1/mt} S_s)^* y."""
    y = _c(y, np.complex128)
    out = np.empty_like(y)
    _load().or_mag_adj(y.shape[0], float(mt), float(sx), float(sy), _p(y), _p(out))
    return out


def _geo_args(geom: Geometry, K, L, N, shifts):
    shifts = _c(shifts, np.float64).reshape(K, geom.nz, 2)
    return shifts, [K, geom.nz, L, N, geom.wavelength, geom.p0, _p(geom.mt), _p(geom.zdet), _p(geom.omega), _p(shifts)]


def fwd(geom: Geometry, psi, q, shifts, N):
    """O6-O7: w[k][j] = C P_{zdet_j}(q_j . M_{1/mt_j} S_{s_kj} psi_k), q_j = P_{omega_j} q."""
    psi = _c(psi, np.complex128)
    q = _c(q, np.complex128)
    K, L = psi.shape[0], psi.shape[1]
    shifts, ga = _geo_args(geom, K, L, N, shifts)
    w = np.empty((K, geom.nz, N, N), np.complex128)
    _load().or_fwd(*ga, _p(psi), _p(q), _p(w))
    return w


def adj(geom: Geometry, y, psi, q, shifts, want_psi=True, want_q=True):
    """Adjoints of the two linearisations at (psi, q) (no factor 2)."""
    psi = _c(psi, np.complex128)
    q = _c(q, np.complex128)
    y = _c(y, np.complex128)
    K, L = psi.shape[0], psi.shape[1]
    N = y.shape[-1]
    shifts, ga = _geo_args(geom, K, L, N, shifts)
    ap = np.empty_like(psi) if want_psi else None
    aq = np.empty_like(q) if want_q else None
    _load().or_adj(*ga, _p(y), _p(psi), _p(q), _p(ap), _p(aq))
    return ap, aq


def grad(geom: Geometry, psi, q, shifts, sqrt_d, want_psi=True, want_q=True):
    """O8-O12: (F, grad_psi, grad_q) of F1 (Eq. (10)) at (psi, q)."""
    psi = _c(psi, np.complex128)
    q = _c(q, np.complex128)
    sqrt_d = _c(sqrt_d, np.float64)
    K, L = psi.shape[0], psi.shape[1]
    N = sqrt_d.shape[-1]
    shifts, ga = _geo_args(geom, K, L, N, shifts)
    gp = np.empty_like(psi) if want_psi else None
    gq = np.empty_like(q) if want_q else None
    F = _load().or_grad(*ga, _p(psi), _p(q), _p(sqrt_d), _p(gp), _p(gq))
    return F, gp, gq


def grad_ref(geom: Geometry, q, ref_shifts, sqrt_dref, want_q=True):
    """O14: reference arm F_ref and its q-gradient 2 sum_r S_{-s_r} P_{-zeta0} Z rho^r."""
    q = _c(q, np.complex128)
    sqrt_dref = _c(sqrt_dref, np.float64)
    R, N = sqrt_dref.shape[0], sqrt_dref.shape[-1]
    L = q.shape[0]
    rs = _c(ref_shifts, np.float64).reshape(R, 2)
    gq = np.zeros_like(q) if want_q else None
    F = _load().or_grad_ref(R, L, N, geom.wavelength, geom.p0, float(geom.zeta[0]), _p(rs), _p(q),
                            _p(sqrt_dref), _p(gq))
    return F, gq


def crop(x, N):
    """C: central N x N window of an L x L array, offset o = (L - N)/2 (O7)."""
    L = x.shape[-1]
    o = (L - N) // 2
    return x[..., o:o + N, o:o + N]


def zpad(x, L):
    """Z = C^T: zero-pad an N x N array into the centre of an L x L torus."""
    N = x.shape[-1]
    o = (L - N) // 2
    out = np.zeros(x.shape[:-2] + (L, L), dtype=np.result_type(x, np.complex128))
    out[..., o:o + N, o:o + N] = x
    return out


def upsample2(x):
    """O15: Fourier 2x upsampling [L][L] -> [2L][2L], coarse sample n at fine coordinate
    2n + 1/2 (multiresolution schedule P:258-259; reading R1).  Naive sums."""
    x = _c(x, np.complex128)
    L = x.shape[-1]
    out = np.empty((2 * L, 2 * L), np.complex128)
    _load().or_upsample2(L, _p(x), _p(out))
    return out


def bin2(a):
    """O16: 2x2 binning of amplitudes a = sqrt(d~) [M][2N][2N] -> [M][N][N]: the binned
    intensity is the block mean of the four intensities (reading R2)."""
    a = _c(a, np.float64)
    M, N = a.shape[0], a.shape[-1] // 2
    out = np.empty((M, N, N), np.float64)
    _load().or_bin2(M, N, _p(a), _p(out))
    return out


def init_probe(geom: Geometry, ref_shifts, sqrt_dref, L):
    """O17: q0 = (1/R) sum_r S_{-s_r} P_{-zeta0} Z_{c_r}(sqrt d~^r_r), ring = frame mean (reading R3)."""
    sqrt_dref = _c(sqrt_dref, np.float64)
    R, N = sqrt_dref.shape[0], sqrt_dref.shape[-1]
    rs = _c(ref_shifts, np.float64).reshape(R, 2)
    q0 = np.empty((L, L), np.complex128)
    _load().or_init_probe(R, L, N, geom.wavelength, geom.p0, float(geom.zeta[0]), _p(rs), _p(sqrt_dref), _p(q0))
    return q0


def multipaganin(geom: Geometry, L, shifts_k, sqrt_d_k, sqrt_dref, delta_beta):
    """O18: multi-distance Paganin initial object of one angle (reading R4); shifts_k [nz][2],
    sqrt_d_k [nz][N][N], sqrt_dref [N][N]."""
    sqrt_d_k = _c(sqrt_d_k, np.float64)
    sqrt_dref = _c(sqrt_dref, np.float64)
    sk = _c(shifts_k, np.float64).reshape(geom.nz, 2)
    N = sqrt_dref.shape[-1]
    out = np.empty((L, L), np.complex128)
    _load().or_multipaganin(geom.nz, L, N, geom.wavelength, geom.p0, _p(geom.mt), _p(geom.zeta), _p(sk),
                            _p(sqrt_d_k), _p(sqrt_dref), float(delta_beta), _p(out))
    return out


def grad_full(geom: Geometry, psi, q, shifts, pshifts, sqrt_d, ref_shifts=None, sqrt_dref=None,
              want_psi=True, want_q=True):
    """O19: F and gradients of the full Eq. (10) objective -- per-frame probe shifts s^p_kj
    (q_kj = P_omega S_{s^p} q) and, when sqrt_dref is given, the reference term (O14)."""
    psi = _c(psi, np.complex128)
    q = _c(q, np.complex128)
    sqrt_d = _c(sqrt_d, np.float64)
    K, L = psi.shape[0], psi.shape[1]
    N = sqrt_d.shape[-1]
    shifts, ga = _geo_args(geom, K, L, N, shifts)
    ps = _c(pshifts, np.float64).reshape(K, geom.nz, 2)
    R = 0 if sqrt_dref is None else sqrt_dref.shape[0]
    rs = _c(ref_shifts if R else np.zeros((1, 2)), np.float64).reshape(-1, 2)
    dr = _c(sqrt_dref if R else np.zeros((1, N, N)), np.float64)
    gp = np.empty_like(psi) if want_psi else None
    gq = np.empty_like(q) if want_q else None
    F = _load().or_grad_full(*ga, _p(ps), _p(psi), _p(q), _p(sqrt_d), R, float(geom.zeta[0]), _p(rs), _p(dr),
                             _p(gp), _p(gq))
    return F, gp, gq
