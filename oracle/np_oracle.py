"""numpy fp64 oracle for large tori -- TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Same definitions as holo_oracle.c (O3..O12), with two library
primitives standing in for naive sums so that L = 2048 / 4096 frames finish in
seconds: ``numpy.fft`` for the DFT (O2) and a dense matrix product for the O5
evaluation sum.  Nothing here is blocked, fused or reordered beyond that.

    O5:  Xc[f] = sum_n x[n] e^{-2 pi i fbar u(n)/L} = e^{i pi fbar} FFT(x)[f]   (u(n) = n - L/2)
         y[n]  = (1/L) sum_f E[n, f] kappa[f] r_s[f] Xc[f],  E[n, f] = e^{+2 pi i mt fbar u(n)/L}
"""
from __future__ import annotations

import numpy as np


def fbar(L):
    f = np.arange(L)
    return np.where(f < L // 2, f, f - L)


def transfer(L, wavelength, p0, z):
    """O3: h_z[f] = exp(-i pi lambda z (fbar/(L p0))^2)."""
    fr = fbar(L) / (L * p0)
    return np.exp(-1j * np.pi * wavelength * z * fr * fr)


def ramp(L, s):
    """O4: r_s[f] = exp(-2 pi i fbar s / L)."""
    return np.exp(-2j * np.pi * fbar(L) * s / L)


def kappa(L, mt):
    v = mt * fbar(L)
    return ((v >= -(L // 2)) & (v < L // 2)).astype(np.float64)


def prop(x, wavelength, p0, z):
    L = x.shape[-1]
    h = transfer(L, wavelength, p0, z)
    return np.fft.ifft2(np.fft.fft2(x) * h[:, None] * h[None, :])


def shift(x, sx, sy):
    L = x.shape[-1]
    return np.fft.ifft2(np.fft.fft2(x) * ramp(L, sy)[:, None] * ramp(L, sx)[None, :])


class MagOp:
    """O5 for one (L, mt): E[n, f] = exp(+2 pi i mt fbar u(n) / L), phase reduced mod L."""

    def __init__(self, L, mt):
        self.L, self.mt = L, float(mt)
        u = np.arange(L) - L // 2
        fb = fbar(L)
        p = self.mt * (u[:, None] * fb[None, :]).astype(np.float64)
        p -= L * np.floor(p / L)
        self.E = np.exp(2j * np.pi * p / L)
        self.kap = kappa(L, mt)
        self.centre = np.exp(1j * np.pi * fb)  # e^{i pi fbar} = (-1)^fbar

    def _axis_fwd(self, x, s, axis):
        X = np.fft.fft(x, axis=axis)
        c = self.centre * self.kap * ramp(self.L, s)
        if axis == 1:
            return (X * c[None, :]) @ self.E.T / self.L
        return self.E @ (X * c[:, None]) / self.L

    def _axis_adj(self, y, s, axis):
        c = np.conj(self.centre) * self.kap * np.conj(ramp(self.L, s))
        if axis == 1:
            Zf = y @ np.conj(self.E)
            return np.fft.ifft(Zf * c[None, :], axis=1)
        Zf = np.conj(self.E).T @ y
        return np.fft.ifft(Zf * c[:, None], axis=0)

    def fwd(self, x, sx, sy):
        """M_{1/mt} S_(sx,sy) x: along x with sx, then along y with sy."""
        return self._axis_fwd(self._axis_fwd(x, sx, 1), sy, 0)

    def adj(self, y, sx, sy):
        return self._axis_adj(self._axis_adj(y, sy, 0), sx, 1)


def crop(x, N):
    L = x.shape[-1]
    o = (L - N) // 2
    return x[..., o:o + N, o:o + N]


def zpad(x, L):
    N = x.shape[-1]
    o = (L - N) // 2
    out = np.zeros(x.shape[:-2] + (L, L), np.complex128)
    out[..., o:o + N, o:o + N] = x
    return out


class Problem:
    """Frame-level forward / residual / gradient contributions (O6..O12).

    ``geom`` carries wavelength, p0, mt[], zdet[], omega[] (oracle.Geometry)."""

    def __init__(self, geom, L, N):
        self.g, self.L, self.N = geom, L, N
        self._mag = {}

    def mag(self, j):
        if j not in self._mag:
            self._mag[j] = MagOp(self.L, self.g.mt[j])
        return self._mag[j]

    def qj(self, q, j):
        return prop(q, self.g.wavelength, self.g.p0, self.g.omega[j])

    def frame_fwd(self, psi_k, qj, j, s):
        a = self.mag(j).fwd(psi_k, s[0], s[1])
        return crop(prop(qj * a, self.g.wavelength, self.g.p0, self.g.zdet[j]), self.N), a

    def frame_grad(self, psi_k, qj, j, s, sqrt_d, tau=1):
        """One frame (k, j): returns F_kj, 2 L_kj^* rho, and conj(a) v (the G_j term, no 2, no P_{-omega}).
        tau = 1: F_1 (Eq. (10)), rho = w - sqrt_d w/|w|;  tau = 2: F_2 (Eq. (9)), F = (|w|^2 - d)^2,
        rho = h'(|w|^2) w = 2 (|w|^2 - d) w  (App. A.3 proposition with h(t) = (t - d)^2); any other
        tau: the general penalty G_tau (residual_tau)."""
        w, a = self.frame_fwd(psi_k, qj, j, s)
        m = np.abs(w)
        if tau == 2:
            dm = m ** 2 - sqrt_d ** 2
            F = float(np.sum(dm ** 2))
            rho = 2.0 * dm * w
        elif tau != 1:  # general G_tau (App. A.3)
            F, rho = residual_tau(w, np.asarray(sqrt_d, np.float64), tau)
        else:
            F = float(np.sum((m - sqrt_d) ** 2))
            with np.errstate(invalid="ignore", divide="ignore"):
                rho = np.where(m > 0, w - sqrt_d * w / np.where(m > 0, m, 1), 0)
        v = prop(zpad(rho, self.L), self.g.wavelength, self.g.p0, -self.g.zdet[j])
        gpsi = 2.0 * self.mag(j).adj(np.conj(qj) * v, s[0], s[1])
        return F, gpsi, np.conj(a) * v

    def grad(self, psi, q, shifts, sqrt_d, frames=None, tau=1):
        """F, grad_psi, grad_q over all frames (or a subset: list of (k, j))."""
        K, nz = psi.shape[0], self.g.nz
        frames = frames if frames is not None else [(k, j) for j in range(nz) for k in range(K)]
        F = 0.0
        gpsi = np.zeros_like(psi, dtype=np.complex128)
        G = {}
        qjs = {}
        for (k, j) in frames:
            if j not in qjs:
                qjs[j] = self.qj(q, j)
            Fk, gk, Gk = self.frame_grad(psi[k], qjs[j], j, shifts[k, j], sqrt_d[k, j], tau)
            F += Fk
            gpsi[k] += gk
            G[j] = G.get(j, 0) + Gk
        gq = np.zeros((self.L, self.L), np.complex128)
        for j in sorted(G):
            gq += 2.0 * prop(G[j], self.g.wavelength, self.g.p0, -self.g.omega[j])
        return F, gpsi, gq

    def qkj(self, q, j, sp):
        """O19: q_kj = P_{omega_j} S_{s^p_kj} q (Eq. (10), probe shift s^p)."""
        return prop(shift(q, float(sp[0]), float(sp[1])), self.g.wavelength, self.g.p0, self.g.omega[j])

    def grad_full(self, psi, q, shifts, pshifts, sqrt_d, ref_shifts=None, sqrt_dref=None, tau=1, frames=None):
        """O19: F, grad_psi, grad_q of Eq. (10) with probe shifts (Q_kj^* = S_{-s^p} P_{-omega} (.)) and,
        when sqrt_dref is given, the reference term (O14) -- Eq. (12) P:125-129."""
        K, nz = psi.shape[0], self.g.nz
        frames = frames if frames is not None else [(k, j) for j in range(nz) for k in range(K)]
        F = 0.0
        gpsi = np.zeros_like(psi, dtype=np.complex128)
        gq = np.zeros((self.L, self.L), np.complex128)
        for (k, j) in frames:
            sp = pshifts[k, j]
            Fk, gk, Gk = self.frame_grad(psi[k], self.qkj(q, j, sp), j, shifts[k, j], sqrt_d[k, j], tau)
            F += Fk
            gpsi[k] += gk
            gq += 2.0 * shift(prop(Gk, self.g.wavelength, self.g.p0, -self.g.omega[j]), -float(sp[0]), -float(sp[1]))
        if sqrt_dref is not None:
            Fr, gr = grad_ref(self.g.wavelength, self.g.p0, self.g.zeta[0], q, ref_shifts, sqrt_dref, tau=tau)
            F += Fr
            gq += gr
        return F, gpsi, gq

    def fwd_full(self, psi, q, shifts, pshifts):
        K, nz = psi.shape[0], self.g.nz
        return {(k, j): self.frame_fwd(psi[k], self.qkj(q, j, pshifts[k, j]), j, shifts[k, j])[0]
                for k in range(K) for j in range(nz)}

    def fwd(self, psi, q, shifts, frames=None):
        K, nz = psi.shape[0], self.g.nz
        frames = frames if frames is not None else [(k, j) for k in range(K) for j in range(nz)]
        out = {}
        qjs = {}
        for (k, j) in frames:
            if j not in qjs:
                qjs[j] = self.qj(q, j)
            out[(k, j)] = self.frame_fwd(psi[k], qjs[j], j, shifts[k, j])[0]
        return out


def grad_ref(wavelength, p0, zeta0, q, ref_shifts, sqrt_dref, want_q=True, tau=1):
    """O14 (reference constraint P:102; Eq. (10) reference term P:115; Eq. (12)),
    numpy.fft as the DFT:  w_r = C(P_{zeta0} S_{s_r} q),  F = sum_r || |w_r| - sqrt_dref_r ||^2,
    grad_q = 2 sum_r S_{-s_r} P_{-zeta0} Z rho_r,  rho = w - a w/|w| (0 at w = 0)."""
    L = q.shape[-1]
    N = sqrt_dref.shape[-1]
    F = 0.0
    gq = np.zeros((L, L), np.complex128) if want_q else None
    for r in range(sqrt_dref.shape[0]):
        sx, sy = float(ref_shifts[r][0]), float(ref_shifts[r][1])
        w = crop(prop(shift(q, sx, sy), wavelength, p0, zeta0), N)
        a = np.asarray(sqrt_dref[r], np.float64)
        m = np.abs(w)
        if tau == 2:  # F_2 reference term (Eq. (9)): (|w|^2 - d)^2, rho = 2 (|w|^2 - d) w
            dm = m ** 2 - a ** 2
            F += float(np.sum(dm ** 2))
            rho = 2.0 * dm * w
        elif tau != 1:  # general G_tau (App. A.3)
            Fr, rho = residual_tau(w, a, tau)
            F += Fr
        else:
            F += float(np.sum((m - a) ** 2))
            rho = np.where(m > 0, w - a * w / np.where(m > 0, m, 1.0), 0.0)
        if want_q:
            gq += 2.0 * shift(prop(zpad(rho, L), wavelength, p0, -zeta0), -sx, -sy)
    return F, gq


def residual_tau(w, a, tau):
    """G_tau penalty of App. A.3 for general tau > 0, written out from the proposition:
    h(phi) = (phi^{tau/2} - a^tau)^2, phi = |w|^2  ->  F = sum h(|w|^2),
    h'(phi) = tau (phi^{tau/2} - a^tau) phi^{tau/2 - 1}  ->  rho = h'(|w|^2) w  (0 where w = 0, reading C7).
    The gradient is 2 L^*(rho) (the proposition's 2 L^*(H'(|L psi|^2) . L psi))."""
    phi = np.abs(w) ** 2
    with np.errstate(invalid="ignore", divide="ignore"):
        dm = np.where(phi > 0, phi ** (tau / 2.0), 0.0) - a ** tau
        hp = np.where(phi > 0, tau * dm * np.where(phi > 0, phi, 1.0) ** (tau / 2.0 - 1.0), 0.0)
    return float(np.sum(dm ** 2)), hp * w


def upsample2(x):
    """O15 with numpy.fft as the DFT: per axis Y[F] = 2 X[F] e^{-i pi Fbar/(2L)} on the 2L grid for
    Fbar in [-L/2, L/2) (zero elsewhere), y = IFFT_2L(Y)  (coarse n at fine 2n + 1/2, reading R1)."""
    def last_axis(a):
        L = a.shape[-1]
        fbv = fbar(L)
        Y = np.zeros(a.shape[:-1] + (2 * L,), np.complex128)
        Y[..., np.where(fbv >= 0, fbv, fbv + 2 * L)] = np.fft.fft(a, axis=-1) * 2.0 * np.exp(-1j * np.pi * fbv / (2 * L))
        return np.fft.ifft(Y, axis=-1)
    y = last_axis(np.asarray(x, np.complex128))  # x (rows)
    return last_axis(y.swapaxes(-1, -2)).swapaxes(-1, -2)  # then y (columns)


def bin2(a):
    """O16: a_c = sqrt(block mean of a^2) over 2x2 blocks, [..., 2N, 2N] -> [..., N, N]."""
    a = np.asarray(a, np.float64)
    s = a[..., 0::2, 0::2] ** 2 + a[..., 1::2, 0::2] ** 2 + a[..., 0::2, 1::2] ** 2 + a[..., 1::2, 1::2] ** 2
    return np.sqrt(0.25 * s)


def pad_const(a, L, c):
    """Z_c: the N x N frame a centred on the L x L torus, the ring filled with the constant c."""
    N = a.shape[-1]
    o = (L - N) // 2
    out = np.full(a.shape[:-2] + (L, L), c, np.complex128)
    out[..., o:o + N, o:o + N] = a
    return out


def init_probe(wavelength, p0, zeta0, ref_shifts, sqrt_dref, L):
    """O17 ("the reference image propagated back to the sample plane 0";
    reference model |P_{zeta0} S_{s_r} q|^2 = d~^r, P:102 / Eq. (10)):
        q0 = (1/R) sum_r S_{-s_r} P_{-zeta0} Z_{c_r}(sqrt d~^r_r),  c_r = mean of sqrt d~^r_r,
    the amplitude with zero phase, each frame padded with its mean amplitude (reading R3)."""
    R = sqrt_dref.shape[0]
    q0 = np.zeros((L, L), np.complex128)
    for r in range(R):
        a = np.asarray(sqrt_dref[r], np.float64)
        x = pad_const(a, L, a.mean())
        q0 += shift(prop(x, wavelength, p0, -zeta0), -float(ref_shifts[r][0]), -float(ref_shifts[r][1]))
    return q0 / R


def multipaganin(geom, L, shifts_k, sqrt_d_k, sqrt_dref, delta_beta):
    """O18: multi-distance Paganin (TIE) initial object for one angle (the formula is
    absent from the paper -- SPEC's documented stand-in, in this build's sign convention, reading R4):
      R_j = (sqrt_d_kj / sqrt_dref)^2 (flat-field; sqrt_dref^2 floored at 1e-6 max), padded with 1;
      I_j = M_{1/mt'} S_{s'} R_j with mt' = 1/mt_j, s' = -s_kj/mt_j   (O5: undo the plane's
            magnification and shift, so I_j ~ |P_{zeta_j} psi_k|^2 on the psi grid, Eq. (7));
      Phi = sum_j DFT2(I_j) / (N_z + pi lambda delta_beta sum_j zeta_j |f|^2),  |f| = fbar / (L p0);
      phi = (delta_beta / 2) ln max(Re IDFT2(Phi), 1e-6);   psi0 = exp((i + 1/delta_beta) phi)."""
    nz = geom.nz
    a_r2 = np.asarray(sqrt_dref, np.float64) ** 2
    a_r2 = np.maximum(a_r2, 1e-6 * a_r2.max())
    fb = fbar(L) / (L * geom.p0)
    f2 = fb[:, None] ** 2 + fb[None, :] ** 2
    num = np.zeros((L, L), np.complex128)
    for j in range(nz):
        Rj = pad_const(np.asarray(sqrt_d_k[j], np.float64) ** 2 / a_r2, L, 1.0)
        mtp = 1.0 / geom.mt[j]
        Ij = MagOp(L, mtp).fwd(Rj, -shifts_k[j][0] * mtp, -shifts_k[j][1] * mtp)
        num += np.fft.fft2(Ij)
    den = nz + np.pi * geom.wavelength * delta_beta * float(np.sum(geom.zeta)) * f2
    T = np.real(np.fft.ifft2(num / den))
    phi = 0.5 * delta_beta * np.log(np.maximum(T, 1e-6))
    return np.exp((1j + 1.0 / delta_beta) * phi)
