"""B200-native hot path of arXiv 2407.20304 (joint object/probe holotomography).

Thin ctypes binding over the C ABI of ``include/holo.h`` (``libholo.so``, sm_100a):
argument marshalling only -- every step of the path runs in the library's CUDA
kernels.  PyTorch supplies device memory, streams and ``torch.distributed``.

There is no CPU fallback: importing this package on a machine without the built
library raises, and every call requires CUDA tensors.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np
import torch

from . import _build

HOLO_OK, HOLO_EINVAL, HOLO_ENOMEM, HOLO_ECUDA, HOLO_EUNSUPPORTED, HOLO_ESTATE = 0, -1, -2, -3, -4, -5
HOLO_ACCUMULATE_Q = 1
HOLO_OBJECTIVE_ONLY = 2
HOLO_INTENSITY = 4  # F_2 (tau = 2)
HOLO_MAX_NZ = 8
HOLO_MAX_BATCH = 16

LIB_PATH = os.environ.get("HOLO_LIB", _build.LIB)  # HOLO_LIB: a tuning-variant build of the same sources
if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"libholo.so not found at {LIB_PATH}: build it with `python paper_2407_20304_b200/_build.py` "
        "(there is no CPU fallback)")
_lib = ctypes.CDLL(LIB_PATH)


class HoloGeometry(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int32), ("npad", ctypes.c_int32), ("nz", ctypes.c_int32),
                ("n_angles", ctypes.c_int32), ("angle_batch", ctypes.c_int32),
                ("wavelength", ctypes.c_double), ("focus_to_detector", ctypes.c_double),
                ("z1", ctypes.c_double * HOLO_MAX_NZ), ("detector_pixel", ctypes.c_double)]


class HoloCgIn(ctypes.Structure):
    _fields_ = [("gPg", ctypes.c_double), ("g_eta_prev", ctypes.c_double), ("gprev_eta_prev", ctypes.c_double),
                ("gamma", ctypes.c_double), ("rho_psi", ctypes.c_double), ("rho_q", ctypes.c_double),
                ("first", ctypes.c_int32), ("reuse_eta", ctypes.c_int32)]


class HoloCgOut(ctypes.Structure):
    _fields_ = [("beta", ctypes.c_double), ("g_eta_new", ctypes.c_double), ("reset", ctypes.c_int32)]


_P = ctypes.c_void_p
_S = ctypes.c_int
_lib.holo_plan_create.argtypes = [ctypes.POINTER(_P), ctypes.POINTER(HoloGeometry), ctypes.c_int, _P]
_lib.holo_plan_create.restype = _S
_lib.holo_plan_destroy.argtypes = [_P]
_lib.holo_plan_destroy.restype = None
_lib.holo_plan_workspace_bytes.argtypes = [_P]
_lib.holo_plan_workspace_bytes.restype = ctypes.c_size_t
_lib.holo_last_error.argtypes = [_P]
_lib.holo_last_error.restype = ctypes.c_char_p
_lib.holo_launch_count.argtypes = [_P]
_lib.holo_launch_count.restype = ctypes.c_uint64
_lib.holo_plan_derived.argtypes = [_P] + [_P] * 6
_lib.holo_plan_derived.restype = _S
_lib.holo_set_shifts.argtypes = [_P, _P]
_lib.holo_set_shifts.restype = _S
_lib.holo_set_ref_shifts.argtypes = [_P, ctypes.c_int32, _P]
_lib.holo_set_ref_shifts.restype = _S
_lib.holo_fwd.argtypes = [_P, _P, _P, _P]
_lib.holo_fwd.restype = _S
_lib.holo_adj.argtypes = [_P, _P, _P, _P, _P, _P]
_lib.holo_adj.restype = _S
_lib.holo_grad.argtypes = [_P, _P, _P, _P, _P, _P, _P, _P, ctypes.c_uint32]
_lib.holo_grad.restype = _S
_lib.holo_grad_ref.argtypes = [_P, _P, _P, _P, _P, ctypes.c_uint32]
_lib.holo_grad_ref.restype = _S
_lib.holo_fwd_ref.argtypes = [_P, _P, _P]
_lib.holo_fwd_ref.restype = _S
_lib.holo_q_dots.argtypes = [_P, _P, _P, _P]
_lib.holo_q_dots.restype = _S
_lib.holo_cg_step.argtypes = [_P, ctypes.POINTER(HoloCgIn), ctypes.POINTER(HoloCgOut)] + [_P] * 8
_lib.holo_cg_step.restype = _S

_lib.holo_upsample2.argtypes = [_P, _P, _P, ctypes.c_int32]
_lib.holo_upsample2.restype = _S
_lib.holo_bin2.argtypes = [_P, _P, _P, ctypes.c_int32]
_lib.holo_bin2.restype = _S

_lib.holo_init_probe.argtypes = [_P, _P, _P]
_lib.holo_init_probe.restype = _S
_lib.holo_init_psi.argtypes = [_P, _P, _P, ctypes.c_double, _P]
_lib.holo_init_psi.restype = _S

_lib.holo_set_probe_shifts.argtypes = [_P, _P]
_lib.holo_set_probe_shifts.restype = _S
_lib.holo_grad_full.argtypes = [_P, _P, _P, _P, _P, _P, _P, _P, _P, ctypes.c_uint32]
_lib.holo_grad_full.restype = _S

_lib.holo_set_gq_event.argtypes = [_P, _P]
_lib.holo_set_gq_event.restype = _S
_lib.holo_set_tau.argtypes = [_P, ctypes.c_double]
_lib.holo_set_tau.restype = _S
_lib.holo_stage_sqrt_d.argtypes = [_P, _P, _P]
_lib.holo_stage_sqrt_d.restype = _S
_lib.holo_stage_sqrt_dref.argtypes = [_P, _P, _P]
_lib.holo_stage_sqrt_dref.restype = _S
_lib.holo_set_cg_fuse.argtypes = [_P, ctypes.c_int32]
_lib.holo_set_cg_fuse.restype = _S
_lib.holo_set_fourier.argtypes = [_P, ctypes.c_int32]
_lib.holo_set_fourier.restype = _S
_lib.holo_fourier.argtypes = [_P, _P, _P, ctypes.c_int32, ctypes.c_int32]
_lib.holo_fourier.restype = _S

_lib.holo_profile_enable.argtypes = [_P, ctypes.c_int]
_lib.holo_profile_enable.restype = _S
_lib.holo_profile_read.argtypes = [_P, _P, _P, _P, _P, ctypes.c_int]
_lib.holo_profile_read.restype = _S

HOLO_NPASS = 10
PASS_NAMES = ["X1", "Y1", "X2", "Y2", "X3", "filter", "reduce", "cg", "ref", "ps"]
PASS_KERNELS = ["k_x1", "k_y1", "k_x2", "k_y2", "k_x3", "k_rows_filter|k_cols_filter|k_p2_convert",
                "k_reduce|k_dots", "k_cg", "k_ref", "k_xq|k_xg"]

EXPORTED = ["holo_plan_create", "holo_plan_destroy", "holo_plan_workspace_bytes", "holo_last_error",
            "holo_plan_derived", "holo_set_shifts", "holo_set_ref_shifts", "holo_fwd", "holo_adj", "holo_grad",
            "holo_grad_ref", "holo_fwd_ref", "holo_q_dots", "holo_cg_step", "holo_launch_count", "holo_profile_enable",
            "holo_profile_read", "holo_upsample2", "holo_bin2", "holo_init_probe", "holo_init_psi",
            "holo_set_probe_shifts", "holo_grad_full", "holo_set_gq_event", "holo_set_tau", "holo_set_fourier", "holo_fourier", "holo_stage_sqrt_d", "holo_stage_sqrt_dref", "holo_set_cg_fuse"]


class HoloError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"holo status {status}: {msg}")
        self.status = status


def _ptr(t, dtype=None, numel=None, name="array"):
    if t is None:
        return None
    if not isinstance(t, torch.Tensor):
        raise TypeError(f"{name}: expected a torch tensor")
    if not t.is_cuda:
        raise ValueError(f"{name}: must be a CUDA tensor (no CPU fallback)")
    if not t.is_contiguous():
        raise ValueError(f"{name}: must be contiguous")
    if dtype is not None and t.dtype != dtype:
        raise TypeError(f"{name}: expected {dtype}, got {t.dtype}")
    if numel is not None and t.numel() != numel:
        raise ValueError(f"{name}: expected {numel} elements, got {t.numel()}")
    return ctypes.c_void_p(t.data_ptr())


class Plan:
    """holo_plan_create: one (device, stream) plan for K angles x nz planes on an npad^2 torus."""

    def __init__(self, n, npad, z1, n_angles, wavelength, focus_to_detector, detector_pixel, device=0,
                 stream=None, angle_batch=None):
        self.fourier_state = False  # holo_set_fourier
        if angle_batch is None:  # default: 8 angles per Y1/X2/Y2 launch
            angle_batch = max(1, min(8, n_angles))
        g = HoloGeometry()
        g.n, g.npad, g.nz, g.n_angles, g.angle_batch = n, npad, len(z1), n_angles, angle_batch
        g.wavelength, g.focus_to_detector, g.detector_pixel = wavelength, focus_to_detector, detector_pixel
        for i, z in enumerate(z1):
            g.z1[i] = z
        self.device = torch.device("cuda", device) if isinstance(device, int) else torch.device(device)
        if stream is None:
            stream = torch.cuda.current_stream(self.device)
        self.stream = stream
        h = _P()
        st = _lib.holo_plan_create(ctypes.byref(h), ctypes.byref(g), self.device.index or 0,
                                   ctypes.c_void_p(stream.cuda_stream))
        if st != HOLO_OK:
            raise HoloError(st, "holo_plan_create failed")
        self._h = h
        self.n, self.npad, self.nz, self.K = n, npad, len(z1), n_angles
        self.angle_batch = angle_batch
        self.n_ref = 0
        self.geometry = g

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            _lib.holo_plan_destroy(h)
            self._h = None

    def _chk(self, st):
        if st != HOLO_OK:
            raise HoloError(st, _lib.holo_last_error(self._h).decode())

    @property
    def workspace_bytes(self):
        return _lib.holo_plan_workspace_bytes(self._h)

    @property
    def launch_count(self):
        return _lib.holo_launch_count(self._h)

    def profile_enable(self, on=True):
        self._chk(_lib.holo_profile_enable(self._h, int(bool(on))))

    def profile_read(self, reset=True):
        """Per-pass {name: dict(ms, launches, bytes, flops)} from CUDA events on the plan's stream."""
        ms = (ctypes.c_double * HOLO_NPASS)()
        n = (ctypes.c_uint64 * HOLO_NPASS)()
        b = (ctypes.c_double * HOLO_NPASS)()
        f = (ctypes.c_double * HOLO_NPASS)()
        self._chk(_lib.holo_profile_read(self._h, ctypes.cast(ms, _P), ctypes.cast(n, _P), ctypes.cast(b, _P),
                                         ctypes.cast(f, _P), int(bool(reset))))
        return {PASS_NAMES[i]: dict(ms=ms[i], launches=n[i], bytes=b[i], flops=f[i]) for i in range(HOLO_NPASS)}

    def derived(self):
        nz = self.nz
        m0, p0 = ctypes.c_double(), ctypes.c_double()
        arrs = [(ctypes.c_double * nz)() for _ in range(4)]
        self._chk(_lib.holo_plan_derived(self._h, ctypes.byref(m0), *[ctypes.cast(a, _P) for a in arrs],
                                         ctypes.byref(p0)))
        mt, zdet, omega, zeta = (np.array(a[:]) for a in arrs)
        return dict(m0=m0.value, mt=mt, zdet=zdet, omega=omega, zeta=zeta, p0=p0.value)

    def set_shifts(self, s):
        s = np.ascontiguousarray(s, dtype=np.float64).reshape(self.K, self.nz, 2)
        self._chk(_lib.holo_set_shifts(self._h, s.ctypes.data_as(_P)))

    def set_gq_event(self, event):
        """holo_set_gq_event: a torch.cuda.Event recorded when grad_q_part is complete (None clears).
        The event is recorded once here so that its CUDA handle exists; keep a reference to it."""
        if event is None:
            self._chk(_lib.holo_set_gq_event(self._h, None))
            self._gq_event = None
            return
        event.record(self.stream)
        self._gq_event = event
        self._chk(_lib.holo_set_gq_event(self._h, ctypes.c_void_p(event.cuda_event)))

    def set_tau(self, tau):
        """holo_set_tau: penalty exponent of G_tau (App. A.3) for later grad calls (1 = F_1, 2 = F_2)."""
        self._chk(_lib.holo_set_tau(self._h, float(tau)))

    def stage_sqrt_d(self, host, dev):
        """holo_stage_sqrt_d: the next grad call reading `dev` streams `host` (pinned CPU float32 tensor of
        the same shape) into it per angle batch, overlapped with the sweep.  Keep `host` alive until then."""
        if host is None:
            self._chk(_lib.holo_stage_sqrt_d(self._h, None, None))
            return
        if host.is_cuda or not host.is_pinned() or not host.is_contiguous() or host.dtype != torch.float32:
            raise ValueError("host: must be a contiguous pinned CPU float32 tensor")
        if host.numel() != dev.numel() or host.numel() != self.K * self.nz * self.n ** 2:
            raise ValueError("host / dev: expected K x nz x n x n elements")
        self._stage_host = host
        self._chk(_lib.holo_stage_sqrt_d(self._h, ctypes.c_void_p(host.data_ptr()),
                                         _ptr(dev, torch.float32, host.numel(), "dev")))

    def stage_sqrt_dref(self, host, dev):
        """holo_stage_sqrt_dref: as stage_sqrt_d for the reference frames [n_ref][n][n]."""
        if host is None:
            self._chk(_lib.holo_stage_sqrt_dref(self._h, None, None))
            return
        if host.is_cuda or not host.is_pinned() or not host.is_contiguous() or host.dtype != torch.float32:
            raise ValueError("host: must be a contiguous pinned CPU float32 tensor")
        if host.numel() != dev.numel() or host.numel() != self.n_ref * self.n ** 2:
            raise ValueError("host / dev: expected n_ref x n x n elements")
        self._stage_host = host
        self._chk(_lib.holo_stage_sqrt_dref(self._h, ctypes.c_void_p(host.data_ptr()),
                                            _ptr(dev, torch.float32, host.numel(), "dev")))

    def set_cg_fuse(self, on):
        """holo_set_cg_fuse: defer holo_cg_step's psi-block update into the next sweep's X1."""
        self._chk(_lib.holo_set_cg_fuse(self._h, int(bool(on))))

    def set_fourier(self, on):
        """holo_set_fourier: object-side arrays of later fwd / adj / grad calls are DFT2(psi) (unnormalised)."""
        self._chk(_lib.holo_set_fourier(self._h, int(bool(on))))
        self.fourier_state = bool(on)

    def fourier(self, x, out=None, inverse=False):
        """holo_fourier: out[m] = DFT2(x[m]) (numpy.fft.fft2) or, inverse, IDFT2 (numpy.fft.ifft2); x [M][npad][npad]."""
        LL = self.npad ** 2
        M = x.numel() // LL
        out = x if out is None else out
        self._chk(_lib.holo_fourier(self._h, _ptr(x, torch.complex64, M * LL, "x"), _ptr(out, torch.complex64, M * LL, "out"),
                                    M, int(bool(inverse))))
        return out

    def set_probe_shifts(self, s):
        """holo_set_probe_shifts: per-frame probe shifts s^p [K][nz][2] (None: plain q_j path)."""
        if s is None:
            self._chk(_lib.holo_set_probe_shifts(self._h, None))
            return
        s = np.ascontiguousarray(s, dtype=np.float64).reshape(self.K, self.nz, 2)
        self._chk(_lib.holo_set_probe_shifts(self._h, s.ctypes.data_as(_P)))

    def set_ref_shifts(self, s):
        s = np.ascontiguousarray(s, dtype=np.float64).reshape(-1, 2)
        self._chk(_lib.holo_set_ref_shifts(self._h, s.shape[0], s.ctypes.data_as(_P)))
        self.n_ref = s.shape[0]

    # ---- hot path
    def fwd(self, psi, q, w):
        LL, NN = self.npad ** 2, self.n ** 2
        self._chk(_lib.holo_fwd(self._h, _ptr(psi, torch.complex64, self.K * LL, "psi"),
                                _ptr(q, torch.complex64, LL, "q"),
                                _ptr(w, torch.complex64, self.K * self.nz * NN, "w")))
        return w

    def adj(self, y, psi, q, adj_psi=None, adj_q=None):
        LL, NN = self.npad ** 2, self.n ** 2
        self._chk(_lib.holo_adj(self._h, _ptr(y, torch.complex64, self.K * self.nz * NN, "y"),
                                _ptr(psi, torch.complex64, self.K * LL, "psi"), _ptr(q, torch.complex64, LL, "q"),
                                _ptr(adj_psi, torch.complex64, self.K * LL, "adj_psi"),
                                _ptr(adj_q, torch.complex64, LL, "adj_q")))

    def grad(self, psi, q, sqrt_d, sc, eta_psi_prev=None, grad_psi=None, grad_q_part=None, flags=0):
        LL, NN = self.npad ** 2, self.n ** 2
        self._chk(_lib.holo_grad(self._h, _ptr(psi, torch.complex64, self.K * LL, "psi"),
                                 _ptr(q, torch.complex64, LL, "q"),
                                 _ptr(sqrt_d, torch.float32, self.K * self.nz * NN, "sqrt_d"),
                                 _ptr(eta_psi_prev, torch.complex64, self.K * LL, "eta_psi_prev"),
                                 _ptr(grad_psi, torch.complex64, self.K * LL, "grad_psi"),
                                 _ptr(grad_q_part, torch.complex64, LL, "grad_q_part"),
                                 _ptr(sc, torch.float64, 3, "sc"), flags))

    def grad_full(self, psi, q, sqrt_d, sqrt_dref, sc, eta_psi_prev=None, grad_psi=None, grad_q_part=None, flags=0):
        """holo_grad_full: the object chain and the n_ref reference frames in one sweep (Eq. (10)/(12))."""
        LL, NN = self.npad ** 2, self.n ** 2
        self._chk(_lib.holo_grad_full(self._h, _ptr(psi, torch.complex64, self.K * LL, "psi"),
                                      _ptr(q, torch.complex64, LL, "q"),
                                      _ptr(sqrt_d, torch.float32, self.K * self.nz * NN, "sqrt_d"),
                                      _ptr(sqrt_dref, torch.float32, self.n_ref * NN, "sqrt_dref"),
                                      _ptr(eta_psi_prev, torch.complex64, self.K * LL, "eta_psi_prev"),
                                      _ptr(grad_psi, torch.complex64, self.K * LL, "grad_psi"),
                                      _ptr(grad_q_part, torch.complex64, LL, "grad_q_part"),
                                      _ptr(sc, torch.float64, 3, "sc"), flags))

    def grad_ref(self, q, sqrt_dref, sc, grad_q_part=None, flags=0):
        self._chk(_lib.holo_grad_ref(self._h, _ptr(q, torch.complex64, self.npad ** 2, "q"),
                                     _ptr(sqrt_dref, torch.float32, self.n_ref * self.n ** 2, "sqrt_dref"),
                                     _ptr(grad_q_part, torch.complex64, self.npad ** 2, "grad_q_part"),
                                     _ptr(sc, torch.float64, 1, "sc"), flags))

    def fwd_ref(self, q, w):
        """holo_fwd_ref: w[r] = C(P_{zeta0} S_{s_r} q) for the n_ref reference frames."""
        self._chk(_lib.holo_fwd_ref(self._h, _ptr(q, torch.complex64, self.npad ** 2, "q"),
                                    _ptr(w, torch.complex64, self.n_ref * self.n ** 2, "w")))
        return w

    def q_dots(self, grad_q, eta_q_prev, out):
        LL = self.npad ** 2
        self._chk(_lib.holo_q_dots(self._h, _ptr(grad_q, torch.complex64, LL, "grad_q"),
                                   _ptr(eta_q_prev, torch.complex64, LL, "eta_q_prev"),
                                   _ptr(out, torch.float64, 2, "out")))

    def cg_step(self, cin: HoloCgIn, psi=None, eta_psi=None, grad_psi=None, psi_trial=None,
                q=None, eta_q=None, grad_q=None, q_trial=None) -> HoloCgOut:
        out = HoloCgOut()
        LL = self.npad ** 2
        self._chk(_lib.holo_cg_step(self._h, ctypes.byref(cin), ctypes.byref(out),
                                    _ptr(psi, torch.complex64, self.K * LL, "psi"),
                                    _ptr(eta_psi, torch.complex64, self.K * LL, "eta_psi"),
                                    _ptr(grad_psi, torch.complex64, self.K * LL, "grad_psi"),
                                    _ptr(psi_trial, torch.complex64, self.K * LL, "psi_trial"),
                                    _ptr(q, torch.complex64, LL, "q"), _ptr(eta_q, torch.complex64, LL, "eta_q"),
                                    _ptr(grad_q, torch.complex64, LL, "grad_q"),
                                    _ptr(q_trial, torch.complex64, LL, "q_trial")))
        return out

    # ---- multiresolution schedule
    def upsample2(self, coarse, fine):
        """holo_upsample2: coarse [M][npad/2][npad/2] -> fine [M][npad][npad] (this plan = fine level)."""
        Lc = self.npad // 2
        M = coarse.numel() // (Lc * Lc)
        self._chk(_lib.holo_upsample2(self._h, _ptr(coarse, torch.complex64, M * Lc * Lc, "coarse"),
                                      _ptr(fine, torch.complex64, M * self.npad ** 2, "fine"), M))
        return fine

    def bin2(self, fine, coarse):
        """holo_bin2: amplitudes fine [M][2n][2n] -> coarse [M][n][n] (this plan = coarse level)."""
        M = coarse.numel() // (self.n * self.n)
        self._chk(_lib.holo_bin2(self._h, _ptr(fine, torch.float32, M * 4 * self.n ** 2, "fine"),
                                 _ptr(coarse, torch.float32, M * self.n ** 2, "coarse"), M))
        return coarse

    # ---- initialisers
    def init_probe(self, sqrt_dref, q0):
        """holo_init_probe (O17): q0 from the n_ref reference frames sqrt_dref [R][n][n]."""
        self._chk(_lib.holo_init_probe(self._h, _ptr(sqrt_dref, torch.float32, self.n_ref * self.n ** 2, "sqrt_dref"),
                                       _ptr(q0, torch.complex64, self.npad ** 2, "q0")))
        return q0

    def init_psi(self, sqrt_d, sqrt_dref, delta_beta, psi0):
        """holo_init_psi (O18): multi-distance Paganin psi0 [K][npad][npad] from sqrt_d [K][nz][n][n] and the
        flat field sqrt_dref [n][n]."""
        self._chk(_lib.holo_init_psi(self._h, _ptr(sqrt_d, torch.float32, self.K * self.nz * self.n ** 2, "sqrt_d"),
                                     _ptr(sqrt_dref, torch.float32, self.n ** 2, "sqrt_dref"), float(delta_beta),
                                     _ptr(psi0, torch.complex64, self.K * self.npad ** 2, "psi0")))
        return psi0
