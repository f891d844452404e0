"""Joint psi/q Dai-Yuan CG driver (Eqs. (13)-(14)) over libholo.

Host-side control only: every array operation runs in libholo's kernels
(holo_grad, holo_q_dots, holo_cg_step); torch provides the buffers and, across
ranks, torch.distributed (NCCL) for the two exchange steps of a sweep:
allreduce(sum) of the local probe-gradient partial and of the 3 fp64 psi-block
scalars.  The q-block dots are then computed redundantly on every rank.

Product-space CG with one shared step (reading C9), block preconditioner
P = diag(rho_psi, rho_q), Re<.,.> everywhere (C11), halving line search with a
monotone-F acceptance test (C10).  One host synchronisation per sweep: the
D2H copy of 5 doubles (F, |g_psi|^2, Re<g_psi, eta_psi>, |g_q|^2, Re<g_q, eta_q>).
"""
from __future__ import annotations

import math

import torch
import torch.distributed as dist

from . import HOLO_ACCUMULATE_Q, HoloCgIn


class JointCG:
    """Product-space Dai-Yuan CG over (psi_local..., q).  ``sqrt_dref`` (optional) adds the
    reference arm (O14, holo_grad_ref) of this rank's reference frames to F and grad_q;
    a plan with n_angles = 0 then runs the probe-only problem of configs[4] (rho_psi unused)."""

    def __init__(self, plan, sqrt_d, psi0, q0, rho_psi=1.0, rho_q=1.0, gamma_init=1.0, max_halvings=12,
                 group=None, distributed=None, sqrt_dref=None, fused=None, overlap=True, fourier=None,
                 fuse_cg=None):
        self.plan = plan
        self.d = sqrt_d
        self.dref = sqrt_dref
        # holo_grad_full when the plan provides it (the CPU test double of the dist tests does not)
        self.fused = hasattr(plan, "grad_full") if fused is None else bool(fused)
        self.rho = (float(rho_psi), float(rho_q))
        # rho_q = 0 freezes the probe (object-only CG, e.g. the second stage of the probe-subset
        # schedule): no probe-gradient work in the library (grad_q_part = NULL skips the
        # Aw stores and the G_j accumulation), no g_q exchange, q never moves.
        self.q_frozen = self.rho[1] == 0.0
        self.gamma_init, self.max_halvings = float(gamma_init), int(max_halvings)
        self.group = group
        self.dist = dist.is_available() and dist.is_initialized() if distributed is None else distributed
        dev = psi0.device
        z = lambda t: torch.zeros_like(t)
        # Fourier-domain object state (holo_set_fourier, Parseval): the psi block (psi, eta, g, trial) is
        # held as DFT2 of the object arrays, which saves the chain's four "into / out of the Fourier
        # domain" transforms per sweep; the CG step is linear and the library returns object-domain dots,
        # so the iteration is the same.  `psi` converts back on access.
        if fourier is None:
            fourier = hasattr(plan, "set_fourier") and psi0.numel() > 0 and psi0.is_cuda
        self.fourier = bool(fourier)
        if hasattr(plan, "set_fourier") and psi0.numel() > 0:
            plan.set_fourier(self.fourier)
        self._psi, self.q = psi0.contiguous().clone(), q0.contiguous().clone()
        if self.fourier:
            plan.fourier(self._psi)
        # holo_set_cg_fuse: the psi-block half of every CG step runs inside the following sweep's X1
        # (correct and bit-identical, but measured slower at cfg3: X1 +40 us/frame > the 28 us/frame
        # pointwise pass it replaces), so off unless asked for
        self.fuse_cg = bool(fuse_cg)
        if hasattr(plan, "set_cg_fuse") and psi0.numel() > 0:
            plan.set_cg_fuse(self.fuse_cg)
        self.psi_t, self.q_t = z(self._psi), z(self.q)
        self.eta_psi, self.eta_q = z(self._psi), z(self.q)
        self.g_psi, self.g_q = z(self._psi), z(self.q)
        self.gt_psi, self.gt_q = z(self._psi), z(self.q)
        self.sc = torch.zeros(5, dtype=torch.float64, device=dev)
        # g_q / X3 overlap: only with CUDA tensors, an NCCL group and a plan exposing the hook
        self.comm = self.gq_ev = None
        if self.dist and dev.type == "cuda" and hasattr(plan, "set_gq_event") and overlap:
            self.comm = torch.cuda.Stream(dev)
            self.gq_ev = torch.cuda.Event()
            plan.set_gq_event(self.gq_ev)
        self.scr = torch.zeros(1, dtype=torch.float64, device=dev)  # F of the reference arm
        self.F = None
        self.dots = None
        self.g_eta = 0.0          # Re<g_m, eta_{m-1}>
        self.gprev_eta = 0.0      # Re<g_{m-1}, eta_{m-1}>
        self.gamma_last = None
        self.stagnated = True
        self.m = 0
        self.sweeps = 0

    @property
    def psi(self):
        """The object block in the object domain (in Fourier mode a NEW converted copy, K x npad^2
        complex64 -- use psi_into(out) to reuse a buffer)."""
        if not self.fourier:
            return self._psi
        return self.plan.fourier(self._psi, torch.empty_like(self._psi), inverse=True)

    def psi_into(self, out):
        """Write the object-domain psi block into `out` (same shape / dtype as psi0); returns out."""
        if not self.fourier:
            return out.copy_(self._psi)
        return self.plan.fourier(self._psi, out, inverse=True)

    # ------------------------------------------------------------------ sweep
    def sweep(self, psi, q, eta_psi, eta_q, g_psi, g_q):
        """F and grad at (psi, q); returns host (F, gg_psi, geta_psi, gg_q, geta_q)."""
        p = self.plan
        sc3 = self.sc[:3]
        if self.q_frozen:
            g_q = None
        # always called, also on a rank without angles: the library then writes F = 0 and a ZERO
        # probe-gradient partial, so no stale (already reduced) g_q enters the allreduce.
        if self.dref is None:
            p.grad(psi, q, self.d, sc3, eta_psi, g_psi, g_q)
        elif self.fused:  # the whole Eq. (10): object frames + reference frames in one sweep
            p.grad_full(psi, q, self.d, self.dref, sc3, eta_psi, g_psi, g_q)
        else:  # reference arm as a second call: F_ref into sc[0], its gradient added to g_q
            p.grad(psi, q, self.d, sc3, eta_psi, g_psi, g_q)
            p.grad_ref(q, self.dref, self.scr, g_q, flags=HOLO_ACCUMULATE_Q)
            sc3[:1] += self.scr
        if self.dist and g_q is None:
            dist.all_reduce(sc3, group=self.group)
        elif self.dist:
            # exchange 1: probe-gradient partial (complex64 viewed as float32), exchange 2: scalars.
            # With an overlap event (CUDA/NCCL), exchange 1 runs on a side stream that waits only for
            # the event the library records as soon as g_q is complete, i.e. while the last angle
            # batch's object-gradient passes still run on the plan's stream.
            if self.comm is not None:
                self.comm.wait_event(self.gq_ev)
                with torch.cuda.stream(self.comm):
                    dist.all_reduce(torch.view_as_real(g_q), group=self.group)
                dist.all_reduce(sc3, group=self.group)
                torch.cuda.current_stream(g_q.device).wait_stream(self.comm)
            else:
                dist.all_reduce(torch.view_as_real(g_q), group=self.group)
                dist.all_reduce(sc3, group=self.group)
        if g_q is None:
            self.sc[3:].zero_()
        else:
            p.q_dots(g_q, eta_q, self.sc[3:])
        s = self.sc.cpu().tolist()  # the single host sync of the sweep
        self.sweeps += 1
        if not math.isfinite(s[0]):
            raise FloatingPointError(f"non-finite objective F = {s[0]} at iteration {self.m}")
        return s

    def start(self):
        s = self.sweep(self._psi, self.q, None, None, self.g_psi, self.g_q)
        self.F = s[0]
        self.dots = s
        return self.F

    def gPg(self):
        return self.rho[0] * self.dots[1] + self.rho[1] * self.dots[3]

    # ------------------------------------------------------------------ one CG iteration
    def iterate(self, forced_gamma=None):
        if self.F is None:
            self.start()
        p = self.plan
        first = self.m == 0 or self.stagnated
        gamma = self.gamma_init if first else self.gamma_last
        if forced_gamma is not None:
            gamma = float(forced_gamma)
        cin = HoloCgIn(self.gPg(), self.g_eta, self.gprev_eta, gamma, self.rho[0], self.rho[1], int(first), 0)
        qb = (None,) * 4 if self.q_frozen else (self.q, self.eta_q, self.g_q, self.q_t)
        out = p.cg_step(cin, self._psi, self.eta_psi, self.g_psi, self.psi_t, *qb)
        g_eta_new = out.g_eta_new
        accepted = False
        tries = 0
        while True:
            s = self.sweep(self.psi_t, self.q if self.q_frozen else self.q_t, self.eta_psi, self.eta_q, self.gt_psi, self.gt_q)
            tries += 1
            if forced_gamma is not None or s[0] < self.F:
                accepted = True
                break
            if tries > self.max_halvings:
                break
            gamma *= 0.5
            cin = HoloCgIn(0.0, 0.0, 0.0, gamma, self.rho[0], self.rho[1], 0, 1)
            qb = (None,) * 4 if self.q_frozen else (self.q, self.eta_q, None, self.q_t)
            p.cg_step(cin, self._psi, self.eta_psi, None, self.psi_t, *qb)
        if accepted:
            self._psi, self.psi_t = self.psi_t, self._psi
            if not self.q_frozen:
                self.q, self.q_t = self.q_t, self.q
            self.g_psi, self.gt_psi = self.gt_psi, self.g_psi
            self.g_q, self.gt_q = self.gt_q, self.g_q
            self.F, self.dots = s[0], s
            self.gprev_eta = g_eta_new
            self.g_eta = s[2] + s[4]
            self.gamma_last, self.stagnated = gamma, False
        else:
            gamma, self.stagnated = 0.0, True
        self.m += 1
        return dict(F=self.F, gamma=gamma, beta=out.beta, reset=bool(out.reset), sweeps=tries)
