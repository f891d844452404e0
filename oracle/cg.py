"""O13 -- Dai-Yuan conjugate gradient with monotone backtracking, plain numpy fp64.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Follows Eqs. (13)-(14) in the product space x = (psi_0..psi_{K-1}, q)
with one shared step gamma (reading C9), the block preconditioner
P = diag(rho_psi I, rho_q I), real inner products Re<.,.> (reading C11) and the
halving line search of reading C10 (F must not increase).

    (i)   m = 0: eta = -P g.  Otherwise den = Re<g_m, eta_{m-1}> - Re<g_{m-1}, eta_{m-1}>;
          if |den| < 1e-30 <g_m, P g_m>: eta = -P g_m
          else beta = <g_m, P g_m> / den, eta = -P g_m + beta eta_{m-1}           (Eq. (14))
    (ii)  if Re<g_m, eta_m> >= 0: eta = -P g_m
    (iii) gamma0 = 1 if m = 0 or the last step stagnated, else gamma_{m-1};
          try gamma = gamma0 2^{-t}, t = 0..12; accept the first with F(x + gamma eta) < F(x_m)
    (iv)  none accepted: gamma = 0, x unchanged, next step restarts with eta = -P g
    (v)   x_{m+1} = x_m + gamma eta                                              (Eq. (13))
"""
from __future__ import annotations

import numpy as np


def rdot(a, b):
    """Re<a, b> = Re sum a conj(b) over all blocks (P:429 convention)."""
    return float(sum(np.vdot(bb, aa).real for aa, bb in zip(a, b)))


def dai_yuan_direction(g, g_prev, eta_prev, rho):
    """Steps (i)-(ii). g, g_prev, eta_prev: lists of blocks (g_prev/eta_prev None at m = 0).

    Returns (eta, beta, reset)."""
    Pg = [r * gg for r, gg in zip(rho, g)]
    gPg = rdot(g, Pg)
    if eta_prev is None:
        return [-x for x in Pg], 0.0, True
    den = rdot(g, eta_prev) - rdot(g_prev, eta_prev)
    if abs(den) < 1e-30 * gPg:
        eta, beta, reset = [-x for x in Pg], 0.0, True
    else:
        beta = gPg / den
        eta = [-p + beta * e for p, e in zip(Pg, eta_prev)]
        reset = False
    if rdot(g, eta) >= 0:
        eta, beta, reset = [-x for x in Pg], 0.0, True
    return eta, beta, reset


def run(sweep, x0, rho, n_iter, max_halvings=12, gamma_init=1.0, forced_gammas=None):
    """Run n_iter CG iterations.  sweep(x) -> (F, g) with x, g lists of blocks.

    forced_gammas: optional list; iteration m then uses exactly gamma = forced_gammas[m]
    (no line search) -- used by parity tests where fp32/fp64 accept decisions may differ.
    Returns (x, history) with history = list of dicts(F, gamma, beta, sweeps)."""
    x = [np.array(b, dtype=np.complex128, copy=True) for b in x0]
    F, g = sweep(x)
    g_prev = eta_prev = None
    gamma_last, stagnated = None, True
    hist = []
    for m in range(n_iter):
        eta, beta, reset = dai_yuan_direction(g, g_prev, eta_prev, rho)
        gamma0 = gamma_init if (m == 0 or stagnated) else gamma_last
        sweeps = 0
        accepted = False
        if forced_gammas is not None:
            cands = [forced_gammas[m]]
        else:
            cands = [gamma0 * 2.0 ** (-t) for t in range(max_halvings + 1)]
        for gamma in cands:
            xt = [a + gamma * e for a, e in zip(x, eta)]
            Ft, gt = sweep(xt)
            sweeps += 1
            if forced_gammas is not None or Ft < F:
                accepted = True
                break
        if accepted:
            x, F, g_prev, g, eta_prev = xt, Ft, g, gt, eta
            gamma_last, stagnated = gamma, False
        else:
            gamma, stagnated = 0.0, True
            g_prev = eta_prev = None  # (iv): restart with eta = -P g
        hist.append(dict(F=F, gamma=gamma, beta=beta, reset=reset, sweeps=sweeps))
    return x, hist
