/*
 * holo.h -- C ABI of the B200 (sm_100a) hot path of arXiv 2407.20304,
 * "X-ray nano-holotomography reconstruction with simultaneous probe retrieval".
 *
 * One iteration of the batched per-projection holography operator of Eq. (8)
 * with the amplitude functional F1 of Eq. (10), its Wirtinger
 * gradients Eqs. (11)-(12) and the pointwise half of the Dai-Yuan
 * conjugate-gradient step Eqs. (13)-(14).  P:n = PAPER.md line n.
 *
 * Conventions (readings C1-C21):
 *  - complex = float2 {re, im} (complex64); every array is row-major [y][x]
 *    (x is the fast index); per-frame arrays are ordered [k][j][y][x], k = angle,
 *    j = sample plane ("distance"), one (k, j) pair = one "frame".
 *  - The object psi_k and probe q live on the npad x npad torus (2x padding, C3);
 *    detector-plane fields and data live on the central n x n window,
 *    offset o = (npad - n)/2 (crop C / zero-pad Z, O7).
 *  - Pointers are DEVICE pointers unless marked [host].  The caller owns every
 *    array buffer; the plan owns its tables and workspace.  No entry point
 *    allocates per call.  Outputs must not alias inputs unless stated.
 *  - Every call enqueues on the plan's stream and returns without synchronising;
 *    scalar outputs stay on the device.
 *  - Errors: all arguments are validated on the host before any launch and a
 *    failure returns HOLO_EINVAL (bad pointer/size/geometry) or
 *    HOLO_EUNSUPPORTED (valid but not implemented size).  A CUDA failure returns
 *    HOLO_ECUDA and puts the plan in a sticky error state: later calls return
 *    HOLO_ESTATE until holo_plan_destroy.  holo_last_error() gives the text.
 *    No C++ exception crosses the ABI.
 *  - A plan is single-threaded and bound to one (device, stream).
 */
#ifndef HOLO_H
#define HOLO_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct holo_plan holo_plan; /* opaque */

typedef enum {
  HOLO_OK = 0,
  HOLO_EINVAL = -1,
  HOLO_ENOMEM = -2,
  HOLO_ECUDA = -3,
  HOLO_EUNSUPPORTED = -4,
  HOLO_ESTATE = -5
} holo_status;

#define HOLO_MAX_NZ 8
#define HOLO_MAX_BATCH 16

/* Acquisition geometry (Table 1; Eq. (6); Eq. (8)). */
typedef struct {
  int32_t n;           /* detector / data side N: even, >= 8, n <= npad, (npad - n) even   */
  int32_t npad;        /* torus side N_p: power of two, 128 <= npad <= 4096
                          (6144 = 3*2^11 for reference-arm-only plans, n_angles == 0)          */
  int32_t nz;          /* number of sample planes ("distances"), 1..HOLO_MAX_NZ               */
  int32_t n_angles;    /* K: angles resident on this device (0: reference-arm-only plan)      */
  int32_t angle_batch; /* B, 1..HOLO_MAX_BATCH: angles whose frames of one plane share a Y1 /
                          X2 / Y2 launch (q_j read once and the probe-gradient accumulator G_j
                          read-modify-written once per batch, Eq. (12)).  Sizes the
                          workspace: ~ (2 nz + 2) B npad^2 complex64.  Results do not depend on B
                          beyond fp32 rounding of the G_j sum order.                          */
  double wavelength;   /* lambda [m] > 0                                                       */
  double focus_to_detector; /* Z [m]                                                          */
  double z1[HOLO_MAX_NZ];   /* focus-to-sample [m], 0 < z1[0] < ... < z1[nz-1] < Z            */
  double detector_pixel;    /* [m] > 0; object-plane pixel p0 = detector_pixel * z1[0] / Z   */
} holo_geometry;

/* Create a plan on `device` that enqueues on `stream` (a cudaStream_t; NULL = legacy
 * default stream).  Derives (O1): m0 = Z/z1_0, mt_j = z1_j/z1_0, zeta_j = z1_j(Z-z1_j)/Z,
 * omega_j = (z1_j - z1_0)/mt_j, zdet_j = zeta_j/mt_j^2, p0 = det_px/m0 (Eq. (8)),
 * builds the fp64-derived fp32 tables (Fresnel transfers, chirp-z chirps and kernel
 * spectra, FFT twiddles) and allocates the workspace.  Errors: HOLO_EINVAL for a bad
 * geometry, HOLO_EUNSUPPORTED for an npad outside the supported set, HOLO_ENOMEM. */
holo_status holo_plan_create(holo_plan **out, const holo_geometry *g /*[host]*/, int device, void *stream);
void holo_plan_destroy(holo_plan *p); /* NULL allowed */
size_t holo_plan_workspace_bytes(const holo_plan *p);
const char *holo_last_error(const holo_plan *p); /* message of the last non-OK status */

/* Derived geometry (O1), all [host] arrays of length nz; any pointer may be NULL. */
holo_status holo_plan_derived(const holo_plan *p, double *m0, double *mt, double *zdet, double *omega,
                              double *zeta, double *p0);

/* Sample shifts s^s_kj (Eq. (10), "S_{s^s_kj}"; reading C4): [host] float64
 * [n_angles][nz][2] = (sx, sy) in object-plane (psi-grid) pixels, applied before the
 * magnification, periodic on the torus; |s| < npad/2 and finite, else HOLO_EINVAL.
 * Copied into the plan (the host buffer may be reused on return).  Default: all zero. */
holo_status holo_set_shifts(holo_plan *p, const double *s /*[host]*/);

/* Per-frame PROBE shifts s^p_kj (Eq. (9)/(10) P:108, "S_{s^p_{k,j}}"; O19):
 * [host] float64 [n_angles][nz][2] = (sx, sy) in psi-grid pixels, |s| < npad/2.  After this call
 * every sweep of the object chain (holo_fwd / holo_adj / holo_grad / holo_grad_full) uses
 *   q_kj = P_{omega_j} S_{s^p_kj} q  instead of  q_j = P_{omega_j} q,
 * and the probe gradient 2 sum_kj S_{-s^p_kj} P_{-omega_j}(conj(M S psi_k) v_kj) is accumulated in the
 * Fourier domain (two extra row passes per angle, one extra transform per frame in Y1 and Y2).
 * The first call allocates the path's workspace (~ (2 nz + 1) angle_batch + 2 complex64 npad^2 arrays);
 * a NULL s switches the path off again (plain q_j).  Power-of-two npad, n_angles > 0. */
holo_status holo_set_probe_shifts(holo_plan *p, const double *s /*[host] | NULL*/);

/* Overlap hook: `event` (a cudaEvent_t created by the caller, or NULL to clear) is
 * recorded on the plan's stream by holo_grad / holo_grad_full / holo_adj as soon as grad_q_part
 * (adj_q) is complete -- before the last angle batch's object-gradient (X3) passes -- so the
 * caller can allreduce the probe-gradient partial on another stream while those passes run.
 * The plan does not own the event. */
holo_status holo_set_gq_event(holo_plan *p, void *event);

/* Reference-frame shifts s^r_r (Eq. (10) reference term P:115; reading C16):
 * [host] float64 [n_ref][2] = (sx, sy).  Sets R = n_ref for holo_grad_ref. */
holo_status holo_set_ref_shifts(holo_plan *p, int32_t n_ref, const double *s /*[host]*/);

/* Forward (O7, Eq. (8) without the detector-frame rescale, reading C8):
 *   w[k][j] = C( P_{zdet_j}( q_j . M_{1/mt_j} S_{s_kj} psi_k ) ),  q_j = P_{omega_j} q.
 * psi [K][npad][npad], q [npad][npad] -> w [K][nz][n][n].                                */
holo_status holo_fwd(holo_plan *p, const void *psi, const void *q, void *w);

/* Adjoints of the two linearisations at (psi, q) for a detector-plane field y:
 *   adj_psi[k] = sum_j L_kj^* y_kj,   L_kj^* = S_{-s} M^*_{1/mt} (conj(q_j) . P_{-zdet_j} Z .)
 *   adj_q      = sum_{k,j} Q_kj^* y_kj = sum_j P_{-omega_j} sum_k conj(M S psi_k) . P_{-zdet_j} Z y_kj
 * (local partial over this plan's angles; no factor 2).  Either output may be NULL.     */
holo_status holo_adj(holo_plan *p, const void *y /*[K][nz][n][n]*/, const void *psi, const void *q,
                     void *adj_psi /*[K][npad][npad] | NULL*/, void *adj_q /*[npad][npad] | NULL*/);

#define HOLO_ACCUMULATE_Q 1u  /* add into grad_q_part instead of overwriting          */
#define HOLO_OBJECTIVE_ONLY 2u /* F only: no adjoint work, grad outputs ignored       */
#define HOLO_INTENSITY 4u      /* holo_grad: intensity objective F_2 (tau = 2, Eq. (9)):
                                  F = sum (|w|^2 - sqrt_d^2)^2, rho = 2 (|w|^2 - sqrt_d^2) w (App. A.3)  */

/* Penalty exponent tau of the objective (App. A.3, Eq. (mintau)):
 *   G_tau = sum_{k,j} || |w_kj|^tau - sqrt_d_kj^tau ||^2  (+ the same for the reference frames),
 *   rho   = h'(|w|^2) w = tau (|w|^tau - sqrt_d^tau) |w|^(tau - 2) w   (0 where w = 0, reading C7),
 * used by every later holo_grad / holo_grad_full / holo_grad_ref call on this plan (the gradient keeps
 * Eq. (11)'s factor 2: grad = 2 L^* rho).  tau = 1 (default) is F_1 (Eq. (10)), tau = 2 is F_2
 * (Eq. (9)).  HOLO_INTENSITY still selects tau = 2 for one call.  HOLO_EINVAL outside [0.25, 4]. */
holo_status holo_set_tau(holo_plan *p, double tau);

/* Fused sweep at (psi, q) over this plan's angles (O8-O12; Eqs. (10)-(12)).
 * Writes fp64 DEVICE scalars sc[3]:
 *   sc[0] = F_local = sum_{k,j} sum_pix (|w_kj| - sqrt_d_kj)^2                 (Eq. (10))
 *   sc[1] = ||grad_psi||^2 over local angles
 *   sc[2] = Re<grad_psi, eta_psi_prev> over local angles (0 if eta_psi_prev NULL) (Eq. (14))
 * grad_psi[k] = 2 sum_j L_kj^*(rho_kj), rho = w - sqrt_d w/|w| (0 where w = 0, C7) (Eq. (11))
 * grad_q_part = 2 sum_j P_{-omega_j} sum_k conj(M S psi_k) P_{-zdet_j} Z rho_kj     (Eq. (12))
 *   (local partial: the caller allreduces it over ranks).
 * grad_psi / grad_q_part may be NULL (not computed).  sqrt_d: float32 [K][nz][n][n] >= 0. */
holo_status holo_grad(holo_plan *p, const void *psi, const void *q, const float *sqrt_d,
                      const void *eta_psi_prev, void *grad_psi, void *grad_q_part, double *sc, uint32_t flags);

/* The complete Eq. (10) objective in ONE sweep (O19; Eq. (12)): the object
 * chain of holo_grad (with the probe shifts of holo_set_probe_shifts, if set) PLUS the n_ref
 * reference frames sqrt_dref [R][n][n] (holo_set_ref_shifts), sharing DFT2(q) and the
 * Fourier-domain probe-gradient accumulator:
 *   sc[0] = F_local + F_ref,  sc[1], sc[2] as holo_grad,
 *   grad_q_part = 2 sum_kj Q_kj^*(rho_kj) + 2 sum_r Q_r^*(rho^r)   (local partial).
 * sqrt_dref may be NULL (then identical to holo_grad).  Flags as holo_grad. */
holo_status holo_grad_full(holo_plan *p, const void *psi, const void *q, const float *sqrt_d,
                           const float *sqrt_dref, const void *eta_psi_prev, void *grad_psi, void *grad_q_part,
                           double *sc, uint32_t flags);

/* Reference arm (O14; reference constraint P:102, Eq. (10)/(12) reference terms):
 *   sc[0] = F_ref = sum_r sum_pix (|C P_{zeta0} S_{s_r} q| - sqrt_dref_r)^2
 *   grad_q_part (+)= 2 sum_r S_{-s_r} P_{-zeta0} Z rho^r_r                       */
holo_status holo_grad_ref(holo_plan *p, const void *q, const float *sqrt_dref /*[R][n][n]*/,
                          void *grad_q_part, double *sc, uint32_t flags);

/* Reference-arm forward (O14): w[r] = C( P_{zeta0} S_{s_r} q ), complex64 [R][n][n] row-major
 * (R = n_ref of holo_set_ref_shifts).  Used to synthesise reference frames.            */
holo_status holo_fwd_ref(holo_plan *p, const void *q, void *w);

/* q-block dot products (run identically on every rank after the allreduce):
 *   out[0] = ||grad_q||^2,  out[1] = Re<grad_q, eta_q_prev> (0 if eta_q_prev NULL).       */
holo_status holo_q_dots(holo_plan *p, const void *grad_q, const void *eta_q_prev, double *out /*[2] device*/);

/* CG step (pointwise; Eqs. (13)-(14), reading C9-C11).  in/out are [host] scalars that
 * the caller computed after the allreduce:
 *   if !reuse_eta:  first: eta = -P g;  else eta = -P g + beta eta,
 *                   beta = gPg / (g_eta_prev - gprev_eta_prev);
 *                   guard |den| < 1e-30 gPg or Re<g, eta_new> >= 0  ->  eta = -P g (reset)
 *   x_trial = x + gamma eta          for the psi block and the q block, P = diag(rho_psi, rho_q)
 * out->g_eta_new = Re<g, eta_new> by scalar algebra.  Any of the psi-block pointers may be
 * NULL together (q-only CG), likewise the q-block pointers.  eta_* are updated in place.  */
typedef struct {
  double gPg;            /* <g, P g> = rho_psi ||g_psi||^2 + rho_q ||g_q||^2            */
  double g_eta_prev;     /* Re<g_m, eta_{m-1}>                                          */
  double gprev_eta_prev; /* Re<g_{m-1}, eta_{m-1}>                                      */
  double gamma;          /* step length                                                 */
  double rho_psi, rho_q; /* block preconditioner P                                      */
  int32_t first;         /* 1: eta = -P g                                               */
  int32_t reuse_eta;     /* 1: keep eta (line-search retry), only x_trial is formed     */
} holo_cg_in;
typedef struct {
  double beta, g_eta_new;
  int32_t reset;
} holo_cg_out;
holo_status holo_cg_step(holo_plan *p, const holo_cg_in *in /*[host]*/, holo_cg_out *out /*[host]*/,
                         const void *psi, void *eta_psi, const void *grad_psi, void *psi_trial,
                         const void *q, void *eta_q, const void *grad_q, void *q_trial);

/* CG-step fusion: holo_set_cg_fuse(p, 1) makes holo_cg_step apply the q block at once but defer the
 * psi block: the next holo_fwd / holo_adj / holo_grad / holo_grad_full whose psi argument is that call's
 * psi_trial performs it inside its first row pass (X1 reads the psi, eta_psi and grad_psi rows, writes
 * the eta_psi and psi_trial rows, and transforms psi_trial) -- the same element-wise arithmetic as the
 * separate pointwise pass, one pass over the psi block fewer per iteration.  Any other entry point of
 * the plan first completes a pending update with the separate kernel, so psi_trial / eta_psi are
 * materialised before anything else of this plan reads them; read them from other code only after
 * the sweep.  Default 0. */
holo_status holo_set_cg_fuse(holo_plan *p, int32_t on);

/* Multiresolution schedule ("binning 8x8 ... 4x4 ... then extrapolate
 * the recovered object with the probe function to a grid twice as dense").
 * holo_upsample2: Fourier 2x upsampling (O15, reading R1) of `count` complex64 fields
 *   coarse [count][npad/2][npad/2] -> fine [count][npad][npad] (row-major, this plan = the FINE
 *   level; npad a power of two).  Per axis y[m] = (1/L) sum_f X[f] e^{2 pi i fbar (m - 1/2)/(2L)},
 *   L = npad/2, fbar in [-L/2, L/2): coarse sample n sits at fine coordinate 2n + 1/2.
 *   Uses the plan's scratch; coarse and fine must not alias.  HOLO_EUNSUPPORTED for npad 6144.
 * holo_bin2: 2x2 binning of amplitudes sqrt(d~) (O16, reading R2): fine [count][2n][2n] ->
 *   coarse [count][n][n] (this plan = the COARSE level, n its data side), a_c = sqrt(mean a_f^2). */
holo_status holo_upsample2(holo_plan *p, const void *coarse, void *fine, int32_t count);
holo_status holo_bin2(holo_plan *p, const float *fine, float *coarse, int32_t count);

/* Initialisers.
 * holo_init_probe (O17): "the reference image propagated back to the sample plane 0":
 *   q0 = (1/R) sum_r S_{-s_r} P_{-zeta0} Z_{c_r}(sqrt_dref_r)   [npad][npad] complex64,
 *   sqrt_dref [R][n][n] (R = n_ref, shifts of holo_set_ref_shifts), each frame padded with its
 *   mean amplitude c_r (reading R3).  HOLO_EINVAL without reference frames.
 * holo_init_psi (O18): multi-distance Paganin initial object of every angle (reading R4):
 *   R_j = (sqrt_d_kj / sqrt_dref)^2 (sqrt_dref^2 floored at 1e-6 of its max), 1 outside the data;
 *   I_j = M_{mt_j} S_{-s_kj} R_j on the psi grid (O5 with mt' = 1/mt_j, s' = -s_kj/mt_j);
 *   phi = (db/2) ln Re IDFT2[ sum_j DFT2(I_j) / (nz + pi lambda db sum_j zeta_j |f|^2) ];
 *   psi0_k = exp((i + 1/db) phi).  sqrt_d [K][nz][n][n], sqrt_dref [n][n] (the flat field of
 *   every plane), delta_beta = delta/beta > 0, psi0 [K][npad][npad].  Uses the plan's
 *   shifts (holo_set_shifts) and its T1/T3 workspace; power-of-two npad only. */
holo_status holo_init_probe(holo_plan *p, const float *sqrt_dref, void *q0);
holo_status holo_init_psi(holo_plan *p, const float *sqrt_d, const float *sqrt_dref, double delta_beta, void *psi0);

/* Staged data (end-to-end streaming): the next holo_grad / holo_grad_full call whose sqrt_d argument
 * is dev_sqrt_d first copies host_sqrt_d (PINNED host memory, [K][nz][n][n] float32) into it, one angle
 * batch at a time on a plan-owned copy stream that starts after everything already queued on the
 * plan's stream; each batch's residual pass waits only for its own slice, so the transfer of batch
 * b + 1 overlaps the passes of batch b.  Later calls read the resident data.  A stage stays pending
 * until a call reads dev_sqrt_d (or it is replaced); NULL pointers cancel it.  The host buffer must stay
 * valid until that call's work has completed. */
holo_status holo_stage_sqrt_d(holo_plan *p, const float *host_sqrt_d, float *dev_sqrt_d);
/* The same for the reference frames (sqrt_dref [R][n][n] of holo_grad_ref / holo_grad_full, R = n_ref of
 * holo_set_ref_shifts, which must precede it): streamed per batch of reference frames, each batch's row
 * pass (R2) waiting for its own slice. */
holo_status holo_stage_sqrt_dref(holo_plan *p, const float *host_sqrt_dref, float *dev_sqrt_dref);

/* Fourier-domain object state (Parseval; SURVEY 8(e) "run CG ... in the Fourier domain").
 * holo_set_fourier(p, 1): every later holo_fwd / holo_adj / holo_grad / holo_grad_full call on this
 * plan takes psi and eta_psi_prev, and returns grad_psi / adj_psi, as the 2-D DFTs of the object-domain
 * arrays (psi~_k = DFT2(psi_k), unnormalised: psi~[fy][fx] = sum_{y,x} psi[y][x] e^{-2 pi i (fy y + fx x)/npad},
 * row-major, natural frequency order), while F, sc[1] = ||grad_psi||^2 and sc[2] = Re<grad_psi, eta_psi_prev>
 * stay the object-domain values (Parseval: the transformed dots / npad^2).  The operators are unchanged;
 * the chain skips the transforms that only move the object in and out of the Fourier domain (X1's row
 * FFT, Y1's column FFT, Y2's column IFFT and X3's row IFFT: 2.5 of ~21.5 line transforms per frame).
 * The CG step is pointwise and linear, so it runs unchanged on the transformed arrays.  Default 0.
 * HOLO_EUNSUPPORTED for npad 6144.
 * holo_fourier: out[m] = DFT2(in[m]) (inverse = 0) or IDFT2(in[m]) = (1/npad^2) sum e^{+...} (inverse = 1)
 * for m < count, row-major [count][npad][npad] complex64; in == out allowed (the plan's scratch sits
 * between the two passes).  Not usable while a sweep of the same plan is pending on another stream;
 * HOLO_EUNSUPPORTED on a plan without angles (it uses the object chain's scratch). */
holo_status holo_set_fourier(holo_plan *p, int32_t on);
holo_status holo_fourier(holo_plan *p, const void *in, void *out, int32_t count, int32_t inverse);

/* Number of kernel launches this plan has enqueued since creation (profiling aid). */
uint64_t holo_launch_count(const holo_plan *p);

/* Per-pass device timing with CUDA events recorded on the plan's stream around every
 * launch (enable = 1 starts recording, 0 stops).  holo_profile_read synchronises on the
 * last recorded event and returns, per pass id, the summed device time [ms], the number
 * of launches and the ALGORITHMIC bytes / flops of those launches (DESIGN.md byte and
 * flop model; flops use 5 L log2 L per length-L complex FFT).  Arrays are [host] of
 * length HOLO_NPASS; any may be NULL.  reset = 1 clears the accumulators.
 * Pass ids: */
#define HOLO_PASS_X1 0
#define HOLO_PASS_Y1 1
#define HOLO_PASS_X2 2
#define HOLO_PASS_Y2 3
#define HOLO_PASS_X3 4
#define HOLO_PASS_FILTER 5 /* q_j = P_omega q and g_q = 2 sum P_-omega G_j */
#define HOLO_PASS_REDUCE 6
#define HOLO_PASS_CG 7
#define HOLO_PASS_REF 8
#define HOLO_PASS_PS 9 /* probe-shift passes XQ / XG (holo_set_probe_shifts) */
#define HOLO_NPASS 10
holo_status holo_profile_enable(holo_plan *p, int enable);
holo_status holo_profile_read(holo_plan *p, double *ms, uint64_t *launches, double *bytes, double *flops, int reset);

#ifdef __cplusplus
}
#endif
#endif /* HOLO_H */
