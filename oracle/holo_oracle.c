/*
 * holo_oracle.c -- fp64 CPU ORACLE for the hot path of arXiv 2407.20304
 * ("X-ray nano-holotomography reconstruction with simultaneous probe retrieval").
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  The product path
 * (paper_2407_20304_b200/) never links, imports or executes it, and the two share
 * no code, headers, tables or constants.
 *
 * Plain definitions, written out: every 1-D transform is a naive O(L^2) DFT sum
 * with exact integer reduction of the twiddle index, no FFT anywhere.  2-D
 * operators are applied separably, x axis (fast index) first, then y.
 * Arrays are row-major [y][x], complex = interleaved fp64 (re, im).
 *
 * Citations: P:n = /root/reference/PAPER.md line n; readings C1..C21 and
 * definitions O1..O14 are listed in DESIGN.md ("Readings of the paper").
 *
 *   O1  geometry                  Eq.(8), Thm 2, Eq.(6)
 *   O2  DFT convention            X[f] = sum_n x[n] e^{-2 pi i f n / L}, inverse 1/L
 *   O3  Fresnel propagation P_z   kernel P_Z P:318-323 (defPz/defGz); Fourier form
 *                                  h_z[f] = exp(-i pi lambda z (fbar/(L p0))^2)
 *   O4  shift S_s                 P:111; (S_s x)(u) = x(u - s), periodic (C4)
 *   O5  magnification M_{1/mt}    M_m f(x) = f(x/m) P:86; band-limited
 *                                  Fourier rescale on the torus (reading C1)
 *   O6  q_j = P_{omega_j} q        Eq.(8)
 *   O7  forward  w = C P_zdet (q_j . M S psi)            Eq.(8), L_kj P:123
 *   O8  F1 = sum (|w| - sqrt d)^2                        Eq.(10)
 *   O9  rho = w - sqrt(d) w/|w|  (0 where w = 0, C7)     Eq.(11), App A.3
 *   O10 v = P_{-zdet} Z rho                              L* P:123
 *   O11 g_psi = 2 sum_j (M S)^* (conj(q_j) v)            Eq.(11)
 *   O12 g_q = 2 sum_j P_{-omega_j} sum_k conj(M S psi) v Eq.(12)
 *   O14 reference arm  w^r = C P_{zeta0} S_{s_r} q       P:102, Eq.(10)/(12)
 */
#include <complex.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>

typedef double complex cplx;

static const double PI = 3.14159265358979323846264338327950288;

/* ------------------------------------------------------------------ O1 ---- */
/* m0 = Z/z1_0; mt_j = z1_j/z1_0; z2_j = Z - z1_j; zeta_j = z1_j z2_j / Z;
 * omega_j = (z1_j - z1_0)/mt_j; zdet_j = zeta_j / mt_j^2; p0 = det_px / m0.   */
int or_geometry(int nz, double Z, const double *z1, double det_px, double *m0,
                double *mt, double *zeta, double *zdet, double *omega, double *p0) {
  if (nz < 1 || !(Z > 0) || !(det_px > 0)) return -1;
  for (int j = 0; j < nz; j++) {
    if (!(z1[j] > 0) || !(z1[j] < Z)) return -1;
    if (j > 0 && !(z1[j] > z1[j - 1])) return -1;
  }
  *m0 = Z / z1[0];
  *p0 = det_px / *m0;
  for (int j = 0; j < nz; j++) {
    double z2 = Z - z1[j];
    mt[j] = z1[j] / z1[0];
    zeta[j] = z1[j] * z2 / Z;
    omega[j] = (z1[j] - z1[0]) / mt[j];
    zdet[j] = zeta[j] / (mt[j] * mt[j]);
  }
  return 0;
}

/* ---------------------------------------------------------- helpers ------- */
static inline long fbar_of(long f, long L) { return f < L / 2 ? f : f - L; }
static inline long mod_l(long a, long L) { long r = a % L; return r < 0 ? r + L : r; }

/* W[t] = exp(-2 pi i t / L), t in [0, L) */
static cplx *twiddles(long L) {
  cplx *W = (cplx *)malloc(sizeof(cplx) * L);
  for (long t = 0; t < L; t++) W[t] = cexp(-2.0 * PI * I * (double)t / (double)L);
  return W;
}

/* ------------------------------------------------------------------ O2 ---- */
/* X[f] = sum_n x[n] W[(f n) mod L];  inverse: x[n] = (1/L) sum_f X[f] conj(W[(f n) mod L]) */
static void dft_line(long L, int inverse, const cplx *W, const cplx *x, cplx *X) {
  for (long f = 0; f < L; f++) {
    cplx acc = 0;
    long t = 0;
    for (long n = 0; n < L; n++) {
      acc += x[n] * (inverse ? conj(W[t]) : W[t]);
      t += f;
      if (t >= L) t -= L;
    }
    X[f] = inverse ? acc / (double)L : acc;
  }
}

void or_dft1(int L, int inverse, const cplx *x, cplx *X) {
  cplx *W = twiddles(L);
  dft_line(L, inverse, W, x, X);
  free(W);
}

/* ------------------------------------------ separable 2-D line machinery -- */
typedef void (*line_op)(const void *ctx, long L, const cplx *in, cplx *out, cplx *scratch);

/* Apply op to every line of an [L][L] array along axis 0 (x: rows, contiguous)
 * or axis 1 (y: columns).  in and out may alias. */
static void apply_axis(long L, int axis_y, const cplx *in, cplx *out, line_op op, const void *ctx) {
#pragma omp parallel
  {
    cplx *li = (cplx *)malloc(sizeof(cplx) * L);
    cplx *lo = (cplx *)malloc(sizeof(cplx) * L);
    cplx *sc = (cplx *)malloc(sizeof(cplx) * 2 * L);
#pragma omp for schedule(static)
    for (long l = 0; l < L; l++) {
      for (long n = 0; n < L; n++) li[n] = axis_y ? in[n * L + l] : in[l * L + n];
      op(ctx, L, li, lo, sc);
      for (long n = 0; n < L; n++) {
        if (axis_y) out[n * L + l] = lo[n];
        else out[l * L + n] = lo[n];
      }
    }
    free(li); free(lo); free(sc);
  }
}

/* ------------------------------------------------------------------ O3 ---- */
/* P_z line: IDFT( h_z . DFT x ),  h_z[f] = exp(-i pi lambda z (fbar/(L p0))^2).
 * The unimodular factor e^{ikz}/i of the kernel P:319 is dropped (the paper's
 * "~=" P:327); P_z^* = P_{-z}.                                        */
typedef struct { const cplx *W; double lam, p0, z; } prop_ctx;

static void prop_line(const void *c, long L, const cplx *in, cplx *out, cplx *sc) {
  const prop_ctx *p = (const prop_ctx *)c;
  dft_line(L, 0, p->W, in, sc);
  for (long f = 0; f < L; f++) {
    double fr = (double)fbar_of(f, L) / ((double)L * p->p0); /* cycles per metre */
    sc[f] *= cexp(-I * PI * p->lam * p->z * fr * fr);
  }
  dft_line(L, 1, p->W, sc, out);
}

void or_prop(int L, double lam, double p0, double z, const cplx *in, cplx *out) {
  prop_ctx c = {twiddles(L), lam, p0, z};
  apply_axis(L, 0, in, out, prop_line, &c);
  apply_axis(L, 1, out, out, prop_line, &c);
  free((void *)c.W);
}

/* ------------------------------------------------------------------ O4 ---- */
/* S_s line: IDFT( r_s . DFT x ),  r_s[f] = exp(-2 pi i fbar s / L); (S_s x)(u) = x(u-s). */
typedef struct { const cplx *W; double s; } shift_ctx;

static void shift_line(const void *c, long L, const cplx *in, cplx *out, cplx *sc) {
  const shift_ctx *p = (const shift_ctx *)c;
  dft_line(L, 0, p->W, in, sc);
  for (long f = 0; f < L; f++) sc[f] *= cexp(-2.0 * PI * I * (double)fbar_of(f, L) * p->s / (double)L);
  dft_line(L, 1, p->W, sc, out);
}

void or_shift(int L, double sx, double sy, const cplx *in, cplx *out) {
  cplx *W = twiddles(L);
  shift_ctx cx = {W, sx}, cy = {W, sy};
  apply_axis(L, 0, in, out, shift_line, &cx);
  apply_axis(L, 1, out, out, shift_line, &cy);
  free(W);
}

/* ------------------------------------------------------------------ O5 ---- */
/* Magnification M_{1/mt} with its preceding shift S_s, one axis (reading C1):
 *   u(n)  = n - L/2                              centred coordinate
 *   Xc[f] = sum_n x[n] e^{-2 pi i fbar u(n)/L}    centred spectrum
 *   kappa[f] = 1 iff -L/2 <= mt fbar < L/2        output band
 *   y[n]  = (1/L) sum_f kappa r_s[f] Xc[f] e^{+2 pi i mt fbar u(n)/L}
 * i.e. output(u) = (S_s x)(mt u): M_m f(x) = f(x/m) with m = 1/mt.
 * Adjoint (exact conjugate transpose):
 *   Z[f]  = sum_n y[n] e^{-2 pi i mt fbar u(n)/L}
 *   x~[n] = (1/L) sum_f e^{+2 pi i fbar u(n)/L} conj(r_s[f]) kappa[f] Z[f]    */
typedef struct { const cplx *W; const cplx *E; double mt, s; } mag_ctx;

static inline int kappa(long fb, long L, double mt) {
  double v = mt * (double)fb;
  return v >= -(double)(L / 2) && v < (double)(L / 2);
}

/* E[n*L + f] = exp(+2 pi i mt fbar u(n) / L); phase reduced mod L before scaling */
static cplx *mag_matrix(long L, double mt) {
  cplx *E = (cplx *)malloc(sizeof(cplx) * L * L);
#pragma omp parallel for schedule(static)
  for (long n = 0; n < L; n++) {
    long u = n - L / 2;
    for (long f = 0; f < L; f++) {
      double p = mt * (double)(fbar_of(f, L) * u);
      p -= (double)L * floor(p / (double)L);
      E[n * L + f] = cexp(2.0 * PI * I * p / (double)L);
    }
  }
  return E;
}

static void mag_line(const void *c, long L, const cplx *in, cplx *out, cplx *sc) {
  const mag_ctx *p = (const mag_ctx *)c;
  for (long f = 0; f < L; f++) {
    long fb = fbar_of(f, L);
    cplx acc = 0;
    for (long n = 0; n < L; n++) acc += in[n] * p->W[mod_l(fb * (n - L / 2), L)];
    sc[f] = kappa(fb, L, p->mt) ? acc * cexp(-2.0 * PI * I * (double)fb * p->s / (double)L) : 0;
  }
  for (long n = 0; n < L; n++) {
    cplx acc = 0;
    const cplx *En = p->E + n * L;
    for (long f = 0; f < L; f++) acc += sc[f] * En[f];
    out[n] = acc / (double)L;
  }
}

static void mag_adj_line(const void *c, long L, const cplx *in, cplx *out, cplx *sc) {
  const mag_ctx *p = (const mag_ctx *)c;
  for (long f = 0; f < L; f++) sc[f] = 0;
  for (long n = 0; n < L; n++) {
    const cplx *En = p->E + n * L;
    for (long f = 0; f < L; f++) sc[f] += in[n] * conj(En[f]);
  }
  for (long f = 0; f < L; f++) {
    long fb = fbar_of(f, L);
    sc[f] = kappa(fb, L, p->mt) ? sc[f] * cexp(2.0 * PI * I * (double)fb * p->s / (double)L) : 0;
  }
  for (long n = 0; n < L; n++) {
    cplx acc = 0;
    for (long f = 0; f < L; f++) acc += sc[f] * conj(p->W[mod_l(fbar_of(f, L) * (n - L / 2), L)]);
    out[n] = acc / (double)L;
  }
}

/* 2-D: along x with (mt, sx), then along y with (mt, sy) */
void or_mag(int L, double mt, double sx, double sy, const cplx *in, cplx *out) {
  cplx *W = twiddles(L), *E = mag_matrix(L, mt);
  mag_ctx cx = {W, E, mt, sx}, cy = {W, E, mt, sy};
  apply_axis(L, 0, in, out, mag_line, &cx);
  apply_axis(L, 1, out, out, mag_line, &cy);
  free(W); free(E);
}

void or_mag_adj(int L, double mt, double sx, double sy, const cplx *in, cplx *out) {
  cplx *W = twiddles(L), *E = mag_matrix(L, mt);
  mag_ctx cx = {W, E, mt, sx}, cy = {W, E, mt, sy};
  apply_axis(L, 1, in, out, mag_adj_line, &cy);
  apply_axis(L, 0, out, out, mag_adj_line, &cx);
  free(W); free(E);
}

/* ------------------------------------------------------- crop / zero-pad -- */
/* C crops rows and columns [o, o+N), o = (L-N)/2;  Z = C^T zero-pads (O7).   */
static void crop(long L, long N, const cplx *in, cplx *out) {
  long o = (L - N) / 2;
  for (long y = 0; y < N; y++)
    for (long x = 0; x < N; x++) out[y * N + x] = in[(y + o) * L + (x + o)];
}
static void zpad(long L, long N, const cplx *in, cplx *out) {
  long o = (L - N) / 2;
  memset(out, 0, sizeof(cplx) * L * L);
  for (long y = 0; y < N; y++)
    for (long x = 0; x < N; x++) out[(y + o) * L + (x + o)] = in[y * N + x];
}

typedef struct {
  int K, nz, L, N;
  double lam, p0;
  const double *mt, *zdet, *omega, *shifts; /* shifts [K][nz][2] = (sx, sy) */
} geom_t;

/* ------------------------------------------------------------- O6, O7 ---- */
void or_fwd(int K, int nz, int L, int N, double lam, double p0, const double *mt,
            const double *zdet, const double *omega, const double *shifts,
            const cplx *psi, const cplx *q, cplx *w) {
  long LL = (long)L * L, NN = (long)N * N;
  cplx *qj = (cplx *)malloc(sizeof(cplx) * LL), *a = (cplx *)malloc(sizeof(cplx) * LL);
  for (int j = 0; j < nz; j++) {
    or_prop(L, lam, p0, omega[j], q, qj);                    /* O6 */
    for (int k = 0; k < K; k++) {
      const double *s = shifts + ((long)k * nz + j) * 2;
      or_mag(L, mt[j], s[0], s[1], psi + k * LL, a);         /* M_{1/mt} S_s psi_k */
      for (long i = 0; i < LL; i++) a[i] *= qj[i];            /* q_j . (.) */
      or_prop(L, lam, p0, zdet[j], a, a);                    /* P_{zdet_j} */
      crop(L, N, a, w + ((long)k * nz + j) * NN);            /* C */
    }
  }
  free(qj); free(a);
}

/* Adjoints of the two linearisations at (psi, q), no factor 2:
 *   adj_psi[k] = sum_j L_kj^* y_kj = sum_j (M S)^*( conj(q_j) P_{-zdet} Z y_kj )
 *   adj_q      = sum_j P_{-omega_j} sum_k conj(M S psi_k) P_{-zdet} Z y_kj        */
void or_adj(int K, int nz, int L, int N, double lam, double p0, const double *mt,
            const double *zdet, const double *omega, const double *shifts,
            const cplx *y, const cplx *psi, const cplx *q, cplx *adj_psi, cplx *adj_q) {
  long LL = (long)L * L, NN = (long)N * N;
  cplx *qj = (cplx *)malloc(sizeof(cplx) * LL), *a = (cplx *)malloc(sizeof(cplx) * LL);
  cplx *v = (cplx *)malloc(sizeof(cplx) * LL), *G = (cplx *)malloc(sizeof(cplx) * LL);
  cplx *t = (cplx *)malloc(sizeof(cplx) * LL);
  if (adj_psi) memset(adj_psi, 0, sizeof(cplx) * LL * K);
  if (adj_q) memset(adj_q, 0, sizeof(cplx) * LL);
  for (int j = 0; j < nz; j++) {
    or_prop(L, lam, p0, omega[j], q, qj);
    memset(G, 0, sizeof(cplx) * LL);
    for (int k = 0; k < K; k++) {
      const double *s = shifts + ((long)k * nz + j) * 2;
      zpad(L, N, y + ((long)k * nz + j) * NN, v);
      or_prop(L, lam, p0, -zdet[j], v, v);
      if (adj_q) {
        or_mag(L, mt[j], s[0], s[1], psi + k * LL, a);
        for (long i = 0; i < LL; i++) G[i] += conj(a[i]) * v[i];
      }
      if (adj_psi) {
        for (long i = 0; i < LL; i++) t[i] = conj(qj[i]) * v[i];
        or_mag_adj(L, mt[j], s[0], s[1], t, t);
        for (long i = 0; i < LL; i++) adj_psi[k * LL + i] += t[i];
      }
    }
    if (adj_q) {
      or_prop(L, lam, p0, -omega[j], G, G);
      for (long i = 0; i < LL; i++) adj_q[i] += G[i];
    }
  }
  free(qj); free(a); free(v); free(G); free(t);
}

/* ------------------------------------------------------------ O8 - O12 ---- */
/* Returns F = sum_{k,j} sum_pix (|w| - sqrt_d)^2; writes grad_psi = 2 sum_j L^* rho
 * and grad_q = 2 sum_j P_{-omega_j} sum_k conj(M S psi_k) v  (either may be NULL).
 * Summation order: F over k, then j, then pixels row-major; G_j over k ascending;
 * g_q over j ascending.                                                        */
double or_grad(int K, int nz, int L, int N, double lam, double p0, const double *mt,
               const double *zdet, const double *omega, const double *shifts,
               const cplx *psi, const cplx *q, const double *sqrt_d,
               cplx *grad_psi, cplx *grad_q) {
  long LL = (long)L * L, NN = (long)N * N;
  cplx *qj = (cplx *)malloc(sizeof(cplx) * LL), *a = (cplx *)malloc(sizeof(cplx) * LL);
  cplx *v = (cplx *)malloc(sizeof(cplx) * LL), *G = (cplx *)malloc(sizeof(cplx) * LL);
  cplx *t = (cplx *)malloc(sizeof(cplx) * LL), *w = (cplx *)malloc(sizeof(cplx) * NN);
  double F = 0;
  if (grad_psi) memset(grad_psi, 0, sizeof(cplx) * LL * K);
  if (grad_q) memset(grad_q, 0, sizeof(cplx) * LL);
  for (int j = 0; j < nz; j++) {
    or_prop(L, lam, p0, omega[j], q, qj);                       /* q_j = P_{omega_j} q */
    memset(G, 0, sizeof(cplx) * LL);
    for (int k = 0; k < K; k++) {
      const double *s = shifts + ((long)k * nz + j) * 2;
      const double *d = sqrt_d + ((long)k * nz + j) * NN;
      or_mag(L, mt[j], s[0], s[1], psi + k * LL, a);            /* a = M S psi_k */
      for (long i = 0; i < LL; i++) t[i] = qj[i] * a[i];
      or_prop(L, lam, p0, zdet[j], t, t);
      crop(L, N, t, w);                                         /* w = L_kj psi_k */
      for (long i = 0; i < NN; i++) {
        double m = cabs(w[i]);
        F += (m - d[i]) * (m - d[i]);                           /* O8 */
        w[i] = m > 0 ? w[i] - d[i] * w[i] / m : 0;              /* O9 (C7) */
      }
      zpad(L, N, w, v);
      or_prop(L, lam, p0, -zdet[j], v, v);                      /* O10 */
      if (grad_q)
        for (long i = 0; i < LL; i++) G[i] += conj(a[i]) * v[i];
      if (grad_psi) {
        for (long i = 0; i < LL; i++) t[i] = conj(qj[i]) * v[i];
        or_mag_adj(L, mt[j], s[0], s[1], t, t);                 /* O11 */
        for (long i = 0; i < LL; i++) grad_psi[k * LL + i] += 2.0 * t[i];
      }
    }
    if (grad_q) {
      or_prop(L, lam, p0, -omega[j], G, G);                     /* O12 */
      for (long i = 0; i < LL; i++) grad_q[i] += 2.0 * G[i];
    }
  }
  free(qj); free(a); free(v); free(G); free(t); free(w);
  return F;
}

/* ------------------------------------------------------------------ O14 --- */
/* Reference arm: w^r_r = C P_{zeta0} S_{s_r} q;  F_ref = sum_r sum (|w^r| - a^r)^2;
 * grad_q += 2 sum_r S_{-s_r} P_{-zeta0} Z rho^r  (accumulated into grad_q if not NULL). */
double or_grad_ref(int R, int L, int N, double lam, double p0, double zeta0,
                   const double *ref_shifts, const cplx *q, const double *sqrt_dref, cplx *grad_q) {
  long LL = (long)L * L, NN = (long)N * N;
  cplx *t = (cplx *)malloc(sizeof(cplx) * LL), *w = (cplx *)malloc(sizeof(cplx) * NN);
  double F = 0;
  for (int r = 0; r < R; r++) {
    const double *s = ref_shifts + 2L * r;
    const double *d = sqrt_dref + (long)r * NN;
    or_shift(L, s[0], s[1], q, t);
    or_prop(L, lam, p0, zeta0, t, t);
    crop(L, N, t, w);
    for (long i = 0; i < NN; i++) {
      double m = cabs(w[i]);
      F += (m - d[i]) * (m - d[i]);
      w[i] = m > 0 ? w[i] - d[i] * w[i] / m : 0;
    }
    if (grad_q) {
      zpad(L, N, w, t);
      or_prop(L, lam, p0, -zeta0, t, t);
      or_shift(L, -s[0], -s[1], t, t);
      for (long i = 0; i < LL; i++) grad_q[i] += 2.0 * t[i];
    }
  }
  free(t); free(w);
  return F;
}

/* ------------------------------------------------------------------ O15 --- */
/* Fourier 2x upsampling of an [L][L] field to [2L][2L] between levels of the
 * multiresolution schedule ("extrapolate the recovered object with the probe
 * function to a grid twice as dense").  Reading R1: the trigonometric
 * interpolant of x, band fbar in [-L/2, L/2) (Nyquist bin at -L/2, reading C2), sampled at
 * half-pixel steps with coarse sample n at fine coordinate 2n + 1/2 (the centre of the fine
 * pixels a 2x2 bin merges, O16):
 *   y[m] = (1/L) sum_f X[f] exp(+2 pi i fbar (m - 1/2) / (2L)),  X = DFT_L(x),  m in [0, 2L)
 * applied along x (rows) then along y (columns).  Naive sums, no FFT.                  */
static void up_line(long L, const cplx *W, const cplx *x, cplx *y, cplx *X) {
  dft_line(L, 0, W, x, X);
  for (long m = 0; m < 2 * L; m++) {
    cplx acc = 0;
    for (long f = 0; f < L; f++) acc += X[f] * cexp(2.0 * PI * I * (double)fbar_of(f, L) * ((double)m - 0.5) / (2.0 * L));
    y[m] = acc / (double)L;
  }
}

void or_upsample2(int L, const cplx *in, cplx *out) {
  const long L2 = 2L * L;
  cplx *W = twiddles(L);
  cplx *mid = (cplx *)malloc(sizeof(cplx) * L * L2); /* [L][2L]: rows done */
#pragma omp parallel
  {
    cplx *li = (cplx *)malloc(sizeof(cplx) * L), *lo = (cplx *)malloc(sizeof(cplx) * L2),
         *X = (cplx *)malloc(sizeof(cplx) * L);
#pragma omp for schedule(static)
    for (long y = 0; y < L; y++) up_line(L, W, in + y * L, mid + y * L2, X);
#pragma omp for schedule(static)
    for (long x = 0; x < L2; x++) {
      for (long y = 0; y < L; y++) li[y] = mid[y * L2 + x];
      up_line(L, W, li, lo, X);
      for (long m = 0; m < L2; m++) out[m * L2 + x] = lo[m];
    }
    free(li); free(lo); free(X);
  }
  free(mid); free(W);
}

/* ------------------------------------------------------------------ O16 --- */
/* 2x2 binning of the measured amplitudes a = sqrt(d~) ("binning 8x8 ... 4x4"): the
 * intensity of a binned pixel is the block MEAN of the four intensities (reading R2, the
 * per-pixel intensity unit is kept; the detector pixel doubles), so
 *   a_c[i][l] = sqrt( (1/4) sum_{a,b in {0,1}} a_f[2i+a][2l+b]^2 ),  count frames of [2N][2N]. */
void or_bin2(int count, int N, const double *fine, double *coarse) {
  const long N2 = 2L * N;
  for (long c = 0; c < count; c++)
    for (long i = 0; i < N; i++)
      for (long l = 0; l < N; l++) {
        double s = 0;
        for (int a = 0; a < 2; a++)
          for (int b = 0; b < 2; b++) {
            const double v = fine[c * N2 * N2 + (2 * i + a) * N2 + 2 * l + b];
            s += v * v;
          }
        coarse[c * (long)N * N + i * N + l] = sqrt(0.25 * s);
      }
}

/* plain DFT line ops for apply_axis (ctx = the twiddle table W) */
static void dft_fwd_line(const void *c, long L, const cplx *in, cplx *out, cplx *sc) {
  (void)sc;
  dft_line(L, 0, (const cplx *)c, in, out);
}
static void dft_inv_line(const void *c, long L, const cplx *in, cplx *out, cplx *sc) {
  (void)sc;
  dft_line(L, 1, (const cplx *)c, in, out);
}

/* ------------------------------------------------------------------ O17 --- */
/* Initial probe ("the reference image propagated back to the sample
 * plane 0"; reference model P:102, Eq. (10)):
 *   q0 = (1/R) sum_r S_{-s_r} P_{-zeta0} Z_{c_r}(a_r),  a_r = sqrt(d~^r_r),  c_r = mean(a_r)
 * (zero phase; the ring around the N x N frame filled with the frame's mean amplitude, R3). */
void or_init_probe(int R, int L, int N, double lam, double p0, double zeta0, const double *ref_shifts,
                   const double *sqrt_dref, cplx *q0) {
  const long LL = (long)L * L, NN = (long)N * N, o = (L - N) / 2;
  cplx *t = (cplx *)malloc(sizeof(cplx) * LL);
  for (long i = 0; i < LL; i++) q0[i] = 0;
  for (int r = 0; r < R; r++) {
    const double *a = sqrt_dref + r * NN;
    double c = 0;
    for (long i = 0; i < NN; i++) c += a[i];
    c /= (double)NN;
    for (long y = 0; y < L; y++)
      for (long x = 0; x < L; x++) {
        const int in = y >= o && y < o + N && x >= o && x < o + N;
        t[y * L + x] = in ? a[(y - o) * N + (x - o)] : c;
      }
    or_prop(L, lam, p0, -zeta0, t, t);
    or_shift(L, -ref_shifts[2 * r], -ref_shifts[2 * r + 1], t, t);
    for (long i = 0; i < LL; i++) q0[i] += t[i] / (double)R;
  }
  free(t);
}

/* ------------------------------------------------------------------ O18 --- */
/* Multi-distance Paganin (TIE) initial object of one angle (formula absent from
 * the paper: SPEC's documented stand-in in this build's sign convention, reading R4):
 *   R_j = (a_kj / a^r)^2, a^r^2 floored at 1e-6 max, padded with 1;
 *   I_j = M_{1/mt'} S_{s'} R_j,  mt' = 1/mt_j, s' = -s_kj / mt_j            (O5)
 *   Phi = sum_j DFT2(I_j) / (nz + pi lambda db sum_j zeta_j |f|^2),  |f| = fbar/(L p0)
 *   phi = (db/2) ln max(Re IDFT2(Phi), 1e-6),  psi0 = exp((i + 1/db) phi).               */
void or_multipaganin(int nz, int L, int N, double lam, double p0, const double *mt, const double *zeta,
                     const double *shifts_k, const double *sqrt_d_k, const double *sqrt_dref, double db,
                     cplx *psi0) {
  const long LL = (long)L * L, NN = (long)N * N, o = (L - N) / 2;
  cplx *t = (cplx *)malloc(sizeof(cplx) * LL), *num = (cplx *)malloc(sizeof(cplx) * LL);
  cplx *W = twiddles(L);
  double amax = 0, zs = 0;
  for (long i = 0; i < NN; i++) amax = fmax(amax, sqrt_dref[i] * sqrt_dref[i]);
  for (int j = 0; j < nz; j++) zs += zeta[j];
  for (long i = 0; i < LL; i++) num[i] = 0;
  for (int j = 0; j < nz; j++) {
    for (long y = 0; y < L; y++)
      for (long x = 0; x < L; x++) {
        const int in = y >= o && y < o + N && x >= o && x < o + N;
        double v = 1.0;
        if (in) {
          const long i = (y - o) * N + (x - o);
          const double ar2 = fmax(sqrt_dref[i] * sqrt_dref[i], 1e-6 * amax);
          v = sqrt_d_k[j * NN + i] * sqrt_d_k[j * NN + i] / ar2;
        }
        t[y * L + x] = v;
      }
    const double mtp = 1.0 / mt[j];
    or_mag(L, mtp, -shifts_k[2 * j] * mtp, -shifts_k[2 * j + 1] * mtp, t, t);
    apply_axis(L, 0, t, t, dft_fwd_line, W);
    apply_axis(L, 1, t, t, dft_fwd_line, W);
    for (long i = 0; i < LL; i++) num[i] += t[i];
  }
  for (long fy = 0; fy < L; fy++)
    for (long fx = 0; fx < L; fx++) {
      const double gy = (double)fbar_of(fy, L) / ((double)L * p0), gx = (double)fbar_of(fx, L) / ((double)L * p0);
      num[fy * L + fx] /= (double)nz + PI * lam * db * zs * (gx * gx + gy * gy);
    }
  apply_axis(L, 0, num, num, dft_inv_line, W);
  apply_axis(L, 1, num, num, dft_inv_line, W);
  for (long i = 0; i < LL; i++) {
    const double phi = 0.5 * db * log(fmax(creal(num[i]), 1e-6));
    psi0[i] = cexp((I + 1.0 / db) * phi);
  }
  free(t); free(num); free(W);
}

/* ------------------------------------------------------------------ O19 --- */
/* The full objective of Eq. (10) with per-frame PROBE shifts s^p_kj and the reference term
 * (Eq. (12)):
 *   q_kj = P_{omega_j} S_{s^p_kj} q,   w_kj = C P_{zdet_j}( q_kj . M_{1/mt_j} S_{s_kj} psi_k )
 *   F = sum_kj sum (|w_kj| - a_kj)^2 + F_ref (O14, when R > 0)
 *   grad_psi_k = 2 sum_j (M S)^*( conj(q_kj) v_kj ),  v = P_{-zdet} Z rho        (L*_kj)
 *   grad_q     = 2 sum_kj S_{-s^p_kj} P_{-omega_j}( conj(M S psi_k) v_kj ) + O14's term
 * pshifts [K][nz][2]; ref_shifts [R][2], sqrt_dref [R][N][N] (R = 0: no reference term).
 * With s^p = 0 this is O8-O12 (+ O14).  Summation: F over j, k, pixels; grad_q over j, k. */
double or_grad_full(int K, int nz, int L, int N, double lam, double p0, const double *mt, const double *zdet,
                    const double *omega, const double *shifts, const double *pshifts, const cplx *psi,
                    const cplx *q, const double *sqrt_d, int R, double zeta0, const double *ref_shifts,
                    const double *sqrt_dref, cplx *grad_psi, cplx *grad_q) {
  long LL = (long)L * L, NN = (long)N * N;
  cplx *qk = (cplx *)malloc(sizeof(cplx) * LL), *a = (cplx *)malloc(sizeof(cplx) * LL);
  cplx *v = (cplx *)malloc(sizeof(cplx) * LL), *t = (cplx *)malloc(sizeof(cplx) * LL);
  cplx *w = (cplx *)malloc(sizeof(cplx) * NN);
  double F = 0;
  if (grad_psi) memset(grad_psi, 0, sizeof(cplx) * LL * K);
  if (grad_q) memset(grad_q, 0, sizeof(cplx) * LL);
  for (int j = 0; j < nz; j++)
    for (int k = 0; k < K; k++) {
      const double *s = shifts + ((long)k * nz + j) * 2, *sp = pshifts + ((long)k * nz + j) * 2;
      const double *d = sqrt_d + ((long)k * nz + j) * NN;
      or_shift(L, sp[0], sp[1], q, qk);
      or_prop(L, lam, p0, omega[j], qk, qk);                    /* q_kj = P_omega S_{s^p} q */
      or_mag(L, mt[j], s[0], s[1], psi + k * LL, a);            /* a = M S psi_k */
      for (long i = 0; i < LL; i++) t[i] = qk[i] * a[i];
      or_prop(L, lam, p0, zdet[j], t, t);
      crop(L, N, t, w);
      for (long i = 0; i < NN; i++) {
        double m = cabs(w[i]);
        F += (m - d[i]) * (m - d[i]);
        w[i] = m > 0 ? w[i] - d[i] * w[i] / m : 0;
      }
      zpad(L, N, w, v);
      or_prop(L, lam, p0, -zdet[j], v, v);
      if (grad_q) {
        for (long i = 0; i < LL; i++) t[i] = conj(a[i]) * v[i];
        or_prop(L, lam, p0, -omega[j], t, t);
        or_shift(L, -sp[0], -sp[1], t, t);                     /* Q_kj^* = S_{-s^p} P_{-omega} (.) */
        for (long i = 0; i < LL; i++) grad_q[i] += 2.0 * t[i];
      }
      if (grad_psi) {
        for (long i = 0; i < LL; i++) t[i] = conj(qk[i]) * v[i];
        or_mag_adj(L, mt[j], s[0], s[1], t, t);
        for (long i = 0; i < LL; i++) grad_psi[k * LL + i] += 2.0 * t[i];
      }
    }
  if (R > 0) F += or_grad_ref(R, L, N, lam, p0, zeta0, ref_shifts, q, sqrt_dref, grad_q);
  free(qk); free(a); free(v); free(t); free(w);
  return F;
}
