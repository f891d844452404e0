// holo_kernels.cuh -- CTA layout, line I/O and the fused magnification
// (Bluestein chirp-z) building blocks of the holotomography sweep (sm_100a).
//
// Per frame (k, j) the operator chain of Eq. (8) and its adjoint
// (L* formula P:123) is applied as five separable line passes ("Pass
// schedule"): X = rows (contiguous), Y = columns:
//
//   X1 (per k)   psi_k row: FFT once, then per plane j:  M_{1/mt_j} S_x   -> T1_j
//   Y1 (k, j)    T1_j col:  M_{1/mt_j} S_y -> a (stored), x q_j, D_y, crop rows -> W1
//   X2 (k, j)    W1 row:    D_x, crop, residual + F (Eq. (10)-(11)), zero-pad, D_x^* -> V1
//   Y2 (k, j)    V1 col:    pad, D_y^* -> v; G_j += conj(a) v; conj(q_j) v, (M S)_y^* -> T3_j
//   X3 (per k)   T3_j rows: (M S)_x^* accumulated over j in the Fourier domain, one
//                inverse FFT, x2 -> grad_psi_k, fused ||g||^2 and Re<g, eta> partials
//
// Every line lives in registers in layout S (fft_engine.cuh) from its load to its
// store; all pointwise factors are applied there.
//
// Magnification M_{1/mt} (reading C1), Bluestein's chirp-z, in layout S:
//   spectrum X = FFT(x);  a[i] = cr[f] X[f],  i = (f + L/2) mod L   (register r -> r^8)
//   cr = kappa (-1)^fbar e^{i pi mt fbar^2/L} r_s[f] / L   (chirp x shift ramp, per (k, j, axis))
//   E = IFFT(FFT(a) Bhat_e),  O = IFFT(FFT(a w) Bhat_o),  w[i] = e^{-i pi i/L}
//   y[o] = cout[o] E[o] + cwo[o] O[o],   cout = e^{i pi mt (o-L/2)^2/L},  cwo = cout conj(w)
// i.e. the 2L-point cyclic convolution with b[d] = e^{-i pi mt d^2/L} split into its
// even/odd spectral halves.  The adjoint runs the same steps conjugated and in reverse.
// All tables are fp64-generated on the host, phases reduced in cycles.
#pragma once
#include "fft_engine.cuh"

namespace holo {

struct Tables {
  const float4 *tw;     // FFT stage twiddle rows (w^m, w^2m | w^4m, w^8m)
  const float2 *hdet;   // [nz][L] h_{zdet_j}[f] / L
  const float2 *homega; // [nz][L] h_{omega_j}[f] (unscaled)
  const float2 *cout;   // [nz][L] e^{i pi mt (o - L/2)^2 / L}
  const float2 *cwo;    // [nz][L] cout[o] conj(w[o])
  const float2 *bke;    // [nz][L] Bhat[2k] / (2L)
  const float2 *bko;    // [nz][L] Bhat[2k+1] / (2L)
  const float2 *wodd;   // [L] e^{-i pi i / L}
  const float2 *cr;     // [K][nz][2][L] spectrum factor per (k, j, axis): mag: cin r_s, else r_s / L
};

// CTA geometry: NT threads, G = NT / T lines per CTA, threads mapped g-major
// (g = tid % G, t = tid / G): one warp covers G adjacent lines (rows or columns)
// at 32/G consecutive positions, which is what the P2 layout below needs for full
// 32-byte sectors in both directions.
template <int L, int NT_ = 512>
struct Cta {
  static constexpr int T = Shape<L>::T;
  static constexpr int NT = NT_;
  static constexpr int G = NT / T;
  static constexpr int LP = Shape<L>::LP;
  static constexpr int LPB = (LP + 15) / 16 * 16;  // one buffer, 16-float2 aligned
  // per-group stride (two buffers) skewed so that the groups sharing a 16-lane
  // phase land on distinct banks
  static constexpr int SKEW = G <= 16 ? 16 / G : 1;
  static constexpr int GS = 2 * LPB + SKEW;
  static constexpr size_t XBYTES = sizeof(float2) * (size_t)GS * G;
  static constexpr size_t PRIV = sizeof(float2) * 16 * NT;  // one thread-private line
  __device__ __forceinline__ static int g() { return threadIdx.x % G; }
  __device__ __forceinline__ static int t() { return threadIdx.x / G; }
  __device__ __forceinline__ static Xch xch(float2 *sm) { return Xch{sm + (size_t)g() * GS, 0, LPB}; }
};

// P2 layout ("column-pair interleaved") of an R x L complex64 workspace array:
// element (y, x) at ((x >> 1) R + y) 2 + (x & 1).  A column pair is one contiguous
// block of 16 R bytes (column passes stream it like a row); two adjacent rows of a
// row pass fill whole 32-byte sectors.
__device__ __forceinline__ size_t p2(int y, int x, int R) { return ((size_t)(x >> 1) * R + y) * 2 + (x & 1); }

// thread-private spill slot of 16 float2 (conflict free: consecutive threads, consecutive slots)
template <int NT>
struct Priv {
  float2 *p;
  __device__ __forceinline__ float2 &operator[](int r) const { return p[r * NT + threadIdx.x]; }
};

// ---- layout-S line I/O ----------------------------------------------------------
template <int L>
__device__ __forceinline__ void ld_row(float2 (&v)[16], const float2 *__restrict__ row, int t) {
#pragma unroll
  for (int r = 0; r < 16; r++) v[r] = ldg2(row + t + r * (L / 16));
}
template <int L>
__device__ __forceinline__ void st_row(const float2 (&v)[16], float2 *__restrict__ row, int t) {
#pragma unroll
  for (int r = 0; r < 16; r++) row[t + r * (L / 16)] = v[r];
}
// column x of a row-major L x L array: element i at col[i * L]
template <int L>
__device__ __forceinline__ void ld_col(float2 (&v)[16], const float2 *__restrict__ col, int t) {
#pragma unroll
  for (int r = 0; r < 16; r++) v[r] = ldg2(col + (size_t)(t + r * (L / 16)) * L);
}
template <int L>
__device__ __forceinline__ void st_col(const float2 (&v)[16], float2 *__restrict__ col, int t) {
#pragma unroll
  for (int r = 0; r < 16; r++) col[(size_t)(t + r * (L / 16)) * L] = v[r];
}
// v *= tab (or conj(tab)) elementwise, tab indexed in layout S
template <int L, bool CONJ>
__device__ __forceinline__ void mul_tab(float2 (&v)[16], const float2 *__restrict__ tab, int t) {
#pragma unroll
  for (int r = 0; r < 16; r++) {
    const float2 w = ldg2(tab + t + r * (L / 16));
    v[r] = CONJ ? cmulc(v[r], w) : cmul(v[r], w);
  }
}

// ---- magnification ----------------------------------------------------------------
struct MagTabs {
  const float2 *cr, *wodd, *bke, *bko, *cout, *cwo;
};
__device__ __forceinline__ MagTabs mag_tabs(const Tables &tb, int L, int j, const float2 *cr) {
  return MagTabs{cr, tb.wodd, tb.bke + (size_t)j * L, tb.bko + (size_t)j * L, tb.cout + (size_t)j * L,
                 tb.cwo + (size_t)j * L};
}

// Forward M S along the line: SRC(r) returns the spectrum X at register r (layout S,
// natural frequency order); v receives the spatial result y.
template <int L, class Src>
__device__ __forceinline__ void mag_fwd(float2 (&v)[16], Src src, const MagTabs &m, Xch &x, int t,
                                        const float4 *__restrict__ tw) {
  constexpr int T = L / 16;
  float2 e[16];
#pragma unroll
  for (int r = 0; r < 16; r++) v[r ^ 8] = cmul(src(r), ldg2(m.cr + t + r * T));
  fft<L, false>(v, x, t, tw);
  mul_tab<L, false>(v, m.bke, t);
  fft<L, true>(v, x, t, tw);
#pragma unroll
  for (int r = 0; r < 16; r++) e[r] = cmul(v[r], ldg2(m.cout + t + r * T));
#pragma unroll
  for (int r = 0; r < 16; r++) v[r ^ 8] = cmul(cmul(src(r), ldg2(m.cr + t + r * T)), ldg2(m.wodd + t + (r ^ 8) * T));
  fft<L, false>(v, x, t, tw);
  mul_tab<L, false>(v, m.bko, t);
  fft<L, true>(v, x, t, tw);
#pragma unroll
  for (int r = 0; r < 16; r++) v[r] = cadd(e[r], cmul(v[r], ldg2(m.cwo + t + r * T)));
}

// Adjoint (M S)^* along the line: SRC(r) returns the spatial input y at register r;
// v receives the SPECTRUM W[f] (natural order) of the result; the caller finishes
// with an inverse FFT (possibly after summing several W).
template <int L, class Src>
__device__ __forceinline__ void mag_adj(float2 (&v)[16], Src src, const MagTabs &m, Xch &x, int t,
                                        const float4 *__restrict__ tw) {
  constexpr int T = L / 16;
  float2 e[16];
#pragma unroll
  for (int r = 0; r < 16; r++) v[r] = cmulc(src(r), ldg2(m.cout + t + r * T));
  fft<L, false>(v, x, t, tw);
  mul_tab<L, true>(v, m.bke, t);
  fft<L, true>(v, x, t, tw);
#pragma unroll
  for (int r = 0; r < 16; r++) e[r] = v[r];
#pragma unroll
  for (int r = 0; r < 16; r++) v[r] = cmulc(src(r), ldg2(m.cwo + t + r * T));
  fft<L, false>(v, x, t, tw);
  mul_tab<L, true>(v, m.bko, t);
  fft<L, true>(v, x, t, tw);
  // Z[i] = E[i] + conj(w[i]) O[i];  W[f] = conj(cr[f]) Z[(f + L/2) mod L]
#pragma unroll
  for (int r = 0; r < 16; r++) e[r] = cadd(e[r], cmulc(v[r], ldg2(m.wodd + t + r * T)));
#pragma unroll
  for (int r = 0; r < 16; r++) v[r] = cmulc(e[r ^ 8], ldg2(m.cr + t + r * T));
}

// ---- deterministic block reduction --------------------------------------------------
__device__ __forceinline__ double block_sum(double v, double *red) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[w] = v;
  __syncthreads();
  double s = 0;
  if (threadIdx.x == 0)
    for (int i = 0; i < nw; i++) s += red[i];
  return s;
}

}  // namespace holo
