// holo_kernels.cuh -- line-pass kernels of the holotomography sweep (sm_100a).
//
// Per frame (k, j) the operator chain of Eq. (8) and its adjoint
// (L* formula P:123) is applied as five separable line passes ("Pass
// schedule"): X = rows (contiguous), Y = columns (CTA tiles of 4 columns):
//
//   X1 (per k)   psi_k row: FFT once, then per plane j:  M_{1/mt_j} S_x   -> T1_j
//   Y1 (k, j)    T1_j col:  M_{1/mt_j} S_y -> a (stored), x q_j, D_y, crop rows -> W1
//   X2 (k, j)    W1 row:    D_x, crop, residual + F (Eq. (10)-(11)), zero-pad, D_x^* -> V1
//   Y2 (k, j)    V1 col:    pad, D_y^* -> v; G_j += conj(a) v; conj(q_j) v, (M S)_y^* -> T3_j
//   X3 (per k)   T3_j rows: (M S)_x^* accumulated over j in the Fourier domain, one
//                inverse FFT, x2 -> grad_psi_k, fused ||g||^2 and Re<g, eta> partials
//
// The magnification M_{1/mt} (reading C1) is evaluated with Bluestein's chirp-z:
// spectrum X = FFT(x); a[i] = c_in[f] r_s[f] X[f] with i = (f + L/2) mod L;
// y[o] = c_out[o] (a * b)[o] where b[d] = exp(-i pi mt d^2 / L) is convolved
// linearly through a 2L-point cyclic convolution split into even/odd halves of
// length L:  (a * b)[o] = IFFT(FFT(a) Bhat_e)[o] + e^{i pi o/L} IFFT(FFT(a w) Bhat_o)[o],
// w[i] = e^{-i pi i/L}.  All tables are fp64-generated on the host.
#pragma once
#include "fft_engine.cuh"

namespace holo {

struct Tables {
  const float2 *tw;     // FFT stage twiddles
  const float2 *hdet;   // [nz][L] h_{zdet_j}[f]
  const float2 *homega; // [nz][L] h_{omega_j}[f]
  const float2 *cin;    // [nz][L] kappa (-1)^fbar e^{i pi mt fbar^2/L} / L
  const float2 *cout;   // [nz][L] e^{i pi mt (o - L/2)^2 / L}
  const float2 *bke;    // [nz][L] Bhat[2k] / (2L)
  const float2 *bko;    // [nz][L] Bhat[2k+1] / (2L)
  const float2 *wodd;   // [L] e^{-i pi i / L}
  const float2 *ramps;  // [K][nz][2][L] r_s[f] = e^{-2 pi i fbar s / L}, axis 0: sx, 1: sy
  const float2 *href;   // [L] h_{zeta0}
};

template <int L>
struct Cfg {
  static constexpr int TPL = L / 16;
  static constexpr int G = 4;  // FFT groups per CTA
  static constexpr int NT = TPL * G;
  static constexpr int LPB = L + L / 16 + 4;  // padded line stride in smem (float2)
  static constexpr int NBUF = 6;
  static constexpr size_t SMEM = sizeof(float2) * LPB * NBUF;
};

// ---- cooperative loads / stores -----------------------------------------------
// rows: nl consecutive rows [y0, y0+nl) of a row-major array with row stride `ld`
template <int L>
__device__ __forceinline__ void load_rows(float2 *const *buf, const float2 *__restrict__ g, size_t ld, int y0, int nl,
                                          int nvalid) {
  for (int e = threadIdx.x; e < nl * L / 2; e += blockDim.x) {
    int l = (2 * e) / L, i = (2 * e) % L;
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (l < nvalid) v = __ldg(reinterpret_cast<const float4 *>(g + (size_t)(y0 + l) * ld + i));
    buf[l][P(i)] = make_float2(v.x, v.y);
    buf[l][P(i + 1)] = make_float2(v.z, v.w);
  }
}

template <int L>
__device__ __forceinline__ void store_rows(float2 *const *buf, float2 *__restrict__ g, size_t ld, int y0, int nl,
                                           int nvalid, float scale) {
  for (int e = threadIdx.x; e < nl * L / 2; e += blockDim.x) {
    int l = (2 * e) / L, i = (2 * e) % L;
    if (l < nvalid) {
      float2 a = buf[l][P(i)], b = buf[l][P(i + 1)];
      *reinterpret_cast<float4 *>(g + (size_t)(y0 + l) * ld + i) =
          make_float4(a.x * scale, a.y * scale, b.x * scale, b.y * scale);
    }
  }
}

// columns x0..x0+3 of rows [r0, r0+nr) of an array with row stride L, into line rows [d0, d0+nr)
template <int L>
__device__ __forceinline__ void load_cols4(float2 *const *buf, const float2 *__restrict__ g, int x0, int r0, int nr,
                                           int d0) {
  for (int e = threadIdx.x; e < 2 * nr; e += blockDim.x) {
    int y = e >> 1, h = e & 1;
    float4 v = __ldg(reinterpret_cast<const float4 *>(g + (size_t)(r0 + y) * L + x0 + 2 * h));
    buf[2 * h][P(d0 + y)] = make_float2(v.x, v.y);
    buf[2 * h + 1][P(d0 + y)] = make_float2(v.z, v.w);
  }
}

template <int L>
__device__ __forceinline__ void store_cols4(float2 *const *buf, float2 *__restrict__ g, int x0, int r0, int nr, int s0,
                                            float scale) {
  for (int e = threadIdx.x; e < 2 * nr; e += blockDim.x) {
    int y = e >> 1, h = e & 1;
    float2 a = buf[2 * h][P(s0 + y)], b = buf[2 * h + 1][P(s0 + y)];
    *reinterpret_cast<float4 *>(g + (size_t)(r0 + y) * L + x0 + 2 * h) =
        make_float4(a.x * scale, a.y * scale, b.x * scale, b.y * scale);
  }
}

// ---- transforms over the CTA's groups -----------------------------------------
// Each of the 4 groups transforms line s[g] (nullptr: idle).
template <int L, bool INV>
__device__ __forceinline__ void fft4(float2 *s0, float2 *s1, float2 *s2, float2 *s3, const float2 *tw) {
  const int g = threadIdx.x / Cfg<L>::TPL, t = threadIdx.x % Cfg<L>::TPL;
  float2 *s = g == 0 ? s0 : g == 1 ? s1 : g == 2 ? s2 : s3;
  fft_line<L, INV>(s ? s : s0, tw, t, s != nullptr);
}

// multiply line by table (optionally conjugated) and scale
template <int L, bool CONJ>
__device__ __forceinline__ void mul_lines(float2 *const *lines, int nl, const float2 *__restrict__ tab, float scale) {
  for (int e = threadIdx.x; e < nl * L; e += blockDim.x) {
    int l = e / L, i = e % L;
    float2 v = lines[l][P(i)], w = __ldg(tab + i);
    v = CONJ ? cmulc(v, w) : cmul(v, w);
    lines[l][P(i)] = cscale(v, scale);
  }
}

// Bluestein prologue (forward M): X holds the spectrum X[f]; writes (A may equal X)
// a[i] = cin[f] r[f] X[f] (i = f + L/2 mod L) and the odd branch b[i] = a[i] w[i].
template <int L>
__device__ __forceinline__ void bl_pre_fwd(float2 *const *X, float2 *const *A, float2 *const *B, int nl,
                                           const float2 *cin, const float2 *const *r, const float2 *wodd) {
  constexpr int H = L / 2;
  for (int e = threadIdx.x; e < nl * H; e += blockDim.x) {
    int l = e / H, f = e % H;
    float2 x0 = X[l][P(f)], x1 = X[l][P(f + H)];
    float2 a_hi = cmul(cmul(x0, __ldg(cin + f)), __ldg(r[l] + f));          // -> i = f + H
    float2 a_lo = cmul(cmul(x1, __ldg(cin + f + H)), __ldg(r[l] + f + H));  // -> i = f
    A[l][P(f)] = a_lo;
    A[l][P(f + H)] = a_hi;
    B[l][P(f)] = cmul(a_lo, __ldg(wodd + f));
    B[l][P(f + H)] = cmul(a_hi, __ldg(wodd + f + H));
  }
}

// Bluestein spectrum multiply: A *= bke, B *= bko (conjugated for the adjoint)
template <int L, bool CONJ>
__device__ __forceinline__ void bl_mul(float2 *const *A, float2 *const *B, int nl, const float2 *bke, const float2 *bko) {
  for (int e = threadIdx.x; e < nl * L; e += blockDim.x) {
    int l = e / L, k = e % L;
    float2 be = __ldg(bke + k), bo = __ldg(bko + k);
    A[l][P(k)] = CONJ ? cmulc(A[l][P(k)], be) : cmul(A[l][P(k)], be);
    B[l][P(k)] = CONJ ? cmulc(B[l][P(k)], bo) : cmul(B[l][P(k)], bo);
  }
}

// forward epilogue: out[o] = cout[o] (A[o] + conj(w[o]) B[o]), in place in A
template <int L>
__device__ __forceinline__ void bl_post_fwd(float2 *const *A, float2 *const *B, int nl, const float2 *cout,
                                            const float2 *wodd) {
  for (int e = threadIdx.x; e < nl * L; e += blockDim.x) {
    int l = e / L, o = e % L;
    float2 v = cadd(A[l][P(o)], cmulc(B[l][P(o)], __ldg(wodd + o)));
    A[l][P(o)] = cmul(v, __ldg(cout + o));
  }
}

// adjoint prologue: A[o] *= conj(cout[o]); B[o] = A[o] w[o]
template <int L>
__device__ __forceinline__ void bl_pre_adj(float2 *const *A, float2 *const *B, int nl, const float2 *cout,
                                           const float2 *wodd) {
  for (int e = threadIdx.x; e < nl * L; e += blockDim.x) {
    int l = e / L, o = e % L;
    float2 v = cmulc(A[l][P(o)], __ldg(cout + o));
    A[l][P(o)] = v;
    B[l][P(o)] = cmul(v, __ldg(wodd + o));
  }
}

// adjoint epilogue: Z[i] = A[i] + conj(w[i]) B[i];  W[f] = conj(cin[f] r[f]) Z[(f + L/2) mod L]
// written to D (may equal A); if ACC, D += W.
template <int L, bool ACC>
__device__ __forceinline__ void bl_post_adj(float2 *const *A, float2 *const *B, float2 *const *D, int nl,
                                            const float2 *cin, const float2 *const *r, const float2 *wodd) {
  constexpr int H = L / 2;
  for (int e = threadIdx.x; e < nl * H; e += blockDim.x) {
    int l = e / H, i = e % H;  // pair (i, i + H)
    float2 z_lo = cadd(A[l][P(i)], cmulc(B[l][P(i)], __ldg(wodd + i)));            // Z[i]     -> f = i + H
    float2 z_hi = cadd(A[l][P(i + H)], cmulc(B[l][P(i + H)], __ldg(wodd + i + H)));  // Z[i + H] -> f = i
    float2 c_lo = cmul(__ldg(cin + i), __ldg(r[l] + i));
    float2 c_hi = cmul(__ldg(cin + i + H), __ldg(r[l] + i + H));
    float2 w_f_lo = cmulc(z_hi, c_lo);  // f = i
    float2 w_f_hi = cmulc(z_lo, c_hi);  // f = i + H
    if (ACC) {
      w_f_lo = cadd(w_f_lo, D[l][P(i)]);
      w_f_hi = cadd(w_f_hi, D[l][P(i + H)]);
    }
    D[l][P(i)] = w_f_lo;
    D[l][P(i + H)] = w_f_hi;
  }
}

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
