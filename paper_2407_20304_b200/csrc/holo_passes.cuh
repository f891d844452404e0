// holo_passes.cuh -- the five line-pass kernels (X1, Y1, X2, Y2, X3), the
// propagation filters for q_j / g_q, reductions and the CG pointwise step.
#pragma once
#include "holo_kernels.cuh"

namespace holo {

enum { X2_GRAD = 0, X2_FWD = 1, X2_ADJ = 2, X2_OBJ = 3 };

// ----------------------------------------------------------------------------- X1
// rows of psi_k (2 rows / CTA):  X = FFT(psi row); per j: T1_j row = M_{1/mt_j} S_{sx} psi row
template <int L>
__global__ void __launch_bounds__(Cfg<L>::NT, 1) k_x1(const float2 *__restrict__ psi_k, float2 *__restrict__ T1,
                                                    Tables tb, int k, int nz, uint32_t magmask) {
  using C = Cfg<L>;
  extern __shared__ float2 sm[];
  float2 *X0 = sm, *X1 = sm + C::LPB, *A0 = sm + 2 * C::LPB, *B0 = sm + 3 * C::LPB, *A1 = sm + 4 * C::LPB,
         *B1 = sm + 5 * C::LPB;
  float2 *Xs[2] = {X0, X1}, *As[2] = {A0, A1}, *Bs[2] = {B0, B1};
  const int y0 = blockIdx.x * 2;
  load_rows<L>(Xs, psi_k, L, y0, 2, 2);
  __syncthreads();
  fft4<L, false>(X0, nullptr, X1, nullptr, tb.tw);
  for (int j = 0; j < nz; j++) {
    const float2 *rx = tb.ramps + ((size_t)(k * nz + j) * 2 + 0) * L;
    const float2 *rr[2] = {rx, rx};
    if ((magmask >> j) & 1u) {
      bl_pre_fwd<L>(Xs, As, Bs, 2, tb.cin + j * L, rr, tb.wodd);
      __syncthreads();
      fft4<L, false>(A0, B0, A1, B1, tb.tw);
      bl_mul<L, false>(As, Bs, 2, tb.bke + j * L, tb.bko + j * L);
      __syncthreads();
      fft4<L, true>(A0, B0, A1, B1, tb.tw);
      bl_post_fwd<L>(As, Bs, 2, tb.cout + j * L, tb.wodd);
    } else {
      for (int e = threadIdx.x; e < 2 * L; e += blockDim.x) {
        int l = e / L, i = e % L;
        As[l][P(i)] = cscale(cmul(Xs[l][P(i)], __ldg(rx + i)), 1.0f / L);
      }
      __syncthreads();
      fft4<L, true>(A0, nullptr, A1, nullptr, tb.tw);
    }
    __syncthreads();
    store_rows<L>(As, T1 + (size_t)j * L * L, L, y0, 2, 2, 1.0f);
    __syncthreads();
  }
}

// ----------------------------------------------------------------------------- Y1
// 4 columns / CTA of T1_j:  a = M_{1/mt_j} S_{sy} (column);  optionally store a;
// optionally  W1 = rows [o, o+N) of D_y(q_j . a)
template <int L>
__global__ void __launch_bounds__(Cfg<L>::NT, 1)
    k_y1(const float2 *__restrict__ T1j, const float2 *__restrict__ qj, float2 *__restrict__ Aout,
         float2 *__restrict__ W1, Tables tb, int k, int j, int nz, int mag, int N) {
  using C = Cfg<L>;
  extern __shared__ float2 sm[];
  float2 *Cl[4] = {sm, sm + C::LPB, sm + 2 * C::LPB, sm + 3 * C::LPB};
  float2 *S0 = sm + 4 * C::LPB, *S1 = sm + 5 * C::LPB;
  const int x0 = blockIdx.x * 4;
  load_cols4<L>(Cl, T1j, x0, 0, L, 0);
  __syncthreads();
  fft4<L, false>(Cl[0], Cl[1], Cl[2], Cl[3], tb.tw);
  const float2 *ry = tb.ramps + ((size_t)(k * nz + j) * 2 + 1) * L;
  if (mag) {
    const float2 *rr[2] = {ry, ry};
    for (int rd = 0; rd < 2; rd++) {
      float2 *Ap[2] = {Cl[2 * rd], Cl[2 * rd + 1]}, *Bp[2] = {S0, S1};
      bl_pre_fwd<L>(Ap, Ap, Bp, 2, tb.cin + j * L, rr, tb.wodd);
      __syncthreads();
      fft4<L, false>(Ap[0], S0, Ap[1], S1, tb.tw);
      bl_mul<L, false>(Ap, Bp, 2, tb.bke + j * L, tb.bko + j * L);
      __syncthreads();
      fft4<L, true>(Ap[0], S0, Ap[1], S1, tb.tw);
      bl_post_fwd<L>(Ap, Bp, 2, tb.cout + j * L, tb.wodd);
      __syncthreads();
    }
  } else {
    mul_lines<L, false>(Cl, 4, ry, 1.0f / L);
    __syncthreads();
    fft4<L, true>(Cl[0], Cl[1], Cl[2], Cl[3], tb.tw);
  }
  if (Aout) store_cols4<L>(Cl, Aout, x0, 0, L, 0, 1.0f);
  if (W1) {
    for (int e = threadIdx.x; e < 2 * L; e += blockDim.x) {
      int y = e >> 1, h = e & 1;
      float4 q = __ldg(reinterpret_cast<const float4 *>(qj + (size_t)y * L + x0 + 2 * h));
      Cl[2 * h][P(y)] = cmul(Cl[2 * h][P(y)], make_float2(q.x, q.y));
      Cl[2 * h + 1][P(y)] = cmul(Cl[2 * h + 1][P(y)], make_float2(q.z, q.w));
    }
    __syncthreads();
    fft4<L, false>(Cl[0], Cl[1], Cl[2], Cl[3], tb.tw);
    mul_lines<L, false>(Cl, 4, tb.hdet + j * L, 1.0f / L);
    __syncthreads();
    fft4<L, true>(Cl[0], Cl[1], Cl[2], Cl[3], tb.tw);
    store_cols4<L>(Cl, W1, x0, 0, N, (L - N) / 2, 1.0f);
  }
}

// ----------------------------------------------------------------------------- X2
// 4 rows / CTA.  GRAD: W1 row -> D_x, crop, residual (+F), pad, D_x^* -> V1
//                FWD : W1 row -> D_x, crop -> w frame [N][N]
//                ADJ : y frame row -> pad, D_x^* -> V1
//                OBJ : W1 row -> D_x, crop, F only
template <int L, int MODE>
__global__ void __launch_bounds__(Cfg<L>::NT, 1)
    k_x2(const float2 *__restrict__ in, const float *__restrict__ sqrt_d, float2 *__restrict__ out,
         double *__restrict__ partial, Tables tb, int j, int N) {
  using C = Cfg<L>;
  extern __shared__ float2 sm[];
  __shared__ double red[32];
  float2 *Cl[4] = {sm, sm + C::LPB, sm + 2 * C::LPB, sm + 3 * C::LPB};
  const int y0 = blockIdx.x * 4;
  const int nvalid = min(4, N - y0);
  const int o = (L - N) / 2;
  if (MODE != X2_ADJ) {
    load_rows<L>(Cl, in, L, y0, 4, nvalid);
    __syncthreads();
    fft4<L, false>(Cl[0], Cl[1], Cl[2], Cl[3], tb.tw);
    mul_lines<L, false>(Cl, 4, tb.hdet + j * L, 1.0f / L);
    __syncthreads();
    fft4<L, true>(Cl[0], Cl[1], Cl[2], Cl[3], tb.tw);
    if (MODE == X2_FWD) {
      for (int e = threadIdx.x; e < 4 * N; e += blockDim.x) {
        int l = e / N, x = e % N;
        if (l < nvalid) out[(size_t)(y0 + l) * N + x] = Cl[l][P(o + x)];
      }
      return;
    }
    double acc = 0.0;
    for (int e = threadIdx.x; e < 4 * L; e += blockDim.x) {
      int l = e / L, x = e % L;
      float2 v = make_float2(0.f, 0.f);
      if (l < nvalid && x >= o && x < o + N) {
        float2 w = Cl[l][P(x)];
        float d = __ldg(sqrt_d + (size_t)(y0 + l) * N + (x - o));
        float m = sqrtf(w.x * w.x + w.y * w.y);
        float dm = m - d;
        acc += (double)(dm * dm);
        float f = m > 0.f ? 1.0f - d / m : 0.f;  // rho = w - d w/|w|, 0 at w = 0 (C7)
        v = cscale(w, f);
      }
      Cl[l][P(x)] = v;
    }
    double s = block_sum(acc, red);
    if (threadIdx.x == 0) partial[blockIdx.x] = s;
    if (MODE == X2_OBJ) return;
  } else {
    for (int e = threadIdx.x; e < 4 * L; e += blockDim.x) {
      int l = e / L, x = e % L;
      float2 v = make_float2(0.f, 0.f);
      if (l < nvalid && x >= o && x < o + N) v = in[(size_t)(y0 + l) * N + (x - o)];
      Cl[l][P(x)] = v;
    }
  }
  __syncthreads();
  fft4<L, false>(Cl[0], Cl[1], Cl[2], Cl[3], tb.tw);
  mul_lines<L, true>(Cl, 4, tb.hdet + j * L, 1.0f / L);
  __syncthreads();
  fft4<L, true>(Cl[0], Cl[1], Cl[2], Cl[3], tb.tw);
  store_rows<L>(Cl, out, L, y0, 4, nvalid, 1.0f);
}

// ----------------------------------------------------------------------------- Y2
// 4 columns / CTA:  v = D_y^* pad(V1 col);  G_j += conj(a) v;  T3_j = (M S)_y^*(conj(q_j) v)
template <int L>
__global__ void __launch_bounds__(Cfg<L>::NT, 1)
    k_y2(const float2 *__restrict__ V1, const float2 *__restrict__ a, const float2 *__restrict__ qj,
         float2 *__restrict__ Gj, float2 *__restrict__ T3j, Tables tb, int k, int j, int nz, int mag, int N) {
  using C = Cfg<L>;
  extern __shared__ float2 sm[];
  float2 *Cl[4] = {sm, sm + C::LPB, sm + 2 * C::LPB, sm + 3 * C::LPB};
  float2 *S0 = sm + 4 * C::LPB, *S1 = sm + 5 * C::LPB;
  const int x0 = blockIdx.x * 4;
  const int o = (L - N) / 2;
  for (int e = threadIdx.x; e < 4 * (L - N); e += blockDim.x) {
    int l = e / (L - N), y = e % (L - N);
    Cl[l][P(y < o ? y : y + N)] = make_float2(0.f, 0.f);
  }
  load_cols4<L>(Cl, V1, x0, 0, N, o);
  __syncthreads();
  fft4<L, false>(Cl[0], Cl[1], Cl[2], Cl[3], tb.tw);
  mul_lines<L, true>(Cl, 4, tb.hdet + j * L, 1.0f / L);
  __syncthreads();
  fft4<L, true>(Cl[0], Cl[1], Cl[2], Cl[3], tb.tw);
  for (int e = threadIdx.x; e < 2 * L; e += blockDim.x) {
    int y = e >> 1, h = e & 1;
    size_t gi = (size_t)y * L + x0 + 2 * h;
    float2 v0 = Cl[2 * h][P(y)], v1 = Cl[2 * h + 1][P(y)];
    if (Gj) {
      float4 av = __ldg(reinterpret_cast<const float4 *>(a + gi));
      float4 g = *reinterpret_cast<float4 *>(Gj + gi);
      float2 g0 = cadd(make_float2(g.x, g.y), cmulc(v0, make_float2(av.x, av.y)));
      float2 g1 = cadd(make_float2(g.z, g.w), cmulc(v1, make_float2(av.z, av.w)));
      *reinterpret_cast<float4 *>(Gj + gi) = make_float4(g0.x, g0.y, g1.x, g1.y);
    }
    if (T3j) {
      float4 q = __ldg(reinterpret_cast<const float4 *>(qj + gi));
      Cl[2 * h][P(y)] = cmulc(v0, make_float2(q.x, q.y));
      Cl[2 * h + 1][P(y)] = cmulc(v1, make_float2(q.z, q.w));
    }
  }
  if (!T3j) return;
  __syncthreads();
  const float2 *ry = tb.ramps + ((size_t)(k * nz + j) * 2 + 1) * L;
  if (mag) {
    const float2 *rr[2] = {ry, ry};
    for (int rd = 0; rd < 2; rd++) {
      float2 *Ap[2] = {Cl[2 * rd], Cl[2 * rd + 1]}, *Bp[2] = {S0, S1};
      bl_pre_adj<L>(Ap, Bp, 2, tb.cout + j * L, tb.wodd);
      __syncthreads();
      fft4<L, false>(Ap[0], S0, Ap[1], S1, tb.tw);
      bl_mul<L, true>(Ap, Bp, 2, tb.bke + j * L, tb.bko + j * L);
      __syncthreads();
      fft4<L, true>(Ap[0], S0, Ap[1], S1, tb.tw);
      bl_post_adj<L, false>(Ap, Bp, Ap, 2, tb.cin + j * L, rr, tb.wodd);
      __syncthreads();
    }
  } else {
    fft4<L, false>(Cl[0], Cl[1], Cl[2], Cl[3], tb.tw);
    mul_lines<L, true>(Cl, 4, ry, 1.0f / L);
    __syncthreads();
  }
  fft4<L, true>(Cl[0], Cl[1], Cl[2], Cl[3], tb.tw);
  store_cols4<L>(Cl, T3j, x0, 0, L, 0, 1.0f);
}

// ----------------------------------------------------------------------------- X3
// 2 rows / CTA: g_k row = scale * IFFT( sum_j W_j ),  W_j = spectrum of (M S)_x^* T3_j row;
// partial[blk][0] = sum |g|^2, partial[blk][1] = sum Re(g conj(eta))
template <int L>
__global__ void __launch_bounds__(Cfg<L>::NT, 1)
    k_x3(const float2 *__restrict__ T3, const float2 *__restrict__ eta, float2 *__restrict__ g,
         double *__restrict__ partial, Tables tb, int k, int nz, uint32_t magmask, float scale) {
  using C = Cfg<L>;
  extern __shared__ float2 sm[];
  __shared__ double red[32];
  float2 *Q0 = sm, *Q1 = sm + C::LPB, *A0 = sm + 2 * C::LPB, *B0 = sm + 3 * C::LPB, *A1 = sm + 4 * C::LPB,
         *B1 = sm + 5 * C::LPB;
  float2 *Qs[2] = {Q0, Q1}, *As[2] = {A0, A1}, *Bs[2] = {B0, B1};
  const int y0 = blockIdx.x * 2;
  for (int j = 0; j < nz; j++) {
    load_rows<L>(As, T3 + (size_t)j * L * L, L, y0, 2, 2);
    __syncthreads();
    const float2 *rx = tb.ramps + ((size_t)(k * nz + j) * 2 + 0) * L;
    const float2 *rr[2] = {rx, rx};
    if ((magmask >> j) & 1u) {
      bl_pre_adj<L>(As, Bs, 2, tb.cout + j * L, tb.wodd);
      __syncthreads();
      fft4<L, false>(A0, B0, A1, B1, tb.tw);
      bl_mul<L, true>(As, Bs, 2, tb.bke + j * L, tb.bko + j * L);
      __syncthreads();
      fft4<L, true>(A0, B0, A1, B1, tb.tw);
      if (j == 0)
        bl_post_adj<L, false>(As, Bs, Qs, 2, tb.cin + j * L, rr, tb.wodd);
      else
        bl_post_adj<L, true>(As, Bs, Qs, 2, tb.cin + j * L, rr, tb.wodd);
    } else {
      fft4<L, false>(A0, nullptr, A1, nullptr, tb.tw);
      for (int e = threadIdx.x; e < 2 * L; e += blockDim.x) {
        int l = e / L, i = e % L;
        float2 w = cscale(cmulc(As[l][P(i)], __ldg(rx + i)), 1.0f / L);
        Qs[l][P(i)] = j == 0 ? w : cadd(Qs[l][P(i)], w);
      }
    }
    __syncthreads();
  }
  fft4<L, true>(Q0, nullptr, Q1, nullptr, tb.tw);
  double gg = 0.0, ge = 0.0;
  for (int e = threadIdx.x; e < L; e += blockDim.x) {  // pairs of elements
    int l = (2 * e) / L, i = (2 * e) % L;
    float2 a = cscale(Qs[l][P(i)], scale), b = cscale(Qs[l][P(i + 1)], scale);
    size_t gi = (size_t)(y0 + l) * L + i;
    *reinterpret_cast<float4 *>(g + gi) = make_float4(a.x, a.y, b.x, b.y);
    gg += (double)(a.x * a.x + a.y * a.y) + (double)(b.x * b.x + b.y * b.y);
    if (eta) {
      float4 ev = __ldg(reinterpret_cast<const float4 *>(eta + gi));
      ge += (double)(a.x * ev.x + a.y * ev.y) + (double)(b.x * ev.z + b.y * ev.w);
    }
  }
  double s0 = block_sum(gg, red);
  double s1 = block_sum(ge, red);
  if (threadIdx.x == 0) {
    partial[2 * blockIdx.x] = s0;
    partial[2 * blockIdx.x + 1] = s1;
  }
}

// ------------------------------------------------------------------ filters
// rows (4 / CTA): out = scale * IFFT(h^(*) FFT(in)) along x
template <int L>
__global__ void __launch_bounds__(Cfg<L>::NT, 1)
    k_rows_filter(const float2 *__restrict__ in, float2 *__restrict__ out, Tables tb, const float2 *__restrict__ h,
                  int conj, float scale) {
  using C = Cfg<L>;
  extern __shared__ float2 sm[];
  float2 *Cl[4] = {sm, sm + C::LPB, sm + 2 * C::LPB, sm + 3 * C::LPB};
  const int y0 = blockIdx.x * 4;
  load_rows<L>(Cl, in, L, y0, 4, 4);
  __syncthreads();
  fft4<L, false>(Cl[0], Cl[1], Cl[2], Cl[3], tb.tw);
  if (conj)
    mul_lines<L, true>(Cl, 4, h, scale / L);
  else
    mul_lines<L, false>(Cl, 4, h, scale / L);
  __syncthreads();
  fft4<L, true>(Cl[0], Cl[1], Cl[2], Cl[3], tb.tw);
  store_rows<L>(Cl, out, L, y0, 4, 4, 1.0f);
}

// columns (4 / CTA): out (+)= scale * IFFT(h^(*) FFT(in)) along y
template <int L>
__global__ void __launch_bounds__(Cfg<L>::NT, 1)
    k_cols_filter(const float2 *__restrict__ in, float2 *__restrict__ out, Tables tb, const float2 *__restrict__ h,
                  int conj, float scale, int accumulate) {
  using C = Cfg<L>;
  extern __shared__ float2 sm[];
  float2 *Cl[4] = {sm, sm + C::LPB, sm + 2 * C::LPB, sm + 3 * C::LPB};
  const int x0 = blockIdx.x * 4;
  load_cols4<L>(Cl, in, x0, 0, L, 0);
  __syncthreads();
  fft4<L, false>(Cl[0], Cl[1], Cl[2], Cl[3], tb.tw);
  if (conj)
    mul_lines<L, true>(Cl, 4, h, scale / L);
  else
    mul_lines<L, false>(Cl, 4, h, scale / L);
  __syncthreads();
  fft4<L, true>(Cl[0], Cl[1], Cl[2], Cl[3], tb.tw);
  if (accumulate) {
    for (int e = threadIdx.x; e < 2 * L; e += blockDim.x) {
      int y = e >> 1, hh = e & 1;
      float4 *p = reinterpret_cast<float4 *>(out + (size_t)y * L + x0 + 2 * hh);
      float4 v = *p;
      float2 a = Cl[2 * hh][P(y)], b = Cl[2 * hh + 1][P(y)];
      *p = make_float4(v.x + a.x, v.y + a.y, v.z + b.x, v.w + b.y);
    }
  } else {
    store_cols4<L>(Cl, out, x0, 0, L, 0, 1.0f);
  }
}

// ------------------------------------------------------------------ pointwise / reductions
__global__ void k_scale_add(const float2 *__restrict__ in, float2 *__restrict__ out, size_t n, float scale,
                            int accumulate) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    float2 v = cscale(in[i], scale);
    out[i] = accumulate ? cadd(out[i], v) : v;
  }
}

// deterministic single-block sum: out[v] = sum_i partial[i * nval + v], v < nval
__global__ void k_reduce(const double *__restrict__ partial, size_t n, int nval, double *__restrict__ out,
                         int accumulate) {
  __shared__ double red[32];
  for (int v = 0; v < nval; v++) {
    double s = 0.0;
    for (size_t i = threadIdx.x; i < n; i += blockDim.x) s += partial[i * nval + v];
    double t = block_sum(s, red);
    if (threadIdx.x == 0) out[v] = accumulate ? out[v] + t : t;
    __syncthreads();
  }
}

// partial dots over n complex: part[b][0] = sum |x|^2, part[b][1] = sum Re(x conj(y))
__global__ void k_dots(const float2 *__restrict__ x, const float2 *__restrict__ y, size_t n, double *__restrict__ part) {
  __shared__ double red[32];
  double a = 0.0, b = 0.0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    float2 v = x[i];
    a += (double)v.x * v.x + (double)v.y * v.y;
    if (y) {
      float2 w = y[i];
      b += (double)v.x * w.x + (double)v.y * w.y;
    }
  }
  double s0 = block_sum(a, red);
  double s1 = block_sum(b, red);
  if (threadIdx.x == 0) {
    part[2 * blockIdx.x] = s0;
    part[2 * blockIdx.x + 1] = s1;
  }
}

// CG pointwise step (Eq. (13)-(14)): mode 0: eta = -rho g; 1: eta = -rho g + beta eta; 2: keep eta.
// xt = x + gamma eta.  Two complex per thread-iteration (float4).
__global__ void k_cg(const float4 *__restrict__ x, float4 *__restrict__ eta, const float4 *__restrict__ g,
                     float4 *__restrict__ xt, size_t n4, float rho, float beta, float gamma, int mode) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
    float4 e;
    if (mode == 2) {
      e = eta[i];
    } else {
      float4 gv = g[i];
      if (mode == 0) {
        e = make_float4(-rho * gv.x, -rho * gv.y, -rho * gv.z, -rho * gv.w);
      } else {
        float4 ev = eta[i];
        e = make_float4(fmaf(beta, ev.x, -rho * gv.x), fmaf(beta, ev.y, -rho * gv.y), fmaf(beta, ev.z, -rho * gv.z),
                        fmaf(beta, ev.w, -rho * gv.w));
      }
      eta[i] = e;
    }
    float4 xv = x[i];
    xt[i] = make_float4(fmaf(gamma, e.x, xv.x), fmaf(gamma, e.y, xv.y), fmaf(gamma, e.z, xv.z),
                        fmaf(gamma, e.w, xv.w));
  }
}

}  // namespace holo
