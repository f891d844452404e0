// holo_ref.cuh -- the reference arm (O14; reference constraint P:102, reference terms
// of Eq. (10) P:115 and Eq. (12)): probe-only frames
//
//   w^r_r = C( P_{zeta_0} S_{s_r} q ),   F_ref = sum_r || |w^r_r| - sqrt_dref_r ||^2,
//   grad_q += 2 sum_r S_{-s_r} P_{-zeta_0} Z rho^r_r,   rho as O9.
//
// Both operators are Fourier multipliers, so q is transformed ONCE per sweep
// (Qhat = DFT2 q) and every frame is: multiply by H_y H_x (H = h_{zeta0} r_s / L per
// axis), inverse along y (keep the N data rows), inverse along x, crop, residual,
// zero-pad, forward along x, multiply by conj(H_x), forward along y, multiply by
// conj(H_y), accumulate in the Fourier domain (Ghat).  One inverse DFT2 of Ghat per
// sweep yields the gradient.  Three line passes per frame (R1 columns, R2 rows,
// R3 columns), all arrays in the P2 layout.
//
// Line engines: power-of-two tori use the register-resident Stockham engine
// (layout S in both domains).  N_p = 6144 = 3 * 2048 (configs[4], reading C16) uses
// LineEng<6144>: three interleaved 2048-point sub-transforms of the decimated
// sequences x[3n + s] (128 threads each) and one radix-3 combine through shared memory:
//   spatial  register r of thread (g3, t)  <->  element 3 (t + 128 r) + g3
//   spectral register r of thread (g3, t)  <->  element t + 128 r + 2048 g3
//   X[k + 2048 m] = sum_s W_3^{s m} W_6144^{s k} FFT_2048(x[3 . + s])[k].
#pragma once
#include "holo_kernels.cuh"

namespace holo {

template <int L>
struct LineEng {  // power of two: the Stockham engine, G lines per 512-thread CTA
  using C = Cta<L, 512>;
  static constexpr int NT = 512, G = C::G, T = L / 16;
  static constexpr size_t SMEM = C::XBYTES;
  struct St {
    Xch x;
    int t, g;
  };
  __device__ __forceinline__ static St init(float2 *sm) { return St{C::xch(sm), C::t(), C::g()}; }
  __device__ __forceinline__ static int isp(const St &s, int r) { return s.t + r * T; }
  __device__ __forceinline__ static int ifr(const St &s, int r) { return s.t + r * T; }
  __device__ __forceinline__ static void fwd(float2 (&v)[16], St &s, const float4 *tw, const float2 *) {
    fft<L, false>(v, s.x, s.t, tw);
  }
  __device__ __forceinline__ static void inv(float2 (&v)[16], St &s, const float4 *tw, const float2 *) {
    fft<L, true>(v, s.x, s.t, tw);
  }
};

template <>
struct LineEng<6144> {
  static constexpr int L = 6144, LS = 2048, NT = 384, G = 1, T = 128;
  using CS = Cta<LS, 128>;  // one 2048-point sub-line per 128 threads
  static constexpr int GS = CS::GS;
  static constexpr size_t SMEM = sizeof(float2) * (size_t)GS * 3;
  static_assert(3 * GS >= 3 * LS, "radix-3 buffer must fit in the exchange space");
  struct St {
    Xch x;
    int t, g, g3;
    float2 *buf;
  };
  __device__ __forceinline__ static St init(float2 *sm) {
    const int g3 = threadIdx.x / 128, t = threadIdx.x % 128;
    return St{Xch{sm + (size_t)g3 * GS, 0, CS::LPB, g3}, t, 0, g3, sm};  // sub-line g3 = warps 4 g3 .. 4 g3 + 3
  }
  __device__ __forceinline__ static int isp(const St &s, int r) { return 3 * (s.t + r * T) + s.g3; }
  __device__ __forceinline__ static int ifr(const St &s, int r) { return s.t + r * T + LS * s.g3; }
  // radix-3 buffer slot of element k of sub-sequence m (padded like the engine)
  __device__ __forceinline__ static int B(int m, int k) { return m * GS + P(k); }
  // tw3[(g3 - 1) * 2048 + k] = W_6144^{g3 k} = e^{-2 pi i g3 k / 6144}, g3 = 1, 2
  __device__ __forceinline__ static void fwd(float2 (&v)[16], St &s, const float4 *tw, const float2 *tw3) {
    fft<LS, false>(v, s.x, s.t, tw);
    if (s.g3) {
#pragma unroll
      for (int r = 0; r < 16; r++) v[r] = cmul(v[r], ldg2(tw3 + (s.g3 - 1) * LS + s.t + r * T));
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < 16; r++) s.buf[B(s.g3, s.t + r * T)] = v[r];
    __syncthreads();
    constexpr float C3 = -0.5f, S3 = 0.86602540378443864676f;  // W_3 = e^{-2 pi i / 3} = C3 - i S3
#pragma unroll
    for (int r = 0; r < 16; r++) {
      const int k = s.t + r * T;
      const float2 y0 = s.buf[B(0, k)], y1 = s.buf[B(1, k)], y2 = s.buf[B(2, k)];
      const float2 a = cadd(y1, y2), d = csub(y1, y2);
      const float2 base = make_float2(y0.x + C3 * a.x, y0.y + C3 * a.y);
      const float2 rot = make_float2(S3 * d.y, -S3 * d.x);  // -i S3 (y1 - y2)
      v[r] = s.g3 == 0 ? cadd(y0, a) : (s.g3 == 1 ? cadd(base, rot) : csub(base, rot));
    }
  }
  __device__ __forceinline__ static void inv(float2 (&v)[16], St &s, const float4 *tw, const float2 *tw3) {
    __syncthreads();
#pragma unroll
    for (int r = 0; r < 16; r++) s.buf[B(s.g3, s.t + r * T)] = v[r];
    __syncthreads();
    constexpr float C3 = -0.5f, S3 = 0.86602540378443864676f;  // conj(W_3) = C3 + i S3
#pragma unroll
    for (int r = 0; r < 16; r++) {
      const int k = s.t + r * T;
      const float2 x0 = s.buf[B(0, k)], x1 = s.buf[B(1, k)], x2 = s.buf[B(2, k)];
      const float2 a = cadd(x1, x2), d = csub(x1, x2);
      const float2 base = make_float2(x0.x + C3 * a.x, x0.y + C3 * a.y);
      const float2 rot = make_float2(-S3 * d.y, S3 * d.x);  // +i S3 (x1 - x2)
      float2 y = s.g3 == 0 ? cadd(x0, a) : (s.g3 == 1 ? cadd(base, rot) : csub(base, rot));
      if (s.g3) y = cmulc(y, ldg2(tw3 + (s.g3 - 1) * LS + k));
      v[r] = y;
    }
    fft<LS, true>(v, s.x, s.t, tw);
  }
};

enum { REF_QHAT = 0, REF_R1 = 1, REF_R2 = 2, REF_R3 = 3, REF_FINAL = 4, REF_FWD = 5, REF_INIT = 6 };

// ---------------------------------------------------------------- column passes
// QHAT : Qx (P2, spectral x / spatial y) -> forward along y -> Qhat (P2), in place
// R1   : v = Qhat col x Hy -> inverse along y -> rows [o, o+N) -> W (P2, N rows)
// R3   : v = pad(V col) -> forward along y -> x conj(Hy) -> Ghat (+)= v (P2)
// FINAL: Ghat col -> inverse along y -> Ghat (P2, spatial y), in place
template <int L, int MODE>
__global__ void __launch_bounds__(LineEng<L>::NT, 1)
    k_ref_cols(const float2 *__restrict__ in, float2 *__restrict__ out, const float2 *__restrict__ Hy,
               const float4 *__restrict__ tw, const float2 *__restrict__ tw3, int N, int first) {
  using E = LineEng<L>;
  extern __shared__ float4 sm4[];
  typename E::St st = E::init(reinterpret_cast<float2 *>(sm4));
  const int col = blockIdx.x * E::G + st.g;
  const int o = (L - N) / 2;
  float2 v[16];
  if (MODE == REF_QHAT) {
#pragma unroll
    for (int r = 0; r < 16; r++) v[r] = ldg2(in + p2(E::isp(st, r), col, L));
    E::fwd(v, st, tw, tw3);
#pragma unroll
    for (int r = 0; r < 16; r++) out[p2(E::ifr(st, r), col, L)] = v[r];
  } else if (MODE == REF_R1) {
#pragma unroll
    for (int r = 0; r < 16; r++) {
      const int f = E::ifr(st, r);
      v[r] = cmul(ldg2(in + p2(f, col, L)), ldg2(Hy + f));
    }
    E::inv(v, st, tw, tw3);
#pragma unroll
    for (int r = 0; r < 16; r++) {
      const int row = E::isp(st, r) - o;
      if (row >= 0 && row < N) out[p2(row, col, N)] = v[r];
    }
  } else if (MODE == REF_R3) {
#pragma unroll
    for (int r = 0; r < 16; r++) {
      const int row = E::isp(st, r) - o;
      v[r] = (row >= 0 && row < N) ? ldg2(in + p2(row, col, N)) : make_float2(0.f, 0.f);
    }
    E::fwd(v, st, tw, tw3);
#pragma unroll
    for (int r = 0; r < 16; r++) {
      const int f = E::ifr(st, r);
      const float2 a = cmulc(v[r], ldg2(Hy + f));
      float2 *p = out + p2(f, col, L);
      *p = first ? a : cadd(*p, a);
    }
  } else {  // FINAL
#pragma unroll
    for (int r = 0; r < 16; r++) v[r] = in[p2(E::ifr(st, r), col, L)];
    E::inv(v, st, tw, tw3);
#pragma unroll
    for (int r = 0; r < 16; r++) out[p2(E::isp(st, r), col, L)] = v[r];
  }
}

// ---------------------------------------------------------------- batched column passes
// B_r reference frames per launch; frame b's tables at Href + 2 L b (x row, then y row).
// R1B: the Qhat column is read ONCE; per frame: x Hy_b, inverse along y, rows [o, o+N) -> W_b
template <int L>
__global__ void __launch_bounds__(LineEng<L>::NT, 1)
    k_ref_r1b(const float2 *__restrict__ Qhat, float2 *__restrict__ W, const float2 *__restrict__ Href, int nb,
              const float4 *__restrict__ tw, const float2 *__restrict__ tw3, int N) {
  using E = LineEng<L>;
  extern __shared__ float4 sm4[];
  typename E::St st = E::init(reinterpret_cast<float2 *>(sm4));
  const int col = blockIdx.x * E::G + st.g;
  const int o = (L - N) / 2;
  float2 q0[16];
#pragma unroll
  for (int r = 0; r < 16; r++) q0[r] = ldg2(Qhat + p2(E::ifr(st, r), col, L));
#pragma unroll 1
  for (int b = 0; b < nb; b++) {
    const float2 *Hy = Href + (size_t)b * 2 * L + L;
    float2 v[16];
#pragma unroll
    for (int r = 0; r < 16; r++) v[r] = cmul(q0[r], ldg2(Hy + E::ifr(st, r)));
    E::inv(v, st, tw, tw3);
    float2 *w = W + (size_t)b * N * L;
#pragma unroll
    for (int r = 0; r < 16; r++) {
      const int row = E::isp(st, r) - o;
      if (row >= 0 && row < N) w[p2(row, col, N)] = v[r];
    }
  }
}

// R3B: per frame: pad(V_b col) -> forward along y -> x conj(Hy_b), summed over the batch in
// registers; Ghat (+)= the sum: one read-modify-write of Ghat per batch instead of per frame
template <int L>
__global__ void __launch_bounds__(LineEng<L>::NT, 1)
    k_ref_r3b(const float2 *__restrict__ V, float2 *__restrict__ Ghat, const float2 *__restrict__ Href, int nb,
              const float4 *__restrict__ tw, const float2 *__restrict__ tw3, int N, int first) {
  using E = LineEng<L>;
  extern __shared__ float4 sm4[];
  typename E::St st = E::init(reinterpret_cast<float2 *>(sm4));
  const int col = blockIdx.x * E::G + st.g;
  const int o = (L - N) / 2;
  float2 acc[16];
#pragma unroll
  for (int r = 0; r < 16; r++) acc[r] = make_float2(0.f, 0.f);
#pragma unroll 1
  for (int b = 0; b < nb; b++) {
    const float2 *vin = V + (size_t)b * N * L;
    const float2 *Hy = Href + (size_t)b * 2 * L + L;
    float2 v[16];
#pragma unroll
    for (int r = 0; r < 16; r++) {
      const int row = E::isp(st, r) - o;
      v[r] = (row >= 0 && row < N) ? ldg2(vin + p2(row, col, N)) : make_float2(0.f, 0.f);
    }
    E::fwd(v, st, tw, tw3);
#pragma unroll
    for (int r = 0; r < 16; r++) acc[r] = cadd(acc[r], cmulc(v[r], ldg2(Hy + E::ifr(st, r))));
  }
#pragma unroll
  for (int r = 0; r < 16; r++) {
    float2 *p = Ghat + p2(E::ifr(st, r), col, L);
    *p = first ? acc[r] : cadd(*p, acc[r]);
  }
}

// ---------------------------------------------------------------- row passes
// QHAT : q row (row-major) -> forward along x -> Qx (P2)
// R2   : W row (P2, N rows) x Hx -> inverse along x -> crop, residual (+F), pad ->
//        forward along x -> x conj(Hx) -> V (P2, N rows); partial[blk] = F of the CTA
// FINAL: Ghat row (P2) -> inverse along x -> out (row-major) (+)= scale v
// FWD  : W row (P2, N rows) x Hx -> inverse along x -> crop -> w frame (row-major N x N)
// INIT : (a - mean) row (partial = &mean, fp64), zero-padded -> forward along x -> x conj(Hx) -> V
template <int L, int MODE>
__global__ void __launch_bounds__(LineEng<L>::NT, 1)
    k_ref_rows(const float2 *__restrict__ in, const float *__restrict__ sqrt_d, float2 *__restrict__ out,
               double *__restrict__ partial, const float2 *__restrict__ Hx, const float4 *__restrict__ tw,
               const float2 *__restrict__ tw3, int N, float scale, int accumulate, float tau = 1.f) {
  using E = LineEng<L>;
  extern __shared__ float4 sm4[];
  __shared__ double red[32];
  typename E::St st = E::init(reinterpret_cast<float2 *>(sm4));
  const int y = blockIdx.x * E::G + st.g;
  const int o = (L - N) / 2;
  if (MODE == REF_R2 || MODE == REF_FWD || MODE == REF_INIT) {  // frame blockIdx.y of a batch
    const size_t fb = blockIdx.y;
    if (in) in += fb * N * L;
    sqrt_d += fb * N * N;
    out += fb * (MODE == REF_FWD ? (size_t)N * N : (size_t)N * L);
    if (partial) partial += MODE == REF_INIT ? fb : fb * gridDim.x;
    Hx += fb * 2 * L;
  }
  float2 v[16];
  if (MODE == REF_QHAT) {
#pragma unroll
    for (int r = 0; r < 16; r++) v[r] = ldg2(in + (size_t)y * L + E::isp(st, r));
    E::fwd(v, st, tw, tw3);
#pragma unroll
    for (int r = 0; r < 16; r++) out[p2(y, E::ifr(st, r), L)] = v[r];
  } else if (MODE == REF_R2) {
    const bool act = y < N;
#pragma unroll
    for (int r = 0; r < 16; r++) {
      const int f = E::ifr(st, r);
      v[r] = act ? cmul(ldg2(in + p2(y, f, N)), ldg2(Hx + f)) : make_float2(0.f, 0.f);
    }
    E::inv(v, st, tw, tw3);
    double acc = 0.0;
#pragma unroll
    for (int r = 0; r < 16; r++) {
      const int c = E::isp(st, r) - o;
      float2 w = make_float2(0.f, 0.f);
      if (act && c >= 0 && c < N) {
        w = residual_tau(v[r], __ldg(sqrt_d + (size_t)y * N + c), tau, acc);  // G_tau, App. A.3
      }
      v[r] = w;
    }
    const double s = block_sum(acc, red);
    if (threadIdx.x == 0) partial[blockIdx.x] = s;
    E::fwd(v, st, tw, tw3);
    if (act) {
#pragma unroll
      for (int r = 0; r < 16; r++) {
        const int f = E::ifr(st, r);
        out[p2(y, f, N)] = cmulc(v[r], ldg2(Hx + f));
      }
    }
  } else if (MODE == REF_INIT) {
    // O17 (initial probe): the frame's amplitude minus its mean c (partial[0], fp64), zero-padded,
    // forward along x, x conj(Hx) -> V (P2, N rows); R3 + FINAL then give S_{-s} P_{-zeta0} Z (a - c)
    const bool act = y < N;
    const float c = (float)partial[0];
#pragma unroll
    for (int r = 0; r < 16; r++) {
      const int cc = E::isp(st, r) - o;
      v[r] = make_float2((act && cc >= 0 && cc < N) ? __ldg(sqrt_d + (size_t)y * N + cc) - c : 0.f, 0.f);
    }
    E::fwd(v, st, tw, tw3);
    if (act) {
#pragma unroll
      for (int r = 0; r < 16; r++) {
        const int f = E::ifr(st, r);
        out[p2(y, f, N)] = cmulc(v[r], ldg2(Hx + f));
      }
    }
  } else if (MODE == REF_FWD) {
    const bool act = y < N;
#pragma unroll
    for (int r = 0; r < 16; r++) {
      const int f = E::ifr(st, r);
      v[r] = act ? cmul(ldg2(in + p2(y, f, N)), ldg2(Hx + f)) : make_float2(0.f, 0.f);
    }
    E::inv(v, st, tw, tw3);
    if (act) {
#pragma unroll
      for (int r = 0; r < 16; r++) {
        const int c = E::isp(st, r) - o;
        if (c >= 0 && c < N) out[(size_t)y * N + c] = v[r];
      }
    }
  } else {  // FINAL
#pragma unroll
    for (int r = 0; r < 16; r++) v[r] = in[p2(y, E::ifr(st, r), L)];
    E::inv(v, st, tw, tw3);
#pragma unroll
    for (int r = 0; r < 16; r++) {
      float2 *p = out + (size_t)y * L + E::isp(st, r);
      const float2 a = cscale(v[r], scale);
      *p = accumulate ? cadd(*p, a) : a;
    }
  }
}

}  // namespace holo
