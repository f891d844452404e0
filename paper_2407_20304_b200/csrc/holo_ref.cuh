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
// LineEng<6144>: each thread runs the three 2048-point sub-transforms of the decimated
// sequences x[3n + s] in lockstep and combines them with a radix-3 step in registers:
//   X[k + 2048 m] = sum_s W_3^{s m} W_6144^{s k} FFT_2048(x[3 . + s])[k].
#pragma once
#include "holo_kernels.cuh"

namespace holo {

template <int L>
struct LineEng {  // power of two: the Stockham engine, G lines per 512-thread CTA
  using C = Cta<L, 512>;
  static constexpr int NT = 512, G = C::G, T = L / 16, R = 16, MINB = 1, MINB_ACC = 1;
  static constexpr bool HOLD_SMEM = false;  // R1B / R3B keep their second line in registers
  static constexpr int FS = R + T;          // ramp factors per frame and axis (A[R], B[T])
  static constexpr size_t SMEM = C::XBYTES, SMEM_ACC = SMEM;
  struct St {
    Xch x;
    int t, g;
  };
  __device__ __forceinline__ static St init(float2 *sm) { return St{C::xch(sm), C::t(), C::g()}; }
  __device__ __forceinline__ static int isp(const St &s, int r) { return s.t + r * T; }
  __device__ __forceinline__ static int ifr(const St &s, int r) { return s.t + r * T; }
  __device__ __forceinline__ static void fwd(float2 (&v)[R], St &s, const float4 *tw, const float2 *) {
    fft<L, false>(v, s.x, s.t, tw);
  }
  __device__ __forceinline__ static void inv(float2 (&v)[R], St &s, const float4 *tw, const float2 *) {
    fft<L, true>(v, s.x, s.t, tw);
  }
};

// N_p = 6144 = 3 x 2048 (configs[4]): ONE line per 128-thread CTA, each thread holding the three
// decimated sub-lines x[3 n + s] (s = 0, 1, 2) of 2048 points in layout S (48 values, v[16 s + r]):
//   spatial  value (s, r) of thread t  <->  element 3 (t + 128 r) + s   (a thread's three values are
//            adjacent: 24 contiguous bytes, a warp covers 768 contiguous bytes per r)
//   spectral value (m, r) of thread t  <->  element t + 128 r + 2048 m
// The three 2048-point sub-transforms run in lockstep (fft_nv: one barrier pair per exchange for
// all three) and the radix-3 combine X[k + 2048 m] = sum_s W_3^{s m} W_6144^{s k} Y_s[k] is done in
// registers (no third exchange).  Several CTAs per SM, so one CTA's exchange overlaps another's
// butterflies.
#ifndef HOLO_REF_MINB
#define HOLO_REF_MINB 3
#endif
template <>
struct LineEng<6144> {
  static constexpr int L = 6144, LS = 2048, NT = 128, G = 1, T = 128, R = 48;
  static constexpr int MINB = HOLO_REF_MINB;  // CTAs per SM of the plain passes (3: <= 170 registers)
  static constexpr int MINB_ACC = 2;  // R1B / R3B keep a second 48-value line (Qhat column / Ghat sum)
  static constexpr int BS = Shape<LS>::LP;  // one sub-line's exchange buffer (float2)
  static constexpr size_t SMEM = sizeof(float2) * (size_t)BS * 3;
  // R1B / R3B: the second line (Qhat column / batch sum) in a thread-private shared-memory slot
  // behind the exchange buffers (value i of thread t at SMEM + 8 (i NT + t): conflict free)
  static constexpr bool HOLD_SMEM = true;
  static constexpr int FS = R + T;  // ramp factors per frame and axis (A[R], B[T])
  static constexpr size_t SMEM_ACC = SMEM + sizeof(float2) * (size_t)R * NT;
  struct St {
    float2 *buf;
    int t, g;
  };
  __device__ __forceinline__ static St init(float2 *sm) { return St{sm, (int)threadIdx.x, 0}; }
  __device__ __forceinline__ static int isp(const St &s, int i) { return 3 * (s.t + (i & 15) * T) + (i >> 4); }
  __device__ __forceinline__ static int ifr(const St &s, int i) { return s.t + (i & 15) * T + LS * (i >> 4); }
  // tw3[(s - 1) * 2048 + k] = W_6144^{s k} = e^{-2 pi i s k / 6144}, s = 1, 2
  __device__ __forceinline__ static void fwd(float2 (&v)[R], St &s, const float4 *tw, const float2 *tw3) {
    fft_nv<LS, false, 3>(v, s.buf, BS, s.t, tw);
    constexpr float C3 = -0.5f, S3 = 0.86602540378443864676f;  // W_3 = e^{-2 pi i / 3} = C3 - i S3
#pragma unroll
    for (int r = 0; r < 16; r++) {
      const int k = s.t + r * T;
      const float2 y0 = v[r], y1 = cmul(v[16 + r], ldg2(tw3 + k)), y2 = cmul(v[32 + r], ldg2(tw3 + LS + k));
      const float2 a = cadd(y1, y2), d = csub(y1, y2);
      const float2 base = make_float2(fmaf(C3, a.x, y0.x), fmaf(C3, a.y, y0.y));
      const float2 rot = make_float2(S3 * d.y, -S3 * d.x);  // -i S3 (y1 - y2)
      v[r] = cadd(y0, a);
      v[16 + r] = cadd(base, rot);
      v[32 + r] = csub(base, rot);
    }
  }
  __device__ __forceinline__ static void inv(float2 (&v)[R], St &s, const float4 *tw, const float2 *tw3) {
    constexpr float C3 = -0.5f, S3 = 0.86602540378443864676f;  // conj(W_3) = C3 + i S3
#pragma unroll
    for (int r = 0; r < 16; r++) {
      const int k = s.t + r * T;
      const float2 x0 = v[r], x1 = v[16 + r], x2 = v[32 + r];
      const float2 a = cadd(x1, x2), d = csub(x1, x2);
      const float2 base = make_float2(fmaf(C3, a.x, x0.x), fmaf(C3, a.y, x0.y));
      const float2 rot = make_float2(-S3 * d.y, S3 * d.x);  // +i S3 (x1 - x2)
      v[r] = cadd(x0, a);
      v[16 + r] = cmulc(cadd(base, rot), ldg2(tw3 + k));
      v[32 + r] = cmulc(csub(base, rot), ldg2(tw3 + LS + k));
    }
    fft_nv<LS, true, 3>(v, s.buf, BS, s.t, tw);
  }
};

enum { REF_QHAT = 0, REF_R1 = 1, REF_R2 = 2, REF_R3 = 3, REF_FINAL = 4, REF_FWD = 5, REF_INIT = 6 };

// ---------------------------------------------------------------- column passes
// QHAT : Qx (P2, spectral x / spatial y) -> forward along y -> Qhat (P2), in place
// R1   : v = Qhat col x Hy -> inverse along y -> rows [o, o+N) -> W (P2, N rows)
// R3   : v = pad(V col) -> forward along y -> x conj(Hy) -> Ghat (+)= v (P2)
// FINAL: Ghat col -> inverse along y -> Ghat (P2, spatial y), in place
template <int L, int MODE>
__global__ void __launch_bounds__(LineEng<L>::NT, LineEng<L>::MINB)
    k_ref_cols(const float2 *__restrict__ in, float2 *__restrict__ out, const float2 *__restrict__ Hy,
               const float4 *__restrict__ tw, const float2 *__restrict__ tw3, int N, int first) {
  using E = LineEng<L>;
  extern __shared__ float4 sm4[];
  typename E::St st = E::init(reinterpret_cast<float2 *>(sm4));
  const int col = blockIdx.x * E::G + st.g;
  const int o = (L - N) / 2;
  float2 v[E::R];
  if (MODE == REF_QHAT) {
#pragma unroll
    for (int r = 0; r < E::R; r++) v[r] = ldg2(in + p2(E::isp(st, r), col, L));
    E::fwd(v, st, tw, tw3);
#pragma unroll
    for (int r = 0; r < E::R; r++) out[p2(E::ifr(st, r), col, L)] = v[r];
  } else if (MODE == REF_R1) {
#pragma unroll
    for (int r = 0; r < E::R; r++) {
      const int f = E::ifr(st, r);
      v[r] = cmul(ldg2(in + p2(f, col, L)), ldg2(Hy + f));
    }
    E::inv(v, st, tw, tw3);
#pragma unroll
    for (int r = 0; r < E::R; r++) {
      const int row = E::isp(st, r) - o;
      if (row >= 0 && row < N) out[p2(row, col, N)] = v[r];
    }
  } else if (MODE == REF_R3) {
#pragma unroll
    for (int r = 0; r < E::R; r++) {
      const int row = E::isp(st, r) - o;
      v[r] = (row >= 0 && row < N) ? ldg2(in + p2(row, col, N)) : make_float2(0.f, 0.f);
    }
    E::fwd(v, st, tw, tw3);
#pragma unroll
    for (int r = 0; r < E::R; r++) {
      const int f = E::ifr(st, r);
      const float2 a = cmulc(v[r], ldg2(Hy + f));
      float2 *p = out + p2(f, col, L);
      *p = first ? a : cadd(*p, a);
    }
  } else {  // FINAL
#pragma unroll
    for (int r = 0; r < E::R; r++) v[r] = in[p2(E::ifr(st, r), col, L)];
    E::inv(v, st, tw, tw3);
#pragma unroll
    for (int r = 0; r < E::R; r++) out[p2(E::isp(st, r), col, L)] = v[r];
  }
}

// ---------------------------------------------------------------- batched column passes
// B_r reference frames per launch; frame b's tables at Href + 2 L b (x row, then y row).
// The frame tables factor as H_b[f] = h[f] / L x r_{s_b}[f] (hz = h_{zeta0} / L, common to all frames)
// and the ramp as r_s[f] = A[i] B[t] over the engine layout f = ifr(t, i) (fac: per frame and axis
// FS = R + T values, ref_factors on the host), so a frame costs one table value per thread plus
// R warp-uniform (L1 broadcast) values instead of a length-L table.
// R1B: the Qhat column x hz is read ONCE; per frame: x ramp_b, inverse along y, rows [o, o+N) -> W_b
#ifndef HOLO_R1B_REREAD
#define HOLO_R1B_REREAD 1  // re-read the Qhat column (L2) every frame instead of holding it: 3 CTAs / SM (measured +7 %)
#endif
template <int L, bool RR = (HOLO_R1B_REREAD && LineEng<L>::HOLD_SMEM)>
__global__ void __launch_bounds__(LineEng<L>::NT, RR ? LineEng<L>::MINB : LineEng<L>::MINB_ACC)
    k_ref_r1b(const float2 *__restrict__ Qhat, float2 *__restrict__ W, const float2 *__restrict__ hz,
              const float2 *__restrict__ fac, int nb, const float4 *__restrict__ tw, const float2 *__restrict__ tw3,
              int N) {
  using E = LineEng<L>;
  extern __shared__ float4 sm4[];
  typename E::St st = E::init(reinterpret_cast<float2 *>(sm4));
  const int col = blockIdx.x * E::G + st.g;
  const int o = (L - N) / 2;
  float2 q0[E::HOLD_SMEM ? 1 : E::R];
  float2 *hold = reinterpret_cast<float2 *>(reinterpret_cast<char *>(sm4) + E::SMEM) + threadIdx.x;
  if constexpr (!RR) {
#pragma unroll
    for (int r = 0; r < E::R; r++) {  // the frame-independent part Qhat h_{zeta0} / L of the column
      const int f = E::ifr(st, r);
      const float2 a = cmul(ldg2(Qhat + p2(f, col, L)), ldg2(hz + f));
      if constexpr (E::HOLD_SMEM) hold[r * E::NT] = a; else q0[r] = a;
    }
  }
#pragma unroll 1
  for (int b = 0; b < nb; b++) {
    const float2 *A = fac + (size_t)(2 * b + 1) * E::FS;  // y-axis ramp factors of frame b
    const float2 Bt = ldg2(A + E::R + st.t);
    float2 v[E::R];
#pragma unroll
    for (int r = 0; r < E::R; r++) {
      float2 qh;
      if constexpr (RR) {
        const int f = E::ifr(st, r);
        qh = cmul(ldg2(Qhat + p2(f, col, L)), ldg2(hz + f));
      } else {
        qh = E::HOLD_SMEM ? hold[r * E::NT] : q0[r];
      }
      v[r] = cmul(qh, cmul(ldg2(A + r), Bt));
    }
    E::inv(v, st, tw, tw3);
    float2 *w = W + (size_t)b * N * L;
#pragma unroll
    for (int r = 0; r < E::R; r++) {
      const int row = E::isp(st, r) - o;
      if (row >= 0 && row < N) w[p2(row, col, N)] = v[r];
    }
  }
}

// R3B: per frame: pad(V_b col) -> forward along y -> x conj(ramp_b), summed over the batch (registers
// or the private smem slot), x conj(hz); Ghat (+)= the sum: one read-modify-write of Ghat per batch
#ifndef HOLO_R3B_RED
#define HOLO_R3B_RED 0  // 1: every frame adds into Ghat with fire-and-forget L2 reductions (no held sum; measured -10 %)
#endif
template <int L, bool RD = (HOLO_R3B_RED && LineEng<L>::HOLD_SMEM)>
__global__ void __launch_bounds__(LineEng<L>::NT, RD ? LineEng<L>::MINB : LineEng<L>::MINB_ACC)
    k_ref_r3b(const float2 *__restrict__ V, float2 *__restrict__ Ghat, const float2 *__restrict__ hz,
              const float2 *__restrict__ fac, int nb, const float4 *__restrict__ tw, const float2 *__restrict__ tw3,
              int N, int first) {
  using E = LineEng<L>;
  extern __shared__ float4 sm4[];
  typename E::St st = E::init(reinterpret_cast<float2 *>(sm4));
  const int col = blockIdx.x * E::G + st.g;
  const int o = (L - N) / 2;
  if constexpr (RD) {  // one owner thread per Ghat element: the same sequential sum, no held batch sum
#pragma unroll 1
    for (int b = 0; b < nb; b++) {
      const float2 *vin = V + (size_t)b * N * L;
      const float2 *A = fac + (size_t)(2 * b + 1) * E::FS;
      const float2 Bt = ldg2(A + E::R + st.t);
      float2 v[E::R];
#pragma unroll
      for (int r = 0; r < E::R; r++) {
        const int row = E::isp(st, r) - o;
        v[r] = (row >= 0 && row < N) ? ldg2(vin + p2(row, col, N)) : make_float2(0.f, 0.f);
      }
      E::fwd(v, st, tw, tw3);
#pragma unroll
      for (int r = 0; r < E::R; r++) {
        const int f = E::ifr(st, r);
        const float2 a = cmulc(cmulc(v[r], cmul(ldg2(A + r), Bt)), ldg2(hz + f));
        float2 *p = Ghat + p2(f, col, L);
        if (first && b == 0) *p = a; else red_add2(p, a);
      }
    }
    return;
  }
  float2 acc[E::HOLD_SMEM ? 1 : E::R];
  float2 *hold = reinterpret_cast<float2 *>(reinterpret_cast<char *>(sm4) + E::SMEM) + threadIdx.x;
#pragma unroll
  for (int r = 0; r < E::R; r++) {
    if constexpr (E::HOLD_SMEM) hold[r * E::NT] = make_float2(0.f, 0.f); else acc[r] = make_float2(0.f, 0.f);
  }
#pragma unroll 1
  for (int b = 0; b < nb; b++) {
    const float2 *vin = V + (size_t)b * N * L;
    const float2 *A = fac + (size_t)(2 * b + 1) * E::FS;
    const float2 Bt = ldg2(A + E::R + st.t);
    float2 v[E::R];
#pragma unroll
    for (int r = 0; r < E::R; r++) {
      const int row = E::isp(st, r) - o;
      v[r] = (row >= 0 && row < N) ? ldg2(vin + p2(row, col, N)) : make_float2(0.f, 0.f);
    }
    E::fwd(v, st, tw, tw3);
#pragma unroll
    for (int r = 0; r < E::R; r++) {
      const float2 a = cmulc(v[r], cmul(ldg2(A + r), Bt));  // x conj(ramp_b); conj(h)/L after the sum
      if constexpr (E::HOLD_SMEM) hold[r * E::NT] = cadd(hold[r * E::NT], a); else acc[r] = cadd(acc[r], a);
    }
  }
#pragma unroll
  for (int r = 0; r < E::R; r++) {
    const int f = E::ifr(st, r);
    const float2 a = cmulc(E::HOLD_SMEM ? hold[r * E::NT] : acc[r], ldg2(hz + f));
    float2 *p = Ghat + p2(f, col, L);
    *p = first ? a : cadd(*p, a);
  }
}

#ifndef HOLO_R2B_PF_W
#define HOLO_R2B_PF_W 0
#endif
// R2B (LineEng<6144>): row y of ALL nb frames of a batch in one CTA (the frame loop inside, as
// R1B / R3B): the code stays hot in the instruction cache, and the next frame's W row and data row
// are prefetched into L2 (one lane per 32-byte sector) while the current frame is transformed.
// Per frame as REF_R2: W row x Hx_b, inverse along x, crop, residual (+F), pad, forward along x,
// x conj(Hx_b) -> V_b; partial[fb * gridDim.x + y] = F of (frame fb, row y).
template <int L, int TM = -1>
__global__ void __launch_bounds__(LineEng<L>::NT, LineEng<L>::MINB)
    k_ref_r2b(const float2 *__restrict__ W, const float *__restrict__ sqrt_d, float2 *__restrict__ V,
              double *__restrict__ partial, const float2 *__restrict__ H, const float4 *__restrict__ tw,
              const float2 *__restrict__ tw3, int N, int nb, float tau) {
  using E = LineEng<L>;
  extern __shared__ float4 sm4[];
  __shared__ double red[32];
  typename E::St st = E::init(reinterpret_cast<float2 *>(sm4));
  const int y = blockIdx.x;  // E::G == 1
  const int o = (L - N) / 2;
#pragma unroll 1
  for (int fb = 0; fb < nb; fb++) {
    const float2 *win = W + (size_t)fb * N * L;
    const float2 *Hx = H + (size_t)fb * 2 * L;
    const float *drow = sqrt_d + (size_t)fb * N * N + (size_t)y * N;
    float2 v[E::R];
#pragma unroll
    for (int r = 0; r < E::R; r++) {
      const int f = E::ifr(st, r);
      v[r] = cmul(ldg2(win + p2(y, f, N)), ldg2(Hx + f));
    }
    if (fb + 1 < nb) {  // the next frame's data row into L2 (its W row: R2B_PF_W)
#if HOLO_R2B_PF_W
      if ((threadIdx.x & 1) == 0) {
#pragma unroll
        for (int r = 0; r < E::R; r++) prefetch_l2_sector(win + (size_t)N * L + p2(y, E::ifr(st, r), N));
      }
#endif
      for (int i = threadIdx.x; i < (N * 4 + 31) / 32; i += E::NT) prefetch_l2_sector(drow + (size_t)N * N + 8 * i);
    }
    E::inv(v, st, tw, tw3);
    double acc = 0.0;
#pragma unroll
    for (int r = 0; r < E::R; r++) {
      const int c = E::isp(st, r) - o;
      float2 w = make_float2(0.f, 0.f);
      if (c >= 0 && c < N) w = residual_tau<TM>(v[r], __ldg(drow + c), tau, acc);  // G_tau, App. A.3
      v[r] = w;
    }
    const double sum = block_sum(acc, red);
    if (threadIdx.x == 0) partial[(size_t)fb * gridDim.x + y] = sum;
    E::fwd(v, st, tw, tw3);
    float2 *vo = V + (size_t)fb * N * L;
#pragma unroll
    for (int r = 0; r < E::R; r++) {
      const int f = E::ifr(st, r);
      vo[p2(y, f, N)] = cmulc(v[r], ldg2(Hx + f));
    }
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
__global__ void __launch_bounds__(LineEng<L>::NT, LineEng<L>::MINB)
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
    if (Hx) Hx += fb * 2 * L;
  }
  float2 v[E::R];
  if (MODE == REF_QHAT) {
#pragma unroll
    for (int r = 0; r < E::R; r++) v[r] = ldg2(in + (size_t)y * L + E::isp(st, r));
    E::fwd(v, st, tw, tw3);
#pragma unroll
    for (int r = 0; r < E::R; r++) out[p2(y, E::ifr(st, r), L)] = v[r];
  } else if (MODE == REF_R2) {  // the full frame table H_x (one frame per blockIdx.y: L2 / L1 resident)
    const bool act = y < N;
#pragma unroll
    for (int r = 0; r < E::R; r++) {
      const int f = E::ifr(st, r);
      v[r] = act ? cmul(ldg2(in + p2(y, f, N)), ldg2(Hx + f)) : make_float2(0.f, 0.f);
    }
    E::inv(v, st, tw, tw3);
    double acc = 0.0;
#pragma unroll
    for (int r = 0; r < E::R; r++) {
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
      for (int r = 0; r < E::R; r++) {
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
    for (int r = 0; r < E::R; r++) {
      const int cc = E::isp(st, r) - o;
      v[r] = make_float2((act && cc >= 0 && cc < N) ? __ldg(sqrt_d + (size_t)y * N + cc) - c : 0.f, 0.f);
    }
    E::fwd(v, st, tw, tw3);
    if (act) {
#pragma unroll
      for (int r = 0; r < E::R; r++) {
        const int f = E::ifr(st, r);
        out[p2(y, f, N)] = cmulc(v[r], ldg2(Hx + f));
      }
    }
  } else if (MODE == REF_FWD) {
    const bool act = y < N;
#pragma unroll
    for (int r = 0; r < E::R; r++) {
      const int f = E::ifr(st, r);
      v[r] = act ? cmul(ldg2(in + p2(y, f, N)), ldg2(Hx + f)) : make_float2(0.f, 0.f);
    }
    E::inv(v, st, tw, tw3);
    if (act) {
#pragma unroll
      for (int r = 0; r < E::R; r++) {
        const int c = E::isp(st, r) - o;
        if (c >= 0 && c < N) out[(size_t)y * N + c] = v[r];
      }
    }
  } else {  // FINAL
#pragma unroll
    for (int r = 0; r < E::R; r++) v[r] = in[p2(y, E::ifr(st, r), L)];
    E::inv(v, st, tw, tw3);
#pragma unroll
    for (int r = 0; r < E::R; r++) {
      float2 *p = out + (size_t)y * L + E::isp(st, r);
      const float2 a = cscale(v[r], scale);
      *p = accumulate ? cadd(*p, a) : a;
    }
  }
}

}  // namespace holo
