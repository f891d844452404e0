// holo_multires.cuh -- kernels of the multiresolution schedule (
// P:258-259 "initiate reconstruction with binning 8x8 ... 4x4 ... then extrapolate the
// recovered object with the probe function to a grid twice as dense").
//
// Fourier 2x upsampling (O15, reading R1): per axis, the trigonometric interpolant of the
// coarse line x (length L, band fbar in [-L/2, L/2)) sampled at half-pixel steps, coarse
// sample n at fine coordinate 2n + 1/2:
//   y[m] = (1/L) sum_f X[f] e^{+2 pi i fbar (m - 1/2)/(2L)},  m < L2 = 2L.
// On the fine engine (length L2): the zero-inserted line z[2n] = x[n] has FFT_L2(z)[F] =
// X[F mod L], so y = IFFT_L2(up[F] FFT_L2(z)) with the table
//   up[F] = [Fbar in [-L/2, L/2)] e^{-i pi Fbar / L2} / L     (the 2 and 1/L2 folded in).
// Rows first (coarse rows -> P2 [L][L2] scratch), then columns (-> row-major [L2][L2]).
//
// 2x2 binning of amplitudes (O16, reading R2): a_c = sqrt(mean of the four a_f^2).
#pragma once
#include "holo_passes.cuh"

namespace holo {

// coarse rows (row-major [L2/2][L2/2]) -> P2 scratch [L2/2 rows][L2]
template <int L2>
__global__ void __launch_bounds__(NT, CTAS_PER_SM)
    k_up_rows(const float2 *__restrict__ in, float2 *__restrict__ mid, const float4 *__restrict__ tw,
              const float2 *__restrict__ up) {
  using C = CtaK<L2>;
  constexpr int T = L2 / 16, L = L2 / 2;
  extern __shared__ float4 sm4[];
  float2 *sm = reinterpret_cast<float2 *>(sm4);
  Xch x = C::xch(sm);
  const int t = C::t(), y = blockIdx.x * C::G + C::g();
  float2 v[16];
#pragma unroll
  for (int r = 0; r < 16; r++) v[r] = (t & 1) ? make_float2(0.f, 0.f) : ldg2(in + (size_t)y * L + (t + r * T) / 2);
  fft<L2, false>(v, x, t, tw);
  mul_tab<L2, false>(v, up, t);
  fft<L2, true>(v, x, t, tw);
  st_p2_row<L2>(v, mid, y, L, t);
}

// columns of the P2 scratch (L2/2 rows) -> fine row-major [L2][L2]
template <int L2>
__global__ void __launch_bounds__(NT, CTAS_PER_SM)
    k_up_cols(const float2 *__restrict__ mid, float2 *__restrict__ out, const float4 *__restrict__ tw,
              const float2 *__restrict__ up) {
  using C = CtaK<L2>;
  constexpr int T = L2 / 16, L = L2 / 2;
  extern __shared__ float4 sm4[];
  float2 *sm = reinterpret_cast<float2 *>(sm4);
  Xch x = C::xch(sm);
  const int t = C::t(), col = blockIdx.x * C::G + C::g();
  float2 v[16];
#pragma unroll
  for (int r = 0; r < 16; r++) v[r] = (t & 1) ? make_float2(0.f, 0.f) : ldg2(mid + p2((t + r * T) / 2, col, L));
  fft<L2, false>(v, x, t, tw);
  mul_tab<L2, false>(v, up, t);
  fft<L2, true>(v, x, t, tw);
#pragma unroll
  for (int r = 0; r < 16; r++) out[(size_t)(t + r * T) * L2 + col] = v[r];
}

// a_c[i][l] = sqrt(0.25 sum a_f[2i+a][2l+b]^2), count frames of [2N][2N] -> [N][N]
static __global__ void k_bin2(const float *__restrict__ fine, float *__restrict__ coarse, int N, size_t count) {
  const size_t NN = (size_t)N * N, total = NN * count;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
    const size_t c = i / NN, rem = i % NN;
    const int r = (int)(rem / N), l = (int)(rem % N);
    const float *f = fine + c * 4 * NN + (size_t)(2 * r) * (2 * N) + 2 * l;
    const float2 a = *reinterpret_cast<const float2 *>(f), b = *reinterpret_cast<const float2 *>(f + 2 * N);
    coarse[i] = sqrtf(0.25f * (a.x * a.x + a.y * a.y + b.x * b.x + b.y * b.y));
  }
}

}  // namespace holo
