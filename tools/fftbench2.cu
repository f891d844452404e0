// fftbench2.cu -- does splitting the CTA overlap one line's shared-memory exchange with another
// line's butterflies?  Same work as fftbench.cu (rows of a 4096^2 array, NPAIR x (FFT, x h, IFFT,
// x g)), launched as NT-thread CTAs (G = NT/256 lines each) with MINB CTAs per SM.
#include <cmath>
#include <cstdio>
#include <vector>

#include "holo_kernels.cuh"
using namespace holo;

constexpr int L = 4096;

template <int NT, int MINB, int NPAIR>
__global__ void __launch_bounds__(NT, MINB) kb(const float2 *__restrict__ in, float2 *__restrict__ out,
                                               const float4 *__restrict__ tw, const float2 *__restrict__ h) {
  using C = Cta<L, NT>;
  constexpr int T = L / 16;
  extern __shared__ float4 sm4[];
  float2 *sm = reinterpret_cast<float2 *>(sm4);
  Xch x = C::xch(sm);
  const int t = C::t(), line = blockIdx.x * C::G + C::g();
  float2 v[16];
#pragma unroll
  for (int r = 0; r < 16; r++) v[r] = __ldg(in + (size_t)line * L + t + r * T);
#pragma unroll 1
  for (int p = 0; p < NPAIR; p++) {
    fft<L, false>(v, x, t, tw);
    mul_tab<L, false>(v, h, t);
    fft<L, true>(v, x, t, tw);
    mul_tab<L, false>(v, h + L, t);
  }
#pragma unroll
  for (int r = 0; r < 16; r++) out[(size_t)line * L + t + r * T] = v[r];
}

template <int NT, int MINB, int NPAIR>
void run(const char *name, const float2 *in, float2 *out, const float4 *tw, const float2 *h) {
  using C = Cta<L, NT>;
  const size_t smem = C::XBYTES;
  auto k = kb<NT, MINB, NPAIR>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int i = 0; i < 3; i++) k<<<L / C::G, NT, smem>>>(in, out, tw, h);
  const int reps = 10;
  cudaEventRecord(e0);
  for (int i = 0; i < reps; i++) k<<<L / C::G, NT, smem>>>(in, out, tw, h);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double us = 1e3 * ms / reps, per_set = us / (2.0 * NPAIR);
  const double tf = 5.0 * L * 12 * L * 2.0 * NPAIR / (us * 1e-6) / 1e12;
  int nb = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k, NT, smem);
  printf("%-34s %9.1f us/launch  %6.2f us/set  %5.1f TFLOP/s  blocks/SM %d smem %zu  %s\n", name, us, per_set, tf, nb,
         smem, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  std::vector<float2> twh;
  for (int Ns = 16; Ns < L; Ns *= 16)
    for (int m = 0; m < Ns; m++)
    {
      for (int e : {1, 2, 4, 8}) {
        double a = -2.0 * M_PI * (double)((long)m * e) / (16.0 * Ns);
        twh.push_back(make_float2((float)cos(a), (float)sin(a)));
      }
      if (TW_ROW_F2 == 8) {  // DIT level twiddles (fft_engine.cuh, HOLO_TW8)
        const double f = -2.0 * M_PI * (double)m / (16.0 * Ns);
        for (double a : {f - M_PI / 8, f - M_PI / 4, f - 3 * M_PI / 8, 2 * f - M_PI / 4})
          twh.push_back(make_float2((float)cos(a), (float)sin(a)));
      }
    }
  std::vector<float2> hh(2 * L), xin((size_t)L * L);
  for (int i = 0; i < 2 * L; i++) hh[i] = make_float2((float)cos(0.001 * i * i) / L, (float)sin(0.001 * i * i) / L);
  for (size_t i = 0; i < xin.size(); i++) xin[i] = make_float2((float)sin(0.37 * i), (float)cos(0.11 * i * 1.3));
  float2 *in, *out, *h;
  float4 *tw;
  cudaMalloc(&in, xin.size() * 8);
  cudaMalloc(&out, xin.size() * 8);
  cudaMalloc(&h, hh.size() * 8);
  cudaMalloc(&tw, twh.size() * 8);
  cudaMemcpy(in, xin.data(), xin.size() * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(h, hh.data(), hh.size() * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(tw, twh.data(), twh.size() * 8, cudaMemcpyHostToDevice);
  for (int rep = 0; rep < 2; rep++) {
    run<512, 1, 8>("NT 512 (2 lines) x1/SM", in, out, tw, h);
    run<256, 2, 8>("NT 256 (1 line)  x2/SM", in, out, tw, h);
    run<256, 3, 8>("NT 256 (1 line)  x3/SM (85 regs)", in, out, tw, h);
    run<1024, 1, 8>("NT 1024 (4 lines) x1/SM", in, out, tw, h);
  }
  return 0;
}
