// fftbench.cu -- microbenchmark of the line-FFT engine (fft_engine.cuh) in isolation.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2407_20304_b200/csrc \
//        [-DHOLO_DIT=0|1] [-DHOLO_SINGLE_BUF=0|1] tools/fftbench.cu -o tools/bin/fftbench_x
// Rows of a 4096^2 complex64 array: load, NPAIR x (FFT, [x h], IFFT, [x g]), store; 512-thread
// CTAs (2 lines), the layout of the product's row passes.  Prints us per 4096^2 set of
// 4096-point transforms and checks one forward transform against an fp64 DFT.
#include <cmath>
#include <cstdio>
#include <vector>

#include "holo_kernels.cuh"
using namespace holo;

constexpr int L = 4096;

template <int NPAIR, bool TABLES, bool FWD_ONLY>
__global__ void __launch_bounds__(512, 1) kbench(const float2 *__restrict__ in, float2 *__restrict__ out,
                                                 const float4 *__restrict__ tw, const float2 *__restrict__ h) {
  using C = Cta<L, 512>;
  constexpr int T = L / 16;
  extern __shared__ float4 sm4[];
  float2 *sm = reinterpret_cast<float2 *>(sm4);
  Xch x = C::xch(sm);
  const int t = C::t(), line = blockIdx.x * C::G + C::g();
  float2 v[16];
#pragma unroll
  for (int r = 0; r < 16; r++) v[r] = __ldg(in + (size_t)line * L + t + r * T);
  if (FWD_ONLY) {
    fft<L, false>(v, x, t, tw);
  } else {
#pragma unroll 1
    for (int p = 0; p < NPAIR; p++) {
      fft<L, false>(v, x, t, tw);
      if (TABLES) mul_tab<L, false>(v, h, t);
      fft<L, true>(v, x, t, tw);
      if (TABLES) mul_tab<L, false>(v, h + L, t);
    }
  }
#pragma unroll
  for (int r = 0; r < 16; r++) out[(size_t)line * L + t + r * T] = v[r];
}

template <int NPAIR, bool TABLES>
void run(const char *name, const float2 *in, float2 *out, const float4 *tw, const float2 *h) {
  using C = Cta<L, 512>;
  const size_t smem = C::XBYTES;
  auto k = kbench<NPAIR, TABLES, false>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int i = 0; i < 3; i++) k<<<L / C::G, 512, smem>>>(in, out, tw, h);
  const int reps = 10;
  cudaEventRecord(e0);
  for (int i = 0; i < reps; i++) k<<<L / C::G, 512, smem>>>(in, out, tw, h);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double us = 1e3 * ms / reps, per_set = us / (2.0 * NPAIR);
  const double tf = 5.0 * L * 12 * L * 2.0 * NPAIR / (us * 1e-6) / 1e12;
  printf("%-28s %9.1f us/launch  %6.2f us per 4096^2 set  %5.1f TFLOP/s (5NlogN)  %s\n", name, us, per_set, tf,
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  printf("knobs: HOLO_DIT=%d HOLO_SINGLE_BUF=%d\n", HOLO_DIT, HOLO_SINGLE_BUF);
  // twiddle rows exactly as holo_plan.cu builds them (Ns = F 16^st, per m: w^m, w^2m, w^4m, w^8m)
  std::vector<float2> twh;
  for (int Ns = 16; Ns < L; Ns *= 16)
    for (int m = 0; m < Ns; m++)
      for (int e : {1, 2, 4, 8}) {
        double a = -2.0 * M_PI * (double)((long)m * e) / (16.0 * Ns);
        twh.push_back(make_float2((float)cos(a), (float)sin(a)));
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
  // correctness: forward transform of row 5 vs an fp64 DFT
  {
    using C = Cta<L, 512>;
    auto k = kbench<1, false, true>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::XBYTES);
    k<<<L / C::G, 512, C::XBYTES>>>(in, out, tw, h);
    std::vector<float2> o(L);
    cudaMemcpy(o.data(), out + 5 * (size_t)L, L * 8, cudaMemcpyDeviceToHost);
    double num = 0, den = 0;
    for (int f = 0; f < L; f++) {
      double re = 0, im = 0;
      for (int n = 0; n < L; n++) {
        const double a = -2.0 * M_PI * (double)(((long)f * n) % L) / L;
        const float2 v = xin[5 * (size_t)L + n];
        re += v.x * cos(a) - v.y * sin(a);
        im += v.x * sin(a) + v.y * cos(a);
      }
      num += (o[f].x - re) * (o[f].x - re) + (o[f].y - im) * (o[f].y - im);
      den += re * re + im * im;
    }
    printf("forward 4096-point vs fp64 DFT: rel L2 error %.3e\n", sqrt(num / den));
  }
  run<8, false>("rows 8 pairs, no tables", in, out, tw, h);
  run<8, true>("rows 8 pairs + tables", in, out, tw, h);
  run<2, true>("rows 2 pairs + tables", in, out, tw, h);
  return 0;
}
