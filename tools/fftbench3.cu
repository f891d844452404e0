// fftbench3.cu -- the N_p = 6144 line engine (holo_ref.cuh LineEng<6144>) in isolation: rows of a
// 6144^2 complex64 array, load, NPAIR x (forward, x h, inverse, x g), store; 128-thread CTAs (one
// line each, 3 per SM).  Prints us per 6144^2 set of 6144-point transforms (5 N log2 N flops).
#include <cmath>
#include <cstdio>
#include <vector>

#include "holo_ref.cuh"
using namespace holo;

constexpr int L = 6144;
using E = LineEng<L>;

template <int NPAIR>
__global__ void __launch_bounds__(E::NT, E::MINB) kb(const float2 *__restrict__ in, float2 *__restrict__ out,
                                                     const float4 *__restrict__ tw, const float2 *__restrict__ tw3,
                                                     const float2 *__restrict__ h) {
  extern __shared__ float4 sm4[];
  E::St st = E::init(reinterpret_cast<float2 *>(sm4));
  const int line = blockIdx.x;
  float2 v[E::R];
#pragma unroll
  for (int r = 0; r < E::R; r++) v[r] = __ldg(in + (size_t)line * L + E::isp(st, r));
#pragma unroll 1
  for (int p = 0; p < NPAIR; p++) {
    E::fwd(v, st, tw, tw3);
#pragma unroll
    for (int r = 0; r < E::R; r++) v[r] = cmul(v[r], __ldg(h + E::ifr(st, r)));
    E::inv(v, st, tw, tw3);
#pragma unroll
    for (int r = 0; r < E::R; r++) v[r] = cmul(v[r], __ldg(h + L + E::isp(st, r)));
  }
#pragma unroll
  for (int r = 0; r < E::R; r++) out[(size_t)line * L + E::isp(st, r)] = v[r];
}

int main() {
  constexpr int LS = 2048;
  std::vector<float2> twh;
  for (int Ns = 8; Ns < LS; Ns *= 16)
    for (int m = 0; m < Ns; m++)
      for (int e : {1, 2, 4, 8}) {
        double a = -2.0 * M_PI * (double)((long)m * e) / (16.0 * Ns);
        twh.push_back(make_float2((float)cos(a), (float)sin(a)));
      }
  std::vector<float2> t3(2 * LS);
  for (int g = 1; g <= 2; g++)
    for (int k = 0; k < LS; k++) {
      double a = -2.0 * M_PI * (double)(g * k) / L;
      t3[(g - 1) * LS + k] = make_float2((float)cos(a), (float)sin(a));
    }
  std::vector<float2> hh(2 * L), xin((size_t)L * L);
  for (int i = 0; i < 2 * L; i++) hh[i] = make_float2((float)cos(0.001 * i * i) / L, (float)sin(0.001 * i * i) / L);
  for (size_t i = 0; i < xin.size(); i++) xin[i] = make_float2((float)sin(0.37 * i), (float)cos(0.11 * i * 1.3));
  float2 *in, *out, *h, *tw3;
  float4 *tw;
  cudaMalloc(&in, xin.size() * 8);
  cudaMalloc(&out, xin.size() * 8);
  cudaMalloc(&h, hh.size() * 8);
  cudaMalloc(&tw, twh.size() * 8);
  cudaMalloc(&tw3, t3.size() * 8);
  cudaMemcpy(in, xin.data(), xin.size() * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(h, hh.data(), hh.size() * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(tw, twh.data(), twh.size() * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(tw3, t3.data(), t3.size() * 8, cudaMemcpyHostToDevice);
  auto k = kb<4>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)E::SMEM);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int i = 0; i < 3; i++) k<<<L, E::NT, E::SMEM>>>(in, out, tw, tw3, h);
  cudaEventRecord(e0);
  for (int i = 0; i < 5; i++) k<<<L, E::NT, E::SMEM>>>(in, out, tw, tw3, h);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double us = 1e3 * ms / 5, per_set = us / 8.0;
  const double tf = 5.0 * L * log2((double)L) * L * 8.0 / (us * 1e-6) / 1e12;
  int nb = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k, E::NT, E::SMEM);
  printf("6144 engine, 4 pairs + tables: %9.1f us/launch  %7.2f us per 6144^2 set  %5.1f TFLOP/s  blocks/SM %d  %s\n",
         us, per_set, tf, nb, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
