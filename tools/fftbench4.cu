// fftbench4.cu -- does a thread holding V x 16 values of ONE line (V "virtual threads", T/V real
// threads per line) beat the 16-values-per-thread engine?  Rows of a 4096^2 array: load, 8 x (FFT,
// x h, IFFT, x g), store.  V = 1: the product engine (fft_engine.cuh, 256 threads / line); V = 2: 128
// threads / line, two radix-16 butterflies per thread per stage, one exchange buffer per line.
#include <cmath>
#include <cstdio>
#include <vector>

#include "holo_kernels.cuh"
using namespace holo;

constexpr int L = 4096;

// Stockham like fft<L>, but thread t runs the butterflies of virtual threads t + TR * u, u < V
template <int L, bool INV, int V, int ST>
__device__ __forceinline__ void stage_vt(float2 (&v)[V * 16], float2 *buf, const int t, const float4 *__restrict__ tw) {
  using S = Shape<L>;
  constexpr int TR = S::T / V;
  constexpr int Ns = S::F * pow16(ST);
  constexpr int ROW0 = S::F * (pow16(ST) - 1) / 15;
#pragma unroll
  for (int u = 0; u < V; u++) {
    const int tv = t + TR * u, m = tv & (Ns - 1);
    const float4 a = __ldg(tw + 2 * (ROW0 + m)), b = __ldg(tw + 2 * (ROW0 + m) + 1);
    dft16_dit_tw<INV>(v + 16 * u, make_float2(a.x, a.y), make_float2(a.z, a.w), make_float2(b.x, b.y),
                      make_float2(b.z, b.w));
  }
  if constexpr (ST + 1 < S::S16) {
    __syncthreads();
#pragma unroll
    for (int u = 0; u < V; u++) {
      const int tv = t + TR * u, m = tv & (Ns - 1), base = (tv - m) * 16 + m;
#pragma unroll
      for (int s = 0; s < 16; s++) buf[P(base + s * Ns)] = v[16 * u + s];
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < V; u++)
#pragma unroll
      for (int r = 0; r < 16; r++) v[16 * u + r] = buf[P(t + TR * u + r * S::T)];
    stage_vt<L, INV, V, ST + 1>(v, buf, t, tw);
  }
}
template <int L, bool INV, int V>
__device__ __forceinline__ void fft_vt(float2 (&v)[V * 16], float2 *buf, const int t, const float4 *__restrict__ tw) {
  using S = Shape<L>;
  constexpr int TR = S::T / V;
  static_assert(S::F == 16, "first stage radix 16 only in this benchmark");
#pragma unroll
  for (int u = 0; u < V; u++) dft16_dit<INV>(v + 16 * u);
  __syncthreads();
#pragma unroll
  for (int u = 0; u < V; u++)
#pragma unroll
    for (int s = 0; s < 16; s++) buf[P((t + TR * u) * 16 + s)] = v[16 * u + s];
  __syncthreads();
#pragma unroll
  for (int u = 0; u < V; u++)
#pragma unroll
    for (int r = 0; r < 16; r++) v[16 * u + r] = buf[P(t + TR * u + r * S::T)];
  stage_vt<L, INV, V, 0>(v, buf, t, tw);
}

// element of register (u, r) of thread t: tv + T r with tv = t + TR u
template <int V, int MINB>
__global__ void __launch_bounds__(L / 16 / V, MINB) kb(const float2 *__restrict__ in, float2 *__restrict__ out,
                                                      const float4 *__restrict__ tw, const float2 *__restrict__ h) {
  constexpr int T = L / 16, TR = T / V;
  extern __shared__ float4 sm4[];
  float2 *buf = reinterpret_cast<float2 *>(sm4);
  const int t = threadIdx.x, line = blockIdx.x;
  float2 v[V * 16];
#pragma unroll
  for (int u = 0; u < V; u++)
#pragma unroll
    for (int r = 0; r < 16; r++) v[16 * u + r] = __ldg(in + (size_t)line * L + t + TR * u + r * T);
#pragma unroll 1
  for (int p = 0; p < 8; p++) {
    fft_vt<L, false, V>(v, buf, t, tw);
#pragma unroll
    for (int u = 0; u < V; u++)
#pragma unroll
      for (int r = 0; r < 16; r++) v[16 * u + r] = cmul(v[16 * u + r], __ldg(h + t + TR * u + r * T));
    fft_vt<L, true, V>(v, buf, t, tw);
#pragma unroll
    for (int u = 0; u < V; u++)
#pragma unroll
      for (int r = 0; r < 16; r++) v[16 * u + r] = cmul(v[16 * u + r], __ldg(h + L + t + TR * u + r * T));
  }
#pragma unroll
  for (int u = 0; u < V; u++)
#pragma unroll
    for (int r = 0; r < 16; r++) out[(size_t)line * L + t + TR * u + r * T] = v[16 * u + r];
}

template <int V, int MINB>
void run(const char *name, const float2 *in, float2 *out, const float4 *tw, const float2 *h, const std::vector<float2> &xin) {
  const size_t smem = sizeof(float2) * Shape<L>::LP;
  auto k = kb<V, MINB>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int nt = L / 16 / V;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int i = 0; i < 3; i++) k<<<L, nt, smem>>>(in, out, tw, h);
  cudaEventRecord(e0);
  for (int i = 0; i < 10; i++) k<<<L, nt, smem>>>(in, out, tw, h);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double us = 1e3 * ms / 10, per_set = us / 16.0;
  int nb = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k, nt, smem);
  // correctness: one FFT+h+IFFT+g pair chain is hard to check; compare V runs against each other
  std::vector<float2> o(L);
  cudaMemcpy(o.data(), out + 7 * (size_t)L, L * 8, cudaMemcpyDeviceToHost);
  double cs = 0;
  for (int i = 0; i < L; i++) cs += o[i].x * (i % 7) - o[i].y * (i % 5);
  printf("%-30s %8.1f us/launch  %6.2f us per 4096^2 set  blocks/SM %d  checksum %.6e  %s\n", name, us, per_set, nb, cs,
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
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
  for (int rep = 0; rep < 2; rep++) {
    run<1, 2>("V=1: 256 thr/line, 2 CTA/SM", in, out, tw, h, xin);
    run<1, 3>("V=1: 256 thr/line, 3 CTA/SM", in, out, tw, h, xin);
    run<2, 3>("V=2: 128 thr/line, 3 CTA/SM", in, out, tw, h, xin);
    run<2, 4>("V=2: 128 thr/line, 4 CTA/SM", in, out, tw, h, xin);
    run<2, 5>("V=2: 128 thr/line, 5 CTA/SM", in, out, tw, h, xin);
    run<4, 4>("V=4: 64 thr/line, 4 CTA/SM", in, out, tw, h, xin);
    run<4, 8>("V=4: 64 thr/line, 8 CTA/SM", in, out, tw, h, xin);
  }
  return 0;
}
