// fftbench.cu -- microbenchmark of the line-FFT engine (fft_engine.cuh) in isolation.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2407_20304_b200/csrc \
//        [-DHOLO_TW_FULL=1] [-DHOLO_SINGLE_BUF=1] [-DNOALLOC=1] tools/fftbench.cu -o fftbench
// Kernels: rows / columns of a 4096^2 complex64 array: load, (FFT, x h, IFFT, x g) x NPAIR, store.
#include <cstdio>
#include <vector>
#include <cmath>
#include "holo_kernels.cuh"
#include "tma.cuh"
#include <cudaTypedefs.h>
using namespace holo;

#ifndef NOALLOC
#define NOALLOC 0
#endif
constexpr int L = 4096;

__device__ __forceinline__ float2 ldd(const float2 *p) {
#if NOALLOC
  float2 v;
  asm volatile("ld.global.nc.L1::no_allocate.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "l"(p));
  return v;
#else
  return __ldg(p);
#endif
}

template <int NT, bool COLS, int NPAIR, bool TABLES>
__global__ void __launch_bounds__(NT, 512 / NT) kbench(const float2 *__restrict__ in, float2 *__restrict__ out,
                                                       const float4 *__restrict__ tw, const float2 *__restrict__ h,
                                                       const float2 *__restrict__ g2) {
  using C = Cta<L, COLS, NT>;
  constexpr int T = L / 16;
  extern __shared__ float4 sm4[];
  float2 *sm = reinterpret_cast<float2 *>(sm4);
  Xch x = C::xch(sm);
  const int t = C::t(), line = blockIdx.x * C::G + C::g();
  float2 v[16];
#pragma unroll
  for (int r = 0; r < 16; r++)
    v[r] = COLS ? ldd(in + (size_t)(t + r * T) * L + line) : ldd(in + (size_t)line * L + t + r * T);
#pragma unroll 1
  for (int p = 0; p < NPAIR; p++) {
    fft<L, false>(v, x, t, tw);
    if (TABLES) mul_tab<L, false>(v, h, t);
    fft<L, true>(v, x, t, tw);
    if (TABLES) mul_tab<L, false>(v, g2, t);
  }
#pragma unroll
  for (int r = 0; r < 16; r++) {
    if (COLS) out[(size_t)(t + r * T) * L + line] = v[r];
    else out[(size_t)line * L + t + r * T] = v[r];
  }
}

template <int NT, bool COLS, int NPAIR, bool TABLES>
void run(const char *name, const float2 *in, float2 *out, const float4 *tw, const float2 *h, const float2 *g2) {
  using C = Cta<L, COLS, NT>;
  size_t smem = C::XBYTES;
  auto k = kbench<NT, COLS, NPAIR, TABLES>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int grid = L / C::G;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int i = 0; i < 3; i++) k<<<grid, NT, smem>>>(in, out, tw, h, g2);
  const int reps = 10;
  cudaEventRecord(e0);
  for (int i = 0; i < reps; i++) k<<<grid, NT, smem>>>(in, out, tw, h, g2);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaError_t err = cudaGetLastError();
  double us = 1e3 * ms / reps;
  double nfft = 2.0 * NPAIR * L;  // line FFTs per launch
  double per_set = us / (2.0 * NPAIR);
  // element-FFTs per SM-cycle at 1.965 GHz (clock not locked; indicative)
  double epc = nfft * L / (us * 1e-6) / (148 * 1.965e9);
  int nb = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k, NT, smem);
  printf("%-34s NT=%d G=%d blocks/SM=%d smem=%zuKB  %9.1f us/launch  %7.1f us per 4096^2 FFT set  %.2f elemFFT/SM-cycle  %s\n",
         name, NT, C::G, nb, smem / 1024, us, per_set, epc, err == cudaSuccess ? "" : cudaGetErrorString(err));
}


// column pairs through TMA: load 16 boxes {BOXC complex, 256 rows} into the exchange region,
// read layout S, NPAIR (FFT, x h, IFFT, x g), write back through 16 boxes {2, 256}.
template <int NPAIR, int BOXC>
__global__ void __launch_bounds__(512, 1) kcol_tma(const __grid_constant__ CUtensorMap tin,
                                                   const __grid_constant__ CUtensorMap tout,
                                                   const float4 *__restrict__ tw, const float2 *__restrict__ h,
                                                   const float2 *__restrict__ g2) {
  using C = Cta<L, true, 512>;
  constexpr int T = L / 16;
  extern __shared__ __align__(1024) float4 sm4[];
  __shared__ uint64_t bar;
  float2 *sm = reinterpret_cast<float2 *>(sm4);
  float2 *stage = sm;  // 16 * 256 * BOXC float2 <= exchange region
  Xch x = C::xch(sm);
  const int t = C::t(), g = C::g();
  const int x0 = blockIdx.x * 2;             // first column of this CTA
  const int xb = x0 & ~(BOXC - 1);           // first column of the box
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    mbar_expect_tx(&bar, 16 * 256 * BOXC * 8);
    for (int r = 0; r < 16; r++) tma_load_2d(stage + r * 256 * BOXC, &tin, 2 * xb, 256 * r, &bar);
  }
  mbar_wait(&bar, 0);
  float2 v[16];
#pragma unroll
  for (int r = 0; r < 16; r++) v[r] = stage[r * 256 * BOXC + t * BOXC + (x0 - xb) + g];
  __syncthreads();
#pragma unroll 1
  for (int p = 0; p < NPAIR; p++) {
    fft<L, false>(v, x, t, tw);
    mul_tab<L, false>(v, h, t);
    fft<L, true>(v, x, t, tw);
    mul_tab<L, false>(v, g2, t);
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < 16; r++) stage[r * 512 + t * 2 + g] = v[r];
  fence_proxy_async();
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int r = 0; r < 16; r++) tma_store_2d(&tout, 2 * x0, 256 * r, stage + r * 512);
    tma_store_commit();
    tma_store_wait_all();
  }
}

CUtensorMap make_map(void *base, int boxc) {
  CUtensorMap m;
  cuuint64_t dims[2] = {(cuuint64_t)2 * L, (cuuint64_t)L};
  cuuint64_t strides[1] = {(cuuint64_t)L * 8};
  cuuint32_t box[2] = {(cuuint32_t)(2 * boxc), 256};
  cuuint32_t es[2] = {1, 1};
  printf("encode base=%p\n", base); fflush(stdout);
  CUresult r = cuTensorMapEncodeTiled(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, base, dims, strides, box, es,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) printf("encode failed %d\n", (int)r);
  return m;
}

template <int NPAIR, int BOXC>
void run_tma(const char *name, float2 *in, float2 *out, const float4 *tw, const float2 *h, const float2 *g2) {
  using C = Cta<L, true, 512>;
  size_t smem = C::XBYTES;
  auto k = kcol_tma<NPAIR, BOXC>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  CUtensorMap mi = make_map(in, BOXC), mo = make_map(out, 2);
  int grid = L / 2;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int i = 0; i < 3; i++) k<<<grid, 512, smem>>>(mi, mo, tw, h, g2);
  const int reps = 10;
  cudaEventRecord(e0);
  for (int i = 0; i < reps; i++) k<<<grid, 512, smem>>>(mi, mo, tw, h, g2);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaError_t err = cudaGetLastError();
  double us = 1e3 * ms / reps;
  printf("%-34s TMA box %d cols               %9.1f us/launch  %7.1f us per 4096^2 FFT set  %s\n", name, BOXC, us,
         us / (2.0 * NPAIR), err == cudaSuccess ? "" : cudaGetErrorString(err));
}

// check: TMA column path == LDG column path (same arithmetic)
void check(float2 *in, float2 *o1, float2 *o2, const float4 *tw, const float2 *h, const float2 *g2) {
  using C = Cta<L, true, 512>;
  auto k1 = kbench<512, true, 1, true>;
  auto k2 = kcol_tma<1, 4>;
  cudaFuncSetAttribute(k1, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::XBYTES);
  cudaFuncSetAttribute(k2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::XBYTES);
  k1<<<L / 2, 512, C::XBYTES>>>(in, o1, tw, h, g2);
  printf("k1 %s\n", cudaGetErrorString(cudaDeviceSynchronize())); fflush(stdout);
  CUtensorMap m1 = make_map(in, 4);
  printf("map1\n"); fflush(stdout);
  CUtensorMap m2 = make_map(o2, 2);
  printf("map2\n"); fflush(stdout);
  k2<<<L / 2, 512, C::XBYTES>>>(m1, m2, tw, h, g2);
  cudaError_t e2 = cudaDeviceSynchronize();
  printf("k2 %s\n", cudaGetErrorString(e2)); fflush(stdout);
  if (e2 != cudaSuccess) exit(1);
  std::vector<float2> a((size_t)L * L), b((size_t)L * L);
  cudaMemcpy(a.data(), o1, a.size() * 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(b.data(), o2, b.size() * 8, cudaMemcpyDeviceToHost);
  double md = 0;
  for (size_t i = 0; i < a.size(); i++) md = std::max(md, (double)std::fabs(a[i].x - b[i].x) + std::fabs(a[i].y - b[i].y));
  printf("TMA vs LDG column path: max |diff| = %g (%s)\n", md, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  const size_t n = (size_t)L * L;
  float2 *in, *out, *h, *g2;
  float4 *tw;
  cudaMalloc(&in, n * 8);
  cudaMalloc(&out, n * 8);
  cudaMalloc(&h, L * 8);
  cudaMalloc(&g2, L * 8);
  cudaMalloc(&tw, 1 << 20);
  std::vector<float2> hv(n);
  for (size_t i = 0; i < n; i++) hv[i] = make_float2(std::sin(0.001 * i), std::cos(0.0013 * i));
  cudaMemcpy(in, hv.data(), n * 8, cudaMemcpyHostToDevice);
  std::vector<float2> t(L);
  for (int i = 0; i < L; i++) t[i] = make_float2(std::cos(1e-3 * i * i), std::sin(1e-3 * i * i));
  cudaMemcpy(h, t.data(), L * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(g2, t.data(), L * 8, cudaMemcpyHostToDevice);
  // twiddles (layout depends on HOLO_TW_FULL); values are what the engine expects for L = 4096
  std::vector<float2> tws;
  for (int Ns = 16; Ns < L; Ns *= 16)
    for (int m = 0; m < Ns; m++) {
#if HOLO_TW_FULL
      for (int e = 0; e < 16; e++) {
#else
      for (int e : {1, 2, 4, 8}) {
#endif
        double a = -2 * M_PI * (double)m * e / (16.0 * Ns);
        tws.push_back(make_float2(std::cos(a), std::sin(a)));
      }
    }
  cudaMemcpy(tw, tws.data(), tws.size() * 8, cudaMemcpyHostToDevice);
  printf("knobs: TW_FULL=%d SINGLE_BUF=%d NOALLOC=%d\n", HOLO_TW_FULL, HOLO_SINGLE_BUF, NOALLOC);
  {
    float2 *o2;
    cudaMalloc(&o2, n * 8);
    printf("check...\n"); fflush(stdout);
    check(in, out, o2, tw, h, g2);
    run<512, true, 1, true>("cols  1 pair + tables (LDG)", in, out, tw, h, g2);
    run_tma<1, 2>("cols  1 pair + tables", in, o2, tw, h, g2);
    run_tma<1, 4>("cols  1 pair + tables", in, o2, tw, h, g2);
    run<512, true, 2, true>("cols  2 pairs + tables (LDG)", in, out, tw, h, g2);
    run_tma<2, 2>("cols  2 pairs + tables", in, o2, tw, h, g2);
    run_tma<2, 4>("cols  2 pairs + tables", in, o2, tw, h, g2);
    run<512, false, 1, true>("rows  1 pair + tables", in, out, tw, h, g2);
    if (getenv("ONLY_TMA")) return 0;
  }
  run<512, false, 2, true>("rows  2 pairs + tables", in, out, tw, h, g2);
  run<256, false, 2, true>("rows  2 pairs + tables", in, out, tw, h, g2);
  run<512, true, 2, true>("cols  2 pairs + tables", in, out, tw, h, g2);
  run<256, true, 2, true>("cols  2 pairs + tables", in, out, tw, h, g2);
  run<512, false, 8, false>("rows  8 pairs, no tables", in, out, tw, h, g2);
  run<256, false, 8, false>("rows  8 pairs, no tables", in, out, tw, h, g2);
  run<512, false, 8, true>("rows  8 pairs + tables", in, out, tw, h, g2);
  run<256, false, 8, true>("rows  8 pairs + tables", in, out, tw, h, g2);
  run<512, true, 8, true>("cols  8 pairs + tables", in, out, tw, h, g2);
  run<256, true, 8, true>("cols  8 pairs + tables", in, out, tw, h, g2);
  run<512, false, 1, false>("rows  1 pair (I/O bound)", in, out, tw, h, g2);
  run<512, true, 1, false>("cols  1 pair (I/O bound)", in, out, tw, h, g2);
  return 0;
}
