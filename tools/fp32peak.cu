// fp32peak.cu -- measured FP32 ALU peak of this GPU (the ALU roof of SURVEY 8(d): P_FP32
// "from an FFMA microbenchmark, with the SM clock recorded").  Built into
// tools/libfp32peak.so by __graft_entry__.build(); bench.py loads it with ctypes.
//
//   fp32_peak(device, ms_target, *ffma_tflops, *mix_tflops, *sm_mhz)
//     ffma_tflops: 2 flop per FFMA, 8 independent chains per thread, 148 x 8 CTAs x 256 threads
//     mix_tflops : FFMA:FADD = 1:1 (an FFT's instruction mix), flops = 2 per FFMA + 1 per FADD
//     sm_mhz     : SM cycles (clock64) / wall ns (globaltimer) inside the FFMA kernel
#include <cuda_runtime.h>
#include <stdint.h>

__device__ __forceinline__ uint64_t gtimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

template <bool MIX>
__global__ void __launch_bounds__(256) k_peak(float *out, unsigned long long *clk, int iters, float a, float b) {
  float x[8];
#pragma unroll
  for (int k = 0; k < 8; k++) x[k] = threadIdx.x * 1e-3f + k;
  const long long c0 = clock64();
  const uint64_t t0 = gtimer();
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int u = 0; u < 16; u++) {
#pragma unroll
      for (int k = 0; k < 8; k++) {
        if (MIX && (u & 1)) x[k] = x[k] + b;
        else x[k] = fmaf(x[k], a, b);
      }
    }
  }
  const long long c1 = clock64();
  const uint64_t t1 = gtimer();
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < 8; k++) s += x[k];
  if (s == 12345.678f) out[threadIdx.x] = s;  // keep the chains alive
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    clk[0] = (unsigned long long)(c1 - c0);
    clk[1] = (unsigned long long)(t1 - t0);
  }
}

extern "C" int fp32_peak(int device, double ms_target, double *ffma_tflops, double *mix_tflops, double *sm_mhz) {
  if (cudaSetDevice(device) != cudaSuccess) return -1;
  cudaDeviceProp pr;
  cudaGetDeviceProperties(&pr, device);
  const int blocks = pr.multiProcessorCount * 8, threads = 256;
  float *out;
  unsigned long long *clk;
  cudaMalloc(&out, 1024 * sizeof(float));
  cudaMalloc(&clk, 2 * sizeof(unsigned long long));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  double res[2] = {0, 0};
  for (int mix = 0; mix < 2; mix++) {
    int iters = 256;
    for (int pass = 0; pass < 6; pass++) {  // grow iters until the kernel runs ~ms_target
      cudaEventRecord(e0);
      if (mix) k_peak<true><<<blocks, threads>>>(out, clk, iters, 0.9999f, 1e-7f);
      else k_peak<false><<<blocks, threads>>>(out, clk, iters, 0.9999f, 1e-7f);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      const double per_thread = (double)iters * 16 * 8;  // instructions per thread
      const double flops = mix ? per_thread * 1.5 : per_thread * 2.0;
      const double tf = flops * blocks * threads / (ms * 1e-3) / 1e12;
      if (tf > res[mix]) res[mix] = tf;
      if (ms < 0.5 * ms_target) iters *= 4;
      if (mix == 0 && pass >= 2) {
        unsigned long long h[2];
        cudaMemcpy(h, clk, sizeof(h), cudaMemcpyDeviceToHost);
        if (h[1] > 0) *sm_mhz = 1e3 * (double)h[0] / (double)h[1];
      }
    }
  }
  *ffma_tflops = res[0];
  *mix_tflops = res[1];
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(out);
  cudaFree(clk);
  return cudaGetLastError() == cudaSuccess ? 0 : -2;
}
