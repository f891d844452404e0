#include <cstdio>
#include <cuda_runtime.h>
// throughput of FP32 instruction forms: MODE 0 FFMA r,r,r (all distinct live regs); 1 FFMA r,r,imm;
// 2 FADD r,r; 3 FMUL r,r; 4 fma.rn.f32x2 (r,r,r); 5 FFMA r,r,r with 2 reads the same reg
template <int MODE>
__global__ void __launch_bounds__(256) k(float *out, int iters, float a0, float b0) {
  float x[8], y[8], z[8];
#pragma unroll
  for (int k = 0; k < 8; k++) { x[k] = threadIdx.x * 1e-3f + k; y[k] = a0 + k * 1e-3f; z[k] = b0 - k * 1e-4f; }
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int u = 0; u < 16; u++) {
#pragma unroll
      for (int k = 0; k < 8; k++) {
        if (MODE == 0) x[k] = fmaf(x[k], y[k], z[k]);
        if (MODE == 1) x[k] = fmaf(x[k], 0.9999f, 1e-7f);
        if (MODE == 2) x[k] = x[k] + y[k];
        if (MODE == 3) x[k] = x[k] * y[k];
        if (MODE == 5) x[k] = fmaf(x[k], x[k], z[k]);
      }
      if (MODE == 4) {
#pragma unroll
        for (int k = 0; k < 8; k += 2) {
          unsigned long long xx, yy, zz;
          asm("mov.b64 %0, {%1, %2};" : "=l"(xx) : "f"(x[k]), "f"(x[k + 1]));
          asm("mov.b64 %0, {%1, %2};" : "=l"(yy) : "f"(y[k]), "f"(y[k + 1]));
          asm("mov.b64 %0, {%1, %2};" : "=l"(zz) : "f"(z[k]), "f"(z[k + 1]));
          asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(xx) : "l"(xx), "l"(yy), "l"(zz));
          asm("mov.b64 {%0, %1}, %2;" : "=f"(x[k]), "=f"(x[k + 1]) : "l"(xx));
        }
      }
    }
  }
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < 8; k++) s += x[k] + y[k] + z[k];
  if (s == 12345.678f) out[threadIdx.x] = s;
}
template <int MODE>
void run(const char *name, float *out) {
  int blocks = 148 * 8, iters = 4096;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  k<MODE><<<blocks, 256>>>(out, iters, 0.999f, 1e-7f);
  cudaEventRecord(e0);
  k<MODE><<<blocks, 256>>>(out, iters, 0.999f, 1e-7f);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double inst = (double)iters * 16 * 8 * blocks * 256 / (MODE == 4 ? 2 : 1);
  printf("%-28s %8.3f ms  %7.2f T lane-instr/s  (%s)\n", name, ms, inst / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
}
int main() {
  float *out; cudaMalloc(&out, 4096);
  for (int r = 0; r < 2; r++) {
    run<0>("FFMA r,r,r", out); run<1>("FFMA r,imm,imm", out); run<2>("FADD r,r", out);
    run<3>("FMUL r,r", out); run<4>("FFMA2 (f32x2) r,r,r", out); run<5>("FFMA r,r(same),r", out);
  }
}
