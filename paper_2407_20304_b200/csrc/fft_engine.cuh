// fft_engine.cuh -- register-resident Stockham line FFT for sm_100a.
//
// A length-L complex64 line (L = F * 16^S16, F in {2, 4, 8, 16}) is held by a
// "group" of T = L/16 threads, 16 values per thread, in LAYOUT S:
//
//     thread t, register r  <->  element t + T*r            (r = 0..15)
//
// Stockham autosort (natural order in and out).  Stage 0 is radix F (Ns = 1,
// no twiddles; thread t runs the 16/F butterflies j = t + T*b); then S16
// radix-16 stages with Ns = F, 16F, ..., L/16.  Every stage reads its inputs in
// layout S, and the LAST stage (Ns = T, so m = t) also WRITES layout S: the
// result stays in the same registers and pointwise factors (chirps, transfer
// functions, probe) are applied there, between transforms, with no shared-memory
// round trip.  Only the S16 exchanges between stages go through shared memory:
// 2 per transform for L = 512 ... 4096 (one STS.64 + one LDS.64 per element each).
//
// Exchange buffers: one per line (HOLO_SINGLE_BUF, default; a barrier before each
// write and one before the reads) or two (exchange e writes buffer e&1, then ONE
// barrier per exchange suffices).  Element i sits at padded slot P(i) = i + i/16, so the
// layout-S reads and the radix-16 / radix-F scatters are bank-conflict free for
// 64-bit accesses within a group.
//
// Stage twiddles w^{m s}, w = exp(-2 pi i / (16 Ns)), s = 1..15: the table holds
// only w^m, w^2m, w^4m, w^8m per m (fp64-generated, one 32-byte row); the other
// eleven are products of at most three of them (<= 3 roundings in fp32).
//
// Every thread of the CTA must call every transform (barriers); lines without
// data simply transform zeros.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

// Build knobs (compile-time, for the engine microbenchmark tools/fftbench.cu):
//   HOLO_TW_FULL   1: load all 15 stage twiddles from a [stage][m][16] table instead of 4 powers
//   HOLO_SINGLE_BUF 1 (default): one exchange buffer per line, two barriers per exchange;
//                   0: double-buffered, one barrier per exchange, twice the shared memory
//                   (measured 4% slower in the full sweep: the freed space serves L1 / table slots)
#ifndef HOLO_TW_FULL
#define HOLO_TW_FULL 0
#endif
#ifndef HOLO_SINGLE_BUF
#define HOLO_SINGLE_BUF 1
#endif

namespace holo {

__device__ __forceinline__ int P(int i) { return i + (i >> 4); }

__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
  return make_float2(fmaf(a.x, b.x, -a.y * b.y), fmaf(a.x, b.y, a.y * b.x));
}
// a * conj(b)
__device__ __forceinline__ float2 cmulc(float2 a, float2 b) {
  return make_float2(fmaf(a.x, b.x, a.y * b.y), fmaf(a.y, b.x, -a.x * b.y));
}
__device__ __forceinline__ float2 cconj(float2 a) { return make_float2(a.x, -a.y); }
__device__ __forceinline__ float2 cscale(float2 a, float s) { return make_float2(a.x * s, a.y * s); }
__device__ __forceinline__ float2 ldg2(const float2 *p) { return __ldg(p); }

// Multiply by W16^e = exp(-+2 pi i e / 16) (forward: minus), e in [0, 8), compile-time.
template <int E, bool INV>
__device__ __forceinline__ float2 tw16(float2 x) {
  constexpr float C1 = 0.92387953251128674f, S1 = 0.38268343236508977f, H = 0.70710678118654752f;
  if constexpr (E == 0) {
    return x;
  } else if constexpr (E == 4) {
    return INV ? make_float2(-x.y, x.x) : make_float2(x.y, -x.x);
  } else if constexpr (E == 2 || E == 6) {
    constexpr float c = (E == 2) ? H : -H;
    constexpr float s = H;
    return INV ? make_float2(c * x.x - s * x.y, c * x.y + s * x.x) : make_float2(c * x.x + s * x.y, c * x.y - s * x.x);
  } else {
    constexpr float c = (E == 1) ? C1 : (E == 3) ? S1 : (E == 5) ? -S1 : -C1;
    constexpr float s = (E == 1) ? S1 : (E == 3) ? C1 : (E == 5) ? C1 : S1;
    return INV ? make_float2(fmaf(c, x.x, -s * x.y), fmaf(c, x.y, s * x.x))
               : make_float2(fmaf(c, x.x, s * x.y), fmaf(c, x.y, -s * x.x));
  }
}

__host__ __device__ constexpr int ilog2c(int n) { return n <= 1 ? 0 : 1 + ilog2c(n / 2); }
__host__ __device__ constexpr int brevc(int i, int bits) { return bits == 0 ? 0 : ((i & 1) << (bits - 1)) | brevc(i >> 1, bits - 1); }
__host__ __device__ constexpr int pow16(int e) { return e == 0 ? 1 : 16 * pow16(e - 1); }

// radix-2 DIF level with half-span H on R registers starting at v[O], stride D
template <int R, int H, bool INV>
struct DifLevel {
  template <int I>
  __device__ __forceinline__ static void bf(float2 *v) {
    if constexpr (I < R) {
      if constexpr ((I & H) == 0) {
        constexpr int k = I & (H - 1);
        constexpr int e = k * (8 / H);  // W_{2H}^k in 16ths
        float2 a = v[I], b = v[I + H];
        v[I] = cadd(a, b);
        v[I + H] = tw16<e, INV>(csub(a, b));
      }
      bf<I + 1>(v);
    }
  }
  __device__ __forceinline__ static void run(float2 *v) {
    bf<0>(v);
    if constexpr (H > 1) DifLevel<R, H / 2, INV>::run(v);
  }
};

template <int R, int I>
struct BrevPerm {
  __device__ __forceinline__ static void run(const float2 *v, float2 *t) {
    if constexpr (I < R) {
      constexpr int J = brevc(I, ilog2c(R));
      t[J] = v[I];
      BrevPerm<R, I + 1>::run(v, t);
    }
  }
};

// In-register DFT of size R (2, 4, 8, 16), natural order in and out.
template <int R, bool INV>
__device__ __forceinline__ void dft_reg(float2 *v) {
  DifLevel<R, R / 2, INV>::run(v);
  float2 t[R];
  BrevPerm<R, 0>::run(v, t);
#pragma unroll
  for (int i = 0; i < R; i++) v[i] = t[i];
}

template <int L>
struct Shape {
  static constexpr int LOG = ilog2c(L);
  static constexpr int S16 = (LOG - 1) / 4;  // radix-16 stages after the first
  static constexpr int F = L >> (4 * S16);   // first radix
  static constexpr int T = L / 16;           // threads per line
  static constexpr int PER = 16 / F;         // stage-0 butterflies per thread
  static constexpr int LP = L + L / 16;      // padded line (float2)
  // twiddle rows (4 float2 = 2 float4 each): sum over radix-16 stages of Ns
  static constexpr int TWROWS = F * (pow16(S16) - 1) / 15;
  static_assert(F == 2 || F == 4 || F == 8 || F == 16, "unsupported L");
  static_assert((1 << LOG) == L && L >= 128, "L must be a power of two >= 128");
};

// Exchange space of one line: two buffers of LP float2 at b and b + LPB.
struct Xch {
  float2 *b;
  int par;
  int stride;
  __device__ __forceinline__ float2 *next() {
#if HOLO_SINGLE_BUF
    __syncthreads();  // previous readers of the single buffer are done
    return b;
#else
    float2 *p = par ? b + stride : b;
    par ^= 1;
    return p;
#endif
  }
};

template <bool INV>
__device__ __forceinline__ void twmul(float2 &v, float2 w) { v = INV ? cmulc(v, w) : cmul(v, w); }

template <int L, bool INV, int ST>
__device__ __forceinline__ void r16_stage(float2 (&v)[16], Xch &x, const int t, const float4 *__restrict__ tw) {
  using S = Shape<L>;
  constexpr int Ns = S::F * pow16(ST);
  constexpr int ROW0 = S::F * (pow16(ST) - 1) / 15;
  const int m = t & (Ns - 1);
#if HOLO_TW_FULL
  {
    // full table: rows of 8 float4 = 16 float2 (entry 0 unused) per (stage, m)
    const float4 *row = tw + 8 * (ROW0 + m);
#pragma unroll
    for (int q = 0; q < 8; q++) {
      const float4 a = __ldg(row + q);
      if (q > 0) twmul<INV>(v[2 * q], make_float2(a.x, a.y));
      twmul<INV>(v[2 * q + 1], make_float2(a.z, a.w));
    }
  }
#else
  {
    const float4 a = __ldg(tw + 2 * (ROW0 + m)), b = __ldg(tw + 2 * (ROW0 + m) + 1);
    const float2 w1 = make_float2(a.x, a.y), w2 = make_float2(a.z, a.w), w4 = make_float2(b.x, b.y),
                 w8 = make_float2(b.z, b.w);
    twmul<INV>(v[1], w1);
    twmul<INV>(v[2], w2);
    twmul<INV>(v[4], w4);
    twmul<INV>(v[8], w8);
    const float2 w3 = cmul(w1, w2), w5 = cmul(w1, w4), w6 = cmul(w2, w4), w7 = cmul(w3, w4);
    twmul<INV>(v[3], w3);
    twmul<INV>(v[5], w5);
    twmul<INV>(v[6], w6);
    twmul<INV>(v[7], w7);
    twmul<INV>(v[9], cmul(w1, w8));
    twmul<INV>(v[10], cmul(w2, w8));
    twmul<INV>(v[11], cmul(w3, w8));
    twmul<INV>(v[12], cmul(w4, w8));
    twmul<INV>(v[13], cmul(w5, w8));
    twmul<INV>(v[14], cmul(w6, w8));
    twmul<INV>(v[15], cmul(w7, w8));
  }
#endif
  dft_reg<16, INV>(v);
  if constexpr (ST + 1 < S::S16) {
    float2 *buf = x.next();
    const int base = (t - m) * 16 + m;
#pragma unroll
    for (int s = 0; s < 16; s++) buf[P(base + s * Ns)] = v[s];
    __syncthreads();
#pragma unroll
    for (int r = 0; r < 16; r++) v[r] = buf[P(t + r * S::T)];
    r16_stage<L, INV, ST + 1>(v, x, t, tw);
  }
}

// In-place transform of the line held in layout S (unnormalised; INV: exp(+...)).
template <int L, bool INV>
__device__ __forceinline__ void fft(float2 (&v)[16], Xch &x, const int t, const float4 *__restrict__ tw) {
  using S = Shape<L>;
  constexpr int F = S::F, PER = S::PER;
#pragma unroll
  for (int b = 0; b < PER; b++) {
    float2 u[F];
#pragma unroll
    for (int s = 0; s < F; s++) u[s] = v[b + PER * s];
    dft_reg<F, INV>(u);
#pragma unroll
    for (int s = 0; s < F; s++) v[b + PER * s] = u[s];
  }
  float2 *buf = x.next();
#pragma unroll
  for (int b = 0; b < PER; b++)
#pragma unroll
    for (int s = 0; s < F; s++) buf[P((t + S::T * b) * F + s)] = v[b + PER * s];
  __syncthreads();
#pragma unroll
  for (int r = 0; r < 16; r++) v[r] = buf[P(t + r * S::T)];
  r16_stage<L, INV, 0>(v, x, t, tw);
}

}  // namespace holo
