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

// Exchange padding.  HOLO_PAD2=1 (measured 3 % slower, off): P(i) = i + 2 (i / 16) keeps every 16-element run
// 16-byte aligned, so a thread's contiguous first-stage run is written with STS.128 (half the
// store instructions of the MIO-throttled exchange); reads stay one 128-byte wavefront per
// 16 lanes.  HOLO_PAD2=0 (default): the round-1 padding i + i/16.
#ifndef HOLO_PAD2
#define HOLO_PAD2 0
#endif
__device__ __forceinline__ int P(int i) { return HOLO_PAD2 ? i + 2 * (i >> 4) : i + (i >> 4); }

// Complex arithmetic.  HOLO_FFMA2=1: Blackwell's packed f32x2 instructions (FADD2 / FMUL2 /
// FFMA2) on the (re, im) pair, whose operand modifiers swap the halves (.LO_HI), negate one half
// (.NP) or broadcast a scalar (.F32): a complex multiply is FMUL2 + FFMA2 (2 issue slots instead
// of 4), a twiddled butterfly 3 FFMA2 instead of 6 FFMA (-35 % FP32 SASS instructions in the
// engine).  MEASURED SLOWER (tools/fftbench2.cu: 39.2 vs 35.45 us per 4096^2 set at 512 threads;
// cfg3 sweep 907.6 vs 949.3 frame-it/s, profiles/r02_ffma2.log): the FP32 pipe is bound by lane
// operations, not by issue slots, so the default stays HOLO_FFMA2=0 (scalar FP32).
#ifndef HOLO_FFMA2
#define HOLO_FFMA2 0
#endif
#if HOLO_FFMA2
__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return __fadd2_rn(a, make_float2(-b.x, -b.y)); }
__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
  // (ax bx - ay by, ax by + ay bx) = ax (bx, by) + ay (-by, bx)
  return __ffma2_rn(make_float2(a.y, a.y), make_float2(-b.y, b.x), __fmul2_rn(make_float2(a.x, a.x), b));
}
// a * conj(b) = (ax bx + ay by, ay bx - ax by) = ax (bx, -by) + ay (by, bx)
__device__ __forceinline__ float2 cmulc(float2 a, float2 b) {
  return __ffma2_rn(make_float2(a.y, a.y), make_float2(b.y, b.x), __fmul2_rn(make_float2(a.x, a.x), make_float2(b.x, -b.y)));
}
__device__ __forceinline__ float2 cscale(float2 a, float s) { return __fmul2_rn(a, make_float2(s, s)); }
#else
__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
  return make_float2(fmaf(a.x, b.x, -a.y * b.y), fmaf(a.x, b.y, a.y * b.x));
}
// a * conj(b)
__device__ __forceinline__ float2 cmulc(float2 a, float2 b) {
  return make_float2(fmaf(a.x, b.x, a.y * b.y), fmaf(a.y, b.x, -a.x * b.y));
}
__device__ __forceinline__ float2 cscale(float2 a, float s) { return make_float2(a.x * s, a.y * s); }
#endif
__device__ __forceinline__ float2 cconj(float2 a) { return make_float2(a.x, -a.y); }
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

// ---- radix-16 as a twiddle-absorbing DIT with FMA-fused butterflies (HOLO_DIT, default) ----
// A twiddled radix-16 Stockham step computes y[k] = sum_s v[s] w^{ms} W16^{sk} = sum_s v[s] z_k^s,
// z_k = omega W16^k (omega = w^m).  Radix-2 DIT on the bit-reversed register order: the level
// with span H combines sub-DFTs with twiddles omega^{8/H} W_{2H}^k, k < H, so the four table
// powers (omega, omega^2, omega^4, omega^8) plus 4 constant products are all the twiddles
// needed, and every butterfly (a + t b, a - t b) costs 6 FP32 instructions (4 FFMA for
// p = a + t b, then q = 2 a - p).  Per 16 points: 208 instructions for a twiddled stage and
// 148 for the untwiddled first stage, against 272 / 168 for DIF + separate twiddle multiplies.
#ifndef HOLO_DIT
#define HOLO_DIT 1
#endif
// HOLO_TW8=1: each stage-twiddle row also holds the DIT level twiddles omega e^{-i pi/8},
// omega e^{-i pi/4}, omega e^{-3 i pi/8}, omega^2 e^{-i pi/4} (fp64-generated, 64-byte rows), so the
// 16 FP32 instructions that derive them per twiddled stage become two more L1-resident loads.
// 0 (default): 32-byte rows (omega, omega^2, omega^4, omega^8), level twiddles derived in registers.
// MEASURED SLOWER with 1 (tools/fftbench2.cu 35.65 vs 35.40 us per 4096^2 set at 512 threads, 35.03 vs
// 32.06 at 2 x 256; cfg3 sweep 926.2 vs 947.7 frame-it/s, profiles/r02_tw8.log): the extra loads
// cost more on the L1 / shared-memory path than the FP32 instructions they remove.
#ifndef HOLO_TW8
#define HOLO_TW8 0
#endif
constexpr int TW_ROW_F2 = HOLO_TW8 ? 8 : 4;  // float2 per twiddle row (the host builds the same rows)

// (a, b) <- (a + t b, a - t b), runtime twiddle t
__device__ __forceinline__ void bfly(float2 &a, float2 &b, float2 t) {
#if HOLO_FFMA2
  // p = a + tx (bx, by) + ty (-by, bx);  q = 2 a - p      (3 FFMA2, the same roundings per lane)
  float2 p = __ffma2_rn(make_float2(t.x, t.x), b, a);
  p = __ffma2_rn(make_float2(t.y, t.y), make_float2(-b.y, b.x), p);
  b = __ffma2_rn(make_float2(2.f, 2.f), a, make_float2(-p.x, -p.y));
  a = p;
#else
  float px = fmaf(t.x, b.x, a.x);
  px = fmaf(-t.y, b.y, px);
  float py = fmaf(t.x, b.y, a.y);
  py = fmaf(t.y, b.x, py);
  b = make_float2(fmaf(2.f, a.x, -px), fmaf(2.f, a.y, -py));
  a = make_float2(px, py);
#endif
}
// (a, b) <- (a + t b, a - t b), t = W16^E (forward, e^{-2 pi i E/16}) or its conjugate (INV)
template <int E, bool INV>
__device__ __forceinline__ void bfly_c(float2 &a, float2 &b) {
  if constexpr (E == 0) {
    const float2 p = cadd(a, b);
    b = csub(a, b);
    a = p;
  } else if constexpr (E == 4) {  // t = -i (fwd) / +i (inv)
    const float2 tb = INV ? make_float2(-b.y, b.x) : make_float2(b.y, -b.x);
    const float2 p = cadd(a, tb);
    b = csub(a, tb);
    a = p;
  } else {
    constexpr float C1 = 0.92387953251128674f, S1 = 0.38268343236508977f, H = 0.70710678118654752f;
    constexpr float c = (E == 1) ? C1 : (E == 2) ? H : (E == 3) ? S1 : (E == 5) ? -S1 : (E == 6) ? -H : -C1;
    constexpr float sn = (E == 1) ? S1 : (E == 2) ? H : (E == 3) ? C1 : (E == 5) ? C1 : (E == 6) ? H : S1;
    bfly(a, b, make_float2(c, INV ? sn : -sn));
  }
}
__host__ __device__ constexpr int brev4(int i) { return ((i & 1) << 3) | ((i & 2) << 1) | ((i & 4) >> 1) | ((i & 8) >> 3); }

// untwiddled 16-point DFT, natural order in and out (first Stockham stage)
template <bool INV>
__device__ __forceinline__ void dft16_dit(float2 *v) {
  float2 a[16];
#pragma unroll
  for (int i = 0; i < 16; i++) a[i] = v[brev4(i)];
#pragma unroll
  for (int j = 0; j < 16; j += 2) bfly_c<0, INV>(a[j], a[j + 1]);
#pragma unroll
  for (int j = 0; j < 16; j += 4) {
    bfly_c<0, INV>(a[j], a[j + 2]);
    bfly_c<4, INV>(a[j + 1], a[j + 3]);
  }
#pragma unroll
  for (int j = 0; j < 16; j += 8) {
    bfly_c<0, INV>(a[j], a[j + 4]);
    bfly_c<2, INV>(a[j + 1], a[j + 5]);
    bfly_c<4, INV>(a[j + 2], a[j + 6]);
    bfly_c<6, INV>(a[j + 3], a[j + 7]);
  }
  bfly_c<0, INV>(a[0], a[8]);
  bfly_c<1, INV>(a[1], a[9]);
  bfly_c<2, INV>(a[2], a[10]);
  bfly_c<3, INV>(a[3], a[11]);
  bfly_c<4, INV>(a[4], a[12]);
  bfly_c<5, INV>(a[5], a[13]);
  bfly_c<6, INV>(a[6], a[14]);
  bfly_c<7, INV>(a[7], a[15]);
#pragma unroll
  for (int i = 0; i < 16; i++) v[i] = a[i];
}

// twiddled 16-point step: y[k] = sum_s v[s] (omega W16^k)^s, given omega^{1,2,4,8} and the level
// twiddles t1 = omega e^{-i pi/8}, t2 = omega e^{-i pi/4}, t3 = omega e^{-3 i pi/8}, s1 = omega^2 e^{-i pi/4}
// (forward convention; INV uses the conjugates)
template <bool INV>
__device__ __forceinline__ void dft16_dit_tw8(float2 *v, float2 w1, float2 w2, float2 w4, float2 w8, float2 t1,
                                              float2 t2, float2 t3, float2 s1) {
  auto mi = [](float2 z) { return make_float2(z.y, -z.x); };  // -i z
  auto cj = [](float2 z) { return INV ? make_float2(z.x, -z.y) : z; };
  const float2 t0 = w1, s0 = w2;
  float2 a[16];
#pragma unroll
  for (int i = 0; i < 16; i++) a[i] = v[brev4(i)];
  {
    const float2 t = cj(w8);
#pragma unroll
    for (int j = 0; j < 16; j += 2) bfly(a[j], a[j + 1], t);
  }
  {
    const float2 u0 = cj(w4), u1 = cj(mi(w4));
#pragma unroll
    for (int j = 0; j < 16; j += 4) {
      bfly(a[j], a[j + 2], u0);
      bfly(a[j + 1], a[j + 3], u1);
    }
  }
  {
    const float2 q0 = cj(s0), q1 = cj(s1), q2 = cj(mi(s0)), q3 = cj(mi(s1));
#pragma unroll
    for (int j = 0; j < 16; j += 8) {
      bfly(a[j], a[j + 4], q0);
      bfly(a[j + 1], a[j + 5], q1);
      bfly(a[j + 2], a[j + 6], q2);
      bfly(a[j + 3], a[j + 7], q3);
    }
  }
  bfly(a[0], a[8], cj(t0));
  bfly(a[1], a[9], cj(t1));
  bfly(a[2], a[10], cj(t2));
  bfly(a[3], a[11], cj(t3));
  bfly(a[4], a[12], cj(mi(t0)));
  bfly(a[5], a[13], cj(mi(t1)));
  bfly(a[6], a[14], cj(mi(t2)));
  bfly(a[7], a[15], cj(mi(t3)));
#pragma unroll
  for (int i = 0; i < 16; i++) v[i] = a[i];
}
// the same with the level twiddles derived from omega in registers (HOLO_TW8 = 0)
template <bool INV>
__device__ __forceinline__ void dft16_dit_tw(float2 *v, float2 w1, float2 w2, float2 w4, float2 w8) {
  constexpr float C1 = 0.92387953251128674f, S1 = 0.38268343236508977f, H = 0.70710678118654752f;
  const float2 t1 = make_float2(fmaf(w1.x, C1, w1.y * S1), fmaf(w1.y, C1, -w1.x * S1)),
               t2 = make_float2((w1.x + w1.y) * H, (w1.y - w1.x) * H),
               t3 = make_float2(fmaf(w1.x, S1, w1.y * C1), fmaf(w1.y, S1, -w1.x * C1));
  const float2 s1 = make_float2((w2.x + w2.y) * H, (w2.y - w2.x) * H);
  dft16_dit_tw8<INV>(v, w1, w2, w4, w8, t1, t2, t3, s1);
}
// one stage-twiddle row (TW_ROW_F2 float2) -> the twiddled 16-point step
template <bool INV>
__device__ __forceinline__ void dft16_row(float2 *v, const float4 *__restrict__ row) {
  const float4 a = __ldg(row), b = __ldg(row + 1);
#if HOLO_TW8
  const float4 c = __ldg(row + 2), d = __ldg(row + 3);
  dft16_dit_tw8<INV>(v, make_float2(a.x, a.y), make_float2(a.z, a.w), make_float2(b.x, b.y), make_float2(b.z, b.w),
                     make_float2(c.x, c.y), make_float2(c.z, c.w), make_float2(d.x, d.y), make_float2(d.z, d.w));
#else
  dft16_dit_tw<INV>(v, make_float2(a.x, a.y), make_float2(a.z, a.w), make_float2(b.x, b.y), make_float2(b.z, b.w));
#endif
}

template <int L>
struct Shape {
  static constexpr int LOG = ilog2c(L);
  static constexpr int S16 = (LOG - 1) / 4;  // radix-16 stages after the first
  static constexpr int F = L >> (4 * S16);   // first radix
  static constexpr int T = L / 16;           // threads per line
  static constexpr int PER = 16 / F;         // stage-0 butterflies per thread
  static constexpr int LP = L + (HOLO_PAD2 ? 2 : 1) * (L / 16);  // padded line (float2)
  // twiddle rows (4 float2 = 2 float4 each): sum over radix-16 stages of Ns
  static constexpr int TWROWS = F * (pow16(S16) - 1) / 15;
  static_assert(F == 2 || F == 4 || F == 8 || F == 16, "unsupported L");
  static_assert((1 << LOG) == L && L >= 128, "L must be a power of two >= 128");
};

// Line-local barrier (HOLO_LINE_BAR): with the thread-major CTA mapping (HOLO_TMAJOR) the
// T threads of a line are whole warps (T >= 64: named barrier 1 + line, T threads) or live
// inside one warp (T <= 32: __syncwarp), so the lines of a CTA synchronise independently and
// one line's shared-memory exchange overlaps another line's butterflies.
#ifndef HOLO_TMAJOR
#define HOLO_TMAJOR 0
#endif
template <int T>
__device__ __forceinline__ void line_sync(int g) {
#if HOLO_TMAJOR
  if constexpr (T <= 32) {
    __syncwarp();
  } else {
    asm volatile("bar.sync %0, %1;" ::"r"(1 + g), "n"(T) : "memory");
  }
#else
  __syncthreads();
#endif
}

// Exchange space of one line: two buffers of LP float2 at b and b + LPB.
struct Xch {
  float2 *b;
  int par;
  int stride;
  int g;  // line of this thread within the CTA (named barrier id - 1)
  template <int T>
  __device__ __forceinline__ float2 *next() {
#if HOLO_SINGLE_BUF
    line_sync<T>(g);  // previous readers of the single buffer are done
    return b;
#else
    float2 *p = par ? b + stride : b;
    par ^= 1;
    return p;
#endif
  }
  template <int T>
  __device__ __forceinline__ void sync() { line_sync<T>(g); }
};

template <bool INV>
__device__ __forceinline__ void twmul(float2 &v, float2 w) { v = INV ? cmulc(v, w) : cmul(v, w); }

template <int L, bool INV, int ST>
__device__ __forceinline__ void r16_stage(float2 (&v)[16], Xch &x, const int t, const float4 *__restrict__ tw) {
  using S = Shape<L>;
  constexpr int Ns = S::F * pow16(ST);
  constexpr int ROW0 = S::F * (pow16(ST) - 1) / 15;
  const int m = t & (Ns - 1);
#if HOLO_DIT
  dft16_row<INV>(v, tw + (TW_ROW_F2 / 2) * (ROW0 + m));
#elif HOLO_TW_FULL
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
    const float4 a = __ldg(tw + (TW_ROW_F2 / 2) * (ROW0 + m)), b = __ldg(tw + (TW_ROW_F2 / 2) * (ROW0 + m) + 1);
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
#if !HOLO_DIT
  dft_reg<16, INV>(v);
#endif
  if constexpr (ST + 1 < S::S16) {
    float2 *buf = x.next<S::T>();
    const int base = (t - m) * 16 + m;
#pragma unroll
    for (int s = 0; s < 16; s++) buf[P(base + s * Ns)] = v[s];
    x.sync<S::T>();
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
    if constexpr (F == 16 && HOLO_DIT)
      dft16_dit<INV>(u);
    else
      dft_reg<F, INV>(u);
#pragma unroll
    for (int s = 0; s < F; s++) v[b + PER * s] = u[s];
  }
  float2 *buf = x.next<S::T>();
#if HOLO_PAD2
  // each run of F outputs is contiguous (and, for L >= 1024 where the line buffers' skew is even,
  // 16-byte aligned) in the padded buffer: STS.128
  if constexpr (L >= 1024) {
#pragma unroll
  for (int b = 0; b < PER; b++) {
    float4 *dst = reinterpret_cast<float4 *>(buf + P((t + S::T * b) * F));
#pragma unroll
    for (int s = 0; s < F; s += 2) {
      const float2 lo = v[b + PER * s], hi = v[b + PER * (s + 1)];
      dst[s / 2] = make_float4(lo.x, lo.y, hi.x, hi.y);
    }
  }
  } else {
#pragma unroll
    for (int b = 0; b < PER; b++)
#pragma unroll
      for (int s = 0; s < F; s++) buf[P((t + S::T * b) * F + s)] = v[b + PER * s];
  }
#else
#pragma unroll
  for (int b = 0; b < PER; b++)
#pragma unroll
    for (int s = 0; s < F; s++) buf[P((t + S::T * b) * F + s)] = v[b + PER * s];
#endif
  x.sync<S::T>();
#pragma unroll
  for (int r = 0; r < 16; r++) v[r] = buf[P(t + r * S::T)];
  r16_stage<L, INV, 0>(v, x, t, tw);
}

}  // namespace holo

namespace holo {

// ---- NV independent lines per thread (the 6144 = 3 x 2048 engine of holo_ref.cuh) -------------
// Thread t holds NV lines of length L in layout S, line s in v[16 s .. 16 s + 15].  The NV
// transforms run stage by stage in lockstep, so each exchange is ONE barrier pair for all NV lines
// (their buffers at buf + s * bstride) and the butterflies of one line overlap the shared-memory
// traffic of another.  Every thread of the CTA must call it (CTA barriers).
template <int L, bool INV, int NV, int ST>
__device__ __forceinline__ void r16_stage_nv(float2 (&v)[NV * 16], float2 *buf, int bstride, const int t,
                                             const float4 *__restrict__ tw) {
  using S = Shape<L>;
  constexpr int Ns = S::F * pow16(ST);
  constexpr int ROW0 = S::F * (pow16(ST) - 1) / 15;
  const int m = t & (Ns - 1);
  {
    const float4 *row = tw + (TW_ROW_F2 / 2) * (ROW0 + m);
    const float4 a = __ldg(row), b = __ldg(row + 1);
    const float2 w1 = make_float2(a.x, a.y), w2 = make_float2(a.z, a.w), w4 = make_float2(b.x, b.y),
                 w8 = make_float2(b.z, b.w);
#if HOLO_TW8
    const float4 c = __ldg(row + 2), d = __ldg(row + 3);
    const float2 t1 = make_float2(c.x, c.y), t2 = make_float2(c.z, c.w), t3 = make_float2(d.x, d.y),
                 s1 = make_float2(d.z, d.w);
#pragma unroll
    for (int s = 0; s < NV; s++) dft16_dit_tw8<INV>(v + 16 * s, w1, w2, w4, w8, t1, t2, t3, s1);
#else
#pragma unroll
    for (int s = 0; s < NV; s++) dft16_dit_tw<INV>(v + 16 * s, w1, w2, w4, w8);
#endif
  }
  if constexpr (ST + 1 < S::S16) {
    const int base = (t - m) * 16 + m;
    __syncthreads();  // the previous exchange's readers are done with buf
#pragma unroll
    for (int s = 0; s < NV; s++)
#pragma unroll
      for (int q = 0; q < 16; q++) buf[s * bstride + P(base + q * Ns)] = v[16 * s + q];
    __syncthreads();
#pragma unroll
    for (int s = 0; s < NV; s++)
#pragma unroll
      for (int r = 0; r < 16; r++) v[16 * s + r] = buf[s * bstride + P(t + r * S::T)];
    r16_stage_nv<L, INV, NV, ST + 1>(v, buf, bstride, t, tw);
  }
}

template <int L, bool INV, int NV>
__device__ __forceinline__ void fft_nv(float2 (&v)[NV * 16], float2 *buf, int bstride, const int t,
                                       const float4 *__restrict__ tw) {
  using S = Shape<L>;
  constexpr int F = S::F, PER = S::PER;
#pragma unroll
  for (int s = 0; s < NV; s++) {
#pragma unroll
    for (int b = 0; b < PER; b++) {
      float2 u[F];
#pragma unroll
      for (int k = 0; k < F; k++) u[k] = v[16 * s + b + PER * k];
      if constexpr (F == 16 && HOLO_DIT)
        dft16_dit<INV>(u);
      else
        dft_reg<F, INV>(u);
#pragma unroll
      for (int k = 0; k < F; k++) v[16 * s + b + PER * k] = u[k];
    }
  }
  __syncthreads();
#pragma unroll
  for (int s = 0; s < NV; s++)
#pragma unroll
    for (int b = 0; b < PER; b++)
#pragma unroll
      for (int k = 0; k < F; k++) buf[s * bstride + P((t + S::T * b) * F + k)] = v[16 * s + b + PER * k];
  __syncthreads();
#pragma unroll
  for (int s = 0; s < NV; s++)
#pragma unroll
    for (int r = 0; r < 16; r++) v[16 * s + r] = buf[s * bstride + P(t + r * S::T)];
  r16_stage_nv<L, INV, NV, 0>(v, buf, bstride, t, tw);
}

}  // namespace holo
