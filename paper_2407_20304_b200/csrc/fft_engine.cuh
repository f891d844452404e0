// fft_engine.cuh -- shared-memory Stockham line FFT for sm_100a.
//
// One "group" of TPL = L/16 threads transforms one length-L complex64 line that
// lives in shared memory.  A CTA runs G groups side by side on G line buffers
// (all groups pass the same __syncthreads(), so every thread of the CTA must call
// the transform even when its group has no line: active = false).
//
// Factorisation: L = F * 16^s with a first radix F in {2, 4, 8, 16} (Ns = 1, no
// twiddles) followed by s radix-16 Stockham stages (self-sorting, natural order
// in and out).  Each radix-16 butterfly is done in registers (radix-2 DIF with
// compile-time twiddles); stage twiddles exp(-2 pi i m r / (16 Ns)) come from an
// fp64-generated table laid out [stage][r-1][m] so consecutive threads read
// consecutive entries.
//
// Shared-memory layout: element i of a line sits at P(i) = i + (i >> 4) (one pad
// slot every 16 complex) which makes both the strided reads and the radix-16 /
// radix-F Stockham scatters bank-conflict free for 64-bit accesses.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace holo {

__device__ __forceinline__ int P(int i) { return i + (i >> 4); }

// Read-only table load that the compiler may not hoist or CSE across transforms
// (keeping a whole stage of twiddles live across FFT calls costs ~60 registers).
__device__ __forceinline__ float2 ldtw(const float2 *p) {
  float2 v;
  asm volatile("ld.global.nc.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "l"(p));
  return v;
}

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

// Multiply by W16^e = exp(-+2 pi i e / 16) (forward: minus), e in [0, 8), compile-time.
template <int E, bool INV>
__device__ __forceinline__ float2 tw16(float2 x) {
  constexpr float C1 = 0.92387953251128674f, S1 = 0.38268343236508977f, H = 0.70710678118654752f;
  // forward: x * (c - i s);  inverse: x * (c + i s)
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

// radix-2 DIF level with half-span H on R registers
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

// compile-time bit-reversal permutation of R registers (pure renaming after inlining)
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
struct FftShape {
  static constexpr int S16 = (ilog2c(L) - 1) / 4;  // radix-16 stages
  static constexpr int F = L >> (4 * S16);          // first radix (2, 4, 8 or 16)
  static constexpr int TPL = L / 16;                                                // threads per line
  static_assert(F == 2 || F == 4 || F == 8 || F == 16, "unsupported L");
  static_assert((1 << ilog2c(L)) == L, "L must be a power of two");
  static constexpr int TW = L - F;  // twiddle table entries (radix-16 stages)
};

// Stage twiddle table: after the first radix-F stage (Ns = 1, no twiddles) the
// radix-16 stages have Ns = F, 16F, 256F, ...; stage Ns uses 15*Ns entries
// [(r-1)*Ns + m] = exp(-2 pi i m r / (16 Ns)) at offset sum_{previous} 15*Ns.

// Transform a padded smem line in place.  t = thread index in the group [0, TPL).
template <int L, bool INV>
__device__ __noinline__ void fft_line(float2 *buf, const float2 *__restrict__ tw, int t, bool active) {
  using S = FftShape<L>;
  constexpr int TPL = S::TPL;
  constexpr int F = S::F;
  // ---- first stage: radix F, Ns = 1, 16/F butterflies per thread
  {
    constexpr int NB = L / F;
    constexpr int PER = 16 / F;
    float2 v[PER][F];
    if (active) {
#pragma unroll
      for (int b = 0; b < PER; b++)
#pragma unroll
        for (int r = 0; r < F; r++) v[b][r] = buf[P(t + b * TPL + r * NB)];
    }
    __syncthreads();
    if (active) {
#pragma unroll
      for (int b = 0; b < PER; b++) {
        dft_reg<F, INV>(v[b]);
        const int j = t + b * TPL;
#pragma unroll
        for (int r = 0; r < F; r++) buf[P(j * F + r)] = v[b][r];
      }
    }
    __syncthreads();
  }
  // ---- radix-16 stages
  int off = 0;
#pragma unroll
  for (int st = 0, Ns = F; st < S::S16; st++, Ns *= 16) {
    constexpr int NB = L / 16;  // == TPL
    float2 v[16];
    if (active) {
#pragma unroll
      for (int r = 0; r < 16; r++) v[r] = buf[P(t + r * NB)];
    }
    __syncthreads();
    if (active) {
      const int m = t & (Ns - 1);
      const float2 *tws = tw + off + m;
#pragma unroll
      for (int r = 1; r < 16; r++) {
        float2 w = ldtw(tws + (r - 1) * Ns);
        v[r] = INV ? cmulc(v[r], w) : cmul(v[r], w);
      }
      dft_reg<16, INV>(v);
      const int base = (t - m) * 16 + m;
#pragma unroll
      for (int r = 0; r < 16; r++) buf[P(base + r * Ns)] = v[r];
    }
    __syncthreads();
    off += 15 * Ns;
  }
}

}  // namespace holo
