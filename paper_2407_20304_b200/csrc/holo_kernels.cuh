// holo_kernels.cuh -- CTA layout, line I/O and the fused magnification
// (Bluestein chirp-z) building blocks of the holotomography sweep (sm_100a).
//
// Per frame (k, j) the operator chain of Eq. (8) and its adjoint
// (L* formula P:123) is applied as five separable line passes ("Pass
// schedule"): X = rows (contiguous), Y = columns:
//
//   X1 (per k)   psi_k row: FFT once, then per plane j:  M_{1/mt_j} S_x   -> T1_j
//   Y1 (k, j)    T1_j col:  M_{1/mt_j} S_y -> a (stored), x q_j, D_y, crop rows -> W1
//   X2 (k, j)    W1 row:    D_x, crop, residual + F (Eq. (10)-(11)), zero-pad, D_x^* -> V1
//   Y2 (k, j)    V1 col:    pad, D_y^* -> v; G_j += conj(a) v; conj(q_j) v, (M S)_y^* -> T3_j
//   X3 (per k)   T3_j rows: (M S)_x^* accumulated over j in the Fourier domain, one
//                inverse FFT, x2 -> grad_psi_k, fused ||g||^2 and Re<g, eta> partials
//
// Every line lives in registers in layout S (fft_engine.cuh) from its load to its
// store; all pointwise factors are applied there.
//
// Magnification M_{1/mt} (reading C1), Bluestein's chirp-z, in layout S:
//   spectrum X = FFT(x);  a[i] = cr[f] X[f],  i = (f + L/2) mod L   (register r -> r^8)
//   cr = kappa (-1)^fbar e^{i pi mt fbar^2/L} r_s[f] / L   (chirp x shift ramp, per (k, j, axis))
//   E = IFFT(FFT(a) Bhat_e),  O = IFFT(FFT(a w) Bhat_o),  w[i] = e^{-i pi i/L}
//   y[o] = cout[o] (E[o] + conj(w[o]) O[o]),   cout = e^{i pi mt (o-L/2)^2/L}
// i.e. the 2L-point cyclic convolution with b[d] = e^{-i pi mt d^2/L} split into its
// even/odd spectral halves.  The adjoint runs the same steps conjugated and in reverse.
// All tables are fp64-generated on the host, phases reduced in cycles.
#pragma once
#include "fft_engine.cuh"
#include "tma.cuh"

namespace holo {

struct Tables {
  const float4 *tw;     // FFT stage twiddle rows (w^m, w^2m | w^4m, w^8m)
  const float2 *hdet;   // [nz][L] h_{zdet_j}[f] / L
  const float2 *homega; // [nz][L] h_{omega_j}[f] (unscaled)
  const float2 *cout;   // [nz][L] e^{i pi mt (o - L/2)^2 / L}
  const float2 *bke;    // [nz][L] Bhat[2k] / (2L)
  const float2 *bko;    // [nz][L] Bhat[2k+1] / (2L)
  const float2 *cr;     // [K][nz][2][L] spectrum factor per (k, j, axis): mag: cin r_s, else r_s / L
};

// CTA geometry: NT threads, G = NT / T lines per CTA, threads mapped g-major
// (g = tid % G, t = tid / G): one warp covers G adjacent lines (rows or columns)
// at 32/G consecutive positions, which is what the P2 layout below needs for full
// 32-byte sectors in both directions.
template <int L, int NT_ = 512>
struct Cta {
  static constexpr int T = Shape<L>::T;
  static constexpr int NT = NT_;
  static constexpr int G = NT / T;
  static constexpr int LP = Shape<L>::LP;
  static constexpr int LPB = (LP + 15) / 16 * 16;  // one buffer, 16-float2 aligned
  // per-group stride (two buffers) skewed so that the groups sharing a 16-lane
  // phase land on distinct banks
  static constexpr int SKEW = G <= 16 ? 16 / G : 1;  // 16 lines/warp-half pairs on distinct banks; even for G <= 8
  static constexpr int GS = (HOLO_SINGLE_BUF ? 1 : 2) * LPB + SKEW;
  static constexpr size_t XBYTES = sizeof(float2) * (size_t)GS * G;
  static constexpr size_t PRIV = sizeof(float2) * 16 * NT;  // one thread-private line
#if HOLO_TMAJOR
  __device__ __forceinline__ static int g() { return threadIdx.x / T; }
  __device__ __forceinline__ static int t() { return threadIdx.x % T; }
#else
  __device__ __forceinline__ static int g() { return threadIdx.x % G; }
  __device__ __forceinline__ static int t() { return threadIdx.x / G; }
#endif
  __device__ __forceinline__ static Xch xch(float2 *sm) { return Xch{sm + (size_t)g() * GS, 0, LPB, g()}; }
};

// P2 layout ("column-pair interleaved") of an R x L complex64 workspace array:
// element (y, x) at ((x >> 1) R + y) 2 + (x & 1).  A column pair is one contiguous
// block of 16 R bytes (column passes stream it like a row); two adjacent rows of a
// row pass fill whole 32-byte sectors.
__device__ __forceinline__ size_t p2(int y, int x, int R) { return ((size_t)(x >> 1) * R + y) * 2 + (x & 1); }

// thread-private spill slot of 16 float2 (conflict free: consecutive threads, consecutive slots)
template <int NT>
struct Priv {
  float2 *p;
  __device__ __forceinline__ float2 &operator[](int r) const { return p[r * NT + threadIdx.x]; }
};

// Fire-and-forget accumulate (REDG.ADD.F32x2): for accumulators with ONE writer thread per
// element (a column's owner across the batch, a row's owner across planes), so the result is the
// same sequential sum as a read-modify-write, without the load round trip (fp32 RN; the L2 ALU
// flushes denormals, irrelevant at |x| >> 1e-38).  A later read by the same thread uses __ldcg.
__device__ __forceinline__ void red_add2(float2 *p, float2 v) {
  asm volatile("red.global.add.v2.f32 [%0], {%1, %2};" ::"l"(p), "f"(v.x), "f"(v.y) : "memory");
}

// ---- residual of the penalty G_tau (App. A.3) ------------------------
// h(phi) = (phi^{tau/2} - a^tau)^2 with phi = |w|^2, a = sqrt(d~):  F += h(|w|^2),
// rho = h'(|w|^2) w = tau (|w|^tau - a^tau) |w|^{tau - 2} w  (the proposition's 2 L^*(H' . Lpsi)
// carries the remaining factor 2 in the gradient).  tau = 1 is F_1 (Eq. (10)): rho = w - a w/|w|;
// tau = 2 is F_2 (Eq. (9)): rho = 2 (|w|^2 - a^2) w.  rho = 0 where w = 0 (reading C7, all tau).
// tau is uniform over the launch, so the branches do not diverge.
// TM: 0 = tau 1, 1 = tau 2, 2 = general tau, -1 = decided at run time.  The kernels on the hot path
// are instantiated per TM so that only one branch is compiled into their (fully unrolled) loops:
// three interleaved unrolled branches cost instruction-cache misses in the 6144-point R2B pass.
template <int TM = -1>
__device__ __forceinline__ float2 residual_tau(float2 w, float a, float tau, double &acc) {
  const float m2 = w.x * w.x + w.y * w.y;
  if (TM == 0 || (TM < 0 && tau == 1.0f)) {
    const float m = sqrtf(m2);
    const float dm = m - a;
    acc += (double)(dm * dm);
    const float f = m > 0.f ? 1.0f - __fdividef(a, m) : 0.f;
    return cscale(w, f);
  }
  if (TM == 1 || (TM < 0 && tau == 2.0f)) {
    const float dm = m2 - a * a;
    acc += (double)dm * (double)dm;
    return cscale(w, 2.0f * dm);
  }
  const float wt = m2 > 0.f ? powf(m2, 0.5f * tau) : 0.f;  // |w|^tau
  const float at = a > 0.f ? powf(a, tau) : 0.f;
  const float dm = wt - at;
  acc += (double)dm * (double)dm;
  return m2 > 0.f ? cscale(w, tau * dm * (wt / m2)) : make_float2(0.f, 0.f);
}

// ---- layout-S line I/O ----------------------------------------------------------
template <int L>
__device__ __forceinline__ void ld_row(float2 (&v)[16], const float2 *__restrict__ row, int t) {
#pragma unroll
  for (int r = 0; r < 16; r++) v[r] = ldg2(row + t + r * (L / 16));
}
template <int L>
__device__ __forceinline__ void st_row(const float2 (&v)[16], float2 *__restrict__ row, int t) {
#pragma unroll
  for (int r = 0; r < 16; r++) row[t + r * (L / 16)] = v[r];
}
// column x of a row-major L x L array: element i at col[i * L]
template <int L>
__device__ __forceinline__ void ld_col(float2 (&v)[16], const float2 *__restrict__ col, int t) {
#pragma unroll
  for (int r = 0; r < 16; r++) v[r] = ldg2(col + (size_t)(t + r * (L / 16)) * L);
}
template <int L>
__device__ __forceinline__ void st_col(const float2 (&v)[16], float2 *__restrict__ col, int t) {
#pragma unroll
  for (int r = 0; r < 16; r++) col[(size_t)(t + r * (L / 16)) * L] = v[r];
}
// v *= tab (or conj(tab)) elementwise, tab indexed in layout S
template <int L, bool CONJ>
__device__ __forceinline__ void mul_tab(float2 (&v)[16], const float2 *__restrict__ tab, int t) {
#pragma unroll
  for (int r = 0; r < 16; r++) {
    const float2 w = ldg2(tab + t + r * (L / 16));
    v[r] = CONJ ? cmulc(v[r], w) : cmul(v[r], w);
  }
}

// ---- table pipeline --------------------------------------------------------------
// The pointwise factors of a launch (chirps, Bluestein kernel spectra, transfer
// functions: one length-L table per step) are streamed into two shared-memory slots
// by 1-D bulk copies (cp.async.bulk + mbarrier), each issued one transform ahead of
// its use: the FFT hides the L2 latency that a direct load would expose.  The
// launch's table sequence is a kernel parameter (built on the host).
constexpr int MAXTAB = 160;  // a batched launch chains the tables of up to 16 frames
struct TabSeq {
  const float2 *p[MAXTAB];
  int n;
};

// L2 prefetch of a contiguous block (16-byte aligned, multiple of 16 bytes)
__device__ __forceinline__ void prefetch_l2(const void *src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}

// the same for any block: its 16-byte-aligned interior (the bulk copy's alignment rule)
__device__ __forceinline__ void prefetch_l2_any(const void *src, uint32_t bytes) {
  const uintptr_t a = reinterpret_cast<uintptr_t>(src), b = (a + 15) & ~(uintptr_t)15, e = (a + bytes) & ~(uintptr_t)15;
  if (e > b) prefetch_l2(reinterpret_cast<const void *>(b), (uint32_t)(e - b));
}

// per-thread L2 prefetch of the sector holding p (no register, no scoreboard)
__device__ __forceinline__ void prefetch_l2_sector(const void *p) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p) : "memory");
}

__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

// Table slots: 2 (default; table i + 1 streams into the other slot while table i is in use)
// or 1 (HOLO_TAB_SLOTS=1, for two CTAs per SM: the slot is refilled by done() right after
// each use, so the load overlaps the transform that follows), or 0 (no slots: the steps read
// the tables from global memory at their use, L2 / L1 resident).
#ifndef HOLO_TAB_SLOTS
#define HOLO_TAB_SLOTS 2
#endif
template <int L>
struct TabPipe {
  static constexpr int SLOTS = HOLO_TAB_SLOTS;
  float2 *slot;   // SLOTS * L float2 of shared memory
  uint64_t *bar;  // SLOTS mbarriers in shared memory
  int used;       // tables taken so far (uniform over the CTA)
  static constexpr size_t BYTES = SLOTS * sizeof(float2) * L;

  __device__ __forceinline__ void issue(const TabSeq &q, int i) {
    if constexpr (SLOTS == 0) return;
    if (threadIdx.x == 0 && i < q.n) {
      fence_proxy_async();  // earlier generic reads of this slot precede the async write
      mbar_expect_tx(bar + (i & (SLOTS - 1)), L * sizeof(float2));
      bulk_g2s(slot + (i & (SLOTS - 1)) * L, q.p[i], L * sizeof(float2), bar + (i & (SLOTS - 1)));
    }
  }
  // all threads; starts the first table(s)
  __device__ __forceinline__ void start(const TabSeq &q, float2 *sm_slots, uint64_t *bars) {
    slot = sm_slots;
    bar = bars;
    used = 0;
    if constexpr (SLOTS == 0) return;  // tables read from global memory (L2 / L1) at their use
    if (threadIdx.x == 0) {
      for (int b = 0; b < SLOTS; b++) mbar_init(bar + b, 1);
      fence_mbar_init();
    }
    __syncthreads();
    for (int b = 0; b < SLOTS; b++) issue(q, b);
  }
  // Table i = used.  Two slots: wait for it, then refill the other slot with table i + 1 (its
  // previous content, table i - 1, was consumed before a transform barrier; pass sync = true
  // when no transform separates the use of table i - 1 from this call).  One slot: just wait
  // (done() refilled it).
  __device__ __forceinline__ const float2 *take(const TabSeq &q, bool sync = false) {
    const int i = used++;
    if constexpr (SLOTS == 0) {
      return q.p[i];
    } else if constexpr (SLOTS == 2) {
      if (i >= 1) {
        // the slot being refilled held table i - 1: every LINE must be done with it.  The
        // transforms' barriers guarantee that only within a line when lines sync
        // independently (HOLO_TMAJOR), so then the CTA syncs here.
        if (sync || HOLO_TMAJOR) __syncthreads();
        issue(q, i + 1);
      }
      mbar_wait(bar + (i & 1), (i >> 1) & 1);
      return slot + (i & 1) * L;
    } else {
      mbar_wait(bar, i & 1);
      return slot;
    }
  }
  // after the last read of the table just taken (all threads): one slot -> refill it now
  __device__ __forceinline__ void done(const TabSeq &q) {
    if constexpr (SLOTS == 1) {
      __syncthreads();
      issue(q, used);
    }
  }
};

// w[i] = e^{-i pi i / L} at i = t + T q (T = L/16): e^{-i pi t/L} e^{-i pi q/16}
__device__ __forceinline__ float2 wodd_base(int t, int L) {
  float s, c;
  sincospif(-(float)t / (float)L, &s, &c);
  return make_float2(c, s);
}
template <int Q>
__device__ __forceinline__ float2 wodd_q(float2 base) {
  // cos / sin (pi Q / 16), Q = 0..15
  constexpr float C[16] = {1.0f, 0.98078528040323044913f, 0.92387953251128675613f, 0.83146961230254523708f,
                           0.70710678118654752440f, 0.55557023301960222474f, 0.38268343236508977173f,
                           0.19509032201612826785f, 0.0f, -0.19509032201612826785f, -0.38268343236508977173f,
                           -0.55557023301960222474f, -0.70710678118654752440f, -0.83146961230254523708f,
                           -0.92387953251128675613f, -0.98078528040323044913f};
  constexpr float S[16] = {0.0f, 0.19509032201612826785f, 0.38268343236508977173f, 0.55557023301960222474f,
                           0.70710678118654752440f, 0.83146961230254523708f, 0.92387953251128675613f,
                           0.98078528040323044913f, 1.0f, 0.98078528040323044913f, 0.92387953251128675613f,
                           0.83146961230254523708f, 0.70710678118654752440f, 0.55557023301960222474f,
                           0.38268343236508977173f, 0.19509032201612826785f};
  return cmul(base, make_float2(C[Q], -S[Q]));
}

// ---- magnification ----------------------------------------------------------------
// Forward M S along the line (reading C1):
//   a[i] = cr[f] X[f] (i = f + L/2 mod L),  E = IFFT(FFT(a) bke),  O = IFFT(FFT(a w) bko),
//   y[o] = cout[o] (E[o] + conj(w[o]) O[o]).
// SRC(r): spectrum X at register r (layout S, natural frequency order).  E is parked
// with STASH(r, e) between the two transform pairs and fetched back with UNSTASH(r);
// SRC(r) is read before STASH(r, .) for the same r, so source and stash may share a
// thread-private slot: only one line is live across each transform.  w is computed on
// the fly; the pipe supplies, in order: cr, bke, cr, bko, cout.  v receives y.
struct NoHook {
  __device__ __forceinline__ void operator()() const {}
};
// SRC_FREED() runs after the transform that follows the last SRC read (its barriers: every thread of
// the CTA is past its SRC reads), e.g. to reuse the source's shared memory.
template <int L, class Src, class Stash, class Unstash, class Freed = NoHook>
__device__ __forceinline__ void mag_fwd(float2 (&v)[16], Src src, Stash stash, Unstash unstash, TabPipe<L> &pipe,
                                        const TabSeq &q, bool sync0, Xch &x, int t, const float4 *__restrict__ tw,
                                        Freed src_freed = {}) {
  constexpr int T = L / 16;
  const float2 *tab = pipe.take(q, sync0);  // cr
#pragma unroll
  for (int r = 0; r < 16; r++) v[r ^ 8] = cmul(src(r), tab[t + r * T]);
  pipe.done(q);
  fft<L, false>(v, x, t, tw);
  tab = pipe.take(q);  // bke
#pragma unroll
  for (int r = 0; r < 16; r++) v[r] = cmul(v[r], tab[t + r * T]);
  pipe.done(q);
  fft<L, true>(v, x, t, tw);
  tab = pipe.take(q);  // cr again
  const float2 wb = wodd_base(t, L);
  float2 s[16];
#pragma unroll
  for (int r = 0; r < 16; r++) {
    s[r] = src(r);
    stash(r, v[r]);
  }
#define HOLO_B(R) v[(R) ^ 8] = cmul(cmul(s[R], tab[t + (R) * T]), wodd_q<(R) ^ 8>(wb));
  HOLO_B(0) HOLO_B(1) HOLO_B(2) HOLO_B(3) HOLO_B(4) HOLO_B(5) HOLO_B(6) HOLO_B(7)
  HOLO_B(8) HOLO_B(9) HOLO_B(10) HOLO_B(11) HOLO_B(12) HOLO_B(13) HOLO_B(14) HOLO_B(15)
#undef HOLO_B
  pipe.done(q);
  fft<L, false>(v, x, t, tw);
  src_freed();
  tab = pipe.take(q);  // bko
#pragma unroll
  for (int r = 0; r < 16; r++) v[r] = cmul(v[r], tab[t + r * T]);
  pipe.done(q);
  fft<L, true>(v, x, t, tw);
  tab = pipe.take(q);  // cout
#define HOLO_C(R) v[R] = cmul(cadd(unstash(R), cmulc(v[R], wodd_q<R>(wb))), tab[t + (R) * T]);
  HOLO_C(0) HOLO_C(1) HOLO_C(2) HOLO_C(3) HOLO_C(4) HOLO_C(5) HOLO_C(6) HOLO_C(7)
  HOLO_C(8) HOLO_C(9) HOLO_C(10) HOLO_C(11) HOLO_C(12) HOLO_C(13) HOLO_C(14) HOLO_C(15)
#undef HOLO_C
  pipe.done(q);
}

// Adjoint (M S)^* along the line (the steps of mag_fwd conjugated, in reverse):
//   A = y conj(cout),  Za = IFFT(FFT(A) conj(bke)),  Zb = IFFT(FFT(A w) conj(bko)),
//   Z[i] = Za[i] + conj(w[i]) Zb[i],  W[f] = conj(cr[f]) Z[(f + L/2) mod L].
// SRC(r): spatial input y at register r; STASH / UNSTASH as in mag_fwd.  The pipe
// supplies, in order: cout, bke, cout, bko, cr.  v receives the SPECTRUM W (natural
// order); the caller finishes with an inverse FFT (possibly after summing several W).
template <int L, class Src, class Stash, class Unstash, class Freed = NoHook>
__device__ __forceinline__ void mag_adj(float2 (&v)[16], Src src, Stash stash, Unstash unstash, TabPipe<L> &pipe,
                                        const TabSeq &q, bool sync0, Xch &x, int t, const float4 *__restrict__ tw,
                                        Freed src_freed = {}) {
  constexpr int T = L / 16;
  const float2 *tab = pipe.take(q, sync0);  // cout
#pragma unroll
  for (int r = 0; r < 16; r++) v[r] = cmulc(src(r), tab[t + r * T]);
  pipe.done(q);
  fft<L, false>(v, x, t, tw);
  tab = pipe.take(q);  // bke
#pragma unroll
  for (int r = 0; r < 16; r++) v[r] = cmulc(v[r], tab[t + r * T]);
  pipe.done(q);
  fft<L, true>(v, x, t, tw);
  tab = pipe.take(q);  // cout again
  const float2 wb = wodd_base(t, L);
  float2 s[16];
#pragma unroll
  for (int r = 0; r < 16; r++) {
    s[r] = src(r);
    stash(r, v[r]);
  }
#define HOLO_B(R) v[R] = cmul(cmulc(s[R], tab[t + (R) * T]), wodd_q<R>(wb));
  HOLO_B(0) HOLO_B(1) HOLO_B(2) HOLO_B(3) HOLO_B(4) HOLO_B(5) HOLO_B(6) HOLO_B(7)
  HOLO_B(8) HOLO_B(9) HOLO_B(10) HOLO_B(11) HOLO_B(12) HOLO_B(13) HOLO_B(14) HOLO_B(15)
#undef HOLO_B
  pipe.done(q);
  fft<L, false>(v, x, t, tw);
  src_freed();
  tab = pipe.take(q);  // bko
#pragma unroll
  for (int r = 0; r < 16; r++) v[r] = cmulc(v[r], tab[t + r * T]);
  pipe.done(q);
  fft<L, true>(v, x, t, tw);
#define HOLO_Z(R) s[R] = cadd(unstash(R), cmulc(v[R], wodd_q<R>(wb)));
  HOLO_Z(0) HOLO_Z(1) HOLO_Z(2) HOLO_Z(3) HOLO_Z(4) HOLO_Z(5) HOLO_Z(6) HOLO_Z(7)
  HOLO_Z(8) HOLO_Z(9) HOLO_Z(10) HOLO_Z(11) HOLO_Z(12) HOLO_Z(13) HOLO_Z(14) HOLO_Z(15)
#undef HOLO_Z
  tab = pipe.take(q);  // cr
#pragma unroll
  for (int r = 0; r < 16; r++) v[r] = cmulc(s[r ^ 8], tab[t + r * T]);
  pipe.done(q);
}

// ---- deterministic block reduction --------------------------------------------------
__device__ __forceinline__ double block_sum(double v, double *red) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[w] = v;
  __syncthreads();
  double s = 0;
  if (threadIdx.x == 0)
    for (int i = 0; i < nw; i++) s += red[i];
  return s;
}

}  // namespace holo
