// holo_passes.cuh -- the five line-pass kernels (X1, Y1, X2, Y2, X3), the
// propagation filters for q_j / g_q, reductions and the CG pointwise step.
//
// Line kernels: 512 threads, G = 512 / (L/16) lines per CTA (g-major), <= 128
// registers per thread; shared memory = double-buffered exchange space + (Bluestein
// kernels) one thread-private line.  Workspace arrays (T1, Aw, W1, V1, T3, G, QJ)
// are in the P2 layout (holo_kernels.cuh); the caller's arrays (psi, q, w, sqrt_d,
// grad, eta) are row-major.
#pragma once
#include "holo_kernels.cuh"

namespace holo {

// Threads per CTA of the object-chain line kernels (HOLO_NT): 512 = G = 8192/L lines per CTA and one
// CTA per SM at <= 128 registers; 256 = half the lines and two CTAs per SM (their shared-memory
// and FP32 phases can overlap; needs HOLO_TAB_SLOTS=1 to fit two CTAs' shared memory at L = 4096).
#ifndef HOLO_NT
#define HOLO_NT 512
#endif
constexpr int NT = HOLO_NT;
constexpr int CTAS_PER_SM = 512 / NT;
template <int L>
using CtaK = Cta<L, NT>;

enum { X2_GRAD = 0, X2_FWD = 1, X2_ADJ = 2, X2_OBJ = 3 };

template <int L>
__device__ __forceinline__ float2 *priv_base(float2 *sm) {
  return sm + CtaK<L>::XBYTES / sizeof(float2);
}
// table slots follow the exchange space (and the private line when PRIV)
template <int L, bool PRIV>
__device__ __forceinline__ float2 *slot_base(float2 *sm) {
  return sm + (CtaK<L>::XBYTES + (PRIV ? CtaK<L>::PRIV : 0)) / sizeof(float2);
}

// layout-S line access of a P2 array with R rows: row y (x = t + T r) / column x (y = t + T r)
template <int L>
__device__ __forceinline__ void ld_p2_row(float2 (&v)[16], const float2 *__restrict__ a, int y, int R, int t) {
#pragma unroll
  for (int r = 0; r < 16; r++) v[r] = ldg2(a + p2(y, t + r * (L / 16), R));
}
template <int L>
__device__ __forceinline__ void st_p2_row(const float2 (&v)[16], float2 *__restrict__ a, int y, int R, int t) {
#pragma unroll
  for (int r = 0; r < 16; r++) a[p2(y, t + r * (L / 16), R)] = v[r];
}
template <int L>
__device__ __forceinline__ void ld_p2_col(float2 (&v)[16], const float2 *__restrict__ a, int x, int R, int t) {
#pragma unroll
  for (int r = 0; r < 16; r++) v[r] = ldg2(a + p2(t + r * (L / 16), x, R));
}
template <int L>
__device__ __forceinline__ void st_p2_col(const float2 (&v)[16], float2 *__restrict__ a, int x, int R, int t) {
#pragma unroll
  for (int r = 0; r < 16; r++) a[p2(t + r * (L / 16), x, R)] = v[r];
}

// Column staging (HOLO_STAGE, default 1).  A column pass's CTA owns G adjacent columns, i.e. ONE
// contiguous block of 8 G L bytes of a P2 array (G/2 column pairs).  The frame's block is bulk-copied
// (cp.async.bulk: the TMA engine, completion on an mbarrier) into the CTA's 64 KB thread-private
// slot, where it also serves as the magnification's source and stash; the copy of frame b + 1 is
// issued as soon as frame b's last access to the slot is behind a CTA barrier (the next transform's
// exchange), so it lands while frame b's remaining transforms run.  It replaces the 16 LDG per
// thread whose L2 latency every frame start exposed.  Element (y, col0 + g) of the block sits at
// 2 L (g >> 1) + 2 y + (g & 1): a warp's (t, g) lanes read consecutive float2 (conflict free, G = 2).
#ifndef HOLO_STAGE
#define HOLO_STAGE 1
#endif
#ifndef HOLO_STAGE_Q
#define HOLO_STAGE_Q 1  // Y1: the q_j block through the slot too (1: behind the magnification; 2: also in the shift-only plane)
#endif
struct ColStage {
  uint64_t *bar;       // the slot's mbarrier
  const float2 *next;  // the next frame's block (nullptr: last frame)
  uint32_t bytes;      // 8 G L
  uint32_t phase;      // parity of this frame's copy
  const float2 *qblk;  // Y1: the CTA's block of q_j, staged behind the magnification (nullptr: read by LDG);
                       // its copy completes parity 1 (then the frame copies complete parity 0)
  // all threads, after a CTA barrier that follows their last access to the slot
  __device__ __forceinline__ void issue_next(float2 *slot) const {
    if (next && threadIdx.x == 0) {
      fence_proxy_async();  // the generic-proxy reads / writes of the slot precede the async write
      mbar_expect_tx(bar, bytes);
      bulk_g2s(slot, next, bytes, bar);
    }
  }
};
template <int L>
__device__ __forceinline__ int stage_idx(int g, int y) { return 2 * L * (g >> 1) + 2 * y + (g & 1); }

// ----------------------------------------------------------------------------- X1
// rows of psi_k (row-major):  X = FFT(psi row) (kept thread-private); per j: T1_j row = M_{1/mt_j} S_{sx} psi row
// (one non-inlined call per plane: only pointers and the pipe state cross it, so the
// magnification keeps the whole register budget)
// Row staging in X1 (HOLO_STAGE_X1, default 1; 2 <= G <= 8, launches without the fused CG update): a
// launch covers the nb angles of a batch, each CTA looping over them for its G rows.  The rows of
// angle b + 1 (row-major psi: G contiguous rows) are bulk-copied into the thread-private slot once
// the last plane's second source read of angle b is behind a barrier (mag_fwd's src_freed hook), so
// the CTA start (launch, table pipeline start, DRAM latency of the row loads) is paid once per batch
// instead of once per angle.  Row g sits at g (L + 16/G) float2: the skew keeps a warp's (t, g) lanes
// on distinct banks.
#ifndef HOLO_STAGE_X1
#define HOLO_STAGE_X1 1
#endif
template <int L>
struct X1Stage {
  static constexpr int SK = CtaK<L>::G <= 16 ? 16 / CtaK<L>::G : 1;  // float2
  static constexpr int RS = L + SK;                                  // staged row stride
  static constexpr bool OK = HOLO_STAGE && HOLO_STAGE_X1 && CtaK<L>::G >= 2 && CtaK<L>::G <= 8;
  // control block at the end of the launch's dynamic shared memory (Smem::XPT1), so that the plane
  // bodies find it from the shared-memory base instead of carrying it in registers
  struct Ctl {
    uint64_t bar;
    const float2 *next;  // first of the CTA's rows of the next angle (nullptr: none)
  };
  static constexpr size_t CTL_OFF = CtaK<L>::XBYTES + CtaK<L>::PRIV + 128 + TabPipe<L>::BYTES;
  __device__ __forceinline__ static Ctl *ctl(float2 *sm) {
    return reinterpret_cast<Ctl *>(reinterpret_cast<char *>(sm) + CTL_OFF);
  }
  // thread 0, behind a CTA barrier that follows every thread's last access to the slot
  __device__ __forceinline__ static void issue(float2 *sm, const float2 *rows) {
    float2 *xs = priv_base<L>(sm);
    uint64_t *bar = &ctl(sm)->bar;
    fence_proxy_async();
    mbar_expect_tx(bar, 8u * CtaK<L>::G * L);
#pragma unroll 1
    for (int g = 0; g < CtaK<L>::G; g++) bulk_g2s(xs + g * RS, rows + (size_t)g * L, 8u * L, bar);
  }
};

template <int L, bool STG>
__device__ __noinline__ TabPipe<L> x1_plane(float2 *__restrict__ T1j, const float4 *__restrict__ tw, const TabSeq &seq,
                                      TabPipe<L> pipe, float2 *sm, bool mag, bool sync0) {
  using C = CtaK<L>;
  constexpr int T = L / 16;
  Xch x = C::xch(sm);
  const Priv<NT> X{priv_base<L>(sm)};
  const int t = C::t(), y = blockIdx.x * C::G + C::g();
  // the spectrum of the row (thread-private smem), reused by every plane
  auto src = [&](int r) -> float2 {
    if constexpr (STG) {
      const float2 z = priv_base<L>(sm)[C::g() * X1Stage<L>::RS + t + r * T];
      if (r == 15) fence_proxy_async();  // this thread's slot accesses precede a later async write
      return z;
    } else {
      return X[r];
    }
  };
  auto freed = [&]() {
    if constexpr (STG) {
      if (threadIdx.x == 0) {
        const float2 *nx = X1Stage<L>::ctl(sm)->next;  // set by the kernel for the angle's last plane
        if (nx) {
          X1Stage<L>::ctl(sm)->next = nullptr;
          X1Stage<L>::issue(sm, nx);
        }
      }
    }
  };
  float2 v[16];
  if (mag) {
    // the first half's term stays in registers
    float2 e[16];
    mag_fwd<L>(
        v, src, [&](int r, float2 val) { e[r] = val; }, [&](int r) { return e[r]; }, pipe, seq, sync0, x, t, tw, freed);
  } else {
    const float2 *cr = pipe.take(seq, sync0);
#pragma unroll
    for (int r = 0; r < 16; r++) v[r] = cmul(src(r), cr[t + r * T]);
    pipe.done(seq);
    fft<L, true>(v, x, t, tw);
    freed();
  }
  st_p2_row<L>(v, T1j, y, L, t);
  return pipe;
}

// The psi-block CG update fused into X1 (holo_set_cg_fuse): mode -1 off; otherwise the row of
// x_trial = x + gamma eta with eta = -rho g (mode 0), -rho g + beta eta (mode 1) or eta (mode 2),
// written to trial (and eta), is the row X1 transforms -- the arithmetic of k_cg, element by element.
struct CgFuse {
  const float2 *g;
  float2 *eta, *trial;
  float rho, beta, gamma;
  int mode;
};

template <int L>
__global__ void __launch_bounds__(NT, CTAS_PER_SM)
    k_x1(const float2 *__restrict__ psi_k, float2 *__restrict__ T1, Tables tb, const __grid_constant__ TabSeq seq,
         int nz, uint32_t magmask, int fourier, CgFuse cg) {
  using C = CtaK<L>;
  extern __shared__ float4 sm4[];
  __shared__ uint64_t bars[2];
  float2 *sm = reinterpret_cast<float2 *>(sm4);
  TabPipe<L> pipe;
  pipe.start(seq, slot_base<L, true>(sm), bars);
  {
    Xch x = C::xch(sm);
    const Priv<NT> X{priv_base<L>(sm)};
    const int t = C::t(), y = blockIdx.x * C::G + C::g();
    float2 v[16];
    ld_row<L>(v, psi_k + (size_t)y * L, t);
    if (cg.mode >= 0) {
      const size_t row = (size_t)y * L;
#pragma unroll
      for (int r = 0; r < 16; r++) {
        const size_t i = row + t + r * (L / 16);
        float2 e;
        if (cg.mode == 2) {
          e = cg.eta[i];
        } else {
          const float2 gv = ldg2(cg.g + i);
          if (cg.mode == 0) {
            e = make_float2(-cg.rho * gv.x, -cg.rho * gv.y);
          } else {
            const float2 ev = cg.eta[i];
            e = make_float2(fmaf(cg.beta, ev.x, -cg.rho * gv.x), fmaf(cg.beta, ev.y, -cg.rho * gv.y));
          }
          cg.eta[i] = e;
        }
        v[r] = make_float2(fmaf(cg.gamma, e.x, v[r].x), fmaf(cg.gamma, e.y, v[r].y));
        cg.trial[i] = v[r];
      }
    }
    if (!fourier) fft<L, false>(v, x, t, tb.tw);  // HOLO_FOURIER: the row of DFT2(psi) IS the x-spectrum
#pragma unroll
    for (int r = 0; r < 16; r++) X[r] = v[r];
  }
#pragma unroll 1
  for (int j = 0; j < nz; j++) pipe = x1_plane<L, false>(T1 + (size_t)j * L * L, tb.tw, seq, pipe, sm, (magmask >> j) & 1u, j > 0);
}

// the staged rows -> their x-spectrum, in place (thread-private positions of the slot)
template <int L>
__device__ __noinline__ void x1_spectrum(float2 *sm, const float4 *__restrict__ tw) {
  using C = CtaK<L>;
  constexpr int T = L / 16;
  Xch x = C::xch(sm);
  float2 *xs = priv_base<L>(sm) + C::g() * X1Stage<L>::RS + C::t();
  float2 v[16];
#pragma unroll
  for (int r = 0; r < 16; r++) v[r] = xs[r * T];
  fft<L, false>(v, x, C::t(), tw);
#pragma unroll
  for (int r = 0; r < 16; r++) xs[r * T] = v[r];
}

// The staged, batched X1: the nb angles of a batch in one launch (psi0: the first angle, angles L^2
// apart; T1 [nb][nz][L][L]), one flat loop over the (angle, plane) pairs so that little state is live
// across the plane calls (kernel-level spills cost L2 round trips: the L1 left beside 198 KB of shared
// memory does not hold the CTA's stack).
template <int L>
__global__ void __launch_bounds__(NT, CTAS_PER_SM)
    k_x1s(const float2 *__restrict__ psi0, float2 *__restrict__ T1, Tables tb, const __grid_constant__ TabSeq seq,
          int nz, uint32_t magmask, int fourier, int nb) {
  using C = CtaK<L>;
  using XS = X1Stage<L>;
  extern __shared__ float4 sm4[];
  __shared__ uint64_t bars[2];
  float2 *sm = reinterpret_cast<float2 *>(sm4);
  typename XS::Ctl *ctl = XS::ctl(sm);
  if (threadIdx.x == 0) {
    mbar_init(&ctl->bar, 1);
    ctl->next = nullptr;
    fence_mbar_init();
  }
  // [exchange][row slot: PRIV + 128 B (skewed rows)][table slots][control block]  (Smem::XPT1)
  TabPipe<L> pipe;
  pipe.start(seq, priv_base<L>(sm) + (C::PRIV + 128) / sizeof(float2), bars);
  __syncthreads();
  if (threadIdx.x == 0) XS::issue(sm, psi0 + (size_t)blockIdx.x * C::G * L);
  const int nm = nb * nz;
#pragma unroll 1
  for (int m = 0, j = 0, b = 0; m < nm; m++) {
    if (j == 0) {  // a new angle: its rows have been staged
      if (threadIdx.x == 0 && b + 1 < nb)  // the copy at the end of this angle reads L2
        prefetch_l2(psi0 + ((size_t)(b + 1) * L + (size_t)blockIdx.x * C::G) * L, 8u * C::G * L);
      mbar_wait(&ctl->bar, b & 1);
      if (!fourier) x1_spectrum<L>(sm, tb.tw);  // HOLO_FOURIER: the row of DFT2(psi) IS the x-spectrum
    }
    // the last plane's src_freed hook (thread 0) copies the next angle's rows
    if (j + 1 == nz && threadIdx.x == 0)
      ctl->next = b + 1 < nb ? psi0 + ((size_t)(b + 1) * L + (size_t)blockIdx.x * C::G) * L : nullptr;
    pipe = x1_plane<L, XS::OK>(T1 + (size_t)m * L * L, tb.tw, seq, pipe, sm, (magmask >> j) & 1u, m > 0);
    if (++j == nz) {
      j = 0;
      b++;
    }
  }
}

// ----------------------------------------------------------------------------- Y1
// Angle-batched (Eq. (12)'s sum over k is what makes a batch pay): nb frames of ONE plane
// j, frame b at T1j + b * fstride.  Each CTA owns G columns and loops over the batch, so
// its q_j columns are re-read from L2, and the next frame's input block (contiguous in P2)
// is prefetched into L2 by a bulk copy while the current frame is transformed.
// Per frame: a = M_{1/mt_j} S_{sy} (column) -> Aout[b] (optional);
//            W1[b] = rows [o, o+N) of D_y(q_j . a) (optional; P2 with N rows)
// The frame body is a separate (non-inlined) function: only the loop state crosses the
// call, so the transforms keep the full register budget (an inlined loop spills).
// PS (per-frame probe shifts): q_kj = P_omega S_{s^p} q is not a
// per-plane constant; its column comes from qt = IDFT_x(Hq_x Qhat) (XQ pass, spectral in y):
// x Hq_y (table), IFFT_y -> q_kj column, stored to qk (Y2 needs conj(q_kj)).
template <int L, bool PS, bool STG>
__device__ __noinline__ TabPipe<L> y1_frame(const float2 *__restrict__ in, const float2 *__restrict__ qj,
                                      const float2 *__restrict__ qt, float2 *__restrict__ qk,
                                      float2 *__restrict__ aout, float2 *__restrict__ w1, const float4 *__restrict__ tw,
                                      const TabSeq &seq, TabPipe<L> pipe, float2 *sm, int mag, int N, int fourier,
                                      ColStage st) {
  using C = CtaK<L>;
  constexpr int T = L / 16;
  Xch x = C::xch(sm);
  const Priv<NT> X{priv_base<L>(sm)};
  float2 *Sb = priv_base<L>(sm);
  const int t = C::t(), col = blockIdx.x * C::G + C::g();
  const int s0 = stage_idx<L>(C::g(), t);
  // the thread-private slot: the staged block (STG) or the Priv layout
  auto slot = [&](int r) -> float2 & { if constexpr (STG) return Sb[s0 + 2 * r * T]; else return X[r]; };
  float2 v[16];
  if constexpr (STG) {
    mbar_wait(st.bar, st.phase);
#pragma unroll
    for (int r = 0; r < 16; r++) v[r] = slot(r);
  } else {
    ld_p2_col<L>(v, in, col, L, t);
  }
  if (!fourier) fft<L, false>(v, x, t, tw);  // HOLO_FOURIER: T1 is already the y-spectrum (X1 ran on DFT2 psi)
  if (mag) {
    if (!STG || !fourier) {  // (staged Fourier-state input: the slot already holds the spectrum)
#pragma unroll
      for (int r = 0; r < 16; r++) slot(r) = v[r];
    }
    if constexpr (STG) {
      // the first half's term stays in registers (as in X1), so the slot is free once the second source
      // read is behind a barrier: the q_j block lands there while the last two transforms run
      float2 e[16];
      mag_fwd<L>(
          v, [&](int r) { const float2 z = slot(r); if (r == 15) fence_proxy_async(); return z; },
          [&](int r, float2 val) { e[r] = val; }, [&](int r) { return e[r]; }, pipe, seq, false, x, t, tw, [&]() {
            if (st.qblk && threadIdx.x == 0) {
              fence_proxy_async();
              mbar_expect_tx(st.bar, st.bytes);
              bulk_g2s(Sb, st.qblk, st.bytes, st.bar);
            }
          });
    } else {
      mag_fwd<L>(
          v, [&](int r) { return slot(r); }, [&](int r, float2 e) { slot(r) = e; }, [&](int r) { return slot(r); },
          pipe, seq, false, x, t, tw);
    }
  } else {
    const float2 *cr = pipe.take(seq);
#pragma unroll
    for (int r = 0; r < 16; r++) v[r] = cmul(v[r], cr[t + r * T]);
    pipe.done(seq);
    if constexpr (STG) {
      if (st.qblk) {  // shift-only plane: the q_j block lands behind the one inverse transform
        fence_proxy_async();
        __syncthreads();  // every thread is past its reads of the staged column
        if (threadIdx.x == 0) {
          fence_proxy_async();
          mbar_expect_tx(st.bar, st.bytes);
          bulk_g2s(Sb, st.qblk, st.bytes, st.bar);
        }
      }
    }
    fft<L, true>(v, x, t, tw);
  }
  if (aout) st_p2_col<L>(v, aout, col, L, t);
  if (PS && qk) {  // q_kj column: park a, transform the qt column
#pragma unroll
    for (int r = 0; r < 16; r++) X[r] = v[r];
    ld_p2_col<L>(v, qt, col, L, t);
    const float2 *hq = pipe.take(seq);  // Hq_y(k, j) = h_omega r_{s^p_y} / L
#pragma unroll
    for (int r = 0; r < 16; r++) v[r] = cmul(v[r], hq[t + r * T]);
    pipe.done(seq);
    fft<L, true>(v, x, t, tw);
    st_p2_col<L>(v, qk, col, L, t);
    if (w1) {
#pragma unroll
      for (int r = 0; r < 16; r++) v[r] = cmul(v[r], X[r]);
    }
  } else if (w1) {
    if (STG && st.qblk) {
      mbar_wait(st.bar, 1);
#pragma unroll
      for (int r = 0; r < 16; r++) v[r] = cmul(v[r], slot(r));
    } else {
#pragma unroll
      for (int r = 0; r < 16; r++) v[r] = cmul(v[r], ldg2(qj + p2(t + r * T, col, L)));
    }
  }
  if (w1) {
    if constexpr (STG) fence_proxy_async();  // this thread's slot accesses before the next async write
    fft<L, false>(v, x, t, tw);
    if constexpr (STG) st.issue_next(Sb);  // every thread is past its last slot access (the FFT's barriers)
    const float2 *h = pipe.take(seq);  // hdet_j / L
#pragma unroll
    for (int r = 0; r < 16; r++) v[r] = cmul(v[r], h[t + r * T]);
    pipe.done(seq);
    fft<L, true>(v, x, t, tw);
    const int o = (L - N) / 2;
#pragma unroll
    for (int r = 0; r < 16; r++) {
      const int row = t + r * T - o;
      if (row >= 0 && row < N) w1[p2(row, col, N)] = v[r];
    }
  } else if constexpr (STG) {
    fence_proxy_async();
    __syncthreads();
    st.issue_next(Sb);
  }
  return pipe;
}

template <int L, bool PS>
__global__ void __launch_bounds__(NT, CTAS_PER_SM)
    k_y1(const float2 *__restrict__ T1j, size_t fstride, const float2 *__restrict__ qj, const float2 *__restrict__ Qt,
         float2 *__restrict__ Qk, float2 *__restrict__ Aout, float2 *__restrict__ W1, Tables tb,
         const __grid_constant__ TabSeq seq, int mag, int N, int nb, int fourier) {
  using C = CtaK<L>;
  constexpr bool STG = HOLO_STAGE && !PS && C::G >= 2;
  extern __shared__ float4 sm4[];
  __shared__ uint64_t bars[2];
  __shared__ uint64_t sbar;
  float2 *sm = reinterpret_cast<float2 *>(sm4);
  const int col0 = blockIdx.x * C::G;
  constexpr uint32_t SBYTES = 8u * C::G * L;
  if (STG && threadIdx.x == 0) {
    mbar_init(&sbar, 1);
    fence_mbar_init();
  }
  TabPipe<L> pipe;
  pipe.start(seq, slot_base<L, true>(sm), bars);
  if (STG) {
    __syncthreads();
    if (threadIdx.x == 0) {
      mbar_expect_tx(&sbar, SBYTES);
      bulk_g2s(priv_base<L>(sm), T1j + p2(0, col0, L), SBYTES, &sbar);
    }
  }
  constexpr int PF_COLS = C::G < 2 ? 2 : C::G;  // whole P2 column pairs (16-byte aligned blocks)
  // q_j staged behind the magnification (HOLO_STAGE_Q >= 1) / the shift-only plane's transform (2)
  const bool qstg = STG && HOLO_STAGE_Q && (mag || HOLO_STAGE_Q >= 2) && W1 && qj;
#pragma unroll 1
  for (int b = 0; b < nb; b++) {
    const float2 *in = T1j + (size_t)b * fstride;
    if (threadIdx.x == 0 && b + 1 < nb) prefetch_l2(in + fstride + p2(0, col0 & ~1, L), 8u * PF_COLS * L);
    const ColStage st{&sbar, b + 1 < nb ? in + fstride + p2(0, col0, L) : nullptr, SBYTES, qstg ? 0u : (uint32_t)(b & 1),
                      qstg ? qj + p2(0, col0, L) : nullptr};
    pipe = y1_frame<L, PS, STG>(in, qj, PS ? Qt + (size_t)b * fstride : nullptr,
                                (PS && Qk) ? Qk + (size_t)b * L * L : nullptr, Aout ? Aout + (size_t)b * L * L : nullptr,
                                W1 ? W1 + (size_t)b * N * L : nullptr, tb.tw, seq, pipe, sm, mag, N, fourier, st);
  }
}

// Row staging (HOLO_STAGE, X3): the CTA's G rows of plane j of T3 (P2: 2048 strided 32-byte pieces at
// L = 4096) are gathered by 4-D tensor copies (TMA, tma.cuh) into the 64 KB thread-private slot; the
// copy of plane j + 1 is issued as soon as the magnification's last source read is behind a CTA
// barrier, so it lands while plane j's last two transforms run.  Element (y0 + g, x) of the staged
// rows sits at 2 (G (x >> 1) + g) + (x & 1) (the box order {x & 1, g, x >> 1}): a warp's (t, g)
// lanes read consecutive float2.
struct RowStage {
  const CUtensorMap *map;  // T3 as {4 floats, L rows, L/2 column pairs, planes}
  uint64_t *bar;
  int next;                // plane index (in the map) of the next copy, -1: none
  int y0;
  uint32_t phase;          // parity of this plane's copy
  template <int L>
  __device__ __forceinline__ void issue(float2 *slot, int plane) const {
    using C = CtaK<L>;
    constexpr int BOXC = L / 2 < 256 ? L / 2 : 256;  // column pairs per box
    if (threadIdx.x == 0) {
      mbar_expect_tx(bar, 8u * C::G * L);
#pragma unroll 1
      for (int c = 0; c < L / 2; c += BOXC) tma_load_4d(slot + 2 * C::G * c, map, 0, y0, c, plane, bar);
    }
  }
};

// ----------------------------------------------------------------------------- X2
// rows y < N of the nb frames of a batch (one plane, so one transfer table for all of them).
//   GRAD: W1 row -> D_x, crop, residual (+F), pad, D_x^* -> V1   (W1, V1: P2, N rows)
//   FWD : W1 row -> D_x, crop -> w frame [N][N] (row-major)
//   ADJ : y frame row (row-major) -> pad, D_x^* -> V1
//   OBJ : W1 row -> D_x, crop, F only
// Strides between the batch's frames: in / out (elements), sqrt_d (elements), partial (CTAs).
// HOLO_X2_LOOP=1 (default): a CTA owns G rows of EVERY frame of the batch (frame loop inside, as
// Y1 / Y2 do): the table hdet_j / L is bulk-copied into shared memory once per CTA instead of once
// per (CTA, frame), and the next frame's rows are prefetched into L2 while this frame is
// transformed, so the row loads stop exposing DRAM latency at every CTA start.
// HOLO_X2_LOOP=0: one frame per CTA (blockIdx.y), the round-1 launch shape.
#ifndef HOLO_X2_LOOP
#define HOLO_X2_LOOP 1
#endif
// Row staging in X2 (HOLO_STAGE_X2, default 1; W1-reading modes with the frame loop): the CTA's G rows
// of the frame's W1 (P2 with N rows: strided 32-byte pieces) are gathered by 4-D tensor copies into a
// 64 KB slot, as X3 does for T3; the copy of frame b + 1 is issued once frame b's first transform is
// past its barriers, so it lands behind the frame's four transforms.  Rows >= N read as zeros (the
// tensor map's out-of-bounds fill).
#ifndef HOLO_STAGE_X2
#define HOLO_STAGE_X2 1
#endif
template <int L, int MODE, int TM>
__device__ __forceinline__ void x2_frame(const float2 *__restrict__ in, const float *__restrict__ sqrt_d,
                                         float2 *__restrict__ out, double *__restrict__ partial, const float2 *h,
                                         Xch &x, const float4 *__restrict__ tw, double *red, int N, float tau,
                                         uint64_t *bar, const float2 *zs, RowStage rs) {
  using C = CtaK<L>;
  constexpr int T = L / 16;
  const int t = C::t(), y = blockIdx.x * C::G + C::g();
  const bool act = y < N;
  const int o = (L - N) / 2;
  float2 v[16];
  float dv[16];  // sqrt_d of this thread's crop positions, fetched before the transforms
  if (MODE == X2_GRAD || MODE == X2_OBJ) {
#pragma unroll
    for (int r = 0; r < 16; r++) {
      const int c = t + r * T - o;
      dv[r] = (act && c >= 0 && c < N) ? __ldg(sqrt_d + (size_t)y * N + c) : 0.f;
    }
  }
  if (MODE != X2_ADJ) {
    if (zs) {
      mbar_wait(rs.bar, rs.phase);
#pragma unroll
      for (int r = 0; r < 16; r++) {
        const int xx = t + r * T;
        v[r] = zs[2 * (C::G * (xx >> 1) + C::g()) + (xx & 1)];
      }
      fft<L, false>(v, x, t, tw);
      if (rs.next >= 0) rs.template issue<L>(const_cast<float2 *>(zs), rs.next);  // every thread is past its slot reads
    } else {
#pragma unroll
      for (int r = 0; r < 16; r++) v[r] = act ? ldg2(in + p2(y, t + r * T, N)) : make_float2(0.f, 0.f);
      fft<L, false>(v, x, t, tw);
    }
    mbar_wait(bar, 0);  // the resident table has arrived (returns at once after the first frame)
#pragma unroll
    for (int r = 0; r < 16; r++) v[r] = cmul(v[r], h[t + r * T]);
    fft<L, true>(v, x, t, tw);
    if (MODE == X2_FWD) {
      if (act) {
#pragma unroll
        for (int r = 0; r < 16; r++) {
          const int c = t + r * T - o;
          if (c >= 0 && c < N) out[(size_t)y * N + c] = v[r];
        }
      }
      return;
    }
    double acc = 0.0;
#pragma unroll
    for (int r = 0; r < 16; r++) {
      const int c = t + r * T - o;
      float2 w = make_float2(0.f, 0.f);
      if (act && c >= 0 && c < N) {
        w = residual_tau<TM>(v[r], dv[r], tau, acc);  // G_tau (App. A.3): F_1 at tau = 1, F_2 at 2
      }
      v[r] = w;
    }
    const double s = block_sum(acc, red);
    if (threadIdx.x == 0) partial[blockIdx.x] = s;
    if (MODE == X2_OBJ) return;
  } else {
#pragma unroll
    for (int r = 0; r < 16; r++) {
      const int c = t + r * T - o;
      v[r] = (act && c >= 0 && c < N) ? ldg2(in + (size_t)y * N + c) : make_float2(0.f, 0.f);
    }
  }
  fft<L, false>(v, x, t, tw);
  mbar_wait(bar, 0);
#pragma unroll
  for (int r = 0; r < 16; r++) v[r] = cmulc(v[r], h[t + r * T]);
  fft<L, true>(v, x, t, tw);
  if (act) st_p2_row<L>(v, out, y, N, t);
}

template <int L, int MODE, int TM = -1>
__global__ void __launch_bounds__(NT, CTAS_PER_SM)
    k_x2(const float2 *__restrict__ in, size_t in_stride, const float *__restrict__ sqrt_d, size_t d_stride,
         float2 *__restrict__ out, size_t out_stride, double *__restrict__ partial, int part_stride, Tables tb,
         const __grid_constant__ TabSeq seq, int N, float tau, int nb, const __grid_constant__ CUtensorMap w1map,
         int staged) {
  using C = CtaK<L>;
  constexpr int T = L / 16;
  constexpr bool STG_OK = HOLO_STAGE && HOLO_STAGE_X2 && HOLO_X2_LOOP && MODE != X2_ADJ && C::G >= 2;
  extern __shared__ float4 sm4[];
  __shared__ double red[32];
  __shared__ uint64_t bars[2];
  __shared__ uint64_t sbar;
  float2 *sm = reinterpret_cast<float2 *>(sm4);
  Xch x = C::xch(sm);
  // the launch's only table (hdet_j / L; seq.p[0]) into the first slot, once
  float2 *h = slot_base<L, false>(sm);
  const bool stg = STG_OK && staged;
  // [exchange][table][<= 112 B pad][row slot, 128-byte aligned: TMA destination] (Smem::XHS)
  float2 *zs = h + L;
  zs += ((128u - (smem_u32(zs) & 127u)) & 127u) / sizeof(float2);
  if (threadIdx.x == 0) {
    mbar_init(bars, 1);
    if (stg) mbar_init(&sbar, 1);
    fence_mbar_init();
  }
  __syncthreads();
  const int t = C::t(), y0 = blockIdx.x * C::G;
  const int f0 = HOLO_X2_LOOP ? 0 : blockIdx.y, f1 = HOLO_X2_LOOP ? nb : blockIdx.y + 1;
  if (stg) RowStage{&w1map, &sbar, -1, y0, 0}.template issue<L>(zs, f0);
  if (threadIdx.x == 0) {
    mbar_expect_tx(bars, L * sizeof(float2));
    bulk_g2s(h, seq.p[0], L * sizeof(float2), bars);
  }
#pragma unroll 1
  for (int fb = f0; fb < f1; fb++) {
    if (HOLO_X2_LOOP && fb + 1 < f1) {  // the next frame's rows into L2 (one lane per 32-byte sector)
      if (MODE == X2_ADJ) {
        if (threadIdx.x == 0 && y0 < N)
          prefetch_l2_any(in + (fb + 1) * in_stride + (size_t)y0 * N, 8u * N * (y0 + C::G <= N ? C::G : N - y0));
      } else if (!stg && (threadIdx.x & 3) == 0 && y0 + C::g() < N) {
        const float2 *nx = in + (fb + 1) * in_stride;
#pragma unroll
        for (int r = 0; r < 16; r++) prefetch_l2_sector(nx + p2(y0 + C::g(), t + r * T, N));
      }
      if ((MODE == X2_GRAD || MODE == X2_OBJ) && threadIdx.x == 32 && y0 < N)
        prefetch_l2_any(sqrt_d + (fb + 1) * d_stride + (size_t)y0 * N, 4u * N * (y0 + C::G <= N ? C::G : N - y0));
    }
    x2_frame<L, MODE, TM>(in + fb * in_stride, sqrt_d ? sqrt_d + fb * d_stride : nullptr,
                          out ? out + fb * out_stride : nullptr, partial + (size_t)fb * part_stride, h, x, tb.tw, red,
                          N, tau, bars, stg ? zs : nullptr,
                          RowStage{&w1map, &sbar, fb + 1 < f1 ? fb + 1 : -1, y0, (uint32_t)((fb - f0) & 1)});
  }
}

// ----------------------------------------------------------------------------- Y2
// Angle-batched like Y1: nb frames of plane j; frame b reads V1 + b N L, a + b L L and
// writes T3j + b * fstride.  The probe-gradient accumulator G_j (Eq. (12)) is
// read-modify-written once per frame by the SAME CTA for its columns, so across the
// batch it stays in L2 (DRAM sees ~one read + one write per batch).
// Per frame:  v = D_y^* pad(V1 col);  G_j += conj(a) v;  T3j = (M S)_y^*(conj(q_j) v)
// PS: instead of G_j += conj(a) v, the frame's probe-gradient term u = conj(a) v is taken to
// the y-spectrum with conj(Hq_y) and stored to ut (XG finishes the x axis and accumulates
// the Fourier-domain sum, Eq. (12) with Q_kj^* = S_{-s^p} P_{-omega}); conj(q_kj) comes from qk.
// Column staging in Y2 (HOLO_STAGE_Y2, default 1; non-PS launches with G >= 2): the CTA's V1 block
// (8 G N bytes, contiguous in P2) and, when the probe gradient is accumulated, its block of a
// (8 G L bytes) are bulk-copied (cp.async.bulk + mbarrier) through the thread-private slot instead
// of 2 x 16 LDG per thread: V1 of frame b + 1 is issued once the magnification's last source read of
// frame b is behind a barrier (mag_adj's src_freed hook; the first half's term is parked in
// registers as in X3), a of frame b once the first transform's barriers are past the V1 reads, so
// it lands behind D_y^*'s two transforms.  Copies complete alternating phases of one mbarrier.
#ifndef HOLO_STAGE_Y2
#define HOLO_STAGE_Y2 1
#endif
#ifndef HOLO_Y2_QEARLY
#define HOLO_Y2_QEARLY 0  // 1: q_j into registers before the wait for the block of a (spills: Y2 249 -> 271 us/frame); 2: L1 prefetch (252); 0: off
#endif
struct Y2Stage {
  uint64_t *bar;
  const float2 *ablk;   // this frame's block of a (nullptr: not staged)
  const float2 *vnext;  // the next frame's V1 block (nullptr: last frame)
  uint32_t vbytes, abytes;
  uint32_t vphase;      // parity of this frame's V1 copy (its a copy, if any, completes parity 1)
};

template <int L, bool PS, bool STG>
__device__ __noinline__ TabPipe<L> y2_frame(const float2 *__restrict__ vin, const float2 *__restrict__ ab,
                                      const float2 *__restrict__ qj, float2 *__restrict__ Gj, float2 *__restrict__ ut,
                                      float2 *__restrict__ t3, const float4 *__restrict__ tw, const TabSeq &seq,
                                      TabPipe<L> pipe, float2 *sm, int mag, int N, int fourier, Y2Stage st) {
  using C = CtaK<L>;
  constexpr int T = L / 16;
  Xch x = C::xch(sm);
  const Priv<NT> Y{priv_base<L>(sm)};
  float2 *Sb = priv_base<L>(sm);
  const int t = C::t(), col = blockIdx.x * C::G + C::g();
  const int o = (L - N) / 2;
  float2 v[16];
  if constexpr (STG) {
    const int v0 = 2 * N * (C::g() >> 1) + (C::g() & 1);  // element (row, col) of the V1 block at v0 + 2 row
    mbar_wait(st.bar, st.vphase);
#pragma unroll
    for (int r = 0; r < 16; r++) {
      const int row = t + r * T - o;
      v[r] = (row >= 0 && row < N) ? Sb[v0 + 2 * row] : make_float2(0.f, 0.f);
    }
    fence_proxy_async();  // this thread's reads of the slot precede the async write of a
  } else {
#pragma unroll
    for (int r = 0; r < 16; r++) {
      const int row = t + r * T - o;
      v[r] = (row >= 0 && row < N) ? ldg2(vin + p2(row, col, N)) : make_float2(0.f, 0.f);
    }
  }
  fft<L, false>(v, x, t, tw);
  if constexpr (STG) {
    if (st.ablk && threadIdx.x == 0) {  // every thread is past its V1 reads (the transform's barriers)
      fence_proxy_async();
      mbar_expect_tx(st.bar, st.abytes);
      bulk_g2s(Sb, st.ablk, st.abytes, st.bar);
    }
  }
  {
    const float2 *h = pipe.take(seq);  // hdet_j / L, conjugated
#pragma unroll
    for (int r = 0; r < 16; r++) v[r] = cmulc(v[r], h[t + r * T]);
    pipe.done(seq);
  }
  fft<L, true>(v, x, t, tw);
  const int s0 = stage_idx<L>(C::g(), t);
  // the thread-private slot: the staged layout (STG; element (y, col) where the block of a has it) or Priv
  auto slot = [&](int r) -> float2 & { if constexpr (STG) return Sb[s0 + 2 * r * T]; else return Y[r]; };
  float2 qv[16];
  bool qearly = false;
  if (PS && ut) {
#pragma unroll
    for (int r = 0; r < 16; r++) {
      Y[r] = v[r];
      v[r] = cmulc(v[r], ldg2(ab + p2(t + r * T, col, L)));  // conj(a) v
    }
    fft<L, false>(v, x, t, tw);
    const float2 *hq = pipe.take(seq);  // Hq_y(k, j), conjugated
#pragma unroll
    for (int r = 0; r < 16; r++) v[r] = cmulc(v[r], hq[t + r * T]);
    pipe.done(seq);
    st_p2_col<L>(v, ut, col, L, t);
#pragma unroll
    for (int r = 0; r < 16; r++) v[r] = Y[r];
  } else if (Gj) {
    if constexpr (STG && HOLO_Y2_QEARLY == 2) {
      if (t3) {  // q_j's sectors into L1 while the block of a is awaited and G_j updated
#pragma unroll
        for (int r = 0; r < 16; r++)
          asm volatile("prefetch.global.L1 [%0];" ::"l"(qj + p2(t + r * T, col, L)) : "memory");
      }
    }
    if constexpr (STG && HOLO_Y2_QEARLY == 1) {
      // q_j's L2 round trip overlaps the wait for the block of a and the G_j updates
      if (t3) {
#pragma unroll
        for (int r = 0; r < 16; r++) qv[r] = ldg2(qj + p2(t + r * T, col, L));
        qearly = true;
      }
    }
    if constexpr (STG) mbar_wait(st.bar, 1);
#pragma unroll
    for (int r = 0; r < 16; r++) {
      const size_t gi = p2(t + r * T, col, L);
      float2 av;
      if constexpr (STG) av = slot(r); else av = ldg2(ab + gi);
      red_add2(Gj + gi, cmulc(v[r], av));  // G_j += conj(a) v (this thread owns gi)
    }
  }
  auto issue_next = [&]() {  // all threads, behind a CTA barrier that follows their last slot access
    if constexpr (STG) {
      if (st.vnext && threadIdx.x == 0) {
        fence_proxy_async();
        mbar_expect_tx(st.bar, st.vbytes);
        bulk_g2s(Sb, st.vnext, st.vbytes, st.bar);
      }
    }
  };
  if (!t3) {
    if constexpr (STG) {
      fence_proxy_async();
      __syncthreads();
      issue_next();
    }
    return pipe;
  }
  if (qearly) {
#pragma unroll
    for (int r = 0; r < 16; r++) v[r] = cmulc(v[r], qv[r]);
  } else {
#pragma unroll
    for (int r = 0; r < 16; r++) v[r] = cmulc(v[r], ldg2(qj + p2(t + r * T, col, L)));  // qj: q_j, or q_kj (PS)
  }
  if (mag) {
#pragma unroll
    for (int r = 0; r < 16; r++) slot(r) = v[r];
    if constexpr (STG) {
      float2 e[16];
      mag_adj<L>(
          v, [&](int r) { const float2 z = slot(r); if (r == 15) fence_proxy_async(); return z; },
          [&](int r, float2 val) { e[r] = val; }, [&](int r) { return e[r]; }, pipe, seq, true, x, t, tw, issue_next);
    } else {
      mag_adj<L>(
          v, [&](int r) { return Y[r]; }, [&](int r, float2 e) { Y[r] = e; }, [&](int r) { return Y[r]; }, pipe, seq,
          true, x, t, tw);
    }
  } else {
    if constexpr (STG) fence_proxy_async();
    fft<L, false>(v, x, t, tw);
    issue_next();
    const float2 *cr = pipe.take(seq);
#pragma unroll
    for (int r = 0; r < 16; r++) v[r] = cmulc(v[r], cr[t + r * T]);
    pipe.done(seq);
  }
  if (!fourier) fft<L, true>(v, x, t, tw);  // HOLO_FOURIER: T3 keeps the y-spectrum (X3 works on it row by row)
  st_p2_col<L>(v, t3, col, L, t);
  return pipe;
}

template <int L, bool PS>
__global__ void __launch_bounds__(NT, CTAS_PER_SM)
    k_y2(const float2 *__restrict__ V1, const float2 *__restrict__ a, const float2 *__restrict__ qj,
         const float2 *__restrict__ Qk, float2 *__restrict__ Gj, float2 *__restrict__ Ut, float2 *__restrict__ T3j,
         size_t fstride, Tables tb, const __grid_constant__ TabSeq seq, int mag, int N, int nb, int fourier) {
  using C = CtaK<L>;
  constexpr bool STG = HOLO_STAGE && HOLO_STAGE_Y2 && !PS && C::G >= 2;
  extern __shared__ float4 sm4[];
  __shared__ uint64_t bars[2];
  __shared__ uint64_t sbar;
  float2 *sm = reinterpret_cast<float2 *>(sm4);
  if (STG && threadIdx.x == 0) {
    mbar_init(&sbar, 1);
    fence_mbar_init();
  }
  TabPipe<L> pipe;
  pipe.start(seq, slot_base<L, true>(sm), bars);
  const int col0 = blockIdx.x * C::G;
  constexpr int PF_COLS = C::G < 2 ? 2 : C::G;  // whole P2 column pairs (16-byte aligned blocks)
  const bool wq = PS ? Ut != nullptr : Gj != nullptr;
  const uint32_t VBYTES = 8u * C::G * N, ABYTES = 8u * C::G * L;
  if (STG) {
    __syncthreads();
    if (threadIdx.x == 0) {
      mbar_expect_tx(&sbar, VBYTES);
      bulk_g2s(priv_base<L>(sm), V1 + p2(0, col0, N), VBYTES, &sbar);
    }
  }
#pragma unroll 1
  for (int b = 0; b < nb; b++) {
    const float2 *vin = V1 + (size_t)b * N * L;
    const float2 *ab = a + (size_t)b * L * L;
    if (threadIdx.x == 0 && b + 1 < nb) {
      prefetch_l2(vin + (size_t)N * L + p2(0, col0 & ~1, N), 8u * PF_COLS * N);
      if (wq) prefetch_l2(ab + (size_t)L * L + p2(0, col0 & ~1, L), 8u * PF_COLS * L);
    }
    const Y2Stage st{&sbar, wq ? ab + p2(0, col0, L) : nullptr, b + 1 < nb ? vin + (size_t)N * L + p2(0, col0, N) : nullptr,
                     VBYTES, ABYTES, wq ? 0u : (uint32_t)(b & 1)};
    pipe = y2_frame<L, PS, STG>(vin, ab, PS ? Qk + (size_t)b * L * L : qj, Gj, (PS && Ut) ? Ut + (size_t)b * fstride : nullptr,
                    T3j ? T3j + (size_t)b * fstride : nullptr, tb.tw, seq, pipe, sm, mag, N, fourier, st);
  }
}

// ----------------------------------------------------------------------------- X3
#ifndef HOLO_X3_TAIL
#define HOLO_X3_TAIL 1  // the earlier planes' sum is read back in the kernel tail, together with eta
#endif
#ifndef HOLO_X3_ZACC
#define HOLO_X3_ZACC 0  // 1: plane sum in the private slot, source read twice from global (L2)
#endif
#if HOLO_X3_ZACC
#undef HOLO_X3_TAIL
#define HOLO_X3_TAIL 0
#endif
// rows: g_k row = scale * IFFT( sum_j W_j ),  W_j = spectrum of (M S)_x^* T3_j row;
// partial[blk][0] = sum |g|^2, partial[blk][1] = sum Re(g conj(eta))   (g, eta row-major)
// The sum over planes is kept in the g row itself (L2-resident between planes); each plane
// is one non-inlined call (spill-free magnification).
template <int L, bool STG>
__device__ __noinline__ TabPipe<L> x3_plane(const float2 *__restrict__ T3j, float2 *__restrict__ grow,
                                      const float4 *__restrict__ tw, const TabSeq &seq, TabPipe<L> pipe, float2 *sm,
                                      bool mag, int j, bool last, RowStage rs, float2 *pv) {
  using C = CtaK<L>;
  constexpr int T = L / 16;
  Xch x = C::xch(sm);
  const Priv<NT> Z{pv};  // the private slot, 128-byte aligned for the tensor copies (k_x3)
  float2 *Zs = pv;
  const int t = C::t(), y = blockIdx.x * C::G + C::g();
  float2 v[16];
  if constexpr (STG) {
    auto S = [&](int r) {
      const int xx = t + r * T;
      return Zs[2 * (C::G * (xx >> 1) + C::g()) + (xx & 1)];
    };
    auto freed = [&]() {
      if (rs.next >= 0) rs.template issue<L>(Zs, rs.next);
    };
    mbar_wait(rs.bar, rs.phase);
    if (mag) {
      float2 e[16];
      mag_adj<L>(
          v, S, [&](int r, float2 val) { e[r] = val; }, [&](int r) { return e[r]; }, pipe, seq, j > 0, x, t, tw,
          freed);
    } else {
#pragma unroll
      for (int r = 0; r < 16; r++) v[r] = S(r);
      fft<L, false>(v, x, t, tw);
      freed();
      const float2 *cr = pipe.take(seq);
#pragma unroll
      for (int r = 0; r < 16; r++) v[r] = cmulc(v[r], cr[t + r * T]);
      pipe.done(seq);
    }
  } else {
#if HOLO_X3_ZACC
  // the plane sum stays in the private slot Z; the magnification reads its source twice from
  // global memory (the second read hits L2)
  if (mag) {
    if (!last && (threadIdx.x & 3) == 0) {
#pragma unroll
      for (int r = 0; r < 16; r++) prefetch_l2_sector(T3j + (size_t)L * L + p2(y, t + r * T, L));
    }
    float2 e[16];
    mag_adj<L>(
        v, [&](int r) { return ldg2(T3j + p2(y, t + r * T, L)); }, [&](int r, float2 val) { e[r] = val; },
        [&](int r) { return e[r]; }, pipe, seq, j > 0, x, t, tw);
  } else {
    ld_p2_row<L>(v, T3j, y, L, t);
    fft<L, false>(v, x, t, tw);
    const float2 *cr = pipe.take(seq);
#pragma unroll
    for (int r = 0; r < 16; r++) v[r] = cmulc(v[r], cr[t + r * T]);
    pipe.done(seq);
  }
#pragma unroll
  for (int r = 0; r < 16; r++) Z[r] = j == 0 ? v[r] : cadd(Z[r], v[r]);
  (void)grow;
  return pipe;
#endif
  if (mag) {
    // the source row is read ONCE into the thread-private slot; the first half's term is
    // parked in registers (as in X1)
#pragma unroll
    for (int r = 0; r < 16; r++) Z[r] = ldg2(T3j + p2(y, t + r * T, L));
    if (!last && (threadIdx.x & 3) == 0) {  // the next plane's rows into L2 (one lane per 32-byte sector)
#pragma unroll
      for (int r = 0; r < 16; r++) prefetch_l2_sector(T3j + (size_t)L * L + p2(y, t + r * T, L));
    }
    float2 e[16];
    mag_adj<L>(
        v, [&](int r) { return Z[r]; }, [&](int r, float2 val) { e[r] = val; }, [&](int r) { return e[r]; }, pipe,
        seq, j > 0, x, t, tw);
  } else {
    ld_p2_row<L>(v, T3j, y, L, t);
    fft<L, false>(v, x, t, tw);
    const float2 *cr = pipe.take(seq);
#pragma unroll
    for (int r = 0; r < 16; r++) v[r] = cmulc(v[r], cr[t + r * T]);
    pipe.done(seq);
  }
  }  // !STG
  // sum over planes in the g row (one owner thread per element): store, then fire-and-forget
  // adds, and the last plane reads the sum back (L2, __ldcg) into the private slot
  if (j == 0 && !last) {
#pragma unroll
    for (int r = 0; r < 16; r++) grow[t + r * T] = v[r];
  } else if (!last) {
#pragma unroll
    for (int r = 0; r < 16; r++) red_add2(grow + t + r * T, v[r]);
  } else {
#if HOLO_X3_TAIL
    // the last plane's term goes to the kernel tail through the slot; the tail adds the L2-resident
    // sum of the earlier planes (one round trip together with its eta reads)
#pragma unroll
    for (int r = 0; r < 16; r++) Z[r] = v[r];
#else
#pragma unroll
    for (int r = 0; r < 16; r++) Z[r] = j > 0 ? cadd(__ldcg(grow + t + r * T), v[r]) : v[r];
#endif
  }
  return pipe;
}

template <int L>
__global__ void __launch_bounds__(NT, CTAS_PER_SM)
    k_x3(const float2 *__restrict__ T3, const float2 *__restrict__ eta, float2 *__restrict__ g,
         double *__restrict__ partial, Tables tb, const __grid_constant__ TabSeq seq, int nz, uint32_t magmask,
         float scale, int fourier, const __grid_constant__ CUtensorMap t3map, int pl0, int staged) {
  using C = CtaK<L>;
  constexpr int T = L / 16;
  constexpr bool STG_OK = HOLO_STAGE && !HOLO_X3_ZACC && C::G >= 2;
  extern __shared__ float4 sm4[];
  __shared__ double red[32];
  __shared__ uint64_t bars[2];
  __shared__ uint64_t sbar;
  float2 *sm = reinterpret_cast<float2 *>(sm4);
  const int y0 = blockIdx.x * C::G;
  const bool stg = STG_OK && staged;
  if (stg && threadIdx.x == 0) {
    mbar_init(&sbar, 1);
    fence_mbar_init();
  }
  // [exchange][<= 112 B pad][private slot, 128-byte aligned: TMA destination][table slots] (Smem::XPT3)
  float2 *pv = priv_base<L>(sm);
  pv += ((128u - (smem_u32(pv) & 127u)) & 127u) / sizeof(float2);
  TabPipe<L> pipe;
  pipe.start(seq, pv + CtaK<L>::PRIV / sizeof(float2), bars);
  if (stg) {
    __syncthreads();
    RowStage{&t3map, &sbar, -1, y0, 0}.template issue<L>(pv, pl0);
  }
  const int t = C::t(), y = blockIdx.x * C::G + C::g();
  float2 *grow = g + (size_t)y * L;  // also the Fourier-domain accumulator of sum_j W_j
  if (eta && threadIdx.x == 0) prefetch_l2(eta + (size_t)blockIdx.x * C::G * L, 8u * C::G * L);  // read at the end
  if (STG_OK && stg) {
#pragma unroll 1
    for (int j = 0; j < nz; j++)
      pipe = x3_plane<L, STG_OK>(T3 + (size_t)j * L * L, grow, tb.tw, seq, pipe, sm, (magmask >> j) & 1u, j,
                                 j + 1 == nz, RowStage{&t3map, &sbar, j + 1 < nz ? pl0 + j + 1 : -1, y0, (uint32_t)(j & 1)},
                                 pv);
  } else {
#pragma unroll 1
    for (int j = 0; j < nz; j++)
      pipe = x3_plane<L, false>(T3 + (size_t)j * L * L, grow, tb.tw, seq, pipe, sm, (magmask >> j) & 1u, j,
                                j + 1 == nz, RowStage{}, pv);
  }
  Xch x = C::xch(sm);
  const Priv<NT> Z{pv};
  float2 v[16];
#if HOLO_X3_TAIL
  if (fourier && eta) {
    // no transform in the tail: the plane sum and eta are fetched together
    double gg = 0.0, ge = 0.0;
    float2 sv[16], ev[16];
#pragma unroll
    for (int r = 0; r < 16; r++) {
      sv[r] = nz > 1 ? __ldcg(grow + t + r * T) : make_float2(0.f, 0.f);
      ev[r] = ldg2(eta + (size_t)y * L + t + r * T);
    }
#pragma unroll
    for (int r = 0; r < 16; r++) {
      const float2 a = cscale(cadd(sv[r], Z[r]), scale);
      grow[t + r * T] = a;
      gg += (double)(a.x * a.x + a.y * a.y);
      ge += (double)(a.x * ev[r].x + a.y * ev[r].y);
    }
    const double s0 = block_sum(gg, red);
    const double s1 = block_sum(ge, red);
    if (threadIdx.x == 0) {
      const double ps = 1.0 / ((double)L * L);
      partial[2 * blockIdx.x] = s0 * ps;
      partial[2 * blockIdx.x + 1] = s1 * ps;
    }
    return;
  }
#pragma unroll
  for (int r = 0; r < 16; r++) v[r] = nz > 1 ? cadd(__ldcg(grow + t + r * T), Z[r]) : Z[r];
#else
#pragma unroll
  for (int r = 0; r < 16; r++) v[r] = Z[r];
#endif
  // HOLO_FOURIER: the rows are y-spectral (T3 from Y2) and the x-spectrum is kept: g = DFT2(grad) / L^2
  // before the caller's scale (2 L^2), and the dots carry Parseval's 1/L^2
  if (!fourier) fft<L, true>(v, x, t, tb.tw);
  double gg = 0.0, ge = 0.0;
#pragma unroll
  for (int r = 0; r < 16; r++) {
    const float2 a = cscale(v[r], scale);
    grow[t + r * T] = a;
    gg += (double)(a.x * a.x + a.y * a.y);
    if (eta) {
      const float2 e = ldg2(eta + (size_t)y * L + t + r * T);
      ge += (double)(a.x * e.x + a.y * e.y);
    }
  }
  const double s0 = block_sum(gg, red);
  const double s1 = block_sum(ge, red);
  if (threadIdx.x == 0) {
    const double ps = fourier ? 1.0 / ((double)L * L) : 1.0;  // Parseval: object-domain dots
    partial[2 * blockIdx.x] = s0 * ps;
    partial[2 * blockIdx.x + 1] = s1 * ps;
  }
}

// The batched X3 (HOLO_X3_BATCH, default 1; needs the T3 tensor map): one launch for the nb angles of a
// batch, each CTA looping over the (angle, plane) pairs for its G rows.  The tensor copy of pair m + 1
// is issued from pair m's src_freed hook also across an angle boundary, and the angle's tail (plane
// sum, scale, g row, the two dots) runs inside the last plane's body on the values in registers, so the
// slot is free for that copy.  Per-launch / per-angle state sits in a control block in shared memory
// (the plane body finds it from the shared-memory base; kernel-level spills cost L2 round trips here).
#ifndef HOLO_X3_BATCH
#define HOLO_X3_BATCH 1
#endif
#ifndef HOLO_X3_PF
#define HOLO_X3_PF 1  // tensor prefetch (L2) of the next (angle, plane) pair's rows at the start of each pair
#endif
#ifndef HOLO_X3_WJ
#define HOLO_X3_WJ 0  // 1: plane terms stored in place of the consumed T3 rows and summed in the tail (measured slower: X3 222 vs 191 us/frame); 0: L2 reductions into g
#endif
template <int L>
struct X3Ctl {
  uint64_t bar;
  const CUtensorMap *map;
  float2 *t3;         // the T3 workspace (plane 0 of the map)
  const float2 *eta;  // this angle's eta (nullptr: none), g and partials
  float2 *g;
  double *partial;
  float scale;
  static constexpr size_t OFF = CtaK<L>::XBYTES + CtaK<L>::PRIV + 128 + TabPipe<L>::BYTES;  // after Smem::XPT3
  __device__ __forceinline__ static X3Ctl *at(float2 *sm) {
    return reinterpret_cast<X3Ctl *>(reinterpret_cast<char *>(sm) + OFF);
  }
};
template <int L>
__device__ __forceinline__ float2 *x3_slot(float2 *sm) {
  float2 *pv = priv_base<L>(sm);
  return pv + ((128u - (smem_u32(pv) & 127u)) & 127u) / sizeof(float2);
}
enum { X3F_MAG = 1, X3F_SYNC0 = 2, X3F_FIRST = 4, X3F_LAST = 8, X3F_FOURIER = 16, X3F_PHASE = 32, X3F_NEXT = 64 };

template <int L>
__device__ __noinline__ TabPipe<L> x3s_plane(const float4 *__restrict__ tw, const TabSeq &seq, TabPipe<L> pipe,
                                       float2 *sm, int flags) {  // flags: X3F_* | j << 8 | map plane << 16
  using C = CtaK<L>;
  constexpr int T = L / 16;
  __shared__ double red[32];
  Xch x = C::xch(sm);
  const int t = C::t();
  float2 v[16];
  {
    // element (y0 + g, x = t + r T) of the staged rows at 2 (G (x >> 1) + g) + (x & 1); T is even
    const float2 *zb = x3_slot<L>(sm) + 2 * (C::G * (t >> 1) + C::g()) + (t & 1);
    auto S = [&](int r) { return zb[r * (C::G * T)]; };
    // the next pair's tensor copies, one per thread (no loop state beside the transforms' registers)
    constexpr int BOXC = L / 2 < 256 ? L / 2 : 256, NC = (L / 2) / BOXC;
    auto freed = [&]() {
      const int i = threadIdx.x;
      if (i < NC && (flags & X3F_NEXT)) {
        X3Ctl<L> *c = X3Ctl<L>::at(sm);
        if (i == 0) mbar_expect_tx(&c->bar, 8u * C::G * L);
        tma_load_4d(x3_slot<L>(sm) + 2 * C::G * BOXC * i, c->map, 0, (int)(blockIdx.x * C::G), BOXC * i,
                    (flags >> 16) + 1, &c->bar);
      }
    };
#if HOLO_X3_PF
    // the next pair's rows into L2 now (a tensor prefetch: 2048 strided 32-byte pieces from DRAM), so the
    // copy issued from the src_freed hook, one transform before it is needed, reads L2
    if ((int)threadIdx.x < NC && (flags & X3F_NEXT))
      tma_prefetch_4d(X3Ctl<L>::at(sm)->map, 0, (int)(blockIdx.x * C::G), BOXC * threadIdx.x, (flags >> 16) + 1);
#endif
    mbar_wait(&X3Ctl<L>::at(sm)->bar, (flags & X3F_PHASE) ? 1u : 0u);
    if (flags & X3F_MAG) {
      float2 e[16];
      mag_adj<L>(
          v, S, [&](int r, float2 val) { e[r] = val; }, [&](int r) { return e[r]; }, pipe, seq, (flags & X3F_SYNC0) != 0, x,
          t, tw, freed);
    } else {
#pragma unroll
      for (int r = 0; r < 16; r++) v[r] = S(r);
      fft<L, false>(v, x, t, tw);
      freed();
      const float2 *cr = pipe.take(seq);
#pragma unroll
      for (int r = 0; r < 16; r++) v[r] = cmulc(v[r], cr[t + r * T]);
      pipe.done(seq);
    }
  }
  const X3Ctl<L> *c = X3Ctl<L>::at(sm);
  const size_t row = (size_t)(blockIdx.x * C::G + C::g()) * L + t;
  float2 *grow = c->g + row;  // also the Fourier-domain accumulator of sum_j W_j (one owner thread per element)
#if HOLO_X3_WJ
  // W_j overwrites this CTA's (consumed) rows of its T3 plane with plain stores; the angle's tail sums
  // the planes (one round trip of independent L2 reads) instead of nz - 1 rounds of L2 reductions
  const int pl = flags >> 16, nprev = (flags >> 8) & 0xff;
  if (!(flags & X3F_LAST)) {
    st_p2_row<L>(v, c->t3 + (size_t)pl * L * L, blockIdx.x * C::G + C::g(), L, t);
    return pipe;
  }
  {
    const float2 *w0 = c->t3 + (size_t)(pl - nprev) * L * L;
    const int y = blockIdx.x * C::G + C::g();
#pragma unroll
    for (int r = 0; r < 16; r++) {
      const size_t i = p2(y, t + r * T, L);
      float2 acc = make_float2(0.f, 0.f);
#pragma unroll
      for (int jj = 0; jj < HOLO_MAX_NZ - 1; jj++)
        if (jj < nprev) acc = cadd(acc, __ldcg(w0 + (size_t)jj * L * L + i));
      v[r] = cadd(acc, v[r]);
    }
    flags |= X3F_FIRST;  // the sum is complete: nothing to read back from the g row
  }
#else
  if (!(flags & X3F_LAST)) {
    if (flags & X3F_FIRST) {
#pragma unroll
      for (int r = 0; r < 16; r++) grow[r * T] = v[r];
    } else {
#pragma unroll
      for (int r = 0; r < 16; r++) red_add2(grow + r * T, v[r]);
    }
    return pipe;
  }
#endif
  // the angle's tail: the earlier planes' sum (L2) and eta are fetched together
  const float2 *erow = c->eta ? c->eta + row : nullptr;
  const float scale = c->scale;
  double gg = 0.0, ge = 0.0;
  if (flags & X3F_FOURIER) {
    // all reads first: the g-row stores below alias the g-row reads, so a single loop would wait for
    // one L2 round trip per element (measured: 9 % of the pass)
#pragma unroll
    for (int r = 0; r < 16; r++)
      if (!(flags & X3F_FIRST)) v[r] = cadd(__ldcg(grow + r * T), v[r]);
    float2 ev[16];
#pragma unroll
    for (int r = 0; r < 16; r++) ev[r] = erow ? ldg2(erow + r * T) : make_float2(0.f, 0.f);
#pragma unroll
    for (int r = 0; r < 16; r++) {
      const float2 a = cscale(v[r], scale);
      grow[r * T] = a;
      gg += (double)(a.x * a.x + a.y * a.y);
      ge += (double)(a.x * ev[r].x + a.y * ev[r].y);
    }
  } else {
    if (!(flags & X3F_FIRST)) {
#pragma unroll
      for (int r = 0; r < 16; r++) v[r] = cadd(__ldcg(grow + r * T), v[r]);
    }
    fft<L, true>(v, x, t, tw);
    float2 ev[16];
#pragma unroll
    for (int r = 0; r < 16; r++) ev[r] = erow ? ldg2(erow + r * T) : make_float2(0.f, 0.f);
#pragma unroll
    for (int r = 0; r < 16; r++) {
      const float2 a = cscale(v[r], scale);
      grow[r * T] = a;
      gg += (double)(a.x * a.x + a.y * a.y);
      ge += (double)(a.x * ev[r].x + a.y * ev[r].y);
    }
  }
  const double s0 = block_sum(gg, red);
  const double s1 = block_sum(ge, red);
  if (threadIdx.x == 0) {
    const double ps = (flags & X3F_FOURIER) ? 1.0 / ((double)L * L) : 1.0;  // Parseval: object-domain dots
    c->partial[2 * blockIdx.x] = s0 * ps;
    c->partial[2 * blockIdx.x + 1] = s1 * ps;
  }
  return pipe;
}

// T3 [nb][nz][L][L] (map planes pl0 ...), eta / g: the batch's first angle (angles L^2 apart),
// partial: 2 gridDim.x doubles per angle
template <int L>
__global__ void __launch_bounds__(NT, CTAS_PER_SM)
    k_x3s(float2 *__restrict__ T3, const float2 *__restrict__ eta, float2 *__restrict__ g, double *__restrict__ partial, Tables tb,
          const __grid_constant__ TabSeq seq, int nz, uint32_t magmask, float scale, int fourier,
          const __grid_constant__ CUtensorMap t3map, int pl0, int nb) {
  using C = CtaK<L>;
  extern __shared__ float4 sm4[];
  __shared__ uint64_t bars[2];
  float2 *sm = reinterpret_cast<float2 *>(sm4);
  X3Ctl<L> *ctl = X3Ctl<L>::at(sm);
  if (threadIdx.x == 0) {
    mbar_init(&ctl->bar, 1);
    ctl->map = &t3map;
    ctl->t3 = T3;
    ctl->scale = scale;
    fence_mbar_init();
  }
  // [exchange][<= 112 B pad][private slot, 128-byte aligned: TMA destination][table slots][control block]
  TabPipe<L> pipe;
  pipe.start(seq, x3_slot<L>(sm) + C::PRIV / sizeof(float2), bars);
  __syncthreads();
  RowStage{&t3map, &ctl->bar, -1, (int)(blockIdx.x * C::G), 0}.template issue<L>(x3_slot<L>(sm), pl0);
#pragma unroll 1
  for (int m = 0; m < nb * nz; m++) {
    const int b = m / nz, j = m - b * nz;
    if (threadIdx.x == 0) {
      if (j == 0) {  // a new angle (every thread is past the previous angle's tail barriers)
        const size_t ao = (size_t)b * L * L;
        ctl->eta = eta ? eta + ao : nullptr;
        ctl->g = g + ao;
        ctl->partial = partial + (size_t)b * 2 * gridDim.x;
        if (eta) prefetch_l2(eta + ao + (size_t)blockIdx.x * C::G * L, 8u * C::G * L);  // read in the angle's tail
      }
    }
    const int flags = (((magmask >> j) & 1u) ? X3F_MAG : 0) | (m > 0 ? X3F_SYNC0 : 0) | (j == 0 ? X3F_FIRST : 0) |
                      (j + 1 == nz ? X3F_LAST : 0) | (fourier ? X3F_FOURIER : 0) | ((m & 1) ? X3F_PHASE : 0) |
                      (m + 1 < nb * nz ? X3F_NEXT : 0) | (j << 8) |
                      ((pl0 + m) << 16);
    pipe = x3s_plane<L>(tb.tw, seq, pipe, sm, flags);
  }
}

// ----------------------------------------------------------------------------- XQ, XG (PS)
// Per-frame probe shifts (O19): with Qhat = DFT2 q (P2 [fy][fx]) and Hq(k,j) = h_omega_j r_{s^p_kj} / L
// per axis, q_kj = IDFT_y(Hq_y IDFT_x(Hq_x Qhat)).
// XQ (rows fy, the angles of a batch): Qt[m] row = IFFT_x(Hq_x(k, j) Qhat row) for the m = b nz + j
// (angle, plane) pairs of the batch (nz argument = their count), Qhat row read once   (P2 [fy][x])
template <int L>
__global__ void __launch_bounds__(NT, CTAS_PER_SM)
    k_xq(const float2 *__restrict__ Qhat, float2 *__restrict__ Qt, Tables tb, const __grid_constant__ TabSeq seq,
         int nz) {
  using C = CtaK<L>;
  constexpr int T = L / 16;
  extern __shared__ float4 sm4[];
  __shared__ uint64_t bars[2];
  float2 *sm = reinterpret_cast<float2 *>(sm4);
  Xch x = C::xch(sm);
  const Priv<NT> X{priv_base<L>(sm)};
  TabPipe<L> pipe;
  pipe.start(seq, slot_base<L, true>(sm), bars);
  const int t = C::t(), y = blockIdx.x * C::G + C::g();
  {
    float2 v[16];
    ld_p2_row<L>(v, Qhat, y, L, t);
#pragma unroll
    for (int r = 0; r < 16; r++) X[r] = v[r];
  }
#pragma unroll 1
  for (int j = 0; j < nz; j++) {
    float2 v[16];
    const float2 *hq = pipe.take(seq, j > 0);
#pragma unroll
    for (int r = 0; r < 16; r++) v[r] = cmul(X[r], hq[t + r * T]);
    pipe.done(seq);
    fft<L, true>(v, x, t, tb.tw);
    st_p2_row<L>(v, Qt + (size_t)j * L * L, y, L, t);
  }
}

// XG (rows fy, the angles of a batch): Ghat row (+)= sum_m conj(Hq_x(k, j)) FFT_x(Ut[m] row) over the
// m = b nz + j pairs (nz argument = their count), one Ghat read-modify-write per batch   (first: overwrite)
template <int L>
__global__ void __launch_bounds__(NT, CTAS_PER_SM)
    k_xg(const float2 *__restrict__ Ut, float2 *__restrict__ Ghat, Tables tb, const __grid_constant__ TabSeq seq,
         int nz, int first) {
  using C = CtaK<L>;
  constexpr int T = L / 16;
  extern __shared__ float4 sm4[];
  __shared__ uint64_t bars[2];
  float2 *sm = reinterpret_cast<float2 *>(sm4);
  Xch x = C::xch(sm);
  const Priv<NT> S{priv_base<L>(sm)};
  TabPipe<L> pipe;
  pipe.start(seq, slot_base<L, true>(sm), bars);
  const int t = C::t(), y = blockIdx.x * C::G + C::g();
#pragma unroll 1
  for (int j = 0; j < nz; j++) {
    float2 v[16];
    ld_p2_row<L>(v, Ut + (size_t)j * L * L, y, L, t);
    fft<L, false>(v, x, t, tb.tw);
    const float2 *hq = pipe.take(seq);
#pragma unroll
    for (int r = 0; r < 16; r++) {
      const float2 a = cmulc(v[r], hq[t + r * T]);
      S[r] = j == 0 ? a : cadd(S[r], a);
    }
    pipe.done(seq);
  }
#pragma unroll
  for (int r = 0; r < 16; r++) {
    const size_t gi = p2(y, t + r * T, L);
    Ghat[gi] = first ? S[r] : cadd(Ghat[gi], S[r]);
  }
}

// ------------------------------------------------------------------ filters (q_j, g_q)
// rows: out = scale/L * IFFT(h^(*) FFT(in)) along x.
// IN_P2 / OUT_P2: layout of in / out (else row-major); ACC: out += ...
template <int L, bool IN_P2, bool OUT_P2, bool ACC>
__global__ void __launch_bounds__(NT, CTAS_PER_SM)
    k_rows_filter(const float2 *__restrict__ in, float2 *__restrict__ out, Tables tb, const float2 *__restrict__ h,
                  int conj, float scale) {
  using C = CtaK<L>;
  constexpr int T = L / 16;
  extern __shared__ float4 sm4[];
  float2 *sm = reinterpret_cast<float2 *>(sm4);
  Xch x = C::xch(sm);
  const int t = C::t(), y = blockIdx.x * C::G + C::g();
  float2 v[16];
  if (IN_P2)
    ld_p2_row<L>(v, in, y, L, t);
  else
    ld_row<L>(v, in + (size_t)y * L, t);
  fft<L, false>(v, x, t, tb.tw);
  const float s = scale / L;
  if (conj)
    mul_tab<L, true>(v, h, t);
  else
    mul_tab<L, false>(v, h, t);
#pragma unroll
  for (int r = 0; r < 16; r++) v[r] = cscale(v[r], s);
  fft<L, true>(v, x, t, tb.tw);
#pragma unroll
  for (int r = 0; r < 16; r++) {
    float2 *p = out + (OUT_P2 ? p2(y, t + r * T, L) : (size_t)y * L + t + r * T);
    *p = ACC ? cadd(*p, v[r]) : v[r];
  }
}

// columns of a P2 array, in place allowed: out = scale/L * IFFT(h^(*) FFT(in)) along y
template <int L>
__global__ void __launch_bounds__(NT, CTAS_PER_SM)
    k_cols_filter(const float2 *__restrict__ in, float2 *__restrict__ out, Tables tb, const float2 *__restrict__ h,
                  int conj, float scale) {
  using C = CtaK<L>;
  extern __shared__ float4 sm4[];
  float2 *sm = reinterpret_cast<float2 *>(sm4);
  Xch x = C::xch(sm);
  const int t = C::t(), col = blockIdx.x * C::G + C::g();
  float2 v[16];
  ld_p2_col<L>(v, in, col, L, t);
  fft<L, false>(v, x, t, tb.tw);
  const float s = scale / L;
  if (conj)
    mul_tab<L, true>(v, h, t);
  else
    mul_tab<L, false>(v, h, t);
#pragma unroll
  for (int r = 0; r < 16; r++) v[r] = cscale(v[r], s);
  fft<L, true>(v, x, t, tb.tw);
  st_p2_col<L>(v, out, col, L, t);
}

// layout conversion (plane without propagation, omega_j = 0):  P2 <-> row-major, out (+)= scale * in
// ------------------------------------------------------------------ Fourier-domain object state
// holo_fourier: out = DFT2(in) (unnormalised, numpy.fft.fft2 convention) or IDFT2(in) (numpy.fft.ifft2,
// 1 / L^2), row-major L x L: a row pass into a P2 scratch, then a column pass writing row-major.
template <int L, bool INV>
__global__ void __launch_bounds__(NT, CTAS_PER_SM)
    k_dft2_rows(const float2 *__restrict__ in, float2 *__restrict__ out, const float4 *__restrict__ tw) {
  using C = CtaK<L>;
  extern __shared__ float4 sm4[];
  Xch x = C::xch(reinterpret_cast<float2 *>(sm4));
  const int t = C::t(), y = blockIdx.x * C::G + C::g();
  float2 v[16];
  ld_row<L>(v, in + (size_t)y * L, t);
  fft<L, INV>(v, x, t, tw);
  st_p2_row<L>(v, out, y, L, t);
}
template <int L, bool INV>
__global__ void __launch_bounds__(NT, CTAS_PER_SM)
    k_dft2_cols(const float2 *__restrict__ in, float2 *__restrict__ out, const float4 *__restrict__ tw, float scale) {
  using C = CtaK<L>;
  extern __shared__ float4 sm4[];
  Xch x = C::xch(reinterpret_cast<float2 *>(sm4));
  const int t = C::t(), col = blockIdx.x * C::G + C::g();
  float2 v[16];
  ld_p2_col<L>(v, in, col, L, t);
  fft<L, INV>(v, x, t, tw);
#pragma unroll
  for (int r = 0; r < 16; r++) v[r] = cscale(v[r], scale);
  st_col<L>(v, out + col, t);
}

static __global__ void k_p2_convert(const float2 *__restrict__ in, float2 *__restrict__ out, int L, int to_p2, float scale,
                             int accumulate) {
  const size_t n = (size_t)L * L;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const int y = (int)(i / L), xx = (int)(i % L);
    const size_t pi = p2(y, xx, L);
    const size_t si = to_p2 ? i : pi, di = to_p2 ? pi : i;
    const float2 v = cscale(in[si], scale);
    out[di] = accumulate ? cadd(out[di], v) : v;
  }
}

// ------------------------------------------------------------------ reductions
// deterministic single-block sum: out[v] = sum_i partial[i * nval + v], v < nval
static __global__ void k_reduce(const double *__restrict__ partial, size_t n, int nval, double *__restrict__ out,
                         int accumulate) {
  __shared__ double red[32];
  for (int v = 0; v < nval; v++) {
    double s = 0.0;
    for (size_t i = threadIdx.x; i < n; i += blockDim.x) s += partial[i * nval + v];
    double t = block_sum(s, red);
    if (threadIdx.x == 0) out[v] = accumulate ? out[v] + t : t;
    __syncthreads();
  }
}

// partial dots over n complex: part[b][0] = sum |x|^2, part[b][1] = sum Re(x conj(y))
static __global__ void k_dots(const float2 *__restrict__ x, const float2 *__restrict__ y, size_t n, double *__restrict__ part) {
  __shared__ double red[32];
  double a = 0.0, b = 0.0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    float2 v = x[i];
    a += (double)v.x * v.x + (double)v.y * v.y;
    if (y) {
      float2 w = y[i];
      b += (double)v.x * w.x + (double)v.y * w.y;
    }
  }
  double s0 = block_sum(a, red);
  double s1 = block_sum(b, red);
  if (threadIdx.x == 0) {
    part[2 * blockIdx.x] = s0;
    part[2 * blockIdx.x + 1] = s1;
  }
}

// CG pointwise step (Eq. (13)-(14)): mode 0: eta = -rho g; 1: eta = -rho g + beta eta; 2: keep eta.
// xt = x + gamma eta.  Two complex per thread-iteration (float4).
static __global__ void k_cg(const float4 *__restrict__ x, float4 *__restrict__ eta, const float4 *__restrict__ g,
                     float4 *__restrict__ xt, size_t n4, float rho, float beta, float gamma, int mode) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
    float4 e;
    if (mode == 2) {
      e = eta[i];
    } else {
      float4 gv = g[i];
      if (mode == 0) {
        e = make_float4(-rho * gv.x, -rho * gv.y, -rho * gv.z, -rho * gv.w);
      } else {
        float4 ev = eta[i];
        e = make_float4(fmaf(beta, ev.x, -rho * gv.x), fmaf(beta, ev.y, -rho * gv.y), fmaf(beta, ev.z, -rho * gv.z),
                        fmaf(beta, ev.w, -rho * gv.w));
      }
      eta[i] = e;
    }
    float4 xv = x[i];
    xt[i] = make_float4(fmaf(gamma, e.x, xv.x), fmaf(gamma, e.y, xv.y), fmaf(gamma, e.z, xv.z),
                        fmaf(gamma, e.w, xv.w));
  }
}

}  // namespace holo
