// holo_run.cuh -- pass orchestration for one torus size L (instantiated by inst_<L>.cu).
//
// Object chain (holo_fwd / holo_adj / holo_grad), per batch of B angles (B = plan->B):
//   X1 per angle (rows)  ->  for each plane j: Y1 (cols, batched), X2 (rows, batched),
//   Y2 (cols, batched)   ->  X3 per angle (rows)
// then, once per sweep, g_q = 2 sum_j P_{-omega_j} G_j (filters).  DESIGN.md "Pass schedule".
// Reference arm (holo_grad_ref / holo_fwd_ref, O14): RefRun.
#pragma once
#include "holo_impl.cuh"
#include "holo_passes.cuh"
#include "holo_multires.cuh"
#include "holo_init.cuh"
#include "holo_ref.cuh"

namespace holo_run {
using namespace holo;

template <int L>
struct Smem {
  static constexpr size_t X = CtaK<L>::XBYTES;                          // exchange space only (filters)
  static constexpr size_t XT = X + TabPipe<L>::BYTES;                    // + two table slots
  static constexpr size_t XPT = X + CtaK<L>::PRIV + TabPipe<L>::BYTES;  // + one thread-private line
  static constexpr size_t XH = X + sizeof(float2) * L;                   // + X2's resident table
  static constexpr size_t XPT3 = XPT + 128;                              // X3: private slot 128-byte aligned
  static constexpr size_t XPT3S = XPT3 + 64;                             // batched X3: + control block
  static constexpr size_t XPT1 = XPT + 128 + 16;                         // X1: row slot with skewed rows + control block
  static constexpr size_t XHS = XH + 128 + CtaK<L>::PRIV;                // X2 with its rows staged (TMA slot)
};

template <int L>
void set_chain_attrs() {
  using S = Smem<L>;
  auto a = [](const void *f, size_t s) { cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s); };
  a((const void *)k_x1<L>, S::XPT);
  a((const void *)k_x1s<L>, S::XPT1);
  a((const void *)k_dft2_rows<L, false>, S::X);
  a((const void *)k_dft2_rows<L, true>, S::X);
  a((const void *)k_dft2_cols<L, false>, S::X);
  a((const void *)k_dft2_cols<L, true>, S::X);
  a((const void *)k_y1<L, false>, S::XPT);
  a((const void *)k_y1<L, true>, S::XPT);
  a((const void *)k_xq<L>, S::XPT);
  a((const void *)k_xg<L>, S::XPT);
  a((const void *)k_x2<L, X2_GRAD, 0>, S::XHS);
  a((const void *)k_x2<L, X2_GRAD, 1>, S::XHS);
  a((const void *)k_x2<L, X2_GRAD, 2>, S::XHS);
  a((const void *)k_x2<L, X2_OBJ, 0>, S::XHS);
  a((const void *)k_x2<L, X2_OBJ, 1>, S::XHS);
  a((const void *)k_x2<L, X2_OBJ, 2>, S::XHS);
  a((const void *)k_x2<L, X2_FWD>, S::XHS);
  a((const void *)k_x2<L, X2_ADJ>, S::XH);
  a((const void *)k_y2<L, false>, S::XPT);
  a((const void *)k_y2<L, true>, S::XPT);
  a((const void *)k_x3<L>, S::XPT3);
  a((const void *)k_x3s<L>, S::XPT3S);
  a((const void *)k_rows_filter<L, false, true, false>, S::X);
  a((const void *)k_rows_filter<L, true, false, false>, S::X);
  a((const void *)k_rows_filter<L, true, false, true>, S::X);
  a((const void *)k_cols_filter<L>, S::X);
  a((const void *)k_up_rows<L>, S::X);
  a((const void *)k_up_cols<L>, S::X);
  a((const void *)k_pag_rows<L>, S::XPT);
  a((const void *)k_pag_cols<L>, S::XPT);
  a((const void *)k_pag_final<L>, S::X);
}

template <int L>
void set_ref_attrs() {
  const int sz = (int)LineEng<L>::SMEM;
  auto a = [&](const void *f) { cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, sz); };
  a((const void *)k_ref_cols<L, REF_QHAT>);
  a((const void *)k_ref_cols<L, REF_R1>);
  a((const void *)k_ref_cols<L, REF_R3>);
  a((const void *)k_ref_cols<L, REF_FINAL>);
  a((const void *)k_ref_rows<L, REF_QHAT>);
  a((const void *)k_ref_rows<L, REF_R2>);
  a((const void *)k_ref_rows<L, REF_FINAL>);
  a((const void *)k_ref_rows<L, REF_FWD>);
  a((const void *)k_ref_rows<L, REF_INIT>);
  a((const void *)k_ref_r2b<L, 0>);
  a((const void *)k_ref_r2b<L, 1>);
  a((const void *)k_ref_r2b<L, 2>);
  const int sza = (int)LineEng<L>::SMEM_ACC;
  cudaFuncSetAttribute((const void *)k_ref_r1b<L>, cudaFuncAttributeMaxDynamicSharedMemorySize, sza);
  cudaFuncSetAttribute((const void *)k_ref_r3b<L>, cudaFuncAttributeMaxDynamicSharedMemorySize, sza);
}

template <int L>
struct RefRun;

// ------------------------------------------------------------------ object chain
template <int L>
struct Run {
  using SM = Smem<L>;
  static constexpr int G = CtaK<L>::G;
  static constexpr double A = 8.0 * L * L;  // bytes of one L x L complex64 array

  // q_j = P_{omega_j} q (O6): row-major q -> P2 QJ_j
  static void qj(holo_plan *p, const float2 *q) {
    const Tables tb = p->tables();
    for (int j = 0; j < p->nz; j++) {
      float2 *dst = p->QJ + (size_t)j * L * L;
      pbeg(p);
      if (p->omega[j] == 0.0) {
        k_p2_convert<<<1184, 256, 0, p->stream>>>(q, dst, L, 1, 1.0f, 0);
        pend(p, HOLO_PASS_FILTER, 2 * A, 0);
        continue;
      }
      k_rows_filter<L, false, true, false><<<L / G, NT, SM::X, p->stream>>>(q, dst, tb, p->homega + j * L, 0, 1.0f);
      k_cols_filter<L><<<L / G, NT, SM::X, p->stream>>>(dst, dst, tb, p->homega + j * L, 0, 1.0f);
      pend(p, HOLO_PASS_FILTER, 4 * A, 4.0 * L * fftf(L), 2);
    }
  }

  // g_q (+)= scale * sum_j P_{-omega_j} G_j   (G_j P2 -> row-major out)
  static void gq(holo_plan *p, float2 *out, float scale, bool accumulate) {
    const Tables tb = p->tables();
    for (int j = 0; j < p->nz; j++) {
      float2 *Gj = p->G + (size_t)j * L * L;
      const bool acc = accumulate || j > 0;
      pbeg(p);
      if (p->omega[j] == 0.0) {
        k_p2_convert<<<1184, 256, 0, p->stream>>>(Gj, out, L, 0, scale, acc ? 1 : 0);
        pend(p, HOLO_PASS_FILTER, (acc ? 3 : 2) * A, 0);
        continue;
      }
      k_cols_filter<L><<<L / G, NT, SM::X, p->stream>>>(Gj, Gj, tb, p->homega + j * L, 1, 1.0f);
      if (acc)
        k_rows_filter<L, true, false, true><<<L / G, NT, SM::X, p->stream>>>(Gj, out, tb, p->homega + j * L, 1, scale);
      else
        k_rows_filter<L, true, false, false><<<L / G, NT, SM::X, p->stream>>>(Gj, out, tb, p->homega + j * L, 1, scale);
      pend(p, HOLO_PASS_FILTER, (acc ? 5 : 4) * A, 4.0 * L * fftf(L), 2);
    }
  }

  // Fourier 2x upsampling of count coarse [L/2][L/2] fields to [L][L] (O15, holo_multires.cuh)
  static void upsample2(holo_plan *p, const float2 *coarse, float2 *fine, int count) {
    const float4 *tw = reinterpret_cast<const float4 *>(p->tw);
    const size_t Lc2 = (size_t)(L / 2) * (L / 2);
    for (int m = 0; m < count; m++) {
      pbeg(p);
      k_up_rows<L><<<(L / 2) / G, NT, SM::X, p->stream>>>(coarse + m * Lc2, p->Up, tw, p->uptab);
      k_up_cols<L><<<L / G, NT, SM::X, p->stream>>>(p->Up, fine + m * (size_t)L * L, tw, p->uptab);
      pend(p, HOLO_PASS_FILTER, A / 4 + A / 2 + A / 2 + A, 2.0 * (L / 2 + L) * fftf(L), 2);
    }
  }

  // holo_fourier: out[m] = DFT2(in[m]) or IDFT2(in[m]) (row-major), via the T1 workspace (P2)
  static void dft2(holo_plan *p, const float2 *in, float2 *out, int count, int inverse) {
    const float4 *tw = reinterpret_cast<const float4 *>(p->tw);
    const size_t LL = (size_t)L * L;
    for (int m = 0; m < count; m++) {
      pbeg(p);
      if (inverse) {
        k_dft2_rows<L, true><<<L / G, NT, SM::X, p->stream>>>(in + m * LL, p->T1, tw);
        k_dft2_cols<L, true><<<L / G, NT, SM::X, p->stream>>>(p->T1, out + m * LL, tw, 1.0f / ((float)L * L));
      } else {
        k_dft2_rows<L, false><<<L / G, NT, SM::X, p->stream>>>(in + m * LL, p->T1, tw);
        k_dft2_cols<L, false><<<L / G, NT, SM::X, p->stream>>>(p->T1, out + m * LL, tw, 1.0f);
      }
      pend(p, HOLO_PASS_FILTER, 4 * A, 2.0 * L * fftf(L), 2);
    }
  }

  // O18: multi-distance Paganin initial object of every angle (holo_init.cuh)
  static void init_psi(holo_plan *p, const float *sqrt_d, const float *sqrt_dref, double db, float2 *psi0) {
    const Tables tb = p->tables();
    const int N = p->N, nz = p->nz;
    const size_t NN = (size_t)N * N, LL = (size_t)L * L;
    double zs = 0;
    for (int j = 0; j < nz; j++) zs += p->zeta[j];
    const double kPi = 3.14159265358979323846;
    const float cden = (float)(kPi * p->g.wavelength * db * zs / ((L * p->p0) * (L * p->p0)));
    TabSeq seq{};
    for (int j = 0; j < nz; j++) {
      const float2 *list[5] = {p->pcin + (size_t)j * L, p->pbke + (size_t)j * L, p->pcin + (size_t)j * L,
                               p->pbko + (size_t)j * L, p->pcout + (size_t)j * L};
      for (auto *e : list) seq.p[seq.n++] = e;
    }
    pbeg(p);
    k_frame_stats<<<1, 256, 0, p->stream>>>(sqrt_dref, NN, nullptr, p->partQ);
    pend(p, HOLO_PASS_REDUCE, 4.0 * NN, 0);
    for (int k = 0; k < p->K; k++) {
      PagArgs pa{};
      for (int j = 0; j < nz; j++) {
        pa.sx[j] = (float)(-p->shifts_host[((size_t)k * nz + j) * 2] / p->mt[j]);
        pa.sy[j] = (float)(-p->shifts_host[((size_t)k * nz + j) * 2 + 1] / p->mt[j]);
      }
      pbeg(p);
      k_pag_rows<L><<<L / G, NT, SM::XPT, p->stream>>>(sqrt_d + (size_t)k * nz * NN, sqrt_dref, p->partQ, p->T1, tb,
                                                        seq, pa, nz, N);
      k_pag_cols<L><<<L / G, NT, SM::XPT, p->stream>>>(p->T1, p->T3, tb, seq, pa, nz, cden, 1.0f / ((float)L * L));
      k_pag_final<L><<<L / G, NT, SM::X, p->stream>>>(p->T3, psi0 + (size_t)k * LL, tb, (float)db);
      pend(p, HOLO_PASS_FILTER, A * (3.0 * nz + 2.0) + 4.0 * NN * (nz + 1), L * fftf(L) * (12.0 * nz + 2.0), 3);
    }
  }

  // the probe-gradient tail of a sweep: reference frames of the fused objective (O14 into the same
  // Ghat / F), then g_q = 2 sum_j P_{-omega_j} G_j (or the final IDFT2 of Ghat); records gq_event
  static void finish_q(holo_plan *p, const float2 *q, float2 *gq_out, float gscale, bool want_q, bool acc_q, int mode,
                       const float *sqrt_dref) {
    const bool ps = p->ps, gq_pass = want_q && (mode == 0 || mode == 2);
    const bool ref = sqrt_dref && p->n_ref > 0 && mode == 0;
    if (ref) {
      if (!ps) RefRun<L>::qhat(p, q);
      RefRun<L>::frames(p, sqrt_dref, want_q, /*first=*/!ps);
    }
    if (gq_pass) {
      if (ps) {
        RefRun<L>::final(p, gq_out, gscale, acc_q);
      } else {
        gq(p, gq_out, gscale, acc_q);
        if (ref) RefRun<L>::final(p, gq_out, gscale, true);
      }
      if (p->gq_event) cudaEventRecord(p->gq_event, p->stream);
    }
  }

  // mode: 0 grad, 1 fwd, 2 adj (y given), 3 objective only.
  // With per-frame probe shifts (p->ps, O19) the probe enters through Qhat = DFT2 q (XQ -> Qt ->
  // q_kj in Y1) and the probe gradient is accumulated in the Fourier domain (Y2 -> Ut -> XG ->
  // Ghat); `sqrt_dref` != NULL adds the reference frames (O14) to F and to the same Ghat /
  // g_q in this call (the fused Eq. (10)/(12)); F partials of those frames go to partR.
  static void sweep(holo_plan *p, int mode, const float2 *psi, const float2 *q, const float *sqrt_d,
                    const float2 *yin, float2 *wout, const float2 *eta, float2 *gpsi, float2 *gq_out, float gscale,
                    bool want_q, bool acc_q, const float *sqrt_dref) {
    Tables tb = p->tables();
    const bool ps = p->ps;
    const int N = p->N, nz = p->nz, K = p->K;
    const size_t LL = (size_t)L * L, NL = (size_t)N * L, NN = (size_t)N * N;
    const int nbx2 = p->nbx2;
    const double fl = fftf(L), rN = (double)N / L, NN8 = 8.0 * N * N;
    const bool gq_pass = want_q && (mode == 0 || mode == 2);
    const int fo_ = p->fourier ? 1 : 0;  // holo_set_fourier: psi / eta / grad_psi are DFT2 of the object arrays
    const int tm_ = p->tau == 1.f ? 0 : (p->tau == 2.f ? 1 : 2);  // residual branch compiled into X2
    int nmag = 0;
    for (int j = 0; j < nz; j++) nmag += (p->magmask >> j) & 1;
    if (ps) {
      RefRun<L>::qhat(p, q);
    } else {
      qj(p, q);
      if (want_q) cudaMemsetAsync(p->G, 0, sizeof(float2) * LL * nz, p->stream);
    }
    // table sequences of the pipelined pointwise steps (holo_kernels.cuh, TabPipe)
    auto crp = [&](int k, int j, int ax) { return p->cr + ((size_t)(k * nz + j) * 2 + ax) * L; };
    auto hqp = [&](int k, int j, int ax) { return p->hq + ((size_t)(k * nz + j) * 2 + ax) * L; };
    auto add_fwd = [&](TabSeq &q, int k, int j, int ax) {  // mag_fwd: cr, bke, cr, bko, cout
      const float2 *c = crp(k, j, ax);
      const float2 *list[5] = {c, p->bke + (size_t)j * L, c, p->bko + (size_t)j * L, p->cout + (size_t)j * L};
      for (auto *e : list) q.p[q.n++] = e;
    };
    auto add_adj = [&](TabSeq &q, int k, int j, int ax) {  // mag_adj: cout, bke, cout, bko, cr
      const float2 *c = p->cout + (size_t)j * L;
      const float2 *list[5] = {c, p->bke + (size_t)j * L, c, p->bko + (size_t)j * L, crp(k, j, ax)};
      for (auto *e : list) q.p[q.n++] = e;
    };
    const bool need_fwd_chain = (mode != 2) || want_q || ps;
    // a deferred psi-block CG step (holo_set_cg_fuse) whose trial point is this sweep's psi runs inside X1
    CgFuse cgf{nullptr, nullptr, nullptr, 0.f, 0.f, 0.f, -1};
    const float2 *psi_src = psi;
    if (p->cg_pending) {
      if (need_fwd_chain && psi == p->cg_trial && K > 0) {
        cgf = CgFuse{p->cg_g, p->cg_eta, p->cg_trial, p->cg_rho, p->cg_beta, p->cg_gamma, p->cg_mode};
        psi_src = p->cg_psi;
        p->cg_pending = false;
      } else {
        holo_cg_flush(p);
      }
    }
    // holo_stage_sqrt_d: stream the data in per angle batch on the copy stream (after everything
    // queued so far on the plan's stream, i.e. the previous readers of the device buffer), so batch
    // b + 1's copy overlaps batch b's passes; batch b's first X2 waits for its own event
    const bool staged = !p->stage_ref && p->stage_dev && sqrt_d == p->stage_dev && (mode == 0 || mode == 3);
    if (staged) {
      cudaEventRecord(p->stage_start, p->stream);
      cudaStreamWaitEvent(p->copy_stream, p->stage_start, 0);
      for (int k0 = 0, bi = 0; k0 < K; k0 += p->B, bi++) {
        const int nb = K - k0 < p->B ? K - k0 : p->B;
        const size_t off = (size_t)k0 * nz * NN, cnt = (size_t)nb * nz * NN;
        cudaMemcpyAsync(p->stage_dev + off, p->stage_host + off, cnt * sizeof(float), cudaMemcpyHostToDevice,
                        p->copy_stream);
        cudaEventRecord(p->stage_ev[bi], p->copy_stream);
      }
      p->stage_host = nullptr;
      p->stage_dev = nullptr;
    }
    for (int k0 = 0; k0 < K; k0 += p->B) {
      const int nb = K - k0 < p->B ? K - k0 : p->B;  // ragged last batch
      // ---- X1 (per angle): T1[b][j] = (M S)_x psi_k rows;  PS: XQ, Qt[b][j] = IFFT_x(Hq_x Qhat)
      if (need_fwd_chain) {
        // one launch for the batch (each CTA loops over the angles, the next angle's rows staged behind the
        // last plane) when the chained table sequence fits and the CG update is not fused; else per angle
        const int tabs_per_angle = 5 * nmag + (nz - nmag);
        const bool x1b = X1Stage<L>::OK && cgf.mode < 0 && nb * tabs_per_angle <= MAXTAB;
        if (x1b) {
          TabSeq q{};
          for (int b = 0; b < nb; b++)
            for (int j = 0; j < nz; j++) {
              if ((p->magmask >> j) & 1u)
                add_fwd(q, k0 + b, j, 0);
              else
                q.p[q.n++] = crp(k0 + b, j, 0);
            }
          pbeg(p);
          k_x1s<L><<<L / G, NT, SM::XPT1, p->stream>>>(psi_src + (size_t)k0 * LL, p->T1, tb, q, nz, p->magmask, fo_, nb);
          pend(p, HOLO_PASS_X1, nb * (1 + nz) * A, nb * L * fl * ((fo_ ? 0 : 1) + 4 * nmag + (nz - nmag)));
        }
        for (int b = 0; b < (x1b ? 0 : nb); b++) {
          const int k = k0 + b;
          TabSeq q{};
          for (int j = 0; j < nz; j++) {
            if ((p->magmask >> j) & 1u)
              add_fwd(q, k, j, 0);
            else
              q.p[q.n++] = crp(k, j, 0);
          }
          pbeg(p);
          CgFuse cgk = cgf;
          if (cgk.mode >= 0) {
            if (cgk.g) cgk.g += (size_t)k * LL;
            cgk.eta += (size_t)k * LL;
            cgk.trial += (size_t)k * LL;
          }
          k_x1<L><<<L / G, NT, SM::XPT, p->stream>>>(psi_src + (size_t)k * LL, p->T1 + (size_t)b * nz * LL, tb, q,
                                                      nz, p->magmask, fo_, cgk);
          pend(p, HOLO_PASS_X1, (1 + nz + (cgk.mode < 0 ? 0 : cgk.mode == 2 ? 2 : cgk.mode == 0 ? 3 : 4)) * A,
               L * fl * ((fo_ ? 0 : 1) + 4 * nmag + (nz - nmag)));
        }
        if (ps) {  // XQ for the whole batch: the Qhat row read once, nb x nz row transforms per CTA
          TabSeq qq{};
          for (int b = 0; b < nb; b++)
            for (int j = 0; j < nz; j++) qq.p[qq.n++] = hqp(k0 + b, j, 0);
          pbeg(p);
          k_xq<L><<<L / G, NT, SM::XPT, p->stream>>>(p->Qhat, p->Qt, tb, qq, nz * nb);
          pend(p, HOLO_PASS_PS, (1 + nz * nb) * A, L * fl * nz * nb);
        }
      }
      for (int j = 0; j < nz; j++) {
        const int mag = (p->magmask >> j) & 1;
        const float2 *qjj = ps ? nullptr : p->QJ + (size_t)j * LL;
        // ---- Y1 (batched): Aw[b] = (M S)_y T1[b][j];  W1[b] = crop_y D_y (q_(k)j Aw[b])
        if (need_fwd_chain) {
          float2 *aout = want_q ? p->Aw : nullptr;
          float2 *w1 = (mode == 2) ? nullptr : p->W1;
          TabSeq q{};
          for (int b = 0; b < nb; b++) {
            if (mag)
              add_fwd(q, k0 + b, j, 1);
            else
              q.p[q.n++] = crp(k0 + b, j, 1);
            if (ps) q.p[q.n++] = hqp(k0 + b, j, 1);
            if (w1) q.p[q.n++] = p->hdet + (size_t)j * L;
          }
          pbeg(p);
          if (ps)
            k_y1<L, true><<<L / G, NT, SM::XPT, p->stream>>>(p->T1 + (size_t)j * LL, (size_t)nz * LL, nullptr,
                                                              p->Qt + (size_t)j * LL, p->Qk, aout, w1, tb, q, mag, N,
                                                              nb, fo_);
          else
            k_y1<L, false><<<L / G, NT, SM::XPT, p->stream>>>(p->T1 + (size_t)j * LL, (size_t)nz * LL, qjj, nullptr,
                                                               nullptr, aout, w1, tb, q, mag, N, nb, fo_);
          // bytes: T1 read, Aw write, W1 write per frame; q_j once per batch (L2-resident); PS: Qt read, Qk write
          pend(p, HOLO_PASS_Y1,
               nb * (A + (w1 ? rN * A : 0) + (aout ? A : 0) + (ps ? 2 * A : 0)) + ((w1 && !ps) ? A : 0),
               nb * L * fl * ((fo_ ? 0 : 1) + (mag ? 4 : 1) + (w1 ? 2 : 0) + (ps ? 1 : 0)));
        }
        // ---- X2 (batched over blockIdx.y); a staged batch's data must have arrived (X1 / Y1 overlapped it)
        if (staged && j == 0) cudaStreamWaitEvent(p->stream, p->stage_ev[k0 / p->B], 0);
        double *pf = p->partF + ((size_t)k0 * nz + j) * nbx2;
        TabSeq qh{};
        qh.p[qh.n++] = p->hdet + (size_t)j * L;
        if (mode == 0 || mode == 2) qh.p[qh.n++] = p->hdet + (size_t)j * L;
        const dim3 g2(nbx2, HOLO_X2_LOOP ? 1 : nb);
        const size_t fo = (size_t)k0 * nz + j;  // first frame of the batch in [k][j] order
        pbeg(p);
        const int x2s = (HOLO_X2_LOOP && p->w1map_ok) ? 1 : 0;  // rows staged by tensor copies
        const size_t smx2 = x2s ? SM::XHS : SM::XH;
        if (mode == 1) {
          k_x2<L, X2_FWD><<<g2, NT, smx2, p->stream>>>(p->W1, NL, nullptr, 0, wout + fo * NN, nz * NN, pf,
                                                       nz * nbx2, tb, qh, N, p->tau, nb, p->w1map, x2s);
          pend(p, HOLO_PASS_X2, nb * (rN * A + NN8), nb * N * fl * 2);
          continue;
        }
        if (mode == 3) {
          (tm_ == 0 ? k_x2<L, X2_OBJ, 0> : tm_ == 1 ? k_x2<L, X2_OBJ, 1> : k_x2<L, X2_OBJ, 2>)<<<g2, NT, smx2, p->stream>>>(
              p->W1, NL, sqrt_d + fo * NN, nz * NN, nullptr, 0, pf, nz * nbx2, tb, qh, N, p->tau, nb, p->w1map, x2s);
          pend(p, HOLO_PASS_X2, nb * (rN * A + NN8 / 2), nb * N * fl * 2);
          continue;
        }
        if (mode == 0) {
          (tm_ == 0 ? k_x2<L, X2_GRAD, 0> : tm_ == 1 ? k_x2<L, X2_GRAD, 1> : k_x2<L, X2_GRAD, 2>)<<<g2, NT, smx2, p->stream>>>(
              p->W1, NL, sqrt_d + fo * NN, nz * NN, p->V1, NL, pf, nz * nbx2, tb, qh, N, p->tau, nb, p->w1map, x2s);
          pend(p, HOLO_PASS_X2, nb * (2 * rN * A + NN8 / 2), nb * N * fl * 4);
        } else {
          k_x2<L, X2_ADJ><<<g2, NT, SM::XH, p->stream>>>(yin + fo * NN, nz * NN, nullptr, 0, p->V1, NL, pf,
                                                         nz * nbx2, tb, qh, N, p->tau, nb, p->w1map, 0);
          pend(p, HOLO_PASS_X2, nb * (rN * A + NN8), nb * N * fl * 2);
        }
        // ---- Y2 (batched): v = D_y^* V1[b]; G_j += conj(Aw[b]) v  (PS: Ut[b][j] = Hq_y^* FFT_y(conj(Aw) v));
        //      T3[b][j] = (M S)_y^* (conj(q_(k)j) v)
        float2 *Gj = (want_q && !ps) ? p->G + (size_t)j * LL : nullptr;
        float2 *Utj = (want_q && ps) ? p->Ut + (size_t)j * LL : nullptr;
        float2 *T3j = gpsi ? p->T3 + (size_t)j * LL : nullptr;
        TabSeq q2{};
        for (int b = 0; b < nb; b++) {
          q2.p[q2.n++] = p->hdet + (size_t)j * L;
          if (Utj) q2.p[q2.n++] = hqp(k0 + b, j, 1);
          if (T3j) {
            if (mag)
              add_adj(q2, k0 + b, j, 1);
            else
              q2.p[q2.n++] = crp(k0 + b, j, 1);
          }
        }
        pbeg(p);
        if (ps)
          k_y2<L, true><<<L / G, NT, SM::XPT, p->stream>>>(p->V1, p->Aw, nullptr, p->Qk, nullptr, Utj, T3j,
                                                            (size_t)nz * LL, tb, q2, mag, N, nb, fo_);
        else
          k_y2<L, false><<<L / G, NT, SM::XPT, p->stream>>>(p->V1, p->Aw, qjj, nullptr, Gj, nullptr, T3j,
                                                             (size_t)nz * LL, tb, q2, mag, N, nb, fo_);
        // bytes: V1 read, Aw read (q gradient), T3 write per frame; G_j read + write and q_j once per batch
        // (PS: Qk read per frame, Ut write per frame)
        pend(p, HOLO_PASS_Y2,
             nb * (rN * A + (want_q ? A : 0) + (T3j ? A : 0) + (ps ? ((T3j ? A : 0) + (want_q ? A : 0)) : 0)) +
                 (Gj ? 2 * A : 0) + ((T3j && !ps) ? A : 0),
             nb * L * fl * (2 + (T3j ? (mag ? 5 : 2) - (fo_ ? 1 : 0) : 0) + (Utj ? 1 : 0)));
      }
      // ---- X3 (per angle): g_k = 2 IFFT_x( sum_j W_j ),  W_j = spectrum of (M S)_x^* T3[b][j];
      //      PS: XG, Ghat (+)= sum_j conj(Hq_x) FFT_x(Ut[b][j]).
      // In the LAST batch the probe gradient is completed first (XG, reference frames, g_q filters
      // or the final IDFT2) and p->gq_event recorded, so a caller can allreduce g_q on another
      // stream while this batch's X3 passes run (SURVEY 8e overlap).
      const bool last_batch = k0 + nb >= K;
      auto xg = [&]() {  // the whole batch: nb x nz row transforms summed per CTA, one Ghat update per batch
        TabSeq qg{};
        for (int b = 0; b < nb; b++)
          for (int j = 0; j < nz; j++) qg.p[qg.n++] = hqp(k0 + b, j, 0);
        pbeg(p);
        k_xg<L><<<L / G, NT, SM::XPT, p->stream>>>(p->Ut, p->Ghat, tb, qg, nz * nb, k0 == 0);
        pend(p, HOLO_PASS_PS, (nz * nb + (k0 ? 2 : 1)) * A, L * fl * nz * nb);
      };
      auto x3 = [&](int b) {
        const int k = k0 + b;
        TabSeq q3{};
        for (int j = 0; j < nz; j++) {
          if ((p->magmask >> j) & 1u)
            add_adj(q3, k, j, 0);
          else
            q3.p[q3.n++] = crp(k, j, 0);
        }
        pbeg(p);
        k_x3<L><<<L / G, NT, SM::XPT3, p->stream>>>(p->T3 + (size_t)b * nz * LL, eta ? eta + (size_t)k * LL : nullptr,
                                                    gpsi + (size_t)k * LL, p->partX3 + (size_t)k * 2 * p->nbx3, tb, q3,
                                                    nz, p->magmask, fo_ ? gscale * (float)L * (float)L : gscale, fo_,
                                                    p->t3map, b * nz, p->t3map_ok ? 1 : 0);
        pend(p, HOLO_PASS_X3, (nz + 1 + (eta ? 1 : 0)) * A, L * fl * (4 * nmag + (nz - nmag) + (fo_ ? 0 : 1)));
      };
      // one launch for the batch (k_x3s) when the T3 tensor map exists and the chained tables fit
      auto x3all = [&]() {
        if (HOLO_STAGE && HOLO_X3_BATCH && G >= 2 && p->t3map_ok && nb * (5 * nmag + (nz - nmag)) <= MAXTAB) {
          TabSeq q3{};
          for (int b = 0; b < nb; b++)
            for (int j = 0; j < nz; j++) {
              if ((p->magmask >> j) & 1u)
                add_adj(q3, k0 + b, j, 0);
              else
                q3.p[q3.n++] = crp(k0 + b, j, 0);
            }
          pbeg(p);
          k_x3s<L><<<L / G, NT, SM::XPT3S, p->stream>>>(p->T3, eta ? eta + (size_t)k0 * LL : nullptr, gpsi + (size_t)k0 * LL,
                                                        p->partX3 + (size_t)k0 * 2 * p->nbx3, tb, q3, nz, p->magmask,
                                                        fo_ ? gscale * (float)L * (float)L : gscale, fo_, p->t3map, 0, nb);
          pend(p, HOLO_PASS_X3, nb * (nz + 1 + (eta ? 1 : 0)) * A, nb * L * fl * (4 * nmag + (nz - nmag) + (fo_ ? 0 : 1)));
        } else {
          for (int b = 0; b < nb; b++) x3(b);
        }
      };
      const bool want_x3 = gpsi && (mode == 0 || mode == 2);
      if (!last_batch) {
        if (want_x3) x3all();
        if (ps && gq_pass) xg();
      } else {
        if (ps && gq_pass) xg();
        finish_q(p, q, gq_out, gscale, want_q, acc_q, mode, sqrt_dref);
        if (want_x3) x3all();
      }
    }
    if (K == 0) finish_q(p, q, gq_out, gscale, want_q, acc_q, mode, sqrt_dref);
  }
};

// ------------------------------------------------------------------ reference arm runner (O14)
template <int L>
struct RefRun {
  using E = LineEng<L>;
  // w[r] = C(P_{zeta0} S_{s_r} q), row-major [R][N][N]
  static void fwd(holo_plan *p, const float2 *q, float2 *w) {
    const int N = p->N, R = p->n_ref;
    const size_t SM = E::SMEM;
    const float4 *tw = reinterpret_cast<const float4 *>(p->tw);
    const int gl = L / E::G, gn = (N + E::G - 1) / E::G;
    const double A = 8.0 * L * L, fl = fftf(L);
    pbeg(p);
    k_ref_rows<L, REF_QHAT><<<gl, E::NT, SM, p->stream>>>(q, nullptr, p->Qhat, nullptr, nullptr, tw, p->tw3, N, 1.f, 0);
    k_ref_cols<L, REF_QHAT><<<gl, E::NT, SM, p->stream>>>(p->Qhat, p->Qhat, nullptr, tw, p->tw3, N, 0);
    pend(p, HOLO_PASS_REF, 4 * A, 2.0 * L * fl, 2);
    for (int r0 = 0; r0 < R; r0 += p->BR) {
      const int nb = R - r0 < p->BR ? R - r0 : p->BR;
      const float2 *H = p->Href + (size_t)r0 * 2 * L;
      const float2 *F = p->Hfac + (size_t)r0 * 2 * E::FS;
      pbeg(p);
      k_ref_r1b<L><<<gl, E::NT, (HOLO_R1B_REREAD && E::HOLD_SMEM) ? E::SMEM : E::SMEM_ACC, p->stream>>>(p->Qhat, p->Wr, p->hz, F, nb, tw, p->tw3, N);
      k_ref_rows<L, REF_FWD><<<dim3(gn, nb), E::NT, SM, p->stream>>>(p->Wr, nullptr, w + (size_t)r0 * N * N, nullptr, H,
                                                                       tw, p->tw3, N, 1.f, 0);
      pend(p, HOLO_PASS_REF, A + nb * (A + 8.0 * N * N), nb * fl * (L + N), 2);
    }
  }

  // O17: q0 = mean_r(c_r) + (1/R) sum_r S_{-s_r} P_{-zeta0} Z (a_r - c_r),  c_r = mean(a_r)
  //      (= (1/R) sum_r S_{-s_r} P_{-zeta0} Z_{c_r} a_r: a constant is invariant under S and P)
  static void init_probe(holo_plan *p, const float *sqrt_dref, float2 *q0) {
    const int N = p->N, R = p->n_ref;
    const size_t SM = E::SMEM, NN = (size_t)N * N;
    const float4 *tw = reinterpret_cast<const float4 *>(p->tw);
    const int gl = L / E::G, gn = (N + E::G - 1) / E::G;
    const double A = 8.0 * L * L, fl = fftf(L);
    pbeg(p);
    k_frame_stats<<<R, 256, 0, p->stream>>>(sqrt_dref, NN, p->partR, nullptr);
    pend(p, HOLO_PASS_REDUCE, 4.0 * NN * R, 0);
    for (int r0 = 0; r0 < R; r0 += p->BR) {
      const int nb = R - r0 < p->BR ? R - r0 : p->BR;
      const float2 *H = p->Href + (size_t)r0 * 2 * L;
      const float2 *F = p->Hfac + (size_t)r0 * 2 * E::FS;
      pbeg(p);
      k_ref_rows<L, REF_INIT><<<dim3(gn, nb), E::NT, SM, p->stream>>>(nullptr, sqrt_dref + r0 * NN, p->Vr,
                                                                        p->partR + r0, H, tw, p->tw3, N, 1.f, 0);
      k_ref_r3b<L><<<gl, E::NT, (HOLO_R3B_RED && E::HOLD_SMEM) ? E::SMEM : E::SMEM_ACC, p->stream>>>(p->Vr, p->Ghat, p->hz, F, nb, tw, p->tw3, N, r0 == 0);
      pend(p, HOLO_PASS_REF, nb * A * (0.0625 + 0.5 + 0.5) + A * (r0 ? 2.0 : 1.0), nb * fl * (N + L), 2);
    }
    pbeg(p);
    k_fill_mean<<<1184, 256, 0, p->stream>>>(q0, (size_t)L * L, p->partR, R);
    k_ref_cols<L, REF_FINAL><<<gl, E::NT, SM, p->stream>>>(p->Ghat, p->Ghat, nullptr, tw, p->tw3, N, 0);
    k_ref_rows<L, REF_FINAL><<<gl, E::NT, SM, p->stream>>>(p->Ghat, nullptr, q0, nullptr, nullptr, tw, p->tw3, N,
                                                             1.0f / R, 1);
    pend(p, HOLO_PASS_REF, 6 * A, 2.0 * L * fl, 3);
  }

  // Qhat = DFT2(q)  (P2 [fy][fx])
  static void qhat(holo_plan *p, const float2 *q) {
    const int N = p->N;
    const size_t SM = E::SMEM;
    const float4 *tw = reinterpret_cast<const float4 *>(p->tw);
    const int gl = L / E::G;
    pbeg(p);
    k_ref_rows<L, REF_QHAT><<<gl, E::NT, SM, p->stream>>>(q, nullptr, p->Qhat, nullptr, nullptr, tw, p->tw3, N, 1.f, 0);
    k_ref_cols<L, REF_QHAT><<<gl, E::NT, SM, p->stream>>>(p->Qhat, p->Qhat, nullptr, tw, p->tw3, N, 0);
    pend(p, HOLO_PASS_REF, 4 * 8.0 * L * L, 2.0 * L * fftf(L), 2);
  }

  // the R reference frames: F partials -> partR; with want_q, Ghat (+)= conj(H) DFT2(Z rho^r)
  static void frames(holo_plan *p, const float *sqrt_dref, bool want_q, bool first) {
    const int N = p->N, R = p->n_ref;
    const size_t SM = E::SMEM;
    const float4 *tw = reinterpret_cast<const float4 *>(p->tw);
    const float2 *tw3 = p->tw3;
    const int gl = L / E::G, gn = (N + E::G - 1) / E::G;
    const double A = 8.0 * L * L, fl = fftf(L);
    // holo_stage_sqrt_d on the reference frames: streamed per frame batch on the copy stream, each
    // batch's R2 waiting for its own slice (R1B of the batch overlaps it)
    const size_t NNr = (size_t)N * N;
    const bool staged = p->stage_ref && p->stage_dev && sqrt_dref == p->stage_dev;
    if (staged) {
      cudaEventRecord(p->stage_start, p->stream);
      cudaStreamWaitEvent(p->copy_stream, p->stage_start, 0);
      for (int r0 = 0, bi = 0; r0 < R; r0 += p->BR, bi++) {
        const int nb = R - r0 < p->BR ? R - r0 : p->BR;
        cudaMemcpyAsync(p->stage_dev + r0 * NNr, p->stage_host + r0 * NNr, nb * NNr * sizeof(float),
                        cudaMemcpyHostToDevice, p->copy_stream);
        cudaEventRecord(p->stage_ev[bi], p->copy_stream);
      }
      p->stage_host = nullptr;
      p->stage_dev = nullptr;
    }
    // B_r frames per launch: the Qhat column read once (R1B), Ghat read-modify-written once (R3B)
    for (int r0 = 0; r0 < R; r0 += p->BR) {
      const int nb = R - r0 < p->BR ? R - r0 : p->BR;
      const float2 *H = p->Href + (size_t)r0 * 2 * L;
      const float2 *F = p->Hfac + (size_t)r0 * 2 * E::FS;
      const bool f0 = first && r0 == 0;
      pbeg(p);
      k_ref_r1b<L><<<gl, E::NT, (HOLO_R1B_REREAD && E::HOLD_SMEM) ? E::SMEM : E::SMEM_ACC, p->stream>>>(p->Qhat, p->Wr, p->hz, F, nb, tw, tw3, N);
      if (staged) cudaStreamWaitEvent(p->stream, p->stage_ev[r0 / p->BR], 0);
      if constexpr (E::HOLD_SMEM) {  // LineEng<6144>: one row of every frame of the batch per CTA (gn == N)
        const int tm = p->tau == 1.f ? 0 : (p->tau == 2.f ? 1 : 2);
        (tm == 0 ? k_ref_r2b<L, 0> : tm == 1 ? k_ref_r2b<L, 1> : k_ref_r2b<L, 2>)<<<gn, E::NT, SM, p->stream>>>(
            p->Wr, sqrt_dref + (size_t)r0 * N * N, p->Vr, p->partR + (size_t)r0 * gn, H, tw, tw3, N, nb, p->tau);
      } else {
        k_ref_rows<L, REF_R2><<<dim3(gn, nb), E::NT, SM, p->stream>>>(p->Wr, sqrt_dref + (size_t)r0 * N * N, p->Vr,
                                                                        p->partR + (size_t)r0 * gn, H, tw, tw3, N, 1.f,
                                                                        0, p->tau);
      }
      if (want_q) k_ref_r3b<L><<<gl, E::NT, (HOLO_R3B_RED && E::HOLD_SMEM) ? E::SMEM : E::SMEM_ACC, p->stream>>>(p->Vr, p->Ghat, p->hz, F, nb, tw, tw3, N, f0);
      // bytes: Qhat once, W write + read, sqrt_d, V write + read per frame, Ghat once per batch
      pend(p, HOLO_PASS_REF,
           A + nb * A * (0.5 + 0.5 + 1.0 / 8 + 0.5 + (want_q ? 0.5 : 0.0)) + (want_q ? A * (f0 ? 1.0 : 2.0) : 0.0),
           nb * fl * (L + 2.0 * N + (want_q ? L : 0)), want_q ? 3 : 2);
    }
  }

  // gq (+)= scale * IDFT2(Ghat)
  static void final(holo_plan *p, float2 *gq, float scale, bool acc) {
    const int N = p->N;
    const size_t SM = E::SMEM;
    const float4 *tw = reinterpret_cast<const float4 *>(p->tw);
    const int gl = L / E::G;
    const double A = 8.0 * L * L;
    pbeg(p);
    k_ref_cols<L, REF_FINAL><<<gl, E::NT, SM, p->stream>>>(p->Ghat, p->Ghat, nullptr, tw, p->tw3, N, 0);
    k_ref_rows<L, REF_FINAL><<<gl, E::NT, SM, p->stream>>>(p->Ghat, nullptr, gq, nullptr, nullptr, tw, p->tw3, N,
                                                             scale, acc ? 1 : 0);
    pend(p, HOLO_PASS_REF, (acc ? 5 : 4) * A, 2.0 * L * fftf(L), 2);
  }

  // sc[0] (+)= sum of the reference frames' F partials
  static void reduce(holo_plan *p, double *sc, bool acc) {
    const int gn = (p->N + E::G - 1) / E::G;
    pbeg(p);
    k_reduce<<<1, 1024, 0, p->stream>>>(p->partR, (size_t)p->n_ref * gn, 1, sc, acc ? 1 : 0);
    pend(p, HOLO_PASS_REDUCE, 8.0 * p->n_ref * gn, 0);
  }

  static void run(holo_plan *p, const float2 *q, const float *sqrt_dref, float2 *gq, double *sc, bool acc) {
    qhat(p, q);
    frames(p, sqrt_dref, gq != nullptr, true);
    if (gq) final(p, gq, 2.0f, acc);
    reduce(p, sc, false);
  }
};

}  // namespace holo_run

// One HoloOps per L (object chain + reference arm), and the reference-arm-only size (6144).
#define HOLO_DEFINE_OPS(LV)                                                                                      \
  static void holo_set_attrs_##LV() {                                                                           \
    holo_run::set_ref_attrs<LV>();                                                                              \
    holo_run::set_chain_attrs<LV>();                                                                            \
  }                                                                                                             \
  extern const HoloOps holo_ops_##LV = {LV,                                                                    \
                                        holo_set_attrs_##LV,                                                   \
                                        holo_run::Run<LV>::sweep,                                              \
                                        holo_run::RefRun<LV>::run,                                             \
                                        holo_run::RefRun<LV>::fwd,                                             \
                                        holo_run::Run<LV>::upsample2,                                          \
                                        holo_run::Run<LV>::init_psi,                                           \
                                        holo_run::RefRun<LV>::init_probe,                                      \
                                        holo::LineEng<LV>::G, holo::LineEng<LV>::R, holo::LineEng<LV>::T,      \
                                        holo_run::Run<LV>::dft2};
#define HOLO_DEFINE_REF_OPS(LV)                                                                                  \
  static void holo_set_attrs_##LV() { holo_run::set_ref_attrs<LV>(); }                                          \
  extern const HoloOps holo_ops_##LV = {LV,      holo_set_attrs_##LV,       nullptr, holo_run::RefRun<LV>::run, \
                                        holo_run::RefRun<LV>::fwd, nullptr, nullptr,                           \
                                        holo_run::RefRun<LV>::init_probe, holo::LineEng<LV>::G,                \
                                        holo::LineEng<LV>::R, holo::LineEng<LV>::T, nullptr};
