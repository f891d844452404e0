// holo_impl.cuh -- internals shared by the ABI translation unit (holo_plan.cu) and the
// per-torus-size instantiation units (inst_<L>.cu): the plan object, per-pass event
// profiling, and the table of per-L entry points (HoloOps).  The pass runners
// themselves (holo_run.cuh) are instantiated once per L in their own TU so that the
// seven sizes compile in parallel.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <complex>
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/holo.h"
#include "holo_kernels.cuh"

struct HoloOps;

struct holo_plan {
  int device = 0;
  cudaStream_t stream = nullptr;
  holo_geometry g{};
  int L = 0, N = 0, nz = 0, K = 0, B = 1;  // B: angle batch (frames of one plane per Y1/X2/Y2 launch)
  double m0 = 0, p0 = 0, mt[HOLO_MAX_NZ]{}, zeta[HOLO_MAX_NZ]{}, zdet[HOLO_MAX_NZ]{}, omega[HOLO_MAX_NZ]{};
  uint32_t magmask = 0;
  const HoloOps *ops = nullptr;
  // device tables
  float2 *tw = nullptr, *hdet = nullptr, *homega = nullptr, *cout = nullptr, *bke = nullptr, *bko = nullptr,
         *cr = nullptr;
  std::vector<std::complex<double>> cin_host;  // [nz][L] kappa (-1)^fbar e^{i pi mt fbar^2/L} / L
  // workspace (P2 layout, holo_kernels.cuh):
  //   T1 [B][nz][L][L], Aw [B][L][L], W1 / V1 [B][N][L], T3 [B][nz][L][L], G [nz][L][L], QJ [nz][L][L]
  float2 *T1 = nullptr, *Aw = nullptr, *W1 = nullptr, *V1 = nullptr, *T3 = nullptr, *G = nullptr, *QJ = nullptr;
  // TMA descriptor of T3 for X3's row staging (HOLO_STAGE): {4 floats, L rows, L/2 column pairs, B nz planes}
  CUtensorMap t3map{}, w1map{};
  bool t3map_ok = false, w1map_ok = false;
  double *partF = nullptr, *partX3 = nullptr, *partQ = nullptr;
  int nbx2 = 0, nbx3 = 0;  // CTAs of one frame's X2 launch / one angle's X3 launch (partials per CTA)
  float tau = 1.f;         // penalty exponent of the current call (G_tau, App. A.3): 1 = F_1, 2 = F_2
  double tau_set = 1.0;    // holo_set_tau (HOLO_INTENSITY overrides it with 2 for one call)
  size_t ws_bytes = 0;
  std::vector<void *> allocs;
  std::vector<size_t> alloc_bytes;
  std::string err;
  bool sticky = false;
  uint64_t launches = 0;
  int n_ref = 0;
  std::vector<double> ref_shifts;
  // reference arm (holo_ref.cuh): Qhat, Ghat (P2, L x L), Wr, Vr (P2, N x L), Href [R][2][L], F partials
  float2 *Qhat = nullptr, *Ghat = nullptr, *Wr = nullptr, *Vr = nullptr, *Href = nullptr, *tw3 = nullptr;
  // factored frame tables of the sweep passes (holo_ref.cuh R1B / R2 / R3B): hz [L] = h_{zeta0} / L and
  // Hfac [R][2][FS] = per frame and axis the shift ramp as A[ref_R] (per engine value) x B[ref_T] (per thread)
  float2 *hz = nullptr, *Hfac = nullptr;
  double *partR = nullptr;
  int ref_cap = 0;  // frames Href / partR are sized for
  int BR = 1;       // reference frames per batched launch (Wr / Vr hold BR frames)
  // multiresolution schedule (holo_multires.cuh): up-sampling table [L] and row-pass scratch P2 [L/2][L]
  float2 *uptab = nullptr, *Up = nullptr;
  // initial object (O18, holo_init.cuh): inverse-magnification Bluestein tables [nz][L] (mt' = 1/mt_j)
  float2 *pcin = nullptr, *pcout = nullptr, *pbke = nullptr, *pbko = nullptr;
  std::vector<double> shifts_host;  // [K][nz][2] as last set by holo_set_shifts
  // per-frame probe shifts (O19, holo_set_probe_shifts): Hq [K][nz][2][L] = h_omega_j r_{s^p_kj} / L per axis;
  // Qt [B][nz][L][L] (IDFT_x(Hq_x Qhat), P2), Qk [B][L][L] (q_kj, P2), Ut [B][nz][L][L] (probe-gradient terms)
  bool ps = false;
  bool fourier = false;  // holo_set_fourier: the object-side arrays are DFT2(psi) (Fourier-domain CG state)
  // holo_set_cg_fuse: the psi-block half of holo_cg_step deferred into the next sweep's X1
  bool cg_fuse = false, cg_pending = false;
  const float2 *cg_psi = nullptr, *cg_g = nullptr;
  float2 *cg_eta = nullptr, *cg_trial = nullptr;
  float cg_rho = 0.f, cg_beta = 0.f, cg_gamma = 0.f;
  int cg_mode = -1;
  // holo_stage_sqrt_d: a pending host -> device copy of the data, streamed per angle batch on a copy
  // stream by the next sweep that reads stage_dev (each batch's X2 waits for its own event)
  const float *stage_host = nullptr;
  float *stage_dev = nullptr;
  bool stage_ref = false;  // the staged array is the reference frames (holo_stage_sqrt_dref)
  cudaStream_t copy_stream = nullptr;
  cudaEvent_t stage_start = nullptr;
  std::vector<cudaEvent_t> stage_ev;
  cudaEvent_t gq_event = nullptr;  // holo_set_gq_event: recorded when grad_q_part is complete
  float2 *hq = nullptr, *Qt = nullptr, *Qk = nullptr, *Ut = nullptr;
  // per-pass event profiling (holo_profile_*)
  struct Rec {
    int id;
    double bytes, flops;
    size_t ev;
  };
  bool prof_on = false;
  std::vector<cudaEvent_t> evpool;
  size_t evused = 0;
  std::vector<Rec> recs;
  double pms[HOLO_NPASS]{}, pbytes[HOLO_NPASS]{}, pflops[HOLO_NPASS]{};
  uint64_t pcnt[HOLO_NPASS]{};

  holo::Tables tables() const {
    holo::Tables t;
    t.tw = reinterpret_cast<const float4 *>(tw);
    t.hdet = hdet;
    t.homega = homega;
    t.cout = cout;
    t.bke = bke;
    t.bko = bko;
    t.cr = cr;
    return t;
  }
};

// Entry points of one torus size L (defined in inst_<L>.cu).  sweep is NULL for L = 6144
// (reference-arm-only size).
struct HoloOps {
  int L;
  void (*set_attrs)();
  // mode: 0 grad, 1 fwd, 2 adj (y given), 3 objective only
  void (*sweep)(holo_plan *p, int mode, const float2 *psi, const float2 *q, const float *sqrt_d, const float2 *yin,
                float2 *wout, const float2 *eta, float2 *gpsi, float2 *gq_out, float gscale, bool want_q, bool acc_q,
                const float *sqrt_dref);
  void (*ref_run)(holo_plan *p, const float2 *q, const float *sqrt_dref, float2 *gq, double *sc, bool acc);
  void (*ref_fwd)(holo_plan *p, const float2 *q, float2 *w);
  void (*upsample2)(holo_plan *p, const float2 *coarse, float2 *fine, int count);  // NULL: unsupported L
  void (*init_psi)(holo_plan *p, const float *sqrt_d, const float *sqrt_dref, double db, float2 *psi0);  // O18
  void (*init_probe)(holo_plan *p, const float *sqrt_dref, float2 *q0);                               // O17
  int ref_lines_per_cta;  // rows per CTA of the reference-arm row kernels (partials per frame)
  int ref_R, ref_T;       // values per thread / threads per line of the reference-arm line engine
  void (*dft2)(holo_plan *p, const float2 *in, float2 *out, int count, int inverse);  // holo_fourier; NULL: 6144
};

const HoloOps *holo_ops_for(int L);  // NULL if L is not built
void holo_cg_flush(holo_plan *p);     // launch a deferred psi-block CG update (holo_set_cg_fuse) now

// ------------------------------------------------------------------ profiling
// pbeg / pend bracket one pass (one or more kernels); pend counts `nk` launches.
inline void prof_flush(holo_plan *p) {
  if (p->recs.empty()) return;
  cudaEventSynchronize(p->evpool[p->recs.back().ev + 1]);
  for (const auto &r : p->recs) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, p->evpool[r.ev], p->evpool[r.ev + 1]);
    p->pms[r.id] += ms;
    p->pbytes[r.id] += r.bytes;
    p->pflops[r.id] += r.flops;
    p->pcnt[r.id]++;
  }
  p->recs.clear();
  p->evused = 0;
}

inline void pbeg(holo_plan *p) {
  if (!p->prof_on) return;
  if (p->evused + 2 > 32768) prof_flush(p);
  while (p->evpool.size() < p->evused + 2) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    p->evpool.push_back(e);
  }
  cudaEventRecord(p->evpool[p->evused], p->stream);
}

inline void pend(holo_plan *p, int id, double bytes, double flops, int nk = 1) {
  p->launches += nk;
  if (!p->prof_on) return;
  cudaEventRecord(p->evpool[p->evused + 1], p->stream);
  p->recs.push_back({id, bytes, flops, p->evused});
  p->evused += 2;
}

inline double fftf(int L) {  // 5 L log2 L flops per length-L complex FFT
  int lg = 0;
  while ((1 << lg) < L) lg++;
  return 5.0 * L * lg;
}
