// holo_plan.cu -- host side of libholo: plan, fp64 table generation, argument
// validation, pass orchestration and the C ABI of include/holo.h.
#include <cuda_runtime.h>

#include <cmath>
#include <complex>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/holo.h"
#include "holo_passes.cuh"
#include "holo_ref.cuh"

using namespace holo;
using cd = std::complex<double>;

namespace {

constexpr double kPi = 3.14159265358979323846264338327950288;

struct Buf {
  void *p = nullptr;
  size_t bytes = 0;
};

}  // namespace

struct holo_plan {
  int device = 0;
  cudaStream_t stream = nullptr;
  holo_geometry g{};
  int L = 0, N = 0, nz = 0, K = 0;
  double m0 = 0, p0 = 0, mt[HOLO_MAX_NZ]{}, zeta[HOLO_MAX_NZ]{}, zdet[HOLO_MAX_NZ]{}, omega[HOLO_MAX_NZ]{};
  uint32_t magmask = 0;
  // device tables
  float2 *tw = nullptr, *hdet = nullptr, *homega = nullptr, *cout = nullptr, *cwo = nullptr, *bke = nullptr,
         *bko = nullptr, *wodd = nullptr, *cr = nullptr;
  std::vector<std::complex<double>> cin_host;  // [nz][L] kappa (-1)^fbar e^{i pi mt fbar^2/L} / L
  // workspace
  float2 *T1 = nullptr, *Aw = nullptr, *W1 = nullptr, *V1 = nullptr, *T3 = nullptr, *G = nullptr, *QJ = nullptr;
  double *partF = nullptr, *partX3 = nullptr, *partQ = nullptr;
  int nbx2 = 0, nbx3 = 0;
  int tau2 = 0;  // objective of the current holo_grad call: 0 = F_1 (amplitude), 1 = F_2 (intensity)  // CTAs of the X2 / X3 launches (partials per frame / per angle)
  size_t ws_bytes = 0;
  std::vector<void *> allocs;
  std::string err;
  bool sticky = false;
  uint64_t launches = 0;
  int n_ref = 0;
  std::vector<double> ref_shifts;
  // reference arm (holo_ref.cuh): Qhat, Ghat (P2, L x L), Wr, Vr (P2, N x L), Href [R][2][L], F partials
  float2 *Qhat = nullptr, *Ghat = nullptr, *Wr = nullptr, *Vr = nullptr, *Href = nullptr, *tw3 = nullptr;
  double *partR = nullptr;
  int ref_cap = 0;  // frames Href / partR are sized for
  // per-pass event profiling (holo_profile_*)
  struct Rec { int id; double bytes, flops; size_t ev; };
  bool prof_on = false;
  std::vector<cudaEvent_t> evpool;
  size_t evused = 0;
  std::vector<Rec> recs;
  double pms[HOLO_NPASS]{}, pbytes[HOLO_NPASS]{}, pflops[HOLO_NPASS]{};
  uint64_t pcnt[HOLO_NPASS]{};

  Tables tables() const {
    Tables t;
    t.tw = reinterpret_cast<const float4 *>(tw); t.hdet = hdet; t.homega = homega; t.cout = cout; t.cwo = cwo;
    t.bke = bke; t.bko = bko; t.wodd = wodd; t.cr = cr;
    return t;
  }
};

namespace {

holo_status fail(holo_plan *p, holo_status s, const std::string &msg) {
  if (p) p->err = msg;
  return s;
}

holo_status cuda_check(holo_plan *p, cudaError_t e, const char *what) {
  if (e == cudaSuccess) return HOLO_OK;
  p->sticky = true;
  p->err = std::string(what) + ": " + cudaGetErrorString(e);
  return HOLO_ECUDA;
}

#define HC(call)                                                     \
  do {                                                               \
    holo_status _s = cuda_check(p, (call), #call);                   \
    if (_s != HOLO_OK) return _s;                                    \
  } while (0)

template <class T>
holo_status dalloc(holo_plan *p, T **ptr, size_t bytes) {
  void *q = nullptr;
  cudaError_t e = cudaMalloc(&q, bytes ? bytes : 16);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(p, HOLO_ENOMEM, "cudaMalloc of " + std::to_string(bytes) + " bytes failed");
  }
  p->allocs.push_back(q);
  p->ws_bytes += bytes;
  *ptr = reinterpret_cast<T *>(q);
  return HOLO_OK;
}

holo_status upload(holo_plan *p, float2 *dst, const std::vector<cd> &v) {
  std::vector<float2> f(v.size());
  for (size_t i = 0; i < v.size(); i++) f[i] = make_float2((float)v[i].real(), (float)v[i].imag());
  HC(cudaMemcpy(dst, f.data(), f.size() * sizeof(float2), cudaMemcpyHostToDevice));
  return HOLO_OK;
}

long fbar(long f, long L) { return f < L / 2 ? f : f - L; }

// exp(i * 2 pi * num / den) with the integer part of num/den removed in fp64
cd expi2pi_frac(double x) {  // x in cycles
  x -= std::floor(x);
  return std::polar(1.0, 2.0 * kPi * x);
}

// in-place iterative radix-2 fp64 FFT (forward, unnormalised), n power of two
void fft64(std::vector<cd> &a) {
  const size_t n = a.size();
  for (size_t i = 1, j = 0; i < n; i++) {
    size_t bit = n >> 1;
    for (; j & bit; bit >>= 1) j ^= bit;
    j ^= bit;
    if (i < j) std::swap(a[i], a[j]);
  }
  for (size_t len = 2; len <= n; len <<= 1) {
    for (size_t i = 0; i < n; i += len)
      for (size_t k = 0; k < len / 2; k++) {
        cd w = std::polar(1.0, -2.0 * kPi * (double)k / (double)len);
        cd u = a[i + k], v = a[i + k + len / 2] * w;
        a[i + k] = u + v;
        a[i + k + len / 2] = u - v;
      }
  }
}

int radix16_stages(int L) {  // must match Shape<L>: S16 = (log2 L - 1) / 4, F = L / 16^S16
  int lg = 0;
  while ((1 << lg) < L) lg++;
  return (lg - 1) / 4;
}

// transfer h_z[f] = exp(-i pi lambda z (fbar/(L p0))^2), phase reduced in cycles
std::vector<cd> transfer(int L, double lam, double p0, double z) {
  std::vector<cd> h(L);
  for (int f = 0; f < L; f++) {
    double fr = (double)fbar(f, L) / ((double)L * p0);
    h[f] = expi2pi_frac(-0.5 * lam * z * fr * fr);
  }
  return h;
}

bool supported_L(int L) {
  return L == 128 || L == 256 || L == 512 || L == 1024 || L == 2048 || L == 4096 || L == 6144;
}
// the object chain (holo_fwd / holo_adj / holo_grad) needs a power-of-two torus; N_p = 6144
// (configs[4], reading C16) serves reference-arm-only plans (n_angles = 0)
bool chain_L(int L) { return (L & (L - 1)) == 0; }

template <int L>
struct Smem {
  static constexpr size_t X = CtaK<L>::XBYTES;                      // exchange space only (filters)
  static constexpr size_t XT = X + TabPipe<L>::BYTES;                // + two table slots
  static constexpr size_t XPT = X + CtaK<L>::PRIV + TabPipe<L>::BYTES;  // + one thread-private line
};

template <int L>
void set_smem_attrs() {
  using S = Smem<L>;
  auto a = [](const void *f, size_t s) { cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s); };
  a((const void *)k_x1<L>, S::XPT);
  a((const void *)k_y1<L>, S::XPT);
  a((const void *)k_x2<L, X2_GRAD>, S::XT);
  a((const void *)k_x2<L, X2_FWD>, S::XT);
  a((const void *)k_x2<L, X2_ADJ>, S::XT);
  a((const void *)k_x2<L, X2_OBJ>, S::XT);
  a((const void *)k_y2<L>, S::XPT);
  a((const void *)k_x3<L>, S::XPT);
  a((const void *)k_rows_filter<L, false, true, false>, S::X);
  a((const void *)k_rows_filter<L, true, false, false>, S::X);
  a((const void *)k_rows_filter<L, true, false, true>, S::X);
  a((const void *)k_cols_filter<L>, S::X);
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
}

void set_attrs(int L) {
  switch (L) {
    case 128: set_ref_attrs<128>(); break;
    case 256: set_ref_attrs<256>(); break;
    case 512: set_ref_attrs<512>(); break;
    case 1024: set_ref_attrs<1024>(); break;
    case 2048: set_ref_attrs<2048>(); break;
    case 4096: set_ref_attrs<4096>(); break;
    case 6144: set_ref_attrs<6144>(); return;
  }
  switch (L) {
    case 128: set_smem_attrs<128>(); break;
    case 256: set_smem_attrs<256>(); break;
    case 512: set_smem_attrs<512>(); break;
    case 1024: set_smem_attrs<1024>(); break;
    case 2048: set_smem_attrs<2048>(); break;
    case 4096: set_smem_attrs<4096>(); break;
  }
}

// ------------------------------------------------------------------ profiling
void prof_flush(holo_plan *p) {
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

void pbeg(holo_plan *p) {
  if (!p->prof_on) return;
  if (p->evused + 2 > 32768) prof_flush(p);
  while (p->evpool.size() < p->evused + 2) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    p->evpool.push_back(e);
  }
  cudaEventRecord(p->evpool[p->evused], p->stream);
}

void pend(holo_plan *p, int id, double bytes, double flops) {
  p->launches++;
  if (!p->prof_on) return;
  cudaEventRecord(p->evpool[p->evused + 1], p->stream);
  p->recs.push_back({id, bytes, flops, p->evused});
  p->evused += 2;
}

double fftf(int L) {  // 5 L log2 L flops per length-L complex FFT
  int lg = 0;
  while ((1 << lg) < L) lg++;
  return 5.0 * L * lg;
}

// ------------------------------------------------------------------ pass runners
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
      pend(p, HOLO_PASS_FILTER, 2 * A, 2.0 * L * fftf(L));
      pbeg(p);
      k_cols_filter<L><<<L / G, NT, SM::X, p->stream>>>(dst, dst, tb, p->homega + j * L, 0, 1.0f);
      pend(p, HOLO_PASS_FILTER, 2 * A, 2.0 * L * fftf(L));
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
      pend(p, HOLO_PASS_FILTER, 2 * A, 2.0 * L * fftf(L));
      pbeg(p);
      if (acc)
        k_rows_filter<L, true, false, true><<<L / G, NT, SM::X, p->stream>>>(Gj, out, tb, p->homega + j * L, 1, scale);
      else
        k_rows_filter<L, true, false, false><<<L / G, NT, SM::X, p->stream>>>(Gj, out, tb, p->homega + j * L, 1, scale);
      pend(p, HOLO_PASS_FILTER, (acc ? 3 : 2) * A, 2.0 * L * fftf(L));
    }
  }

  // mode: 0 grad, 1 fwd, 2 adj (y given), 3 objective only
  static void sweep(holo_plan *p, int mode, const float2 *psi, const float2 *q, const float *sqrt_d,
                    const float2 *yin, float2 *wout, const float2 *eta, float2 *gpsi, float2 *gq_out, float gscale,
                    bool want_q) {
    Tables tb = p->tables();
    const int N = p->N, nz = p->nz, K = p->K;
    const size_t LL = (size_t)L * L;
    const int nbx2 = (N + G - 1) / G;
    const double fl = fftf(L), rN = (double)N / L, NN8 = 8.0 * N * N;
    int nmag = 0;
    for (int j = 0; j < nz; j++) nmag += (p->magmask >> j) & 1;
    qj(p, q);
    if (want_q) cudaMemsetAsync(p->G, 0, sizeof(float2) * LL * nz, p->stream);
    // table sequences of the pipelined pointwise steps (holo_kernels.cuh, TabPipe)
    auto crp = [&](int k, int j, int ax) { return p->cr + ((size_t)(k * nz + j) * 2 + ax) * L; };
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
    for (int k = 0; k < K; k++) {
      const float2 *psik = psi + (size_t)k * LL;
      const bool need_fwd_chain = (mode != 2) || want_q;
      if (need_fwd_chain) {
        TabSeq q{};
        for (int j = 0; j < nz; j++) {
          if ((p->magmask >> j) & 1u)
            add_fwd(q, k, j, 0);
          else
            q.p[q.n++] = crp(k, j, 0);
        }
        pbeg(p);
        k_x1<L><<<L / G, NT, SM::XPT, p->stream>>>(psik, p->T1, tb, q, nz, p->magmask);
        pend(p, HOLO_PASS_X1, (1 + nz) * A, L * fl * (1 + 4 * nmag + (nz - nmag)));
      }
      for (int j = 0; j < nz; j++) {
        const int mag = (p->magmask >> j) & 1;
        const float2 *T1j = p->T1 + (size_t)j * LL;
        const float2 *qjj = p->QJ + (size_t)j * LL;
        const size_t fr = (size_t)k * nz + j;
        if (need_fwd_chain) {
          float2 *aout = want_q ? p->Aw : nullptr;
          float2 *w1 = (mode == 2) ? nullptr : p->W1;
          TabSeq q{};
          if (mag)
            add_fwd(q, k, j, 1);
          else
            q.p[q.n++] = crp(k, j, 1);
          if (w1) q.p[q.n++] = p->hdet + (size_t)j * L;
          pbeg(p);
          k_y1<L><<<L / G, NT, SM::XPT, p->stream>>>(T1j, qjj, aout, w1, tb, q, mag, N);
          pend(p, HOLO_PASS_Y1, A + (w1 ? A + rN * A : 0) + (aout ? A : 0),
               L * fl * (1 + (mag ? 4 : 1) + (w1 ? 2 : 0)));
        }
        double *pf = p->partF + fr * nbx2;
        TabSeq qh{};
        qh.p[qh.n++] = p->hdet + (size_t)j * L;
        if (mode == 0) qh.p[qh.n++] = p->hdet + (size_t)j * L;
        pbeg(p);
        if (mode == 1) {
          k_x2<L, X2_FWD><<<nbx2, NT, SM::XT, p->stream>>>(p->W1, nullptr, wout + fr * N * N, pf, tb, qh, N, p->tau2);
          pend(p, HOLO_PASS_X2, rN * A + NN8, N * fl * 2);
          continue;
        }
        if (mode == 3) {
          k_x2<L, X2_OBJ><<<nbx2, NT, SM::XT, p->stream>>>(p->W1, sqrt_d + fr * N * N, nullptr, pf, tb, qh, N, p->tau2);
          pend(p, HOLO_PASS_X2, rN * A + NN8 / 2, N * fl * 2);
          continue;
        }
        if (mode == 0) {
          k_x2<L, X2_GRAD><<<nbx2, NT, SM::XT, p->stream>>>(p->W1, sqrt_d + fr * N * N, p->V1, pf, tb, qh, N, p->tau2);
          pend(p, HOLO_PASS_X2, 2 * rN * A + NN8 / 2, N * fl * 4);
        } else {
          k_x2<L, X2_ADJ><<<nbx2, NT, SM::XT, p->stream>>>(yin + fr * N * N, nullptr, p->V1, pf, tb, qh, N, p->tau2);
          pend(p, HOLO_PASS_X2, rN * A + NN8, N * fl * 2);
        }
        float2 *Gj = want_q ? p->G + (size_t)j * LL : nullptr;
        float2 *T3j = gpsi ? p->T3 + (size_t)j * LL : nullptr;
        TabSeq q2{};
        q2.p[q2.n++] = p->hdet + (size_t)j * L;
        if (T3j) {
          if (mag)
            add_adj(q2, k, j, 1);
          else
            q2.p[q2.n++] = crp(k, j, 1);
        }
        pbeg(p);
        k_y2<L><<<L / G, NT, SM::XPT, p->stream>>>(p->V1, p->Aw, qjj, Gj, T3j, tb, q2, mag, N);
        pend(p, HOLO_PASS_Y2, rN * A + (Gj ? 3 * A : 0) + (T3j ? 2 * A : 0),
             L * fl * (2 + (T3j ? (mag ? 5 : 2) : 0)));
      }
      if (gpsi && (mode == 0 || mode == 2)) {
        TabSeq q3{};
        for (int j = 0; j < nz; j++) {
          if ((p->magmask >> j) & 1u)
            add_adj(q3, k, j, 0);
          else
            q3.p[q3.n++] = crp(k, j, 0);
        }
        pbeg(p);
        k_x3<L><<<L / G, NT, SM::XPT, p->stream>>>(p->T3, eta ? eta + (size_t)k * LL : nullptr, gpsi + (size_t)k * LL,
                                                p->partX3 + (size_t)k * 2 * p->nbx3, tb, q3, nz, p->magmask, gscale);
        pend(p, HOLO_PASS_X3, (nz + 1 + (eta ? 1 : 0)) * A, L * fl * (4 * nmag + (nz - nmag) + 1));
      }
    }
    if (want_q && (mode == 0 || mode == 2)) gq(p, gq_out, gscale, false);
  }
};

template <template <int> class R, class... A>
void dispatch_sweep(holo_plan *p, A... a) {
  switch (p->L) {
    case 128: R<128>::sweep(p, a...); break;
    case 256: R<256>::sweep(p, a...); break;
    case 512: R<512>::sweep(p, a...); break;
    case 1024: R<1024>::sweep(p, a...); break;
    case 2048: R<2048>::sweep(p, a...); break;
    case 4096: R<4096>::sweep(p, a...); break;
  }
}

// spectrum factor per (k, j, axis): cr[f] = cin_j[f] r_s[f] for magnified planes, r_s[f] / L at mt = 1,
// r_s[f] = e^{-2 pi i fbar s / L} (O4 / O5; the shift precedes the magnification, reading C4)
holo_status upload_cr(holo_plan *p, const double *s) {
  const int L = p->L, nz = p->nz, K = p->K;
  std::vector<float2> r((size_t)K * nz * 2 * L);
  for (int k = 0; k < K; k++)
    for (int j = 0; j < nz; j++) {
      const bool mag = (p->magmask >> j) & 1u;
      for (int ax = 0; ax < 2; ax++) {
        const double sv = s[((size_t)k * nz + j) * 2 + ax];
        float2 *dst = r.data() + (((size_t)k * nz + j) * 2 + ax) * L;
        for (int f = 0; f < L; f++) {
          cd v = expi2pi_frac(-(double)fbar(f, L) * sv / (double)L);
          v = mag ? v * p->cin_host[(size_t)j * L + f] : v / (double)L;
          dst[f] = make_float2((float)v.real(), (float)v.imag());
        }
      }
    }
  HC(cudaMemcpy(p->cr, r.data(), r.size() * sizeof(float2), cudaMemcpyHostToDevice));
  return HOLO_OK;
}

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
    pend(p, HOLO_PASS_REF, 4 * A, 2.0 * L * fl);
    for (int r = 0; r < R; r++) {
      const float2 *Hx = p->Href + (size_t)r * 2 * L, *Hy = Hx + L;
      pbeg(p);
      k_ref_cols<L, REF_R1><<<gl, E::NT, SM, p->stream>>>(p->Qhat, p->Wr, Hy, tw, p->tw3, N, 0);
      k_ref_rows<L, REF_FWD><<<gn, E::NT, SM, p->stream>>>(p->Wr, nullptr, w + (size_t)r * N * N, nullptr, Hx, tw,
                                                             p->tw3, N, 1.f, 0);
      pend(p, HOLO_PASS_REF, A * 2.0 + 8.0 * N * N, fl * (L + N));
    }
  }

  static void run(holo_plan *p, const float2 *q, const float *sqrt_dref, float2 *gq, double *sc, bool acc) {
    const int N = p->N, R = p->n_ref;
    const size_t SM = E::SMEM;
    const float4 *tw = reinterpret_cast<const float4 *>(p->tw);
    const float2 *tw3 = p->tw3;
    const int gl = L / E::G, gn = (N + E::G - 1) / E::G;
    const double A = 8.0 * L * L, fl = fftf(L);
    // Qhat = DFT2(q)
    pbeg(p);
    k_ref_rows<L, REF_QHAT><<<gl, E::NT, SM, p->stream>>>(q, nullptr, p->Qhat, nullptr, nullptr, tw, tw3, N, 1.f, 0);
    k_ref_cols<L, REF_QHAT><<<gl, E::NT, SM, p->stream>>>(p->Qhat, p->Qhat, nullptr, tw, tw3, N, 0);
    pend(p, HOLO_PASS_REF, 4 * A, 2.0 * L * fl);
    for (int r = 0; r < R; r++) {
      const float2 *Hx = p->Href + (size_t)r * 2 * L, *Hy = Hx + L;
      pbeg(p);
      k_ref_cols<L, REF_R1><<<gl, E::NT, SM, p->stream>>>(p->Qhat, p->Wr, Hy, tw, tw3, N, 0);
      k_ref_rows<L, REF_R2><<<gn, E::NT, SM, p->stream>>>(p->Wr, sqrt_dref + (size_t)r * N * N, p->Vr,
                                                            p->partR + (size_t)r * gn, Hx, tw, tw3, N, 1.f, 0,
                                                            p->tau2);
      if (gq) k_ref_cols<L, REF_R3><<<gl, E::NT, SM, p->stream>>>(p->Vr, p->Ghat, Hy, tw, tw3, N, r == 0);
      pend(p, HOLO_PASS_REF, A * (1.0 + 0.5 + 0.5 + 1.0 / 8 + 0.5 + (gq ? 0.5 + (r ? 2.0 : 1.0) : 0.0)),
           fl * (L + 2.0 * N + (gq ? L : 0)));
    }
    if (gq) {
      pbeg(p);
      k_ref_cols<L, REF_FINAL><<<gl, E::NT, SM, p->stream>>>(p->Ghat, p->Ghat, nullptr, tw, tw3, N, 0);
      k_ref_rows<L, REF_FINAL><<<gl, E::NT, SM, p->stream>>>(p->Ghat, nullptr, gq, nullptr, nullptr, tw, tw3, N,
                                                               2.0f, acc ? 1 : 0);
      pend(p, HOLO_PASS_REF, (acc ? 5 : 4) * A, 2.0 * L * fl);
    }
    pbeg(p);
    k_reduce<<<1, 1024, 0, p->stream>>>(p->partR, (size_t)R * gn, 1, sc, 0);
    pend(p, HOLO_PASS_REDUCE, 8.0 * R * gn, 0);
  }
};

holo_status precheck(holo_plan *p) {
  if (!p) return HOLO_EINVAL;
  if (p->sticky) return fail(p, HOLO_ESTATE, "plan is in an error state: " + p->err);
  cudaError_t e = cudaSetDevice(p->device);
  if (e != cudaSuccess) return cuda_check(p, e, "cudaSetDevice");
  return HOLO_OK;
}

holo_status postcheck(holo_plan *p) { return cuda_check(p, cudaGetLastError(), "kernel launch"); }

}  // namespace

// =================================================================== C ABI
extern "C" {

holo_status holo_plan_create(holo_plan **out, const holo_geometry *g, int device, void *stream) {
  if (!out || !g) return HOLO_EINVAL;
  *out = nullptr;
  const int L = g->npad, N = g->n, nz = g->nz, K = g->n_angles;
  if (nz < 1 || nz > HOLO_MAX_NZ || N < 8 || N % 2 || N > L || (L - N) % 2 || K < 0) return HOLO_EINVAL;
  if (!(g->wavelength > 0) || !(g->detector_pixel > 0) || !(g->focus_to_detector > 0) || !std::isfinite(g->wavelength))
    return HOLO_EINVAL;
  for (int j = 0; j < nz; j++) {
    if (!(g->z1[j] > 0) || !(g->z1[j] < g->focus_to_detector)) return HOLO_EINVAL;
    if (j > 0 && !(g->z1[j] > g->z1[j - 1])) return HOLO_EINVAL;
  }
  if (!supported_L(L)) return HOLO_EUNSUPPORTED;
  if (!chain_L(L) && K > 0) return HOLO_EUNSUPPORTED;
  if (N % 4) return HOLO_EUNSUPPORTED;  // float4 row I/O of N-wide frames
  holo_plan *p = new holo_plan();
  p->device = device;
  p->stream = reinterpret_cast<cudaStream_t>(stream);
  p->g = *g;
  p->L = L; p->N = N; p->nz = nz; p->K = K;
  // ---- O1 geometry (Eq. (8))
  const double Z = g->focus_to_detector;
  p->m0 = Z / g->z1[0];
  p->p0 = g->detector_pixel / p->m0;
  for (int j = 0; j < nz; j++) {
    p->mt[j] = g->z1[j] / g->z1[0];
    p->zeta[j] = g->z1[j] * (Z - g->z1[j]) / Z;
    p->omega[j] = (g->z1[j] - g->z1[0]) / p->mt[j];
    p->zdet[j] = p->zeta[j] / (p->mt[j] * p->mt[j]);
    if (p->mt[j] != 1.0) p->magmask |= 1u << j;
  }
  if (cudaSetDevice(device) != cudaSuccess) { delete p; return HOLO_ECUDA; }
  set_attrs(L);
  holo_status s = HOLO_OK;
  const size_t LL = (size_t)L * L;
  auto A = [&](auto **ptr, size_t bytes) { if (s == HOLO_OK) s = dalloc(p, ptr, bytes); };
  const int GR = 16 * NT / L;  // lines per CTA of the line kernels (CtaK<L>::G)
  p->nbx2 = (N + GR - 1) / GR;
  p->nbx3 = L / GR;
  const size_t Kc = (size_t)(K > 0 ? K : 1);
  const int LT = chain_L(L) ? L : L / 3;  // line length of the Stockham engine (6144 = 3 x 2048)
  const int S16 = radix16_stages(LT), F = LT >> (4 * S16);
  const size_t twrows = (size_t)F * (((size_t)1 << (4 * S16)) - 1) / 15;  // F (16^S16 - 1) / 15
  A(&p->tw, sizeof(float2) * 4 * twrows);
  A(&p->hdet, sizeof(float2) * L * nz);
  A(&p->homega, sizeof(float2) * L * nz);
  A(&p->cout, sizeof(float2) * L * nz);
  A(&p->cwo, sizeof(float2) * L * nz);
  A(&p->bke, sizeof(float2) * L * nz);
  A(&p->bko, sizeof(float2) * L * nz);
  A(&p->wodd, sizeof(float2) * L);
  A(&p->cr, sizeof(float2) * L * 2 * nz * Kc);
  const size_t LLc = K > 0 ? LL : 0;  // object-chain workspace only when the plan holds angles
  A(&p->T1, sizeof(float2) * LLc * nz);
  A(&p->Aw, sizeof(float2) * LLc);
  A(&p->W1, sizeof(float2) * (K > 0 ? (size_t)N * L : 0));
  A(&p->V1, sizeof(float2) * (K > 0 ? (size_t)N * L : 0));
  A(&p->T3, sizeof(float2) * LLc * nz);
  A(&p->G, sizeof(float2) * LLc * nz);
  A(&p->QJ, sizeof(float2) * LLc * nz);
  A(&p->partF, sizeof(double) * Kc * nz * p->nbx2);
  A(&p->partX3, sizeof(double) * Kc * 2 * p->nbx3);
  A(&p->partQ, sizeof(double) * 2 * 1184);
  if (s != HOLO_OK) { holo_plan_destroy(p); return s; }
  // ---- tables (fp64 -> fp32)
  {
    // FFT stage twiddle rows: radix-16 stage with Ns = F 16^st holds, per m < Ns,
    // (w^m, w^2m, w^4m, w^8m), w = exp(-2 pi i / (16 Ns))   (fft_engine.cuh)
    std::vector<cd> tw;
    for (int Ns = F; Ns < LT; Ns *= 16)
      for (int m = 0; m < Ns; m++)
        for (int e : {1, 2, 4, 8}) tw.push_back(expi2pi_frac(-(double)((long)m * e) / (16.0 * Ns)));
    if (tw.size() != 4 * twrows) { holo_plan_destroy(p); return HOLO_EUNSUPPORTED; }
    if (s == HOLO_OK) s = upload(p, p->tw, tw);
    std::vector<cd> wo(L);
    for (int i = 0; i < L; i++) wo[i] = expi2pi_frac(-(double)i / (2.0 * L));  // w[i] = e^{-i pi i / L}
    std::vector<cd> hd, ho, co, cw, be, bo;
    p->cin_host.clear();
    if (!chain_L(L)) {  // radix-3 combine twiddles W_6144^{g k}, g = 1, 2 (holo_ref.cuh)
      std::vector<cd> t3;
      for (int g3 = 1; g3 <= 2; g3++)
        for (int k = 0; k < L / 3; k++) t3.push_back(expi2pi_frac(-(double)(g3 * k) / (double)L));
      if (s == HOLO_OK) s = dalloc(p, &p->tw3, sizeof(float2) * t3.size());
      if (s == HOLO_OK) s = upload(p, p->tw3, t3);
    }
    for (int j = 0; j < nz && chain_L(L); j++) {
      auto h1 = transfer(L, g->wavelength, p->p0, p->zdet[j]);
      for (auto &h : h1) h /= (double)L;  // the 1/L of the inverse DFT folded in
      auto h2 = transfer(L, g->wavelength, p->p0, p->omega[j]);
      hd.insert(hd.end(), h1.begin(), h1.end());
      ho.insert(ho.end(), h2.begin(), h2.end());
      const double mt = p->mt[j];
      // cin[f] = kappa (-1)^fbar e^{i pi mt fbar^2 / L} / L ; phase in cycles: mt fbar^2 / (2L)
      for (int f = 0; f < L; f++) {
        long fb = fbar(f, L);
        double v = mt * (double)fb;
        bool kap = v >= -(double)(L / 2) && v < (double)(L / 2);
        double cyc = std::fmod(mt * (double)(fb * fb), 2.0 * L) / (2.0 * L) + (fb & 1 ? 0.5 : 0.0);
        p->cin_host.push_back(kap ? expi2pi_frac(cyc) / (double)L : cd(0, 0));
      }
      for (int o = 0; o < L; o++) {
        long n = o - L / 2;
        cd c = expi2pi_frac(std::fmod(mt * (double)(n * n), 2.0 * L) / (2.0 * L));
        co.push_back(c);
        cw.push_back(c * std::conj(wo[o]));
      }
      // b[d] = exp(-i pi mt d^2 / L), |d| < L, on a 2L cycle; Bhat = FFT_2L(b) / (2L)
      std::vector<cd> b(2 * L, cd(0, 0));
      for (int d = 0; d < L; d++) {
        cd v = expi2pi_frac(-std::fmod(mt * (double)((long)d * d), 2.0 * L) / (2.0 * L));
        b[d] = v;
        if (d > 0) b[2 * L - d] = v;
      }
      fft64(b);
      for (int kk = 0; kk < L; kk++) {
        be.push_back(b[2 * kk] / (2.0 * L));
        bo.push_back(b[2 * kk + 1] / (2.0 * L));
      }
    }
    if (chain_L(L)) {
      if (s == HOLO_OK) s = upload(p, p->hdet, hd);
      if (s == HOLO_OK) s = upload(p, p->homega, ho);
      if (s == HOLO_OK) s = upload(p, p->cout, co);
      if (s == HOLO_OK) s = upload(p, p->cwo, cw);
      if (s == HOLO_OK) s = upload(p, p->bke, be);
      if (s == HOLO_OK) s = upload(p, p->bko, bo);
    }
    if (s == HOLO_OK) s = upload(p, p->wodd, wo);
  }
  if (s == HOLO_OK && K > 0) {  // zero shifts until holo_set_shifts
    std::vector<double> zero((size_t)K * nz * 2, 0.0);
    s = upload_cr(p, zero.data());
  }
  if (s != HOLO_OK) { holo_plan_destroy(p); return s; }
  *out = p;
  return HOLO_OK;
}

void holo_plan_destroy(holo_plan *p) {
  if (!p) return;
  cudaSetDevice(p->device);
  for (cudaEvent_t e : p->evpool) cudaEventDestroy(e);
  for (void *a : p->allocs) cudaFree(a);
  delete p;
}

size_t holo_plan_workspace_bytes(const holo_plan *p) { return p ? p->ws_bytes : 0; }

const char *holo_last_error(const holo_plan *p) { return p ? p->err.c_str() : "null plan"; }

uint64_t holo_launch_count(const holo_plan *p) { return p ? p->launches : 0; }

holo_status holo_profile_enable(holo_plan *p, int enable) {
  holo_status st = precheck(p);
  if (st != HOLO_OK) return st;
  p->prof_on = enable != 0;
  return HOLO_OK;
}

holo_status holo_profile_read(holo_plan *p, double *ms, uint64_t *launches, double *bytes, double *flops, int reset) {
  holo_status st = precheck(p);
  if (st != HOLO_OK) return st;
  prof_flush(p);
  for (int i = 0; i < HOLO_NPASS; i++) {
    if (ms) ms[i] = p->pms[i];
    if (launches) launches[i] = p->pcnt[i];
    if (bytes) bytes[i] = p->pbytes[i];
    if (flops) flops[i] = p->pflops[i];
    if (reset) { p->pms[i] = 0; p->pcnt[i] = 0; p->pbytes[i] = 0; p->pflops[i] = 0; }
  }
  return postcheck(p);
}

holo_status holo_plan_derived(const holo_plan *p, double *m0, double *mt, double *zdet, double *omega, double *zeta,
                              double *p0) {
  if (!p) return HOLO_EINVAL;
  if (m0) *m0 = p->m0;
  if (p0) *p0 = p->p0;
  for (int j = 0; j < p->nz; j++) {
    if (mt) mt[j] = p->mt[j];
    if (zdet) zdet[j] = p->zdet[j];
    if (omega) omega[j] = p->omega[j];
    if (zeta) zeta[j] = p->zeta[j];
  }
  return HOLO_OK;
}

holo_status holo_set_shifts(holo_plan *p, const double *s) {
  holo_status st = precheck(p);
  if (st != HOLO_OK) return st;
  if (!s) return fail(p, HOLO_EINVAL, "null shifts");
  const int L = p->L, nz = p->nz, K = p->K;
  for (size_t i = 0; i < (size_t)K * nz * 2; i++)
    if (!std::isfinite(s[i]) || std::fabs(s[i]) >= L / 2) return fail(p, HOLO_EINVAL, "shift not finite or >= npad/2");
  return upload_cr(p, s);
}

holo_status holo_set_ref_shifts(holo_plan *p, int32_t n_ref, const double *s) {
  holo_status st = precheck(p);
  if (st != HOLO_OK) return st;
  if (n_ref < 0 || (n_ref > 0 && !s)) return fail(p, HOLO_EINVAL, "bad reference shifts");
  for (int i = 0; i < 2 * n_ref; i++)
    if (!std::isfinite(s[i]) || std::fabs(s[i]) >= p->L / 2) return fail(p, HOLO_EINVAL, "shift not finite or >= npad/2");
  const int L = p->L, N = p->N;
  const size_t LL = (size_t)L * L;
  // workspace of the reference arm, allocated on first use
  if (!p->Qhat) {
    st = dalloc(p, &p->Qhat, sizeof(float2) * LL);
    if (st == HOLO_OK) st = dalloc(p, &p->Ghat, sizeof(float2) * LL);
    if (st == HOLO_OK) st = dalloc(p, &p->Wr, sizeof(float2) * (size_t)N * L);
    if (st == HOLO_OK) st = dalloc(p, &p->Vr, sizeof(float2) * (size_t)N * L);
    if (st != HOLO_OK) return st;
  }
  if (n_ref > p->ref_cap) {
    const int nbr = (N + 15) / 1;  // >= R2 CTAs per frame for every engine (G >= 1)
    st = dalloc(p, &p->Href, sizeof(float2) * 2 * L * (size_t)n_ref);
    if (st == HOLO_OK) st = dalloc(p, &p->partR, sizeof(double) * (size_t)nbr * n_ref);
    if (st != HOLO_OK) return st;
    p->ref_cap = n_ref;
  }
  // H[r][ax][f] = h_{zeta0}[f] r_{s_ax}[f] / L  (O3 x O4 per axis; ax 0: x, 1: y)
  const auto h = transfer(L, p->g.wavelength, p->p0, p->zeta[0]);
  std::vector<float2> H((size_t)2 * L * n_ref);
  for (int r = 0; r < n_ref; r++)
    for (int ax = 0; ax < 2; ax++) {
      const double sv = s[2 * r + ax];
      for (int f = 0; f < L; f++) {
        const cd v = h[f] * expi2pi_frac(-(double)fbar(f, L) * sv / (double)L) / (double)L;
        H[((size_t)r * 2 + ax) * L + f] = make_float2((float)v.real(), (float)v.imag());
      }
    }
  if (n_ref > 0) HC(cudaMemcpy(p->Href, H.data(), H.size() * sizeof(float2), cudaMemcpyHostToDevice));
  p->n_ref = n_ref;
  p->ref_shifts.assign(s, s + 2 * n_ref);
  return HOLO_OK;
}

holo_status holo_fwd(holo_plan *p, const void *psi, const void *q, void *w) {
  holo_status st = precheck(p);
  if (st != HOLO_OK) return st;
  if (!psi || !q || !w) return fail(p, HOLO_EINVAL, "null pointer");
  dispatch_sweep<Run>(p, 1, (const float2 *)psi, (const float2 *)q, (const float *)nullptr, (const float2 *)nullptr,
                      (float2 *)w, (const float2 *)nullptr, (float2 *)nullptr, (float2 *)nullptr, 1.0f, false);
  return postcheck(p);
}

holo_status holo_adj(holo_plan *p, const void *y, const void *psi, const void *q, void *adj_psi, void *adj_q) {
  holo_status st = precheck(p);
  if (st != HOLO_OK) return st;
  if (!y || !psi || !q) return fail(p, HOLO_EINVAL, "null pointer");
  if (!adj_psi && !adj_q) return HOLO_OK;
  dispatch_sweep<Run>(p, 2, (const float2 *)psi, (const float2 *)q, (const float *)nullptr, (const float2 *)y,
                      (float2 *)nullptr, (const float2 *)nullptr, (float2 *)adj_psi, (float2 *)adj_q, 1.0f,
                      adj_q != nullptr);
  return postcheck(p);
}

holo_status holo_grad(holo_plan *p, const void *psi, const void *q, const float *sqrt_d, const void *eta_psi_prev,
                      void *grad_psi, void *grad_q_part, double *sc, uint32_t flags) {
  holo_status st = precheck(p);
  if (st != HOLO_OK) return st;
  const int K = p->K, nz = p->nz, N = p->N, L = p->L;
  if (!q || !sc || (K > 0 && (!psi || !sqrt_d))) return fail(p, HOLO_EINVAL, "null pointer");
  if (flags & HOLO_ACCUMULATE_Q) return fail(p, HOLO_EUNSUPPORTED, "HOLO_ACCUMULATE_Q not implemented for holo_grad");
  const bool obj = (flags & HOLO_OBJECTIVE_ONLY) != 0;
  p->tau2 = (flags & HOLO_INTENSITY) ? 1 : 0;
  HC(cudaMemsetAsync(sc, 0, 3 * sizeof(double), p->stream));
  if (K == 0) {  // empty shard: F = 0 and a zero probe-gradient partial (sums over no angles)
    if (!obj && grad_q_part) HC(cudaMemsetAsync(grad_q_part, 0, sizeof(float2) * (size_t)L * L, p->stream));
    return HOLO_OK;
  }
  dispatch_sweep<Run>(p, obj ? 3 : 0, (const float2 *)psi, (const float2 *)q, sqrt_d, (const float2 *)nullptr,
                      (float2 *)nullptr, (const float2 *)eta_psi_prev, obj ? nullptr : (float2 *)grad_psi,
                      obj ? nullptr : (float2 *)grad_q_part, 2.0f, !obj && grad_q_part != nullptr);
  pbeg(p);
  k_reduce<<<1, 1024, 0, p->stream>>>(p->partF, (size_t)K * nz * p->nbx2, 1, sc, 0);
  pend(p, HOLO_PASS_REDUCE, 8.0 * K * nz * ((N + 3) / 4), 0);
  if (!obj && grad_psi) {
    pbeg(p);
    k_reduce<<<1, 1024, 0, p->stream>>>(p->partX3, (size_t)K * p->nbx3, 2, sc + 1, 0);
    pend(p, HOLO_PASS_REDUCE, 8.0 * K * L, 0);
  }
  return postcheck(p);
}

holo_status holo_grad_ref(holo_plan *p, const void *q, const float *sqrt_dref, void *grad_q_part, double *sc,
                          uint32_t flags) {
  holo_status st = precheck(p);
  if (st != HOLO_OK) return st;
  if (!q || !sc || (p->n_ref > 0 && !sqrt_dref)) return fail(p, HOLO_EINVAL, "null pointer");
  HC(cudaMemsetAsync(sc, 0, sizeof(double), p->stream));
  const bool obj = (flags & HOLO_OBJECTIVE_ONLY) != 0, acc = (flags & HOLO_ACCUMULATE_Q) != 0;
  p->tau2 = (flags & HOLO_INTENSITY) ? 1 : 0;
  float2 *gq = obj ? nullptr : (float2 *)grad_q_part;
  if (p->n_ref == 0) {
    if (gq && !acc) HC(cudaMemsetAsync(gq, 0, sizeof(float2) * (size_t)p->L * p->L, p->stream));
    return HOLO_OK;
  }
  switch (p->L) {
    case 128: RefRun<128>::run(p, (const float2 *)q, sqrt_dref, gq, sc, acc); break;
    case 256: RefRun<256>::run(p, (const float2 *)q, sqrt_dref, gq, sc, acc); break;
    case 512: RefRun<512>::run(p, (const float2 *)q, sqrt_dref, gq, sc, acc); break;
    case 1024: RefRun<1024>::run(p, (const float2 *)q, sqrt_dref, gq, sc, acc); break;
    case 2048: RefRun<2048>::run(p, (const float2 *)q, sqrt_dref, gq, sc, acc); break;
    case 4096: RefRun<4096>::run(p, (const float2 *)q, sqrt_dref, gq, sc, acc); break;
    case 6144: RefRun<6144>::run(p, (const float2 *)q, sqrt_dref, gq, sc, acc); break;
  }
  return postcheck(p);
}

holo_status holo_fwd_ref(holo_plan *p, const void *q, void *w) {
  holo_status st = precheck(p);
  if (st != HOLO_OK) return st;
  if (!q || (p->n_ref > 0 && !w)) return fail(p, HOLO_EINVAL, "null pointer");
  if (p->n_ref == 0) return HOLO_OK;
  switch (p->L) {
    case 128: RefRun<128>::fwd(p, (const float2 *)q, (float2 *)w); break;
    case 256: RefRun<256>::fwd(p, (const float2 *)q, (float2 *)w); break;
    case 512: RefRun<512>::fwd(p, (const float2 *)q, (float2 *)w); break;
    case 1024: RefRun<1024>::fwd(p, (const float2 *)q, (float2 *)w); break;
    case 2048: RefRun<2048>::fwd(p, (const float2 *)q, (float2 *)w); break;
    case 4096: RefRun<4096>::fwd(p, (const float2 *)q, (float2 *)w); break;
    case 6144: RefRun<6144>::fwd(p, (const float2 *)q, (float2 *)w); break;
  }
  return postcheck(p);
}

holo_status holo_q_dots(holo_plan *p, const void *grad_q, const void *eta_q_prev, double *out) {
  holo_status st = precheck(p);
  if (st != HOLO_OK) return st;
  if (!grad_q || !out) return fail(p, HOLO_EINVAL, "null pointer");
  const size_t n = (size_t)p->L * p->L;
  pbeg(p);
  k_dots<<<1184, 256, 0, p->stream>>>((const float2 *)grad_q, (const float2 *)eta_q_prev, n, p->partQ);
  pend(p, HOLO_PASS_REDUCE, 8.0 * n * (eta_q_prev ? 2 : 1), 0);
  pbeg(p);
  k_reduce<<<1, 1024, 0, p->stream>>>(p->partQ, 1184, 2, out, 0);
  pend(p, HOLO_PASS_REDUCE, 16.0 * 1184, 0);
  return postcheck(p);
}

holo_status holo_cg_step(holo_plan *p, const holo_cg_in *in, holo_cg_out *out, const void *psi, void *eta_psi,
                         const void *grad_psi, void *psi_trial, const void *q, void *eta_q, const void *grad_q,
                         void *q_trial) {
  holo_status st = precheck(p);
  if (st != HOLO_OK) return st;
  if (!in || !out) return fail(p, HOLO_EINVAL, "null pointer");
  if (!std::isfinite(in->gamma) || !std::isfinite(in->gPg)) return fail(p, HOLO_EINVAL, "non-finite CG scalar");
  int mode = 2;
  double beta = 0.0, gen = in->g_eta_prev;  // for reuse_eta the caller tracks its own scalars
  int reset = 0;
  if (!in->reuse_eta) {
    if (in->first) {
      mode = 0; reset = 1; gen = -in->gPg;
    } else {
      double den = in->g_eta_prev - in->gprev_eta_prev;
      if (!(std::fabs(den) >= 1e-30 * in->gPg)) {
        mode = 0; reset = 1; gen = -in->gPg;
      } else {
        beta = in->gPg / den;
        gen = -in->gPg + beta * in->g_eta_prev;  // Re<g, -P g + beta eta_prev>
        if (!(gen < 0.0)) { mode = 0; reset = 1; beta = 0.0; gen = -in->gPg; } else mode = 1;
      }
    }
  }
  out->beta = beta;
  out->g_eta_new = gen;
  out->reset = reset;
  const size_t LL = (size_t)p->L * p->L;
  if (psi && eta_psi && psi_trial && (grad_psi || mode == 2)) {
    pbeg(p);
    k_cg<<<1184, 256, 0, p->stream>>>((const float4 *)psi, (float4 *)eta_psi, (const float4 *)grad_psi,
                                      (float4 *)psi_trial, LL * p->K / 2, (float)in->rho_psi, (float)beta,
                                      (float)in->gamma, mode);
    pend(p, HOLO_PASS_CG, 8.0 * LL * p->K * (mode == 2 ? 3 : mode == 0 ? 4 : 5), 0);
  }
  if (q && eta_q && q_trial && (grad_q || mode == 2)) {
    pbeg(p);
    k_cg<<<1184, 256, 0, p->stream>>>((const float4 *)q, (float4 *)eta_q, (const float4 *)grad_q, (float4 *)q_trial,
                                      LL / 2, (float)in->rho_q, (float)beta, (float)in->gamma, mode);
    pend(p, HOLO_PASS_CG, 8.0 * LL * (mode == 2 ? 3 : mode == 0 ? 4 : 5), 0);
  }
  return postcheck(p);
}

}  // extern "C"
