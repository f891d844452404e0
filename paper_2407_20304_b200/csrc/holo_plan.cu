// holo_plan.cu -- host side of libholo: plan creation, fp64 table generation, argument
// validation and the C ABI of include/holo.h.  The per-L pass runners live in
// inst_<L>.cu (holo_run.cuh); this unit only dispatches through HoloOps.
#include <cuda_runtime.h>

#include <cmath>
#include <complex>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "holo_impl.cuh"
#include "holo_passes.cuh"  // only the non-template helpers (k_reduce, k_dots, k_cg) are instantiated here
#include "holo_multires.cuh"  // k_bin2

using namespace holo;
using cd = std::complex<double>;

extern const HoloOps holo_ops_128, holo_ops_256, holo_ops_512, holo_ops_1024, holo_ops_2048, holo_ops_4096,
    holo_ops_6144;

const HoloOps *holo_ops_for(int L) {
  switch (L) {
    case 128: return &holo_ops_128;
    case 256: return &holo_ops_256;
    case 512: return &holo_ops_512;
    case 1024: return &holo_ops_1024;
    case 2048: return &holo_ops_2048;
    case 4096: return &holo_ops_4096;
    case 6144: return &holo_ops_6144;
  }
  return nullptr;
}

namespace {

constexpr double kPi = 3.14159265358979323846264338327950288;

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
  p->alloc_bytes.push_back(bytes);
  p->ws_bytes += bytes;
  *ptr = reinterpret_cast<T *>(q);
  return HOLO_OK;
}

void dfree(holo_plan *p, void **ptr) {  // free one workspace buffer and forget it
  if (!*ptr) return;
  for (size_t i = 0; i < p->allocs.size(); i++)
    if (p->allocs[i] == *ptr) {
      p->ws_bytes -= p->alloc_bytes[i];
      p->allocs.erase(p->allocs.begin() + i);
      p->alloc_bytes.erase(p->alloc_bytes.begin() + i);
      break;
    }
  cudaFree(*ptr);
  *ptr = nullptr;
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

// Bluestein chirp-z tables of M_{1/mt} on an L torus (reading C1, holo_kernels.cuh mag_fwd), appended:
//   cin[f]  = kappa (-1)^fbar e^{i pi mt fbar^2 / L} / L      (kappa: -L/2 <= mt fbar < L/2)
//   cout[o] = e^{i pi mt (o - L/2)^2 / L}
//   b[d] = e^{-i pi mt d^2 / L}, |d| < L, on a 2L cycle; Bhat = FFT_2L(b) / (2L) split even / odd
// phases reduced in cycles in fp64 before rounding.
void czt_tables(int L, double mt, std::vector<cd> &cin, std::vector<cd> &co, std::vector<cd> &be,
                std::vector<cd> &bo) {
  for (int f = 0; f < L; f++) {
    long fb = fbar(f, L);
    double v = mt * (double)fb;
    bool kap = v >= -(double)(L / 2) && v < (double)(L / 2);
    double cyc = std::fmod(mt * (double)(fb * fb), 2.0 * L) / (2.0 * L) + (fb & 1 ? 0.5 : 0.0);
    cin.push_back(kap ? expi2pi_frac(cyc) / (double)L : cd(0, 0));
  }
  for (int o = 0; o < L; o++) {
    long n = o - L / 2;
    co.push_back(expi2pi_frac(std::fmod(mt * (double)(n * n), 2.0 * L) / (2.0 * L)));
  }
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

bool supported_L(int L) {
  return L == 128 || L == 256 || L == 512 || L == 1024 || L == 2048 || L == 4096 || L == 6144;
}
// the object chain (holo_fwd / holo_adj / holo_grad) needs a power-of-two torus; N_p = 6144
// (configs[4], reading C16) serves reference-arm-only plans (n_angles = 0)
bool chain_L(int L) { return (L & (L - 1)) == 0; }

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

holo_status ensure_fourier_ws(holo_plan *p);  // below

// keep_cg: the sweep entry points decide themselves whether a deferred CG step fuses into their X1
holo_status precheck(holo_plan *p, bool keep_cg = false) {
  if (!p) return HOLO_EINVAL;
  if (p->sticky) return fail(p, HOLO_ESTATE, "plan is in an error state: " + p->err);
  cudaError_t e = cudaSetDevice(p->device);
  if (e != cudaSuccess) return cuda_check(p, e, "cudaSetDevice");
  if (p->cg_pending && !keep_cg) holo_cg_flush(p);
  return HOLO_OK;
}

holo_status postcheck(holo_plan *p) { return cuda_check(p, cudaGetLastError(), "kernel launch"); }

}  // namespace

// =================================================================== C ABI
void holo_cg_flush(holo_plan *p) {
  if (!p->cg_pending) return;
  p->cg_pending = false;
  const size_t LL = (size_t)p->L * p->L;
  const int mode = p->cg_mode;
  pbeg(p);
  k_cg<<<1184, 256, 0, p->stream>>>((const float4 *)p->cg_psi, (float4 *)p->cg_eta, (const float4 *)p->cg_g,
                                    (float4 *)p->cg_trial, LL * p->K / 2, p->cg_rho, p->cg_beta, p->cg_gamma, mode);
  pend(p, HOLO_PASS_CG, 8.0 * LL * p->K * (mode == 2 ? 3 : mode == 0 ? 4 : 5), 0);
}

extern "C" {

// TMA descriptor of a P2 workspace (T3 for X3's row staging, W1 for X2's; holo_passes.cuh RowStage): the
// P2 plane as a 4-D fp32 tensor {4 floats = one column pair of one row, R rows, L/2 column pairs, planes}, box
// {4, G, min(256, L/2), 1}.  The encoder comes from the driver through the runtime (no -lcuda link).
// false (X3 then loads its rows with LDG) if the driver entry point or the encoding is unavailable.
static bool make_p2map(CUtensorMap *map, void *base, int L, int R, int planes) {
  typedef CUresult (*EncodeTiled)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                  const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  void *fn = nullptr;
  cudaDriverEntryPointQueryResult q{};
  if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn ||
      q != cudaDriverEntryPointSuccess) {
    cudaGetLastError();
    return false;
  }
  const int G = 8192 / L;  // lines per 512-thread CTA (holo_kernels.cuh Cta)
  if (G < 2 || G > 256) return false;
  const cuuint64_t dims[4] = {4, (cuuint64_t)R, (cuuint64_t)L / 2, (cuuint64_t)planes};
  const cuuint64_t strides[3] = {16, 16ull * R, 8ull * R * L};  // bytes, dims 1..3
  const cuuint32_t box[4] = {4, (cuuint32_t)G, (cuuint32_t)(L / 2 < 256 ? L / 2 : 256), 1};
  const cuuint32_t estr[4] = {1, 1, 1, 1};
  const CUresult r = reinterpret_cast<EncodeTiled>(fn)(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, base, dims, strides,
                                                      box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                                      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

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
  if (g->angle_batch < 1 || g->angle_batch > HOLO_MAX_BATCH) return HOLO_EINVAL;
  const HoloOps *ops = holo_ops_for(L);
  if (!ops || (K > 0 && !ops->sweep)) return HOLO_EUNSUPPORTED;
  holo_plan *p = new holo_plan();
  p->ops = ops;
  p->B = g->angle_batch < (K > 0 ? K : 1) ? g->angle_batch : (K > 0 ? K : 1);
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
  ops->set_attrs();
  holo_status s = HOLO_OK;
  const size_t LL = (size_t)L * L;
  auto A = [&](auto **ptr, size_t bytes) { if (s == HOLO_OK) s = dalloc(p, ptr, bytes); };
  const int GR = 16 * NT / L;  // lines per CTA of the object-chain line kernels (CtaK<L>::G)
  p->nbx2 = (N + GR - 1) / GR;
  p->nbx3 = L / GR;
  const size_t Kc = (size_t)(K > 0 ? K : 1);
  const int LT = chain_L(L) ? L : L / 3;  // line length of the Stockham engine (6144 = 3 x 2048)
  const int S16 = radix16_stages(LT), F = LT >> (4 * S16);
  const size_t twrows = (size_t)F * (((size_t)1 << (4 * S16)) - 1) / 15;  // F (16^S16 - 1) / 15
  A(&p->tw, sizeof(float2) * holo::TW_ROW_F2 * twrows);
  A(&p->hdet, sizeof(float2) * L * nz);
  A(&p->homega, sizeof(float2) * L * nz);
  A(&p->cout, sizeof(float2) * L * nz);
  A(&p->bke, sizeof(float2) * L * nz);
  A(&p->bko, sizeof(float2) * L * nz);
  A(&p->cr, sizeof(float2) * L * 2 * nz * Kc);
  const size_t LLc = K > 0 ? LL : 0;  // object-chain workspace only when the plan holds angles
  const size_t Bc = (size_t)p->B;     // batch-sized per-frame workspace (holo_run.cuh)
  A(&p->T1, sizeof(float2) * LLc * nz * Bc);
  A(&p->Aw, sizeof(float2) * LLc * Bc);
  A(&p->W1, sizeof(float2) * (K > 0 ? (size_t)N * L * Bc : 0));
  A(&p->V1, sizeof(float2) * (K > 0 ? (size_t)N * L * Bc : 0));
  A(&p->T3, sizeof(float2) * LLc * nz * Bc);
  A(&p->G, sizeof(float2) * LLc * nz);
  A(&p->QJ, sizeof(float2) * LLc * nz);
  if (s == HOLO_OK && p->T3 && chain_L(L)) {
    p->t3map_ok = make_p2map(&p->t3map, p->T3, L, L, nz * (int)Bc);
    p->w1map_ok = make_p2map(&p->w1map, p->W1, L, N, (int)Bc);  // X2's row staging (rows >= N read as zeros)
  }
  A(&p->partF, sizeof(double) * Kc * nz * p->nbx2);
  A(&p->partX3, sizeof(double) * Kc * 2 * p->nbx3);
  A(&p->partQ, sizeof(double) * 2 * 1184);
  if (chain_L(L) && K > 0) {  // initial object (O18): inverse-magnification chirp-z tables
    A(&p->pcin, sizeof(float2) * L * nz);
    A(&p->pcout, sizeof(float2) * L * nz);
    A(&p->pbke, sizeof(float2) * L * nz);
    A(&p->pbko, sizeof(float2) * L * nz);
  }
  if (chain_L(L)) {  // multiresolution: up-sampling table and the row-pass scratch P2 [L/2][L]
    A(&p->uptab, sizeof(float2) * L);
    A(&p->Up, sizeof(float2) * LL / 2);
  }
  if (s != HOLO_OK) { holo_plan_destroy(p); return s; }
  // ---- tables (fp64 -> fp32)
  {
    // FFT stage twiddle rows: radix-16 stage with Ns = F 16^st holds, per m < Ns,
    // (w^m, w^2m, w^4m, w^8m), w = exp(-2 pi i / (16 Ns)), and with HOLO_TW8 the DIT level twiddles
    // w^m e^{-i pi/8}, w^m e^{-i pi/4}, w^m e^{-3 i pi/8}, w^2m e^{-i pi/4}   (fft_engine.cuh)
    std::vector<cd> tw;
    for (int Ns = F; Ns < LT; Ns *= 16)
      for (int m = 0; m < Ns; m++) {
        const double f = -(double)m / (16.0 * Ns);  // cycles of w^m
        for (int e : {1, 2, 4, 8}) tw.push_back(expi2pi_frac(-(double)((long)m * e) / (16.0 * Ns)));
        if (holo::TW_ROW_F2 == 8) {
          tw.push_back(expi2pi_frac(f - 1.0 / 16));
          tw.push_back(expi2pi_frac(f - 1.0 / 8));
          tw.push_back(expi2pi_frac(f - 3.0 / 16));
          tw.push_back(expi2pi_frac(2 * f - 1.0 / 8));
        }
      }
    if (tw.size() != (size_t)holo::TW_ROW_F2 * twrows) { holo_plan_destroy(p); return HOLO_EUNSUPPORTED; }
    if (s == HOLO_OK) s = upload(p, p->tw, tw);
    std::vector<cd> hd, ho, co, be, bo, pci, pco, pbe, pbo;
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
      czt_tables(L, p->mt[j], p->cin_host, co, be, bo);
      if (K > 0) czt_tables(L, 1.0 / p->mt[j], pci, pco, pbe, pbo);  // O18: inverse magnification
    }
    if (chain_L(L)) {
      // up[F] = [Fbar in [-L/4, L/4)] e^{-i pi Fbar / L} / (L/2): Fourier 2x upsampling from L/2 (O15)
      std::vector<cd> up(L);
      for (int f = 0; f < L; f++) {
        const long fb = fbar(f, L);
        up[f] = (fb >= -(L / 4) && fb < L / 4) ? expi2pi_frac(-(double)fb / (2.0 * L)) / (double)(L / 2) : cd(0, 0);
      }
      if (s == HOLO_OK) s = upload(p, p->uptab, up);
      if (s == HOLO_OK) s = upload(p, p->hdet, hd);
      if (s == HOLO_OK) s = upload(p, p->homega, ho);
      if (s == HOLO_OK) s = upload(p, p->cout, co);
      if (s == HOLO_OK) s = upload(p, p->bke, be);
      if (s == HOLO_OK) s = upload(p, p->bko, bo);
      if (K > 0) {
        if (s == HOLO_OK) s = upload(p, p->pcin, pci);
        if (s == HOLO_OK) s = upload(p, p->pcout, pco);
        if (s == HOLO_OK) s = upload(p, p->pbke, pbe);
        if (s == HOLO_OK) s = upload(p, p->pbko, pbo);
      }
    }
  }
  if (s == HOLO_OK && K > 0) {  // zero shifts until holo_set_shifts
    p->shifts_host.assign((size_t)K * nz * 2, 0.0);
    s = upload_cr(p, p->shifts_host.data());
  }
  if (s != HOLO_OK) { holo_plan_destroy(p); return s; }
  *out = p;
  return HOLO_OK;
}

void holo_plan_destroy(holo_plan *p) {
  if (!p) return;
  cudaSetDevice(p->device);
  for (cudaEvent_t e : p->evpool) cudaEventDestroy(e);
  for (cudaEvent_t e : p->stage_ev) cudaEventDestroy(e);
  if (p->stage_start) cudaEventDestroy(p->stage_start);
  if (p->copy_stream) cudaStreamDestroy(p->copy_stream);
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
  p->shifts_host.assign(s, s + (size_t)K * nz * 2);
  return upload_cr(p, s);
}

holo_status holo_set_ref_shifts(holo_plan *p, int32_t n_ref, const double *s) {
  holo_status st = precheck(p);
  if (st != HOLO_OK) return st;
  if (n_ref < 0 || (n_ref > 0 && !s)) return fail(p, HOLO_EINVAL, "bad reference shifts");
  for (int i = 0; i < 2 * n_ref; i++)
    if (!std::isfinite(s[i]) || std::fabs(s[i]) >= p->L / 2) return fail(p, HOLO_EINVAL, "shift not finite or >= npad/2");
  const int L = p->L, N = p->N;
  // workspace of the reference arm, allocated on first use (shared with the probe-shift path)
  st = ensure_fourier_ws(p);
  if (st != HOLO_OK) return st;
  {  // frame workspace of the batched reference passes: W_r, V_r [BR][N][L]
    const int BR = n_ref < 8 ? (n_ref > 0 ? n_ref : 1) : 8;
    if (!p->Wr || BR > p->BR) {
      HC(cudaStreamSynchronize(p->stream));
      dfree(p, (void **)&p->Wr);
      dfree(p, (void **)&p->Vr);
      st = dalloc(p, &p->Wr, sizeof(float2) * (size_t)N * L * BR);
      if (st == HOLO_OK) st = dalloc(p, &p->Vr, sizeof(float2) * (size_t)N * L * BR);
      if (st != HOLO_OK) return st;
      p->BR = BR;
    }
  }
  if (n_ref > p->ref_cap) {  // (re)size the per-frame tables; the old ones are freed, not leaked
    const int G = p->ops->ref_lines_per_cta;
    const int nbr = (N + G - 1) / G;  // CTAs of one frame's R2 row pass (one F partial each)
    HC(cudaStreamSynchronize(p->stream));  // a queued reference sweep may still read them
    dfree(p, (void **)&p->Href);
    dfree(p, (void **)&p->Hfac);
    dfree(p, (void **)&p->partR);
    p->ref_cap = 0;
    st = dalloc(p, &p->Href, sizeof(float2) * 2 * L * (size_t)n_ref);
    if (st == HOLO_OK)
      st = dalloc(p, &p->Hfac, sizeof(float2) * 2 * (size_t)(p->ops->ref_R + p->ops->ref_T) * n_ref);
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
  // factored form for the sweep passes: hz[f] = h_{zeta0}[f] / L, and per frame / axis the ramp
  // r_s[f] = A[i] B[t] over the engine layout f = t + base(i) (t < ref_T: thread, i < ref_R: value):
  // A[i] = e^{-2 pi i fbar(base(i)) s / L} (fbar's Nyquist wrap depends on i only: base(i) is a multiple
  // of ref_T and so is L/2), B[t] = e^{-2 pi i t s / L}.  holo_ref.cuh LineEng<L>::ifr defines base(i).
  if (!p->hz) {
    st = dalloc(p, &p->hz, sizeof(float2) * L);
    if (st != HOLO_OK) return st;
    std::vector<float2> hzv(L);
    for (int f = 0; f < L; f++) {
      const cd v = h[f] / (double)L;
      hzv[f] = make_float2((float)v.real(), (float)v.imag());
    }
    HC(cudaMemcpy(p->hz, hzv.data(), hzv.size() * sizeof(float2), cudaMemcpyHostToDevice));
  }
  {
    const int RE = p->ops->ref_R, TE = p->ops->ref_T, FS = RE + TE;
    auto base = [&](int i) { return RE == 48 ? TE * (i % 16) + (L / 3) * (i / 16) : TE * i; };
    std::vector<float2> Fv((size_t)2 * FS * n_ref);
    for (int r = 0; r < n_ref; r++)
      for (int ax = 0; ax < 2; ax++) {
        const double sv = s[2 * r + ax];
        float2 *o = Fv.data() + ((size_t)r * 2 + ax) * FS;
        for (int i = 0; i < RE; i++) {
          const cd v = expi2pi_frac(-(double)fbar(base(i), L) * sv / (double)L);
          o[i] = make_float2((float)v.real(), (float)v.imag());
        }
        for (int t = 0; t < TE; t++) {
          const cd v = expi2pi_frac(-(double)t * sv / (double)L);
          o[RE + t] = make_float2((float)v.real(), (float)v.imag());
        }
      }
    if (n_ref > 0) HC(cudaMemcpy(p->Hfac, Fv.data(), Fv.size() * sizeof(float2), cudaMemcpyHostToDevice));
  }
  p->n_ref = n_ref;
  p->ref_shifts.assign(s, s + 2 * n_ref);
  return HOLO_OK;
}

holo_status holo_fwd(holo_plan *p, const void *psi, const void *q, void *w) {
  holo_status st = precheck(p, true);
  if (st != HOLO_OK) return st;
  if (!psi || !q || !w) return fail(p, HOLO_EINVAL, "null pointer");
  if (p->K == 0) return HOLO_OK;
  p->ops->sweep(p, 1, (const float2 *)psi, (const float2 *)q, nullptr, nullptr, (float2 *)w, nullptr, nullptr,
                nullptr, 1.0f, false, false, nullptr);
  return postcheck(p);
}

holo_status holo_adj(holo_plan *p, const void *y, const void *psi, const void *q, void *adj_psi, void *adj_q) {
  holo_status st = precheck(p, true);
  if (st != HOLO_OK) return st;
  if (!y || !psi || !q) return fail(p, HOLO_EINVAL, "null pointer");
  if (!adj_psi && !adj_q) return HOLO_OK;
  if (p->K == 0) {  // sums over no angles
    if (adj_q) HC(cudaMemsetAsync(adj_q, 0, sizeof(float2) * (size_t)p->L * p->L, p->stream));
    return HOLO_OK;
  }
  p->ops->sweep(p, 2, (const float2 *)psi, (const float2 *)q, nullptr, (const float2 *)y, nullptr, nullptr,
                (float2 *)adj_psi, (float2 *)adj_q, 1.0f, adj_q != nullptr, false, nullptr);
  return postcheck(p);
}

}  // extern "C"

namespace {
// holo_grad / holo_grad_full: the object chain (+ the fused reference frames when sqrt_dref)
holo_status grad_impl(holo_plan *p, const void *psi, const void *q, const float *sqrt_d, const float *sqrt_dref,
                      const void *eta_psi_prev, void *grad_psi, void *grad_q_part, double *sc, uint32_t flags) {
  const int K = p->K, nz = p->nz, N = p->N, L = p->L;
  if (!q || !sc || (K > 0 && (!psi || !sqrt_d))) return fail(p, HOLO_EINVAL, "null pointer");
  const bool obj = (flags & HOLO_OBJECTIVE_ONLY) != 0, acc = (flags & HOLO_ACCUMULATE_Q) != 0;
  const bool ref = sqrt_dref != nullptr && p->n_ref > 0;
  p->tau = (flags & HOLO_INTENSITY) ? 2.f : (float)p->tau_set;
  HC(cudaMemsetAsync(sc, 0, 3 * sizeof(double), p->stream));
  float2 *gq = obj ? nullptr : (float2 *)grad_q_part;
  if (K == 0) {  // empty shard: F = 0 and a zero probe-gradient partial (sums over no angles)
    if (gq && !acc) HC(cudaMemsetAsync(gq, 0, sizeof(float2) * (size_t)L * L, p->stream));
    if (ref) {  // a reference-only shard: the reference arm alone
      p->ops->ref_run(p, (const float2 *)q, sqrt_dref, gq, sc, true);
    }
    if (gq && p->gq_event) HC(cudaEventRecord(p->gq_event, p->stream));
    return postcheck(p);
  }
  p->ops->sweep(p, obj ? 3 : 0, (const float2 *)psi, (const float2 *)q, sqrt_d, nullptr, nullptr,
                (const float2 *)eta_psi_prev, obj ? nullptr : (float2 *)grad_psi, gq, 2.0f, gq != nullptr, acc,
                ref ? sqrt_dref : nullptr);
  pbeg(p);
  k_reduce<<<1, 1024, 0, p->stream>>>(p->partF, (size_t)K * nz * p->nbx2, 1, sc, 0);
  pend(p, HOLO_PASS_REDUCE, 8.0 * K * nz * ((N + 3) / 4), 0);
  if (ref) {
    const int G = p->ops->ref_lines_per_cta, gn = (N + G - 1) / G;
    pbeg(p);
    k_reduce<<<1, 1024, 0, p->stream>>>(p->partR, (size_t)p->n_ref * gn, 1, sc, 1);
    pend(p, HOLO_PASS_REDUCE, 8.0 * p->n_ref * gn, 0);
  }
  if (!obj && grad_psi) {
    pbeg(p);
    k_reduce<<<1, 1024, 0, p->stream>>>(p->partX3, (size_t)K * p->nbx3, 2, sc + 1, 0);
    pend(p, HOLO_PASS_REDUCE, 8.0 * K * L, 0);
  }
  return postcheck(p);
}

// reference-arm workspace (Qhat, Ghat: P2 L x L; Wr, Vr: P2 N x L), shared with the probe-shift path
holo_status ensure_fourier_ws(holo_plan *p) {
  if (p->Qhat) return HOLO_OK;
  const size_t LL = (size_t)p->L * p->L, NL = (size_t)p->N * p->L;
  holo_status st = dalloc(p, &p->Qhat, sizeof(float2) * LL);
  if (st == HOLO_OK) st = dalloc(p, &p->Ghat, sizeof(float2) * LL);
  (void)NL;
  return st;
}
}  // namespace

extern "C" {

holo_status holo_grad(holo_plan *p, const void *psi, const void *q, const float *sqrt_d, const void *eta_psi_prev,
                      void *grad_psi, void *grad_q_part, double *sc, uint32_t flags) {
  holo_status st = precheck(p, true);
  if (st != HOLO_OK) return st;
  return grad_impl(p, psi, q, sqrt_d, nullptr, eta_psi_prev, grad_psi, grad_q_part, sc, flags);
}

holo_status holo_grad_full(holo_plan *p, const void *psi, const void *q, const float *sqrt_d, const float *sqrt_dref,
                           const void *eta_psi_prev, void *grad_psi, void *grad_q_part, double *sc, uint32_t flags) {
  holo_status st = precheck(p, true);
  if (st != HOLO_OK) return st;
  return grad_impl(p, psi, q, sqrt_d, sqrt_dref, eta_psi_prev, grad_psi, grad_q_part, sc, flags);
}

holo_status holo_set_gq_event(holo_plan *p, void *event) {
  holo_status st = precheck(p);
  if (st != HOLO_OK) return st;
  p->gq_event = reinterpret_cast<cudaEvent_t>(event);
  return HOLO_OK;
}

holo_status holo_set_tau(holo_plan *p, double tau) {
  holo_status st = precheck(p);
  if (st != HOLO_OK) return st;
  if (!(tau >= 0.25 && tau <= 4.0)) return fail(p, HOLO_EINVAL, "tau must lie in [0.25, 4]");
  p->tau_set = tau;
  return HOLO_OK;
}

holo_status holo_set_probe_shifts(holo_plan *p, const double *s) {
  holo_status st = precheck(p);
  if (st != HOLO_OK) return st;
  const int L = p->L, nz = p->nz, K = p->K;
  if (!s) {
    p->ps = false;
    return HOLO_OK;
  }
  if (K == 0 || !p->ops->sweep) return fail(p, HOLO_EUNSUPPORTED, "probe shifts need angles on a power-of-two torus");
  for (size_t i = 0; i < (size_t)K * nz * 2; i++)
    if (!std::isfinite(s[i]) || std::fabs(s[i]) >= L / 2) return fail(p, HOLO_EINVAL, "shift not finite or >= npad/2");
  if (!p->hq) {
    const size_t LL = (size_t)L * L, Bc = (size_t)p->B;
    st = ensure_fourier_ws(p);
    if (st == HOLO_OK) st = dalloc(p, &p->hq, sizeof(float2) * L * 2 * nz * (size_t)K);
    if (st == HOLO_OK) st = dalloc(p, &p->Qt, sizeof(float2) * LL * nz * Bc);
    if (st == HOLO_OK) st = dalloc(p, &p->Qk, sizeof(float2) * LL * Bc);
    if (st == HOLO_OK) st = dalloc(p, &p->Ut, sizeof(float2) * LL * nz * Bc);
    if (st != HOLO_OK) return st;
  }
  // Hq[k][j][ax][f] = h_{omega_j}[f] r_{s^p_kj,ax}[f] / L  (O3 x O4 per axis; the 1/L of the inverse DFT)
  std::vector<float2> H((size_t)K * nz * 2 * L);
  for (int j = 0; j < nz; j++) {
    const auto h = transfer(L, p->g.wavelength, p->p0, p->omega[j]);
    for (int k = 0; k < K; k++)
      for (int ax = 0; ax < 2; ax++) {
        const double sv = s[((size_t)k * nz + j) * 2 + ax];
        float2 *dst = H.data() + (((size_t)k * nz + j) * 2 + ax) * L;
        for (int f = 0; f < L; f++) {
          const cd v = h[f] * expi2pi_frac(-(double)fbar(f, L) * sv / (double)L) / (double)L;
          dst[f] = make_float2((float)v.real(), (float)v.imag());
        }
      }
  }
  HC(cudaMemcpy(p->hq, H.data(), H.size() * sizeof(float2), cudaMemcpyHostToDevice));
  p->ps = true;
  return HOLO_OK;
}

holo_status holo_grad_ref(holo_plan *p, const void *q, const float *sqrt_dref, void *grad_q_part, double *sc,
                          uint32_t flags) {
  holo_status st = precheck(p);
  if (st != HOLO_OK) return st;
  if (!q || !sc || (p->n_ref > 0 && !sqrt_dref)) return fail(p, HOLO_EINVAL, "null pointer");
  HC(cudaMemsetAsync(sc, 0, sizeof(double), p->stream));
  const bool obj = (flags & HOLO_OBJECTIVE_ONLY) != 0, acc = (flags & HOLO_ACCUMULATE_Q) != 0;
  p->tau = (flags & HOLO_INTENSITY) ? 2.f : (float)p->tau_set;
  float2 *gq = obj ? nullptr : (float2 *)grad_q_part;
  if (p->n_ref == 0) {
    if (gq && !acc) HC(cudaMemsetAsync(gq, 0, sizeof(float2) * (size_t)p->L * p->L, p->stream));
    return HOLO_OK;
  }
  p->ops->ref_run(p, (const float2 *)q, sqrt_dref, gq, sc, acc);
  return postcheck(p);
}

holo_status holo_fwd_ref(holo_plan *p, const void *q, void *w) {
  holo_status st = precheck(p);
  if (st != HOLO_OK) return st;
  if (!q || (p->n_ref > 0 && !w)) return fail(p, HOLO_EINVAL, "null pointer");
  if (p->n_ref == 0) return HOLO_OK;
  p->ops->ref_fwd(p, (const float2 *)q, (float2 *)w);
  return postcheck(p);
}

holo_status holo_upsample2(holo_plan *p, const void *coarse, void *fine, int32_t count) {
  holo_status st = precheck(p);
  if (st != HOLO_OK) return st;
  if (count < 0 || (count > 0 && (!coarse || !fine))) return fail(p, HOLO_EINVAL, "bad upsample2 arguments");
  if (!p->ops->upsample2) return fail(p, HOLO_EUNSUPPORTED, "upsample2 needs a power-of-two npad");
  if (count == 0) return HOLO_OK;
  p->ops->upsample2(p, (const float2 *)coarse, (float2 *)fine, count);
  return postcheck(p);
}

namespace {
holo_status stage_impl(holo_plan *p, const float *host, float *dev, bool ref) {
  holo_status st = precheck(p);
  if (st != HOLO_OK) return st;
  p->stage_host = nullptr;
  p->stage_dev = nullptr;
  if (!host || !dev) return HOLO_OK;  // cancel
  const int nbatch = ref ? (p->n_ref + p->BR - 1) / p->BR : (p->K + p->B - 1) / p->B;
  if (nbatch == 0) return HOLO_OK;
  if (!p->copy_stream) {
    HC(cudaStreamCreateWithFlags(&p->copy_stream, cudaStreamNonBlocking));
    HC(cudaEventCreateWithFlags(&p->stage_start, cudaEventDisableTiming));
  }
  while ((int)p->stage_ev.size() < nbatch) {
    cudaEvent_t e;
    HC(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    p->stage_ev.push_back(e);
  }
  p->stage_host = host;
  p->stage_dev = dev;
  p->stage_ref = ref;
  return HOLO_OK;
}
}  // namespace

holo_status holo_stage_sqrt_d(holo_plan *p, const float *host_sqrt_d, float *dev_sqrt_d) {
  return stage_impl(p, host_sqrt_d, dev_sqrt_d, false);
}

holo_status holo_stage_sqrt_dref(holo_plan *p, const float *host_sqrt_dref, float *dev_sqrt_dref) {
  return stage_impl(p, host_sqrt_dref, dev_sqrt_dref, true);
}

holo_status holo_set_cg_fuse(holo_plan *p, int32_t on) {
  holo_status st = precheck(p);  // completes a pending update first
  if (st != HOLO_OK) return st;
  p->cg_fuse = on != 0;
  return HOLO_OK;
}

holo_status holo_set_fourier(holo_plan *p, int32_t on) {
  holo_status st = precheck(p);
  if (st != HOLO_OK) return st;
  if (on && !p->ops->dft2) return fail(p, HOLO_EUNSUPPORTED, "the Fourier-domain object state needs a power-of-two npad");
  p->fourier = on != 0;
  return HOLO_OK;
}

holo_status holo_fourier(holo_plan *p, const void *in, void *out, int32_t count, int32_t inverse) {
  holo_status st = precheck(p);
  if (st != HOLO_OK) return st;
  if (count < 0 || (count > 0 && (!in || !out))) return fail(p, HOLO_EINVAL, "bad holo_fourier arguments");
  if (!p->ops->dft2) return fail(p, HOLO_EUNSUPPORTED, "holo_fourier needs a power-of-two npad");
  if (count == 0) return HOLO_OK;
  if (p->K == 0) return fail(p, HOLO_EUNSUPPORTED, "holo_fourier needs a plan with angles (object-chain scratch)");
  p->ops->dft2(p, (const float2 *)in, (float2 *)out, count, inverse != 0);
  return postcheck(p);
}

holo_status holo_bin2(holo_plan *p, const float *fine, float *coarse, int32_t count) {
  holo_status st = precheck(p);
  if (st != HOLO_OK) return st;
  if (count < 0 || (count > 0 && (!fine || !coarse))) return fail(p, HOLO_EINVAL, "bad bin2 arguments");
  if (count == 0) return HOLO_OK;
  pbeg(p);
  k_bin2<<<1184, 256, 0, p->stream>>>(fine, coarse, p->N, (size_t)count);
  pend(p, HOLO_PASS_FILTER, 20.0 * count * (double)p->N * p->N, 0);
  return postcheck(p);
}

holo_status holo_init_probe(holo_plan *p, const float *sqrt_dref, void *q0) {
  holo_status st = precheck(p);
  if (st != HOLO_OK) return st;
  if (!q0 || (p->n_ref > 0 && !sqrt_dref)) return fail(p, HOLO_EINVAL, "null pointer");
  if (p->n_ref == 0) return fail(p, HOLO_EINVAL, "no reference frames (holo_set_ref_shifts)");
  p->ops->init_probe(p, sqrt_dref, (float2 *)q0);
  return postcheck(p);
}

holo_status holo_init_psi(holo_plan *p, const float *sqrt_d, const float *sqrt_dref, double delta_beta, void *psi0) {
  holo_status st = precheck(p);
  if (st != HOLO_OK) return st;
  if (!sqrt_d || !sqrt_dref || !psi0) return fail(p, HOLO_EINVAL, "null pointer");
  if (!(delta_beta > 0) || !std::isfinite(delta_beta)) return fail(p, HOLO_EINVAL, "delta_beta must be > 0");
  if (p->K == 0) return HOLO_OK;
  if (!p->ops->init_psi) return fail(p, HOLO_EUNSUPPORTED, "init_psi needs a power-of-two npad");
  p->ops->init_psi(p, sqrt_d, sqrt_dref, delta_beta, (float2 *)psi0);
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
  if (psi && eta_psi && psi_trial && (grad_psi || mode == 2) && p->K > 0) {
    p->cg_psi = (const float2 *)psi;
    p->cg_g = (const float2 *)grad_psi;
    p->cg_eta = (float2 *)eta_psi;
    p->cg_trial = (float2 *)psi_trial;
    p->cg_rho = (float)in->rho_psi;
    p->cg_beta = (float)beta;
    p->cg_gamma = (float)in->gamma;
    p->cg_mode = mode;
    p->cg_pending = true;
    if (!p->cg_fuse) holo_cg_flush(p);  // otherwise the next sweep at psi_trial runs it inside X1
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
