// C ABI of strom_b200 (include/strom_b200.h): handle management, template
// dispatch over (law, p, volume rule, face rule), launch configuration.
#include <cuda_runtime.h>
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>
#include "../../include/strom_b200.h"
#include "element_kernels.cuh"
#include "derivs_warp.cuh"
#include "lm_kernels.cuh"

using namespace strom;

static thread_local std::string g_err;

static int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define CK(x)                                                                      \
  do {                                                                             \
    cudaError_t _e = (x);                                                          \
    if (_e != cudaSuccess) return fail(-2, std::string(#x ": ") + cudaGetErrorString(_e)); \
  } while (0)

struct strom_handle {
  int device = 0;
  int ne = 0, nv = 0;
  const int* elem_nodes = nullptr;
  const double* nodes = nullptr;
  const int* nbr = nullptr;
  const uint8_t* finfo = nullptr;
  strom_law_desc law{};
  int p = 0, nb = 0, nq = 0, ns = 0, nf = 0;
  std::vector<double> phi, dphi, wq, bary, trace, ws;
  double wsum = 0.0;
  double kappa = 1.0, eps = 1e-8;
  double* eta_ref = nullptr;
  const double *Phi = nullptr, *Psi = nullptr, *xref = nullptr, *u0 = nullptr;
  int ku = 0, kx = 0;
  double* part = nullptr;
  size_t part_cap = 0;
  int* degen_fill = nullptr;
  int* degen_list = nullptr;
  int degen_cap = 0;
  int* degen_scratch = nullptr;
  int degen_scratch_cap = 0;
  std::vector<std::vector<int>> last_degen;
  int num_sms = 148;
  LmWork lm;
  // benchmark probe
  bool prof = false;
  std::vector<cudaEvent_t> ev;
  int nprof = 0;
};

static void prof_mark(strom_handle* h, cudaStream_t st, int which) {
  if (!h->prof) return;
  const int i = 2 * h->nprof + which;
  if (i >= (int)h->ev.size()) return;
  cudaEventRecord(h->ev[i], st);
  if (which == 1) ++h->nprof;
}

extern "C" int strom_profile(strom_handle* h, int32_t enable) {
  if (!h) return fail(-1, "null handle");
  if (enable && h->ev.empty()) {
    h->ev.resize(2 * 4096);
    for (auto& e : h->ev) CK(cudaEventCreate(&e));
  }
  h->prof = enable != 0;
  h->nprof = 0;
  return 0;
}

extern "C" double strom_profile_ms(strom_handle* h, int32_t* launches) {
  if (!h) return -1.0;
  double ms = 0.0;
  int n = std::min(h->nprof, (int)h->ev.size() / 2);
  for (int i = 0; i < n; ++i) {
    float t = 0.f;
    cudaEventSynchronize(h->ev[2 * i + 1]);
    cudaEventElapsedTime(&t, h->ev[2 * i], h->ev[2 * i + 1]);
    ms += t;
  }
  if (launches) *launches = n;
  return ms;
}

extern "C" const char* strom_last_error(void) { return g_err.c_str(); }

static int ensure_part(strom_handle* h, size_t n) {
  if (n <= h->part_cap) return 0;
  if (h->part) cudaFree(h->part);
  h->part = nullptr;
  CK(cudaMalloc(&h->part, n * sizeof(double)));
  h->part_cap = n;
  return 0;
}

static int ensure_degen(strom_handle* h, int P) {
  if (P > h->degen_scratch_cap) {
    if (h->degen_scratch) cudaFree(h->degen_scratch);
    CK(cudaMalloc(&h->degen_scratch, sizeof(int) * P));
    h->degen_scratch_cap = P;
  }
  return 0;
}

extern "C" int strom_create(const strom_mesh_desc* mesh, const strom_law_desc* law, const strom_quad_desc* quad,
                            const strom_dist_desc* dist, int device, strom_handle** out) {
  if (!mesh || !law || !quad || !dist || !out) return fail(-1, "null argument");
  if (quad->p < 1 || quad->p > 2) return fail(-1, "solution degree must be 1 or 2");
  if (law->n_comp < 1 || law->n_comp > 4) return fail(-1, "n_comp out of range");
  if (law->n_mu > NMU) return fail(-1, "too many parameters per mu");
  if (dist->kappa <= 0.0 || dist->eps <= 0.0) return fail(-1, "kappa and eps must be positive");
  CK(cudaSetDevice(device));
  auto* h = new strom_handle();
  h->device = device;
  h->ne = mesh->num_elements;
  h->nv = mesh->num_nodes;
  h->elem_nodes = mesh->elem_nodes;
  h->nodes = mesh->nodes;
  h->nbr = mesh->nbr_elem;
  h->finfo = mesh->face_info;
  h->law = *law;
  h->p = quad->p; h->nb = quad->nb; h->nq = quad->nq; h->ns = quad->ns; h->nf = quad->nf;
  h->phi.assign(quad->phi, quad->phi + quad->nq * quad->nb);
  h->dphi.assign(quad->dphi, quad->dphi + quad->nq * quad->nb * 2);
  h->wq.assign(quad->wq, quad->wq + quad->nq);
  h->bary.assign(quad->bary, quad->bary + quad->nq * 3);
  h->trace.assign(quad->trace, quad->trace + 3 * quad->ns * quad->nf);
  h->ws.assign(quad->ws, quad->ws + quad->ns);
  h->wsum = 0.0;
  for (double v : h->wq) h->wsum += v;
  h->kappa = dist->kappa;
  h->eps = dist->eps;
  cudaDeviceGetAttribute(&h->num_sms, cudaDevAttrMultiProcessorCount, device);
  if (h->ne > 0) {
    if (cudaMalloc(&h->eta_ref, sizeof(double) * h->ne) != cudaSuccess) { delete h; return fail(-2, "eta_ref alloc"); }
    eta_ref_kernel<<<(h->ne + 127) / 128, 128>>>(h->ne, h->elem_nodes, h->nodes, h->wsum, h->eps, h->eta_ref);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) { delete h; return fail(-2, cudaGetErrorString(e)); }
  }
  h->degen_cap = std::max(1024, h->ne);
  if (cudaMalloc(&h->degen_list, sizeof(int) * 2 * h->degen_cap) != cudaSuccess ||
      cudaMalloc(&h->degen_fill, sizeof(int)) != cudaSuccess) {
    delete h;
    return fail(-2, "degenerate list alloc");
  }
  *out = h;
  return 0;
}

extern "C" int strom_set_bases(strom_handle* h, const double* phi, int32_t ku, const double* psi, int32_t kx,
                               const double* ref_coords, const double* state_offset) {
  if (!h) return fail(-1, "null handle");
  if (ku < 0 || kx < 0 || kx > KXMAX || ku + kx > KMAX) return fail(-1, "k_u + k_x must be <= 40 and k_x <= 16");
  if (ku > DERIV_THREADS) return fail(-1, "k_u too large");
  if ((ku && !phi) || (kx && !psi) || !ref_coords) return fail(-1, "missing basis pointer");
  h->Phi = phi; h->ku = ku; h->Psi = psi; h->kx = kx; h->xref = ref_coords; h->u0 = state_offset;
  return 0;
}

template <int NB, int NQ, int NS, int NF>
static void fill_tabs(const strom_handle* h, Tabs<NB, NQ, NS, NF>& t) {
  for (int q = 0; q < NQ; ++q) {
    for (int n = 0; n < NB; ++n) {
      t.phi[q][n] = h->phi[q * NB + n];
      t.dphi[q][n][0] = h->dphi[(q * NB + n) * 2 + 0];
      t.dphi[q][n][1] = h->dphi[(q * NB + n) * 2 + 1];
    }
    t.wq[q] = h->wq[q];
    for (int g = 0; g < 3; ++g) t.bary[q][g] = h->bary[q * 3 + g];
  }
  for (int f = 0; f < 3; ++f)
    for (int s = 0; s < NS; ++s)
      for (int j = 0; j < NF; ++j) t.trace[f][s][j] = h->trace[(f * NS + s) * NF + j];
  for (int s = 0; s < NS; ++s) t.ws[s] = h->ws[s];
  t.wsum = h->wsum;
  for (int f = 0; f < 3; ++f)
    for (int j = 0; j < NF; ++j) t.fnode[f][j] = fnode_of(NB == 3 ? 1 : 2, f, j);
}

struct EvalArgs {
  int mode;
  const double *w, *tau, *mu;
  int P;
  const int* active;
  const double* rho;
  int A;
  double* out;
  int* degen;
  cudaStream_t stream;
};

template <class LAW, int NB, int NQ, int NS, int TPU>
static int launch_warp(strom_handle* h, const EvalArgs& a, Params<NB, NQ, NS, WShape<LAW, NB, NQ, NS>::NF>& prm,
                       int nunits) {
  using SH = WShape<LAW, NB, NQ, NS>;
  Run& r = prm.r;
  constexpr int UPW = 32 / TPU;
  r.U = UPW;
  r.unit_stride = SH::unit_stride(r.LDJ);
  r.gx_warp_stride = SH::warp_stride(r.LDJ, r.KP, UPW);
  const int smem_cap = 227 * 1024;
  const size_t warp_bytes = (size_t)r.gx_warp_stride * sizeof(double);
  int nwarps = std::min<int>(WTHREADS / 32, (int)(smem_cap / warp_bytes));
  if (nwarps < 1) return fail(-1, "element group does not fit in shared memory");
  const size_t smem = nwarps * warp_bytes;
  auto kern = derivs_warp_kernel<LAW, NB, NQ, NS, TPU>;
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int per_sm = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, nwarps * 32, smem));
  per_sm = std::max(per_sm, 1);
  const int ngroups = (nunits + UPW - 1) / UPW;
  const int target = h->num_sms * per_sm;
  const int maxb = std::max(1, (ngroups + nwarps - 1) / nwarps);
  int gx = std::max(1, std::min(maxb, (target + a.P - 1) / a.P));
  r.gx = gx;
  r.ntiles = ngroups;
  const int PSZ = 1 + r.K + r.KP * r.KP;
  if (a.mode == MODE_DERIVS) {
    if (ensure_part(h, (size_t)a.P * gx * PSZ)) return -2;
    r.part = h->part;
  }
  prof_mark(h, a.stream, 0);
  kern<<<dim3(gx, a.P), nwarps * 32, smem, a.stream>>>(prm);
  prof_mark(h, a.stream, 1);
  CK(cudaGetLastError());
  if (a.mode == MODE_DERIVS) {
    const int OSZ = 1 + r.K + r.K * r.K;
    finalize_derivs_kernel<<<dim3((OSZ + 127) / 128, a.P), 128, 0, a.stream>>>(h->part, gx, r.K, r.KP, a.P, a.out);
    CK(cudaGetLastError());
  }
  return 0;
}

template <class LAW, int NB, int NQ, int NS>
static int eval_impl(strom_handle* h, const EvalArgs& a) {
  using SH = Shape<LAW, NB, NQ, NS>;
  constexpr int NF = SH::NF;
  Params<NB, NQ, NS, NF> prm;
  fill_tabs<NB, NQ, NS, NF>(h, prm.t);
  Run& r = prm.r;
  memset(&r, 0, sizeof(r));
  r.ne = h->ne; r.elem_nodes = h->elem_nodes; r.nodes = h->nodes; r.nbr = h->nbr; r.finfo = h->finfo;
  r.eta_ref = h->eta_ref;
  r.phi = h->Phi; r.psi = h->Psi; r.xref = h->xref; r.u0 = h->u0; r.ku = h->ku; r.kx = h->kx;
  r.K = h->ku + h->kx;
  r.KP = (r.K + 7) / 8 * 8;
  if (r.KP < 8) r.KP = 8;
  r.LDJ = (r.KP % 16 == 0) ? r.KP + 8 : r.KP;
  r.w = a.w; r.tau = a.tau; r.mu = a.mu; r.nmu = h->law.n_mu; r.P = a.P;
  r.active = a.active; r.rho = a.rho; r.A = a.A;
  r.out = a.out;
  r.degen = a.degen; r.degen_list = h->degen_list; r.degen_cap = h->degen_cap; r.degen_fill = h->degen_fill;
  r.mode = a.mode;
  r.kappa = h->kappa; r.eps = h->eps;
  for (int i = 0; i < 8; ++i) r.lawp[i] = h->law.params[i];
  const int nunits = a.active ? a.A : h->ne;
  if (nunits == 0) return 0;
  if (a.mode == MODE_OBJECTIVE || a.mode == MODE_RESNORM2 || a.mode == MODE_RESIDUAL) {
    const int gx = (nunits + 127) / 128;
    if (a.mode != MODE_RESIDUAL) {
      if (ensure_part(h, (size_t)a.P * gx)) return -2;
      r.part = h->part;
    }
    prof_mark(h, a.stream, 0);
    value_kernel<LAW, NB, NQ, NS><<<dim3(gx, a.P), 128, 0, a.stream>>>(prm);
    prof_mark(h, a.stream, 1);
    CK(cudaGetLastError());
    if (a.mode != MODE_RESIDUAL) {
      sum_partials_kernel<<<(a.P + 127) / 128, 128, 0, a.stream>>>(h->part, gx, a.P, a.out);
      CK(cudaGetLastError());
    }
    return 0;
  }
  if (h->ku < 1) return fail(-1, "derivative modes need k_u >= 1");
  if (h->ku > 32) return fail(-1, "derivative modes need k_u <= 32");
  if (h->ku <= 16) return launch_warp<LAW, NB, NQ, NS, 16>(h, a, prm, nunits);
  return launch_warp<LAW, NB, NQ, NS, 32>(h, a, prm, nunits);
}

template <class LAW>
static int dispatch_shape(strom_handle* h, const EvalArgs& a) {
  if (h->nb == 6 && h->nq == 12 && h->ns == 4) return eval_impl<LAW, 6, 12, 4>(h, a);
  if (h->nb == 6 && h->nq == 25 && h->ns == 4) return eval_impl<LAW, 6, 25, 4>(h, a);
  if (h->nb == 3 && h->nq == 7 && h->ns == 3) return eval_impl<LAW, 3, 7, 3>(h, a);
  return fail(-1, "no compiled kernel for (p, n_q, n_s) = (" + std::to_string(h->p) + ", " + std::to_string(h->nq) +
                      ", " + std::to_string(h->ns) + ")");
}

static int dispatch(strom_handle* h, const EvalArgs& a) {
  switch (h->law.law_id) {
    case 0: return dispatch_shape<LinAdv>(h, a);
    case 1: return dispatch_shape<BurgersST>(h, a);
    case 2: return dispatch_shape<BurgersStrip>(h, a);
    case 3: return dispatch_shape<Euler>(h, a);
    default: return fail(-1, "unknown law id");
  }
}

extern "C" int strom_reserve(strom_handle* h, int32_t max_P, int32_t max_active) {
  if (!h) return fail(-1, "null handle");
  const int K = h->ku + h->kx, KP = std::max(8, (K + 7) / 8 * 8);
  const size_t PSZ = 1 + K + (size_t)KP * KP;
  size_t need = std::max((size_t)(h->num_sms * 16 + max_P) * PSZ, (size_t)max_P * ((max_active + 127) / 128 + 1));
  if (ensure_part(h, need)) return -2;
  if (ensure_degen(h, max_P)) return -2;
  return 0;
}

static int collect_degen(strom_handle* h, int P, int* degen, cudaStream_t st) {
  std::vector<int> cnt(P);
  CK(cudaMemcpyAsync(cnt.data(), degen, sizeof(int) * P, cudaMemcpyDeviceToHost, st));
  int fill = 0;
  CK(cudaMemcpyAsync(&fill, h->degen_fill, sizeof(int), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  h->last_degen.assign(P, {});
  bool any = false;
  for (int p = 0; p < P; ++p) any |= cnt[p] > 0;
  if (!any) return 0;
  fill = std::min(fill, h->degen_cap);
  std::vector<int> lst(2 * (size_t)fill);
  CK(cudaMemcpy(lst.data(), h->degen_list, sizeof(int) * 2 * fill, cudaMemcpyDeviceToHost));
  for (int i = 0; i < fill; ++i) h->last_degen[lst[2 * i]].push_back(lst[2 * i + 1]);
  for (auto& v : h->last_degen) {
    std::sort(v.begin(), v.end());
    v.erase(std::unique(v.begin(), v.end()), v.end());
  }
  return 1;
}

extern "C" int strom_eval(strom_handle* h, int32_t mode, const double* w, const double* tau, const double* mu,
                          int32_t P, const int32_t* active, const double* rho, int32_t A, double* out,
                          int32_t* degen, void* stream, int32_t sync) {
  if (!h) return fail(-1, "null handle");
  if (mode < 0 || mode > MODE_CONTRIB_LPROWS) return fail(-1, "bad mode");
  if (P < 1) return fail(-1, "P must be >= 1");
  if (!out) return fail(-1, "null output");
  if (!h->xref) return fail(-1, "bases not set");
  if ((h->ku && !w) || (h->kx && !tau) || (h->law.n_mu && !mu)) return fail(-1, "null coordinates");
  if (active && (!rho || A < 0)) return fail(-1, "active set needs weights");
  if (active && (mode == MODE_CONTRIB || mode == MODE_CONTRIB_SPLIT || mode == MODE_CONTRIB_LPROWS))
    return fail(-1, "element contributions are evaluated over all elements");
  cudaStream_t st = (cudaStream_t)stream;
  if (!degen) {
    if (ensure_degen(h, P)) return -2;
    degen = h->degen_scratch;
  }
  CK(cudaMemsetAsync(degen, 0, sizeof(int) * P, st));
  CK(cudaMemsetAsync(h->degen_fill, 0, sizeof(int), st));
  EvalArgs a{mode, w, tau, mu, P, active, rho, A, out, degen, st};
  int rc = dispatch(h, a);
  if (rc) return rc;
  if (sync) return collect_degen(h, P, degen, st);
  return 0;
}

extern "C" int strom_degenerate_elements(strom_handle* h, int32_t p, int32_t* ids, int32_t cap) {
  if (!h || p < 0 || p >= (int)h->last_degen.size()) return 0;
  const auto& v = h->last_degen[p];
  int n = std::min<int>(cap, (int)v.size());
  for (int i = 0; i < n; ++i) ids[i] = v[i];
  return (int)v.size();
}

extern "C" void strom_destroy(strom_handle* h) {
  if (!h) return;
  cudaSetDevice(h->device);
  if (h->eta_ref) cudaFree(h->eta_ref);
  if (h->part) cudaFree(h->part);
  if (h->degen_list) cudaFree(h->degen_list);
  if (h->degen_fill) cudaFree(h->degen_fill);
  if (h->degen_scratch) cudaFree(h->degen_scratch);
  lm_free(h->lm);
  for (auto& e : h->ev) cudaEventDestroy(e);
  delete h;
}

#include "lm_capi.inc"
