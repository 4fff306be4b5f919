// C ABI of strom_b200 (include/strom_b200.h): handle management, dispatch,
// benchmark probe and the batched LM host loop.
#include <cstdio>
#include "handle.h"
#include "lm_kernels.cuh"

using namespace strom;
using namespace strom_host;

static thread_local std::string g_err;

namespace strom_host {
int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}
int ensure_part(strom_handle* h, size_t n) {
  if (n <= h->part_cap) return 0;
  if (h->part) cudaFree(h->part);
  h->part = nullptr;
  CK(cudaMalloc(&h->part, n * sizeof(double)));
  h->part_cap = n;
  return 0;
}

void prof_mark(strom_handle* h, cudaStream_t st, int which) {
  if (!h->prof) return;
  const int i = 2 * h->nprof + which;
  if (i >= (int)h->ev.size()) return;
  cudaEventRecord(h->ev[i], st);
  if (which == 1) ++h->nprof;
}

}  // namespace strom_host

static int dispatch(strom_handle* h, const EvalArgs& a) {
  switch (h->law.law_id) {
    case 0: return eval_linadv(h, a);
    case 1: return eval_burgers_st(h, a);
    case 2: return eval_strip(h, a);
    case 3: return eval_euler(h, a);
    case 4: return eval_euler_roe(h, a);
    case 5: return eval_euler_wall(h, a);
    case 6: return eval_linadv_ms(h, a);
    default: return fail(-1, "unknown law id");
  }
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
  if (h->ne > 0) {  // slip walls present? (their Jacobians exist on the DMMA path only)
    std::vector<uint8_t> fi((size_t)h->ne * 3);
    if (cudaMemcpy(fi.data(), h->finfo, fi.size(), cudaMemcpyDeviceToHost) != cudaSuccess) {
      delete h;
      return fail(-2, "face info read");
    }
    for (uint8_t v : fi) h->has_wall |= (v >> 3) == BC_REFLECT;
  }
  // slip walls need a wall-capable Euler instantiation: 4 (Roe) or 5 (LLF with walls)
  if (h->has_wall && law->law_id != 4 && law->law_id != 5) { delete h; return fail(-1, "slip walls need law id 4 or 5"); }
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
  h->u0_stride = 0; h->x_stride = 0;
  h->epoch++;
  return 0;
}

extern "C" int strom_set_offsets(strom_handle* h, const double* state_offset, int64_t state_stride,
                                 const double* ref_coords, int64_t coord_stride) {
  if (!h || !ref_coords) return fail(-1, "strom_set_offsets: null argument");
  if (state_stride < 0 || coord_stride < 0) return fail(-1, "strom_set_offsets: negative stride");
  h->u0 = state_offset; h->u0_stride = state_offset ? state_stride : 0;
  h->xref = ref_coords; h->x_stride = coord_stride;
  h->epoch++;
  return 0;
}

extern "C" int strom_set_test_space(strom_handle* h, int32_t nbt, const double* phi, const double* dphi,
                                    const double* trace) {
  if (!h) return fail(-1, "null handle");
  if (nbt < 1 || nbt > 64 || !phi || !dphi || !trace) return fail(-1, "strom_set_test_space: bad arguments");
  CK(cudaSetDevice(h->device));
  if (h->test_tab) {
    CK(cudaDeviceSynchronize());  // an asynchronous evaluation may still read the previous table
    cudaFree(h->test_tab);
  }
  h->test_tab = nullptr;
  const size_t nd = (size_t)h->nq * nbt * 2, nt = (size_t)3 * h->ns * nbt, np = (size_t)h->nq * nbt;
  CK(cudaMalloc(&h->test_tab, (nd + nt + np) * sizeof(double)));  // [dphi | trace | phi]
  CK(cudaMemcpy(h->test_tab, dphi, nd * sizeof(double), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(h->test_tab + nd, trace, nt * sizeof(double), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(h->test_tab + nd + nt, phi, np * sizeof(double), cudaMemcpyHostToDevice));
  h->test_nb = nbt;
  return 0;
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
  if (mode < 0 || mode > MODE_ELEMJAC_ENRICHED) return fail(-1, "bad mode");
  const bool ejmode = mode == MODE_ELEMJAC || mode == MODE_ELEMJAC_ENRICHED;
  if (ejmode && P != 1) return fail(-1, "element Jacobians: one parameter point");
  if (mode == MODE_ELEMJAC && (h->law.n_comp != 4 || h->p != 2))
    return fail(-1, "STROM_ELEMJAC: 4-component laws with p = 2 (other laws: STROM_ELEMJAC_ENRICHED with the trial space as the test space)");
  if (mode == MODE_ELEMJAC_ENRICHED && !h->test_tab) return fail(-1, "enriched element Jacobians: test space not set");
  if (P < 1) return fail(-1, "P must be >= 1");
  if (!out) return fail(-1, "null output");
  if (!h->xref) return fail(-1, "bases not set");
  if ((h->ku && !w) || (h->kx && !tau) || (h->law.n_mu && !mu)) return fail(-1, "null coordinates");
  if (active && (!rho || A < 0)) return fail(-1, "active set needs weights");
  if (active && (mode == MODE_CONTRIB || mode == MODE_CONTRIB_SPLIT || mode == MODE_CONTRIB_LPROWS || ejmode))
    return fail(-1, "element contributions are evaluated over all elements");
  cudaStream_t st = (cudaStream_t)stream;
  if (!degen) {
    if (ensure_degen(h, P)) return -2;
    degen = h->degen_scratch;
  }
  CK(cudaMemsetAsync(degen, 0, sizeof(int) * P, st));
  CK(cudaMemsetAsync(h->degen_fill, 0, sizeof(int), st));
  EvalArgs a{mode, nullptr, w, tau, mu, P, active, rho, A, out, degen, st};
  int rc = dispatch(h, a);
  if (rc) return rc;
  if (sync) return collect_degen(h, P, degen, st);
  return 0;
}

// One evaluation through HOST buffers (the public single-point API): the inputs are staged in
// pinned memory, copied with one asynchronous H2D, evaluated, and the result and the per-row
// degenerate counters come back with one D2H and one stream synchronisation.
extern "C" int strom_eval_host(strom_handle* h, int32_t mode, const double* w, const double* tau, const double* mu,
                               int32_t P, const int32_t* active, const double* rho, int32_t A, double* out,
                               int64_t out_n, int32_t* degen_out, void* stream) {
  if (!h || !out || out_n < 0 || P < 1) return fail(-1, "strom_eval_host: bad arguments");
  cudaStream_t st = (cudaStream_t)stream;
  const int nmu = h->law.n_mu;
  const size_t n_in = (size_t)P * (h->ku + h->kx + nmu);
  const size_t need = n_in + (size_t)out_n + (size_t)P;  // doubles: inputs, outputs, counters (as doubles)
  if (need > h->stage_cap) {
    if (h->stage_h) cudaFreeHost(h->stage_h);
    if (h->stage_d) cudaFree(h->stage_d);
    h->stage_h = nullptr;
    h->stage_d = nullptr;
    h->stage_cap = 0;
    CK(cudaMallocHost(&h->stage_h, need * sizeof(double)));
    CK(cudaMalloc(&h->stage_d, need * sizeof(double)));
    h->stage_cap = need;
  }
  double* hin = h->stage_h;
  double* din = h->stage_d;
  const size_t nw = (size_t)P * h->ku, nt = (size_t)P * h->kx, nm = (size_t)P * nmu;
  if (nw) memcpy(hin, w, nw * sizeof(double));
  if (nt) memcpy(hin + nw, tau, nt * sizeof(double));
  if (nm) memcpy(hin + nw + nt, mu, nm * sizeof(double));
  CK(cudaMemcpyAsync(din, hin, n_in * sizeof(double), cudaMemcpyHostToDevice, st));
  double* dout = din + n_in;
  int32_t* ddeg = reinterpret_cast<int32_t*>(dout + out_n);
  int rc = strom_eval(h, mode, nw ? din : nullptr, nt ? din + nw : nullptr, nm ? din + nw + nt : nullptr, P, active,
                      rho, A, dout, ddeg, st, 0);
  if (rc < 0) return rc;
  double* hout = hin + n_in;
  CK(cudaMemcpyAsync(hout, dout, ((size_t)out_n + P) * sizeof(double), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  memcpy(out, hout, (size_t)out_n * sizeof(double));
  const int32_t* hdeg = reinterpret_cast<const int32_t*>(hout + out_n);
  bool any = false;
  for (int p = 0; p < P; ++p) any |= hdeg[p] > 0;
  if (degen_out) memcpy(degen_out, hdeg, P * sizeof(int32_t));
  if (!any) return 0;
  // degenerate elements: re-run synchronously for their ids (rare path)
  return strom_eval(h, mode, nw ? din : nullptr, nt ? din + nw : nullptr, nm ? din + nw + nt : nullptr, P, active, rho,
                    A, dout, nullptr, st, 1);
}

extern "C" int strom_degenerate_elements(strom_handle* h, int32_t p, int32_t* ids, int32_t cap) {
  if (!h || p < 0 || p >= (int)h->last_degen.size()) return 0;
  const auto& v = h->last_degen[p];
  int n = std::min<int>(cap, (int)v.size());
  for (int i = 0; i < n; ++i) ids[i] = v[i];
  return (int)v.size();
}

static void lm_graph_free(strom_handle* h);  // lm_capi.inc

extern "C" void strom_destroy(strom_handle* h) {
  if (!h) return;
  cudaSetDevice(h->device);
  if (h->eta_ref) cudaFree(h->eta_ref);
  if (h->test_tab) cudaFree(h->test_tab);
  if (h->part) cudaFree(h->part);
  if (h->degen_list) cudaFree(h->degen_list);
  if (h->degen_fill) cudaFree(h->degen_fill);
  if (h->degen_scratch) cudaFree(h->degen_scratch);
  lm_graph_free(h);
  lm_free(h->lm);
  if (h->stage_h) cudaFreeHost(h->stage_h);
  if (h->stage_d) cudaFree(h->stage_d);
  if (h->lm_stream) cudaStreamDestroy(h->lm_stream);
  for (auto& e : h->ev) cudaEventDestroy(e);
  delete h;
}

#include "lm_capi.inc"
