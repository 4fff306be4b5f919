// Template launchers for one conservation law (included by the per-law units).
#pragma once
#include "handle.h"
#include "derivs_warp.cuh"
#include "derivs_mma.cuh"
#include "value_mma.cuh"
#include <cstdlib>
#include <cstdio>

namespace strom_host {
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
  for (int j = 0; j < NF; ++j)
    for (int jp = 0; jp < NF; ++jp)
      for (int s = 0; s < NS; ++s) t.t2[j][jp][s] = t.trace[0][s][j] * t.trace[0][s][jp];
  t.wsum = h->wsum;
  for (int f = 0; f < 3; ++f)
    for (int j = 0; j < NF; ++j) t.fnode[f][j] = fnode_of(NB == 3 ? 1 : 2, f, j);
}


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
  static size_t c_smem = 0;
  static int c_dev = -1, c_per_sm = 0;
  if (c_smem != smem || c_dev != h->device) {
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&c_per_sm, kern, nwarps * 32, smem));
    c_smem = smem;
    c_dev = h->device;
  }
  int per_sm = c_per_sm;
  if (getenv("STROM_DEBUG")) {
    cudaFuncAttributes fa;
    CK(cudaFuncGetAttributes(&fa, kern));
    fprintf(stderr, "[strom] mma kernel attrs: %d regs, %zu B static smem, max dyn %d\n", fa.numRegs, fa.sharedSizeBytes,
            fa.maxDynamicSharedSizeBytes);
  }
  per_sm = std::max(per_sm, 1);
  const int ngroups = (nunits + UPW - 1) / UPW;
  const int target = h->num_sms * per_sm;
  const int maxb = std::max(1, (ngroups + nwarps - 1) / nwarps);
  const int live = a.live > 0 ? a.live : a.P;
  int gx = std::max(1, std::min(maxb, (target + live - 1) / live));
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
    finalize_derivs_kernel<<<dim3((1 + r.K + r.KP * r.KP + 31) / 32, a.P), std::min(1024, 32 * std::max(1, std::min(32, gx))),
                             0, a.stream>>>(h->part, gx, r.K, r.KP, a.P, a.out, a.mask);
    CK(cudaGetLastError());
  }
  return 0;
}

template <class LAW, int NQ, int KUT, int KXT>
static int launch_mma_t(strom_handle* h, const EvalArgs& a, Params<6, NQ, 4, 3>& prm, int nunits) {
  using SH = MShape<NQ>;
  Run& r = prm.r;
  r.LDJ = r.KP + 4;  // == 4 mod 8 doubles: conflict-free half-warp fragment loads
  r.U = 1;
  r.unit_stride = 0;
  r.gx_warp_stride = SH::warp_stride(r.LDJ, r.KP, r.kx, SH::hreg(KUT, KXT), SH::phibuf(KUT));
  const int smem_cap = 227 * 1024;
  const size_t warp_bytes = (size_t)r.gx_warp_stride * sizeof(double);
  int nwarps = std::min<int>(2, (int)(smem_cap / warp_bytes));  // 2-warp CTAs (measured fastest)
  if (const char* ev = getenv("STROM_MMA_WARPS")) nwarps = std::max(1, std::min(nwarps, atoi(ev)));
  if (nwarps < 1) return fail(-1, "element does not fit in shared memory");
  const size_t smem = nwarps * warp_bytes;
  auto kern = KUT > 0 ? (a.mode == MODE_DERIVS ? derivs_mma_kernel<LAW, NQ, KUT, KXT, 1> : derivs_mma_kernel<LAW, NQ, KUT, KXT, 0>)
                      : derivs_mma_kernel<LAW, NQ, KUT, KXT>;
  // attribute + occupancy query once per (kernel, shared-memory size, device): host API
  // calls on every launch dominate the small LM rounds
  const int ck = (KUT > 0 && a.mode == MODE_DERIVS) ? 1 : 0;  // one cache slot per kernel variant
  static size_t c_smem[2] = {0, 0};
  static int c_dev[2] = {-1, -1}, c_per_sm[2] = {0, 0};
  if (c_smem[ck] != smem || c_dev[ck] != h->device) {
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    if (const char* ev = getenv("STROM_MMA_CARVEOUT"))  // experiment knob: shared-memory carveout (%)
      CK(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, atoi(ev)));
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&c_per_sm[ck], kern, nwarps * 32, smem));
    c_smem[ck] = smem;
    c_dev[ck] = h->device;
  }
  int per_sm = c_per_sm[ck];
  if (getenv("STROM_DEBUG")) {
    cudaFuncAttributes fa;
    CK(cudaFuncGetAttributes(&fa, kern));
    fprintf(stderr, "[strom] mma kernel attrs: %d regs, %zu B static smem, max dyn %d\n", fa.numRegs, fa.sharedSizeBytes,
            fa.maxDynamicSharedSizeBytes);
  }
  per_sm = std::max(per_sm, 1);
  // k_u > 16: the larger per-warp footprint leaves too little L1 for the basis rows above
  // 8 warps/SM (measured: cfg3/4/5 fastest at 4 two-warp CTAs per SM; cfg2 at 6)
  if (r.ku > 16) per_sm = std::min(per_sm, 4);
  if (const char* ev = getenv("STROM_MMA_BPS")) per_sm = std::max(1, std::min(per_sm, atoi(ev)));  // blocks/SM cap
  const int target = h->num_sms * per_sm;
  const int maxb = std::max(1, (nunits + nwarps - 1) / nwarps);
  const int live = a.live > 0 ? a.live : a.P;
  // one wave: at most `target` co-resident CTAs (a partial second wave doubles the pass time)
  int gx = std::max(1, std::min(maxb, target / live));
  if (const char* ev = getenv("STROM_MMA_UPW")) {  // experiment knob: at least this many units per warp
    const int upw = std::max(1, atoi(ev));
    gx = std::max(1, std::min(gx, (nunits + nwarps * upw - 1) / (nwarps * upw)));
  }
  r.gx = gx;
  r.ntiles = nunits;
  if (getenv("STROM_DEBUG"))
    fprintf(stderr, "[strom] mma kernel: %d warps/CTA, %zu B smem/CTA, %d CTAs/SM, grid %d x %d\n", nwarps, smem, per_sm,
            gx, a.P);
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
    finalize_derivs_kernel<<<dim3((1 + r.K + r.KP * r.KP + 31) / 32, a.P), std::min(1024, 32 * std::max(1, std::min(32, gx))),
                             0, a.stream>>>(h->part, gx, r.K, r.KP, a.P, a.out, a.mask);
    CK(cudaGetLastError());
  }
  return 0;
}

template <class LAW, int NQ>
static int launch_mma(strom_handle* h, const EvalArgs& a, Params<6, NQ, 4, 3>& prm, int nunits) {
  // compile-time reduced dimensions for the BASELINE configs (addressing folds to immediates)
  if (!getenv("STROM_GENERIC_K")) {
    if (h->ku == 16 && h->kx == 8) return launch_mma_t<LAW, NQ, 16, 8>(h, a, prm, nunits);
    if (h->ku == 20 && h->kx == 10) return launch_mma_t<LAW, NQ, 20, 10>(h, a, prm, nunits);
    if (h->ku == 24 && h->kx == 12) return launch_mma_t<LAW, NQ, 24, 12>(h, a, prm, nunits);
  }
  return launch_mma_t<LAW, NQ, 0, 0>(h, a, prm, nunits);
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
  r.phi = h->Phi; r.psi = h->Psi; r.xref = h->xref; r.u0 = h->u0; r.u0_stride = h->u0_stride; r.x_stride = h->x_stride; r.ku = h->ku; r.kx = h->kx;
  r.K = h->ku + h->kx;
  r.KP = (r.K + 7) / 8 * 8;
  if (r.KP < 8) r.KP = 8;
  r.LDJ = (r.KP % 16 == 0) ? r.KP + 8 : r.KP;
  r.w = a.w; r.tau = a.tau; r.mu = a.mu; r.nmu = h->law.n_mu; r.P = a.P;
  r.active = a.active; r.rho = a.rho; r.A = a.A;
  r.out = a.out;
  r.degen = a.degen; r.degen_list = h->degen_list; r.degen_cap = h->degen_cap; r.degen_fill = h->degen_fill;
  r.mode = a.mode;
  r.mask = a.mask;
  r.kappa = h->kappa; r.eps = h->eps;
  for (int i = 0; i < 8; ++i) r.lawp[i] = h->law.params[i];
  const int nunits = a.active ? a.A : h->ne;
  if (nunits == 0) {
    size_t n = 0;
    if (a.mode == MODE_OBJECTIVE || a.mode == MODE_RESNORM2) n = a.P;
    if (a.mode == MODE_DERIVS) n = (size_t)a.P * (1 + r.K + r.K * r.K);
    if (n) CK(cudaMemsetAsync(a.out, 0, n * sizeof(double), a.stream));
    return 0;
  }
  if (a.mode == MODE_OBJECTIVE || a.mode == MODE_RESNORM2 || a.mode == MODE_RESIDUAL) {
    const bool multi = a.P >= 8;  // many parameter points: warp per element, lanes over mu
    const bool listed = multi && a.list != nullptr && a.live > 0;  // lanes over the compacted enabled rows
    if (listed) { r.list = a.list; r.nlist = a.live; }
    const int gy = multi ? ((listed ? a.live : a.P) + 31) / 32 : a.P;
    const int gx = multi ? std::max(1, std::min((nunits + 3) / 4, (h->num_sms * 16 + gy - 1) / gy)) : (nunits + 127) / 128;
    if (a.mode != MODE_RESIDUAL) {
      if (ensure_part(h, (size_t)a.P * gx)) return -2;
      r.part = h->part;
    }
    prof_mark(h, a.stream, 0);
    static const bool old_value = getenv("STROM_VALUE_OLD") != nullptr;
    if (multi && h->ku <= 32 && !old_value) {
      using VS = VShape<LAW, NB>;
      constexpr int vsmem = (VM_THREADS / 32) * VS::TILE * sizeof(double);
      static int c_dev = -1;
      if (c_dev != h->device) {
        CK(cudaFuncSetAttribute(value_mma_kernel<LAW, NB, NQ, NS>, cudaFuncAttributeMaxDynamicSharedMemorySize, vsmem));
        c_dev = h->device;
      }
      value_mma_kernel<LAW, NB, NQ, NS><<<dim3(gy, gx), VM_THREADS, vsmem, a.stream>>>(prm);
    } else if (multi)
      value_mu_kernel<LAW, NB, NQ, NS><<<dim3(gx, gy), 128, 0, a.stream>>>(prm);
    else
      value_kernel<LAW, NB, NQ, NS><<<dim3(gx, a.P), 128, 0, a.stream>>>(prm);
    prof_mark(h, a.stream, 1);
    CK(cudaGetLastError());
    if (a.mode != MODE_RESIDUAL) {
      sum_partials_kernel<<<(a.P + 3) / 4, 128, 0, a.stream>>>(h->part, gx, a.P, a.out, a.mask);
      CK(cudaGetLastError());
    }
    return 0;
  }
  if (h->ku < 1) return fail(-1, "derivative modes need k_u >= 1");
  if (h->ku > 32) return fail(-1, "derivative modes need k_u <= 32");
  if constexpr (LAW::M == 4 && NB == 6 && NS == 4) {
    if (!h->force_warp_kernel) return launch_mma<LAW, NQ>(h, a, prm, nunits);
  }
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


}  // namespace strom_host
