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


// Launch a derivatives / contribution pass split into `gx` element chunks per parameter row
// (grid (gx, P), rows masked), or, for a device-sized pass (a.dyn_count: graph-resident LM
// rounds, row count read on the device), a 1-D grid of target + P CTAs that the kernel splits
// over the live rows with the same formula (dyn_gx); partials are indexed by the live slot, so
// their buffer is bounded by (target + P) * PSZ however few rows are live.
template <class KERN, class PRM>
static int launch_pass(strom_handle* h, const EvalArgs& a, KERN kern, PRM& prm, int nwarps, size_t smem, int target,
                       int maxb, int ceil_div) {
  Run& r = prm.r;
  const int PSZ = 1 + r.K + r.KP * r.KP;
  const bool dyn = a.dyn_count != nullptr;
  int gx = 0;
  dim3 grid;
  if (dyn) {
    r.dyn_count = a.dyn_count; r.list = a.list;
    r.dyn_target = target; r.dyn_maxb = maxb; r.dyn_ceil = ceil_div;
    grid = dim3(target + a.P);
  } else {
    gx = std::max(1, std::min(maxb, ceil_div ? (target + a.P - 1) / a.P : target / a.P));
    grid = dim3(gx, a.P);
  }
  r.gx = gx;
  if (a.mode == MODE_DERIVS) {
    const size_t need = dyn ? (size_t)(target + a.P) * PSZ : (size_t)a.P * gx * PSZ;
    if (dyn && need > h->part_cap) return fail(-2, "device-sized pass: partial buffer not reserved");
    if (ensure_part(h, need)) return -2;
    r.part = h->part;
  }
  if (!dyn) prof_mark(h, a.stream, 0);
  kern<<<grid, nwarps * 32, smem, a.stream>>>(prm);
  if (!dyn) prof_mark(h, a.stream, 1);
  CK(cudaGetLastError());
  if (a.mode == MODE_DERIVS) {
    const DynRows dr{a.dyn_count, a.list, target, maxb, ceil_div};
    const int fthreads = dyn ? 1024 : std::min(1024, 32 * std::max(1, std::min(32, gx)));
    finalize_derivs_kernel<<<dim3((PSZ + 31) / 32, a.P), fthreads, 0, a.stream>>>(h->part, gx, r.K, r.KP, a.P, a.out,
                                                                                  a.mask, dr);
    CK(cudaGetLastError());
  }
  return 0;
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
  const int per_sm = std::max(c_per_sm, 1);
  const int ngroups = (nunits + UPW - 1) / UPW;
  r.ntiles = ngroups;
  return launch_pass(h, a, kern, prm, nwarps, smem, h->num_sms * per_sm, std::max(1, (ngroups + nwarps - 1) / nwarps), 1);
}

template <class LAW, int NQ, int KUT, int KXT>
static int launch_mma_t(strom_handle* h, const EvalArgs& a, Params<6, NQ, 4, 3>& prm, int nunits) {
  using SH = MShape<NQ>;
  Run& r = prm.r;
  r.LDJ = r.KP + 4;  // == 4 mod 8 doubles: conflict-free half-warp fragment loads
  r.U = 1;
  r.unit_stride = 0;
  r.gx_warp_stride = SH::warp_stride(r.LDJ, r.KP, r.kx, SH::hreg(KUT, KXT));
  const int smem_cap = 227 * 1024;
  const size_t warp_bytes = (size_t)r.gx_warp_stride * sizeof(double);
  const int nwarps = std::min<int>(2, (int)(smem_cap / warp_bytes));  // 2-warp CTAs (measured fastest)
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
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&c_per_sm[ck], kern, nwarps * 32, smem));
    c_smem[ck] = smem;
    c_dev[ck] = h->device;
  }
  int per_sm = std::max(c_per_sm[ck], 1);
  // k_u > 16: the larger per-warp footprint leaves too little L1 for the basis rows above
  // 8 warps/SM (measured: cfg3/4/5 fastest at 4 two-warp CTAs per SM; cfg2 at 6)
  if (r.ku > 16) per_sm = std::min(per_sm, 4);
  r.ntiles = nunits;
  // one wave: at most `target` co-resident CTAs (a partial second wave doubles the pass time)
  return launch_pass(h, a, kern, prm, nwarps, smem, h->num_sms * per_sm, std::max(1, (nunits + nwarps - 1) / nwarps), 0);
}

template <class LAW, int NQ>
static int launch_mma(strom_handle* h, const EvalArgs& a, Params<6, NQ, 4, 3>& prm, int nunits) {
  // compile-time reduced dimensions for the BASELINE configs (addressing folds to immediates)
  // element-Jacobian records come from the generic instantiation (the specialised ones carry
  // only the projected modes)
  if (a.mode == MODE_ELEMJAC || a.mode == MODE_ELEMJAC_ENRICHED) return launch_mma_t<LAW, NQ, 0, 0>(h, a, prm, nunits);
  if (h->ku == 16 && h->kx == 8) return launch_mma_t<LAW, NQ, 16, 8>(h, a, prm, nunits);
  if (h->ku == 20 && h->kx == 10) return launch_mma_t<LAW, NQ, 20, 10>(h, a, prm, nunits);
  if (h->ku == 24 && h->kx == 12) return launch_mma_t<LAW, NQ, 24, 12>(h, a, prm, nunits);
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
  if (a.mode == MODE_ELEMJAC_ENRICHED) { r.test_tab = h->test_tab; r.test_nb = h->test_nb; }
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
    const bool multi = a.P >= 8 && h->ku <= 32;  // many parameter points: warp per element, lanes over mu
    const bool dyn = multi && a.dyn_count != nullptr;  // lanes over the device-counted compacted rows
    prof_mark(h, a.stream, 0);
    if (multi) {
      using VS = VShape<LAW, NB>;
      constexpr int vsmem = (VM_THREADS / 32) * VS::TILE * sizeof(double);
      static int c_dev = -1;
      if (c_dev != h->device) {
        CK(cudaFuncSetAttribute(value_mma_kernel<LAW, NB, NQ, NS>, cudaFuncAttributeMaxDynamicSharedMemorySize, vsmem));
        c_dev = h->device;
      }
      // point groups x element chunks of 4 warps; a device-sized pass splits a 1-D grid of
      // target + groups CTAs over the live groups (dyn_gx with the same target / cap)
      const int gy = (a.P + 31) / 32, target = h->num_sms * 16, cap = std::max(1, (nunits + 3) / 4);
      const int gx = std::max(1, std::min(cap, (target + gy - 1) / gy));
      if (a.mode != MODE_RESIDUAL) {
        const size_t need = dyn ? (size_t)(target + gy) * 32 : (size_t)a.P * gx;
        if (dyn && need > h->part_cap) return fail(-2, "device-sized pass: partial buffer not reserved");
        if (ensure_part(h, need)) return -2;
        r.part = h->part;
      }
      if (dyn) {
        r.list = a.list; r.dyn_count = a.dyn_count; r.dyn_target = target; r.dyn_maxb = cap; r.dyn_ceil = 1;
        value_mma_kernel<LAW, NB, NQ, NS><<<dim3(target + gy), VM_THREADS, vsmem, a.stream>>>(prm);
      } else {
        if (a.list) { r.list = a.list; r.nlist = a.P; }
        value_mma_kernel<LAW, NB, NQ, NS><<<dim3(gy, gx), VM_THREADS, vsmem, a.stream>>>(prm);
      }
      prof_mark(h, a.stream, 1);
      CK(cudaGetLastError());
      if (a.mode != MODE_RESIDUAL) {
        const DynRows dr{dyn ? a.dyn_count : nullptr, a.list, target, cap, 1};
        sum_partials_kernel<<<(a.P + 3) / 4, 128, 0, a.stream>>>(h->part, gx, a.P, a.out, a.mask, dr);
        CK(cudaGetLastError());
      }
      return 0;
    }
    const int gx = (nunits + 127) / 128;
    if (a.mode != MODE_RESIDUAL) {
      if (ensure_part(h, (size_t)a.P * gx)) return -2;
      r.part = h->part;
    }
    value_kernel<LAW, NB, NQ, NS><<<dim3(gx, a.P), 128, 0, a.stream>>>(prm);
    prof_mark(h, a.stream, 1);
    CK(cudaGetLastError());
    if (a.mode != MODE_RESIDUAL) {
      sum_partials_kernel<<<(a.P + 3) / 4, 128, 0, a.stream>>>(h->part, gx, a.P, a.out, a.mask, DynRows{});
      CK(cudaGetLastError());
    }
    return 0;
  }
  if (h->ku < 1) return fail(-1, "derivative modes need k_u >= 1");
  if (h->ku > 32) return fail(-1, "derivative modes need k_u <= 32");
  if constexpr (LAW::M == 4 && NB == 6 && NS == 4) {
    return launch_mma<LAW, NQ>(h, a, prm, nunits);
  }
  // the Roe flux and slip-wall Jacobians exist on the DMMA path (4 components, p = 2) only
  if (LAW::ROE || h->has_wall) return fail(-1, "Roe flux / slip-wall derivatives need p = 2 (DMMA path)");
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
