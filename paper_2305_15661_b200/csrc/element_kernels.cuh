// B200 (sm_100a) fp64 element kernels for the EQP-IFT reduced operator.
//
// Replaces the reference's dual-number element pass (strom/dg.py:82-181 via
// strom/reduced.py:143-229 and strom/distortion.py:33-68).  Straight-sided
// (q = 1) geometry makes the mapping affine per element, so every geometric
// quantity is a function of the three deformed vertices:
//   Jx = [x1-x0, x2-x0] (d x / d xi),  det Jx = g * det_ref,
//   sum_j wdphi0 F = w_q sum_k dphi_k (f . adj(Jx)^T)_k           (volume)
//   nu_f = rot(x_b - x_a) = adj(G)^T N_f |face_ref|                 (faces)
// (derivation in DESIGN.md §3).  Results equal the reference to rounding.
//
// Two kernels:
//   value_kernel   one thread per (element, mu): residual, distortion and the
//                  objective / global residual / residual norm (K2).
//   derivs_kernel  one CTA per tile of U elements at one mu; phases
//                  P0 gather, P1 pointwise physics + Jacobians (point-parallel),
//                  P2 state tangents (one thread per (element, w-direction),
//                     reference-element tables as constant-bank operands),
//                  P3 mesh tangents (6 local directions, projected on Psi),
//                  P4 rho-weighted Gram on DMMA (mma.sync m8n8k4 f64) + S,T,J
//                     in registers across tiles -> deterministic partials (K1),
//                  or per-element contributions (K3).
#include <cuda_runtime.h>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>
#include <algorithm>
#pragma once
#include "element.cuh"

namespace strom {

__host__ __device__ constexpr int fnode_of(int p, int f, int j) {
  // face f runs vertex f -> vertex (f+1)%3, then its edge-interior nodes
  return j == 0 ? f : (j == 1 ? (f + 1) % 3 : 3 + f * (p - 1) + (j - 2));
}

template <class LAW, int NB, int NQ, int NS>
struct Shape {
  static constexpr int M = LAW::M;
  static constexpr int P = NB == 3 ? 1 : (NB == 6 ? 2 : 3);
  static constexpr int NF = P + 1;
  static constexpr int NU = NB * M;
  static constexpr int NR = (NU + 3) / 4 * 4;
  // per-unit shared-memory layout (doubles)
  static constexpr int META = 0;   // x[6] Jx[4] adj[4] detJ nu[6] nlen[3] nhat[6] N rho detr
  static constexpr int DNX = 40;
  static constexpr int DNP = 48;
  static constexpr int UE = DNP + KXMAX;
  static constexpr int UNF = UE + NU;
  static constexpr int RT = UNF + 3 * NF * M;
  static constexpr int RV = RT + NU;
  static constexpr int RF = RV + NU;
  static constexpr int FQ = RF + NU;
  static constexpr int TQ = FQ + NQ * M * 2;
  static constexpr int FXS = 3 * M + 3;
  static constexpr int FX = TQ + NB * M * 4;
  static constexpr int HS = FX + 3 * NS * FXS;
  static constexpr int SW = HS + 3 * NS * M;
  static constexpr int SP = SW + (LAW::SRC != SRC_NONE ? NQ * M : 0);
  static constexpr int WORK = SP + (LAW::SRC == SRC_POS ? NQ * M * 2 : 0);
  // work phase A
  static constexpr int BQ = 0;
  static constexpr int BS = NQ * M * 2 * M;
  static constexpr int CF = BS + (LAW::SRC == SRC_U ? NQ * M * M : 0);
  static constexpr int WORKA = CF + 3 * NS * 2 * M * M;
  __host__ __device__ static int stride(int LDJ) {
    int wb = NR * LDJ + 6 * NU;
    int s = WORK + (WORKA > wb ? WORKA : wb);
    s = (s + 15) / 16 * 16 + 2;  // 16-byte offset between units: bank-disjoint broadcasts
    return s;
  }
};

// meta slots
enum { MX = 0, MJ = 6, MADJ = 10, MDET = 14, MNU = 15, MNLEN = 21, MNHAT = 24, MN = 30, MRHO = 31, MDETR = 32 };

struct UnitInts { int e, nbr[3], fi[3], valid; };

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}

// ---- geometry + distortion of one element ------------------------------------
// x: deformed vertices (x0,y0,x1,y1,x2,y2); X: reference vertices
// Jx[i][k] = x_{k+1}[i] - x_0[i];  adj(Jx) = [[J11,-J01],[-J10,J00]]
struct Geo {
  double J[2][2], adj[2][2], detJ, detr, invr[2][2], G[2][2], g;
};

__device__ __forceinline__ void element_geo(const double* x, const double* X, Geo& o) {
  o.J[0][0] = x[2] - x[0]; o.J[0][1] = x[4] - x[0];
  o.J[1][0] = x[3] - x[1]; o.J[1][1] = x[5] - x[1];
  o.adj[0][0] = o.J[1][1]; o.adj[0][1] = -o.J[0][1];
  o.adj[1][0] = -o.J[1][0]; o.adj[1][1] = o.J[0][0];
  o.detJ = o.J[0][0] * o.J[1][1] - o.J[0][1] * o.J[1][0];
  double r00 = X[2] - X[0], r01 = X[4] - X[0], r10 = X[3] - X[1], r11 = X[5] - X[1];
  o.detr = r00 * r11 - r01 * r10;
  double id = 1.0 / o.detr;
  o.invr[0][0] = r11 * id; o.invr[0][1] = -r01 * id; o.invr[1][0] = -r10 * id; o.invr[1][1] = r00 * id;
  for (int i = 0; i < 2; ++i)
    for (int j = 0; j < 2; ++j) o.G[i][j] = o.J[i][0] * o.invr[0][j] + o.J[i][1] * o.invr[1][j];
  o.g = o.G[0][0] * o.G[1][1] - o.G[0][1] * o.G[1][0];
}

// distortion integral, distortion.py:33-50 (d = 2, affine: ratio constant in q)
__device__ __forceinline__ double distortion_eta(const Geo& o, double wsum, double eps, double* ratio_out,
                                                 double* den_out) {
  double fro2 = o.G[0][0] * o.G[0][0] + o.G[0][1] * o.G[0][1] + o.G[1][0] * o.G[1][0] + o.G[1][1] * o.G[1][1];
  double den = o.g >= eps ? o.g : eps;
  double ratio = fro2 / den;
  if (ratio_out) *ratio_out = ratio;
  if (den_out) *den_out = den;
  return wsum * o.detr * ratio * ratio;
}

__device__ __forceinline__ void distortion_grad(const Geo& o, double wsum, double eps, double kappa, double* dN) {
  double ratio, den;
  distortion_eta(o, wsum, eps, &ratio, &den);
#pragma unroll
  for (int d = 0; d < 6; ++d) {
    const int gv = d >> 1, ic = d & 1;
    const double c0 = (gv == 1) - (gv == 0), c1 = (gv == 2) - (gv == 0);
    const double dJ[2][2] = {{ic == 0 ? c0 : 0.0, ic == 0 ? c1 : 0.0}, {ic == 1 ? c0 : 0.0, ic == 1 ? c1 : 0.0}};
    double dG[2][2];
    for (int i = 0; i < 2; ++i)
      for (int j = 0; j < 2; ++j) dG[i][j] = dJ[i][0] * o.invr[0][j] + dJ[i][1] * o.invr[1][j];
    double dg = dG[0][0] * o.G[1][1] + o.G[0][0] * dG[1][1] - dG[0][1] * o.G[1][0] - o.G[0][1] * dG[1][0];
    double dfro = 2.0 * (o.G[0][0] * dG[0][0] + o.G[0][1] * dG[0][1] + o.G[1][0] * dG[1][0] + o.G[1][1] * dG[1][1]);
    double dden = o.g >= eps ? dg : 0.0;
    double dratio = (dfro - ratio * dden) / den;
    dN[d] = kappa * wsum * o.detr * 2.0 * ratio * dratio;
  }
}

__global__ void eta_ref_kernel(int ne, const int* __restrict__ en, const double* __restrict__ nodes, double wsum,
                               double eps, double* __restrict__ eta) {
  int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= ne) return;
  double X[6];
  for (int g = 0; g < 3; ++g) {
    int n = en[3 * e + g];
    X[2 * g] = nodes[2 * n];
    X[2 * g + 1] = nodes[2 * n + 1];
  }
  Geo o;
  element_geo(X, X, o);
  eta[e] = distortion_eta(o, wsum, eps, nullptr, nullptr);
}

__device__ __forceinline__ void flag_degenerate(const Run& r, int p, int e) {
  atomicAdd(&r.degen[p], 1);
  int pos = atomicAdd(r.degen_fill, 1);
  if (pos < r.degen_cap) {
    r.degen_list[2 * pos] = p;
    r.degen_list[2 * pos + 1] = e;
  }
}

// face normal data: nu_f = rot(x_b - x_a) = (t_y, -t_x)
__device__ __forceinline__ void face_normal(const double* x, int f, double* nu, double& len, double* nh) {
  int a = f, b = (f + 1) % 3;
  double tx = x[2 * b] - x[2 * a], ty = x[2 * b + 1] - x[2 * a + 1];
  nu[0] = ty; nu[1] = -tx;
  len = sqrt(nu[0] * nu[0] + nu[1] * nu[1]);
  nh[0] = nu[0] / len; nh[1] = nu[1] / len;
}

// ============================================================================
// K2: value kernel — one thread per (element, mu)
// ============================================================================
template <class LAW, int NB, int NQ, int NS>
__global__ void __launch_bounds__(128) value_kernel(const __grid_constant__ Params<NB, NQ, NS, Shape<LAW, NB, NQ, NS>::NF> prm) {
  using SH = Shape<LAW, NB, NQ, NS>;
  constexpr int M = SH::M, NU = SH::NU, NF = SH::NF, PD = SH::P;
  const auto& T = prm.t;
  const Run& r = prm.r;
  const int p = blockIdx.y;
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  const int nunits = r.active ? r.A : r.ne;
  double contrib = 0.0;
  if (idx < nunits) {
    const int e = r.active ? r.active[idx] : idx;
    const double rho = r.active ? r.rho[idx] : 1.0;
    LawArgs la;
    for (int i = 0; i < 8; ++i) la.p[i] = r.lawp[i];
    for (int i = 0; i < NMU; ++i) la.mu[i] = i < r.nmu ? r.mu[p * r.nmu + i] : 0.0;
    const double* w = r.w + (size_t)p * r.ku;
    const double* tau = r.tau + (size_t)p * r.kx;
    double x[6], X[6];
#pragma unroll
    for (int g = 0; g < 3; ++g) {
      int n = r.elem_nodes[3 * e + g];
      X[2 * g] = r.nodes[2 * n];
      X[2 * g + 1] = r.nodes[2 * n + 1];
#pragma unroll
      for (int ic = 0; ic < 2; ++ic) {
        int row = 2 * n + ic;
        double v = r.xref[row];
        const double* ps = r.psi + (size_t)row * r.kx;
        for (int a = 0; a < r.kx; ++a) v = fma(ps[a], tau[a], v);
        x[2 * g + ic] = v;
      }
    }
    double U[NU];
    {
      const double* ph = r.phi + (size_t)e * NU * r.ku;
#pragma unroll
      for (int i = 0; i < NU; ++i) {
        double v = r.u0 ? r.u0[(size_t)e * NU + i] : 0.0;
        for (int k = 0; k < r.ku; ++k) v = fma(ph[i * r.ku + k], w[k], v);
        U[i] = v;
      }
    }
    Geo o;
    element_geo(x, X, o);
    if (o.g <= 0.0) flag_degenerate(r, p, e);
    double R[NU];
#pragma unroll
    for (int i = 0; i < NU; ++i) R[i] = 0.0;
    // volume (dg.py:105-125)
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      double uq[M];
#pragma unroll
      for (int c = 0; c < M; ++c) {
        double v = 0.0;
#pragma unroll
        for (int n = 0; n < NB; ++n) v = fma(T.phi[q][n], U[n * M + c], v);
        uq[c] = v;
      }
      double f[M][2];
      LAW::flux(uq, f, la);
#pragma unroll
      for (int c = 0; c < M; ++c) {
        double F0 = T.wq[q] * (f[c][0] * o.adj[0][0] + f[c][1] * o.adj[0][1]);
        double F1 = T.wq[q] * (f[c][0] * o.adj[1][0] + f[c][1] * o.adj[1][1]);
#pragma unroll
        for (int n = 0; n < NB; ++n) R[n * M + c] -= T.dphi[q][n][0] * F0 + T.dphi[q][n][1] * F1;
      }
      if (LAW::SRC != SRC_NONE) {
        double pos[2];
#pragma unroll
        for (int i = 0; i < 2; ++i) pos[i] = T.bary[q][0] * x[i] + T.bary[q][1] * x[2 + i] + T.bary[q][2] * x[4 + i];
        double s[M];
        LAW::source(pos, uq, s, la);
#pragma unroll
        for (int c = 0; c < M; ++c) {
          double sv = T.wq[q] * o.detJ * s[c];
#pragma unroll
          for (int n = 0; n < NB; ++n) R[n * M + c] -= T.phi[q][n] * sv;
        }
      }
    }
    // faces (dg.py:127-175)
#pragma unroll
    for (int f = 0; f < 3; ++f) {
      double nu[2], len, nh[2];
      face_normal(x, f, nu, len, nh);
      const int nb = r.nbr[3 * e + f];
      const int fi = r.finfo[3 * e + f];
      const int bc = fi >> 3;
      double Un[NF][M];
      int flip = 0;
      if (bc == 0) {
        const int nf = fi & 3;
        flip = (fi >> 2) & 1;
        const double* ph = r.phi + (size_t)nb * NU * r.ku;
#pragma unroll
        for (int j = 0; j < NF; ++j) {
          int node = j == 0 ? nf : (j == 1 ? (nf + 1) % 3 : 3 + nf * (PD - 1) + (j - 2));
#pragma unroll
          for (int c = 0; c < M; ++c) {
            int row = node * M + c;
            double v = r.u0 ? r.u0[(size_t)nb * NU + row] : 0.0;
            for (int k = 0; k < r.ku; ++k) v = fma(ph[row * r.ku + k], w[k], v);
            Un[j][c] = v;
          }
        }
      }
      double ghost[M];
      if (bc >= 2) LAW::ghost(bc - 2, la, ghost);
#pragma unroll
      for (int s = 0; s < NS; ++s) {
        double ui[M], uo[M];
#pragma unroll
        for (int c = 0; c < M; ++c) {
          double v = 0.0;
#pragma unroll
          for (int j = 0; j < NF; ++j) v = fma(T.trace[f][s][j], U[fnode_of(PD, f, j) * M + c], v);
          ui[c] = v;
        }
        if (bc == 0) {
          const int sp = flip ? NS - 1 - s : s;
#pragma unroll
          for (int c = 0; c < M; ++c) {
            double v = 0.0;
#pragma unroll
            for (int j = 0; j < NF; ++j) v = fma(T.trace[0][sp][j], Un[j][c], v);
            uo[c] = v;
          }
        } else if (bc == 1) {
#pragma unroll
          for (int c = 0; c < M; ++c) uo[c] = ui[c];
        } else {
#pragma unroll
          for (int c = 0; c < M; ++c) uo[c] = ghost[c];
        }
        double fi_[M][2], fo[M][2];
        LAW::flux(ui, fi_, la);
        LAW::flux(uo, fo, la);
        double wi = LAW::wavespeed(ui, nh, la), wo = LAW::wavespeed(uo, nh, la);
        double lam = wi >= wo ? wi : wo;
#pragma unroll
        for (int c = 0; c < M; ++c) {
          double fn = (fi_[c][0] * nu[0] + fi_[c][1] * nu[1]) + (fo[c][0] * nu[0] + fo[c][1] * nu[1]);
          double H = T.ws[s] * (0.5 * fn - 0.5 * (lam * len) * (uo[c] - ui[c]));
#pragma unroll
          for (int j = 0; j < NF; ++j) R[fnode_of(PD, f, j) * M + c] = fma(T.trace[f][s][j], H, R[fnode_of(PD, f, j) * M + c]);
        }
      }
    }
    if (r.mode == MODE_RESIDUAL) {
      double* o_ = r.out + ((size_t)p * r.ne + e) * NU;
#pragma unroll
      for (int i = 0; i < NU; ++i) o_[i] = R[i];
    } else {
      double r2 = 0.0;
#pragma unroll
      for (int i = 0; i < NU; ++i) r2 = fma(R[i], R[i], r2);
      if (r.mode == MODE_OBJECTIVE) {
        double N = r.kappa * (distortion_eta(o, T.wsum, r.eps, nullptr, nullptr) - r.eta_ref[e]);
        contrib = 0.5 * rho * (r2 + N * N);
      } else {
        contrib = r2;
      }
    }
  }
  if (r.mode != MODE_RESIDUAL) {
    // deterministic block reduction -> one partial per block
    __shared__ double red[128];
    red[threadIdx.x] = contrib;
    __syncthreads();
    for (int s = 64; s > 0; s >>= 1) {
      if (threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
      __syncthreads();
    }
    if (threadIdx.x == 0) r.part[(size_t)p * gridDim.x + blockIdx.x] = red[0];
  }
}

__global__ void sum_partials_kernel(const double* __restrict__ part, int nparts, int P, double* __restrict__ out) {
  int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= P) return;
  double s = 0.0;
  for (int i = 0; i < nparts; ++i) s += part[(size_t)p * nparts + i];
  out[p] = s;
}

// ============================================================================
// K1 / K3: derivatives kernel — one CTA per tile of U elements at one mu
// ============================================================================
template <class LAW, int NB, int NQ, int NS>
__global__ void __launch_bounds__(DERIV_THREADS) derivs_kernel(const __grid_constant__ Params<NB, NQ, NS, Shape<LAW, NB, NQ, NS>::NF> prm) {
  using SH = Shape<LAW, NB, NQ, NS>;
  constexpr int M = SH::M, NU = SH::NU, NF = SH::NF, NR = SH::NR, PD = SH::P;
  const auto& T = prm.t;
  const Run& r = prm.r;
  extern __shared__ __align__(16) double smem[];
  __shared__ UnitInts UI[DERIV_THREADS];
  __shared__ double s_wt[2 * KMAX];  // w then tau of this mu
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int p = blockIdx.y;
  const int U = r.U, ku = r.ku, kx = r.kx, K = r.K, KP = r.KP, LDJ = r.LDJ, STR = r.unit_stride;
  const int nunits_total = r.active ? r.A : r.ne;

  LawArgs la;
  for (int i = 0; i < 8; ++i) la.p[i] = r.lawp[i];
  for (int i = 0; i < NMU; ++i) la.mu[i] = i < r.nmu ? r.mu[p * r.nmu + i] : 0.0;
  for (int i = tid; i < ku; i += blockDim.x) s_wt[i] = r.w[(size_t)p * ku + i];
  for (int i = tid; i < kx; i += blockDim.x) s_wt[KMAX + i] = r.tau[(size_t)p * kx + i];

  // persistent accumulators (DERIVS)
  constexpr int MAXT = 4;
  double hacc[MAXT][2];
#pragma unroll
  for (int s = 0; s < MAXT; ++s) hacc[s][0] = hacc[s][1] = 0.0;
  double gacc = 0.0, tacc[2] = {0.0, 0.0}, jacc = 0.0;
  const int nt8 = KP / 8;
  const int ntri = nt8 * (nt8 + 1) / 2;

  for (int tile = blockIdx.x; tile < r.ntiles; tile += gridDim.x) {
    __syncthreads();
    const int base = tile * U;
    const int nvalid = min(U, nunits_total - base);
    // ---- P0: unit metadata + gathers ------------------------------------------
    if (tid < U) {
      UnitInts& ui = UI[tid];
      ui.valid = tid < nvalid;
      int e = 0;
      double rho = 0.0;
      if (ui.valid) {
        int ix = base + tid;
        e = r.active ? r.active[ix] : ix;
        rho = r.active ? r.rho[ix] : 1.0;
      }
      ui.e = e;
      for (int f = 0; f < 3; ++f) { ui.nbr[f] = r.nbr[3 * e + f]; ui.fi[f] = r.finfo[3 * e + f]; }
      smem[tid * STR + MRHO] = rho;
    }
    __syncthreads();
    // deformed coordinates x = X + Psi tau (6 per unit)
    for (int t = tid; t < nvalid * 6; t += blockDim.x) {
      int u = t / 6, d = t % 6;
      int n = r.elem_nodes[3 * UI[u].e + (d >> 1)];
      int row = 2 * n + (d & 1);
      double v = r.xref[row];
      const double* ps = r.psi + (size_t)row * kx;
      for (int a = 0; a < kx; ++a) v = fma(ps[a], s_wt[KMAX + a], v);
      smem[u * STR + MX + d] = v;
    }
    // element states U_e = U0 + Phi_e w
    for (int t = tid; t < nvalid * NU; t += blockDim.x) {
      int u = t / NU, i = t % NU;
      int e = UI[u].e;
      const double* ph = r.phi + ((size_t)e * NU + i) * ku;
      double v = r.u0 ? r.u0[(size_t)e * NU + i] : 0.0;
      for (int k = 0; k < ku; ++k) v = fma(ph[k], s_wt[k], v);
      smem[u * STR + SH::UE + i] = v;
    }
    // neighbor face-node states
    for (int t = tid; t < nvalid * 3 * NF * M; t += blockDim.x) {
      int u = t / (3 * NF * M), rem = t % (3 * NF * M);
      int f = rem / (NF * M), j = (rem / M) % NF, c = rem % M;
      const UnitInts& ui = UI[u];
      double v = 0.0;
      if ((ui.fi[f] >> 3) == 0) {
        int nf = ui.fi[f] & 3, nb = ui.nbr[f];
        int node = j == 0 ? nf : (j == 1 ? (nf + 1) % 3 : 3 + nf * (PD - 1) + (j - 2));
        int row = node * M + c;
        const double* ph = r.phi + ((size_t)nb * NU + row) * ku;
        v = r.u0 ? r.u0[(size_t)nb * NU + row] : 0.0;
        for (int k = 0; k < ku; ++k) v = fma(ph[k], s_wt[k], v);
      }
      smem[u * STR + SH::UNF + rem] = v;
    }
    __syncthreads();
    // per-unit geometry, normals, distortion (value + 6 local gradients)
    if (tid < nvalid) {
      double* S = smem + tid * STR;
      const int e = UI[tid].e;
      double X[6];
      for (int g = 0; g < 3; ++g) {
        int n = r.elem_nodes[3 * e + g];
        X[2 * g] = r.nodes[2 * n];
        X[2 * g + 1] = r.nodes[2 * n + 1];
      }
      Geo o;
      element_geo(S + MX, X, o);
      if (o.g <= 0.0) flag_degenerate(r, p, e);
      S[MJ + 0] = o.J[0][0]; S[MJ + 1] = o.J[0][1]; S[MJ + 2] = o.J[1][0]; S[MJ + 3] = o.J[1][1];
      S[MADJ + 0] = o.adj[0][0]; S[MADJ + 1] = o.adj[0][1]; S[MADJ + 2] = o.adj[1][0]; S[MADJ + 3] = o.adj[1][1];
      S[MDET] = o.detJ;
      S[MDETR] = o.detr;
      for (int f = 0; f < 3; ++f) face_normal(S + MX, f, S + MNU + 2 * f, S[MNLEN + f], S + MNHAT + 2 * f);
      S[MN] = r.kappa * (distortion_eta(o, T.wsum, r.eps, nullptr, nullptr) - r.eta_ref[e]);
      distortion_grad(o, T.wsum, r.eps, r.kappa, S + SH::DNX);
    }
    __syncthreads();
    // ---- P1: pointwise physics (volume points, then face points) ---------------
    for (int t = tid; t < nvalid * (NQ + 3 * NS); t += blockDim.x) {
      const int u = t / (NQ + 3 * NS), pt = t % (NQ + 3 * NS);
      double* S = smem + u * STR;
      double* W = S + SH::WORK;
      if (pt < NQ) {
        const int q = pt;
        Dn<M> ud[M];
#pragma unroll
        for (int c = 0; c < M; ++c) {
          double v = 0.0;
#pragma unroll
          for (int n = 0; n < NB; ++n) v = fma(T.phi[q][n], S[SH::UE + n * M + c], v);
          ud[c] = seed<M>(v, c);
        }
        Dn<M> f[M][2];
        LAW::flux(ud, f, la);
        const double wq = T.wq[q];
        const double* adj = S + MADJ;
#pragma unroll
        for (int c = 0; c < M; ++c) {
          S[SH::FQ + (q * M + c) * 2 + 0] = wq * f[c][0].v;
          S[SH::FQ + (q * M + c) * 2 + 1] = wq * f[c][1].v;
#pragma unroll
          for (int kk = 0; kk < 2; ++kk)
#pragma unroll
            for (int cp = 0; cp < M; ++cp)
              W[SH::BQ + ((q * M + c) * 2 + kk) * M + cp] = wq * (f[c][0].d[cp] * adj[kk * 2 + 0] + f[c][1].d[cp] * adj[kk * 2 + 1]);
        }
        if (LAW::SRC != SRC_NONE) {
          Dn<M + 2> us[M], ps[2];
#pragma unroll
          for (int c = 0; c < M; ++c) us[c] = seed<M + 2>(ud[c].v, c);
#pragma unroll
          for (int i = 0; i < 2; ++i)
            ps[i] = seed<M + 2>(T.bary[q][0] * S[MX + i] + T.bary[q][1] * S[MX + 2 + i] + T.bary[q][2] * S[MX + 4 + i], M + i);
          Dn<M + 2> sv[M];
          LAW::source(ps, us, sv, la);
          const double detJ = S[MDET];
#pragma unroll
          for (int c = 0; c < M; ++c) {
            S[SH::SW + q * M + c] = wq * sv[c].v;
            if (LAW::SRC == SRC_POS) {
              S[SH::SP + (q * M + c) * 2 + 0] = wq * detJ * sv[c].d[M + 0];
              S[SH::SP + (q * M + c) * 2 + 1] = wq * detJ * sv[c].d[M + 1];
            }
            if (LAW::SRC == SRC_U) {
#pragma unroll
              for (int cp = 0; cp < M; ++cp) W[SH::BS + (q * M + c) * M + cp] = wq * detJ * sv[c].d[cp];
            }
          }
        }
      } else {
        const int fs = pt - NQ, f = fs / NS, s = fs % NS;
        const UnitInts& ui = UI[u];
        const int fi = ui.fi[f], bc = fi >> 3;
        const double* nu = S + MNU + 2 * f;
        const double len = S[MNLEN + f];
        const double* nh = S + MNHAT + 2 * f;
        double ui_[M], uo[M];
        for (int c = 0; c < M; ++c) {
          double v = 0.0;
          for (int j = 0; j < NF; ++j) v = fma(T.trace[f][s][j], S[SH::UE + fnode_of(PD, f, j) * M + c], v);
          ui_[c] = v;
        }
        if (bc == 0) {
          const int sp = ((fi >> 2) & 1) ? NS - 1 - s : s;
          for (int c = 0; c < M; ++c) {
            double v = 0.0;
            for (int j = 0; j < NF; ++j) v = fma(T.trace[0][sp][j], S[SH::UNF + (f * NF + j) * M + c], v);
            uo[c] = v;
          }
        } else if (bc == 1) {
          for (int c = 0; c < M; ++c) uo[c] = ui_[c];
        } else {
          LAW::ghost(bc - 2, la, uo);
        }
        // flux Jacobians (M seeds) and wavespeeds (M + 2 seeds: state, nhat)
        Dn<M> di[M], dO[M];
#pragma unroll
        for (int c = 0; c < M; ++c) { di[c] = seed<M>(ui_[c], c); dO[c] = seed<M>(uo[c], c); }
        Dn<M> fi2[M][2], fo2[M][2];
        LAW::flux(di, fi2, la);
        LAW::flux(dO, fo2, la);
        Dn<M + 2> wi_u[M], wo_u[M], nn[2];
#pragma unroll
        for (int c = 0; c < M; ++c) { wi_u[c] = seed<M + 2>(ui_[c], c); wo_u[c] = seed<M + 2>(uo[c], c); }
        nn[0] = seed<M + 2>(nh[0], M);
        nn[1] = seed<M + 2>(nh[1], M + 1);
        Dn<M + 2> wsi = LAW::wavespeed(wi_u, nn, la), wso = LAW::wavespeed(wo_u, nn, la);
        const bool in_wins = wsi.v >= wso.v;  // dual.maximum tie -> first (dual.py:171)
        const double lam = in_wins ? wsi.v : wso.v;
        const double ws = T.ws[s];
        double* FXp = S + SH::FX + (f * NS + s) * SH::FXS;
        double* Cin = S + SH::WORK + SH::CF + ((f * NS + s) * 2 + 0) * M * M;
        double* Cout = S + SH::WORK + SH::CF + ((f * NS + s) * 2 + 1) * M * M;
#pragma unroll
        for (int c = 0; c < M; ++c) {
          const double du = uo[c] - ui_[c];
          double fn = (fi2[c][0].v * nu[0] + fi2[c][1].v * nu[1]) + (fo2[c][0].v * nu[0] + fo2[c][1].v * nu[1]);
          S[SH::HS + (f * NS + s) * M + c] = ws * (0.5 * fn - 0.5 * (lam * len) * du);
          FXp[2 * c + 0] = 0.5 * ws * (fi2[c][0].v + fo2[c][0].v);
          FXp[2 * c + 1] = 0.5 * ws * (fi2[c][1].v + fo2[c][1].v);
          FXp[2 * M + c] = 0.5 * ws * du;
#pragma unroll
          for (int cp = 0; cp < M; ++cp) {
            double ai = fi2[c][0].d[cp] * nu[0] + fi2[c][1].d[cp] * nu[1];
            double ao = fo2[c][0].d[cp] * nu[0] + fo2[c][1].d[cp] * nu[1];
            double dl_in = in_wins ? wsi.d[cp] : 0.0;
            double dl_out = in_wins ? 0.0 : wso.d[cp];
            double cin = 0.5 * ai + (c == cp ? 0.5 * lam * len : 0.0) - 0.5 * len * du * dl_in;
            double cout = 0.5 * ao - (c == cp ? 0.5 * lam * len : 0.0) - 0.5 * len * du * dl_out;
            if (bc == 1) { cin += cout; cout = 0.0; }
            if (bc >= 2) cout = 0.0;
            Cin[c * M + cp] = ws * cin;
            Cout[c * M + cp] = ws * cout;
          }
        }
        FXp[3 * M + 0] = lam;
        FXp[3 * M + 1] = in_wins ? wsi.d[M] : wso.d[M];
        FXp[3 * M + 2] = in_wins ? wsi.d[M + 1] : wso.d[M + 1];
      }
    }
    __syncthreads();
    // residual (vol / face split) and the x-tangent helper Tq
    for (int t = tid; t < nvalid * NU; t += blockDim.x) {
      const int u = t / NU, i = t % NU, n = i / M, c = i % M;
      double* S = smem + u * STR;
      double tq[2][2] = {{0, 0}, {0, 0}};
#pragma unroll
      for (int q = 0; q < NQ; ++q)
#pragma unroll
        for (int kk = 0; kk < 2; ++kk)
#pragma unroll
          for (int ii = 0; ii < 2; ++ii) tq[kk][ii] = fma(T.dphi[q][n][kk], S[SH::FQ + (q * M + c) * 2 + ii], tq[kk][ii]);
      const double* adj = S + MADJ;
      double rv = -(adj[0] * tq[0][0] + adj[1] * tq[0][1] + adj[2] * tq[1][0] + adj[3] * tq[1][1]);
      if (LAW::SRC != SRC_NONE) {
        double sacc = 0.0;
#pragma unroll
        for (int q = 0; q < NQ; ++q) sacc = fma(T.phi[q][n], S[SH::SW + q * M + c], sacc);
        rv -= S[MDET] * sacc;
      }
      double rf = 0.0;
#pragma unroll
      for (int f = 0; f < 3; ++f)
#pragma unroll
        for (int j = 0; j < NF; ++j)
          if (fnode_of(PD, f, j) == n)
#pragma unroll
            for (int s = 0; s < NS; ++s) rf = fma(T.trace[f][s][j], S[SH::HS + (f * NS + s) * M + c], rf);
      S[SH::TQ + i * 4 + 0] = tq[0][0]; S[SH::TQ + i * 4 + 1] = tq[0][1];
      S[SH::TQ + i * 4 + 2] = tq[1][0]; S[SH::TQ + i * 4 + 3] = tq[1][1];
      S[SH::RV + i] = rv;
      S[SH::RF + i] = rf;
      S[SH::RT + i] = rv + rf;
    }
    __syncthreads();
    // ---- P2: state tangents, one thread per (unit, w-direction) ----------------
    double acc[NU];
    const bool has_tan = tid < U * ku && (tid / ku) < nvalid;
    const int tu = has_tan ? tid / ku : 0, tk = has_tan ? tid % ku : 0;
    if (has_tan) {
      const double* S = smem + tu * STR;
      const double* W = S + SH::WORK;
      const int e = UI[tu].e;
      double pc[NU];
      const double* ph = r.phi + (size_t)e * NU * ku + tk;
#pragma unroll
      for (int i = 0; i < NU; ++i) { pc[i] = __ldg(ph + (size_t)i * ku); acc[i] = 0.0; }
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        double du[M];
#pragma unroll
        for (int c = 0; c < M; ++c) {
          double v = 0.0;
#pragma unroll
          for (int n = 0; n < NB; ++n) v = fma(T.phi[q][n], pc[n * M + c], v);
          du[c] = v;
        }
        const double* B = W + SH::BQ + q * M * 2 * M;
#pragma unroll
        for (int c = 0; c < M; ++c) {
          double g0 = 0.0, g1 = 0.0;
#pragma unroll
          for (int cp = 0; cp < M; ++cp) {
            g0 = fma(B[(c * 2 + 0) * M + cp], du[cp], g0);
            g1 = fma(B[(c * 2 + 1) * M + cp], du[cp], g1);
          }
#pragma unroll
          for (int n = 0; n < NB; ++n) acc[n * M + c] -= T.dphi[q][n][0] * g0 + T.dphi[q][n][1] * g1;
        }
        if (LAW::SRC == SRC_U) {
          const double* Bs = W + SH::BS + q * M * M;
#pragma unroll
          for (int c = 0; c < M; ++c) {
            double sv = 0.0;
#pragma unroll
            for (int cp = 0; cp < M; ++cp) sv = fma(Bs[c * M + cp], du[cp], sv);
#pragma unroll
            for (int n = 0; n < NB; ++n) acc[n * M + c] -= T.phi[q][n] * sv;
          }
        }
      }
#pragma unroll
      for (int f = 0; f < 3; ++f) {
        const int fi = UI[tu].fi[f], bc = fi >> 3;
        double pn[NF][M];
        int flip = 0;
        if (bc == 0) {
          const int nf = fi & 3, nb = UI[tu].nbr[f];
          flip = (fi >> 2) & 1;
          const double* phn = r.phi + (size_t)nb * NU * ku + tk;
#pragma unroll
          for (int j = 0; j < NF; ++j) {
            int node = j == 0 ? nf : (j == 1 ? (nf + 1) % 3 : 3 + nf * (PD - 1) + (j - 2));
#pragma unroll
            for (int c = 0; c < M; ++c) pn[j][c] = __ldg(phn + (size_t)(node * M + c) * ku);
          }
        }
#pragma unroll
        for (int s = 0; s < NS; ++s) {
          double di[M], dO[M];
#pragma unroll
          for (int c = 0; c < M; ++c) {
            double v = 0.0;
#pragma unroll
            for (int j = 0; j < NF; ++j) v = fma(T.trace[f][s][j], pc[fnode_of(PD, f, j) * M + c], v);
            di[c] = v;
          }
          const double* Cin = W + SH::CF + ((f * NS + s) * 2 + 0) * M * M;
          const double* Cout = W + SH::CF + ((f * NS + s) * 2 + 1) * M * M;
          double dH[M];
#pragma unroll
          for (int c = 0; c < M; ++c) {
            double v = 0.0;
#pragma unroll
            for (int cp = 0; cp < M; ++cp) v = fma(Cin[c * M + cp], di[cp], v);
            dH[c] = v;
          }
          if (bc == 0) {
            if (flip) {
#pragma unroll
              for (int c = 0; c < M; ++c) {
                double v = 0.0;
#pragma unroll
                for (int j = 0; j < NF; ++j) v = fma(T.trace[0][NS - 1 - s][j], pn[j][c], v);
                dO[c] = v;
              }
            } else {
#pragma unroll
              for (int c = 0; c < M; ++c) {
                double v = 0.0;
#pragma unroll
                for (int j = 0; j < NF; ++j) v = fma(T.trace[0][s][j], pn[j][c], v);
                dO[c] = v;
              }
            }
#pragma unroll
            for (int c = 0; c < M; ++c) {
              double v = dH[c];
#pragma unroll
              for (int cp = 0; cp < M; ++cp) v = fma(Cout[c * M + cp], dO[cp], v);
              dH[c] = v;
            }
          }
#pragma unroll
          for (int c = 0; c < M; ++c)
#pragma unroll
            for (int j = 0; j < NF; ++j) {
              const int ix = fnode_of(PD, f, j) * M + c;
              acc[ix] = fma(T.trace[f][s][j], dH[c], acc[ix]);
            }
        }
      }
    }
    __syncthreads();  // phase-A work area (B_q, C) is dead from here on
    if (has_tan) {
      double* Jt = smem + tu * STR + SH::WORK;
#pragma unroll
      for (int i = 0; i < NU; ++i) Jt[i * LDJ + tk] = acc[i];
#pragma unroll
      for (int i = NU; i < NR; ++i) Jt[i * LDJ + tk] = 0.0;
    }
    // ---- P3: mesh tangents in the 6 local directions ------------------------------
    for (int t = tid; t < nvalid * 6; t += blockDim.x) {
      const int u = t / 6, d = t % 6, gv = d >> 1, ic = d & 1;
      double* S = smem + u * STR;
      double* dRx = S + SH::WORK + NR * LDJ + d * NU;
      const double c0 = (gv == 1) - (gv == 0), c1 = (gv == 2) - (gv == 0);
      const double dJ[2][2] = {{ic == 0 ? c0 : 0.0, ic == 0 ? c1 : 0.0}, {ic == 1 ? c0 : 0.0, ic == 1 ? c1 : 0.0}};
      const double dadj[4] = {dJ[1][1], -dJ[0][1], -dJ[1][0], dJ[0][0]};
      const double* Jm = S + MJ;
      const double ddet = dJ[0][0] * Jm[3] + Jm[0] * dJ[1][1] - dJ[0][1] * Jm[2] - Jm[1] * dJ[1][0];
      double res[NU];
#pragma unroll
      for (int i = 0; i < NU; ++i) {
        const double* tq = S + SH::TQ + i * 4;
        res[i] = -(dadj[0] * tq[0] + dadj[1] * tq[1] + dadj[2] * tq[2] + dadj[3] * tq[3]);
      }
      if (LAW::SRC != SRC_NONE) {
#pragma unroll
        for (int n = 0; n < NB; ++n)
#pragma unroll
          for (int c = 0; c < M; ++c) {
            double v = 0.0;
#pragma unroll
            for (int q = 0; q < NQ; ++q) {
              double term = ddet * S[SH::SW + q * M + c];
              if (LAW::SRC == SRC_POS) term += S[SH::SP + (q * M + c) * 2 + ic] * T.bary[q][gv];
              v = fma(T.phi[q][n], term, v);
            }
            res[n * M + c] -= v;
          }
      }
#pragma unroll
      for (int f = 0; f < 3; ++f) {
        const int a = f, b = (f + 1) % 3;
        const double del = (gv == b) - (gv == a);
        if (del != 0.0) {
          double dnu[2];
          if (ic == 0) { dnu[0] = 0.0; dnu[1] = -del; } else { dnu[0] = del; dnu[1] = 0.0; }
          const double* nh = S + MNHAT + 2 * f;
          const double len = S[MNLEN + f];
          const double dlen = nh[0] * dnu[0] + nh[1] * dnu[1];
          const double dnh0 = (dnu[0] - nh[0] * dlen) / len, dnh1 = (dnu[1] - nh[1] * dlen) / len;
#pragma unroll
          for (int s = 0; s < NS; ++s) {
            const double* FXp = S + SH::FX + (f * NS + s) * SH::FXS;
            const double lam = FXp[3 * M], dlam = FXp[3 * M + 1] * dnh0 + FXp[3 * M + 2] * dnh1;
            const double coef = dlam * len + lam * dlen;
#pragma unroll
            for (int c = 0; c < M; ++c) {
              double dH = FXp[2 * c] * dnu[0] + FXp[2 * c + 1] * dnu[1] - FXp[2 * M + c] * coef;
#pragma unroll
              for (int j = 0; j < NF; ++j) {
                const int ix = fnode_of(PD, f, j) * M + c;
                res[ix] = fma(T.trace[f][s][j], dH, res[ix]);
              }
            }
          }
        }
      }
#pragma unroll
      for (int i = 0; i < NU; ++i) dRx[i] = res[i];
    }
    __syncthreads();
    // project the local mesh Jacobian on Psi_e; zero the Gram padding columns
    for (int t = tid; t < nvalid * (KP - ku); t += blockDim.x) {
      const int u = t / (KP - ku), a = t % (KP - ku);
      double* S = smem + u * STR;
      double* Jt = S + SH::WORK;
      if (a < kx) {
        const int e = UI[u].e;
        double psv[6];
#pragma unroll
        for (int d = 0; d < 6; ++d) {
          int n = r.elem_nodes[3 * e + (d >> 1)];
          psv[d] = __ldg(r.psi + (size_t)(2 * n + (d & 1)) * kx + a);
        }
        const double* dRx = S + SH::WORK + NR * LDJ;
#pragma unroll
        for (int i = 0; i < NU; ++i) {
          double v = 0.0;
#pragma unroll
          for (int d = 0; d < 6; ++d) v = fma(dRx[d * NU + i], psv[d], v);
          Jt[i * LDJ + ku + a] = v;
        }
#pragma unroll
        for (int i = NU; i < NR; ++i) Jt[i * LDJ + ku + a] = 0.0;
        double dn = 0.0;
#pragma unroll
        for (int d = 0; d < 6; ++d) dn = fma(S[SH::DNX + d], psv[d], dn);
        S[SH::DNP + a] = dn;
      } else {
#pragma unroll
        for (int i = 0; i < NR; ++i) Jt[i * LDJ + ku + a] = 0.0;
      }
    }
    __syncthreads();
    // ---- P4 ---------------------------------------------------------------------
    if (r.mode == MODE_DERIVS) {
      // rho-weighted Gram of the stacked element Jacobians on DMMA
#pragma unroll
      for (int sl = 0; sl < MAXT; ++sl) {
        const int tile8 = warp + 4 * sl;
        if (tile8 < ntri) {
          int ti = 0, rem = tile8;
          while (rem >= nt8 - ti) { rem -= nt8 - ti; ++ti; }
          const int tj = ti + rem;
          for (int u = 0; u < nvalid; ++u) {
            const double* Jt = smem + u * STR + SH::WORK;
            const double rho = smem[u * STR + MRHO];
#pragma unroll
            for (int rs = 0; rs < NR / 4; ++rs) {
              const int row = rs * 4 + (lane & 3);
              const double a = rho * Jt[row * LDJ + ti * 8 + (lane >> 2)];
              const double b = Jt[row * LDJ + tj * 8 + (lane >> 2)];
              dmma(hacc[sl][0], hacc[sl][1], a, b);
            }
          }
        }
      }
      // gradient S/T and objective
      if (tid < K) {
        double g = 0.0;
        for (int u = 0; u < nvalid; ++u) {
          const double* S = smem + u * STR;
          const double* Jt = S + SH::WORK;
          double v = 0.0;
#pragma unroll
          for (int i = 0; i < NU; ++i) v = fma(Jt[i * LDJ + tid], S[SH::RT + i], v);
          if (tid >= ku) v = fma(S[SH::DNP + tid - ku], S[MN], v);
          g = fma(S[MRHO], v, g);
        }
        gacc += g;
      }
#pragma unroll
      for (int sl = 0; sl < 2; ++sl) {
        const int pi = tid + sl * DERIV_THREADS;
        if (pi < kx * kx) {
          const int a = pi / kx, b = pi % kx;
          double h = 0.0;
          for (int u = 0; u < nvalid; ++u) {
            const double* S = smem + u * STR;
            h = fma(S[MRHO] * S[SH::DNP + a], S[SH::DNP + b], h);
          }
          tacc[sl] += h;
        }
      }
      if (tid == 0) {
        double jv = 0.0;
        for (int u = 0; u < nvalid; ++u) {
          const double* S = smem + u * STR;
          double r2 = S[MN] * S[MN];
#pragma unroll
          for (int i = 0; i < NU; ++i) r2 = fma(S[SH::RT + i], S[SH::RT + i], r2);
          jv = fma(S[MRHO], r2, jv);
        }
        jacc += jv;
      }
    } else {
      // per-element contributions (reduced.py:231-251; LP rows eqp.py:97-114)
      const int nk = r.mode == MODE_CONTRIB_SPLIT ? 2 * K : K;
      for (int t = tid; t < nvalid * (nk + (r.mode == MODE_CONTRIB_LPROWS ? 1 : 0)); t += blockDim.x) {
        const int per = nk + (r.mode == MODE_CONTRIB_LPROWS ? 1 : 0);
        const int u = t / per, k2 = t % per;
        const double* S = smem + u * STR;
        const double* Jt = S + SH::WORK;
        const int e = UI[u].e;
        double v = 0.0;
        if (r.mode == MODE_CONTRIB_SPLIT) {
          // layout (Sv[ku], Sf[ku], Tv[kx], Tf[kx])
          int k, part;
          if (k2 < 2 * ku) { k = k2 % ku; part = k2 / ku; }
          else { k = ku + (k2 - 2 * ku) % kx; part = (k2 - 2 * ku) / kx; }
          const double* Rp = S + (part == 0 ? SH::RV : SH::RF);
#pragma unroll
          for (int i = 0; i < NU; ++i) v = fma(Jt[i * LDJ + k], Rp[i], v);
          if (k >= ku && part == 0) v = fma(S[SH::DNP + k - ku], S[MN], v);
          r.out[((size_t)p * r.ne + e) * nk + k2] = v;
        } else if (k2 < K) {
#pragma unroll
          for (int i = 0; i < NU; ++i) v = fma(Jt[i * LDJ + k2], S[SH::RT + i], v);
          if (k2 >= ku) v = fma(S[SH::DNP + k2 - ku], S[MN], v);
          if (r.mode == MODE_CONTRIB) r.out[((size_t)p * r.ne + e) * K + k2] = v;
          else r.out[((size_t)p * (K + 1) + k2) * r.ne + e] = v;
        } else {
          double r2 = S[MN] * S[MN];
#pragma unroll
          for (int i = 0; i < NU; ++i) r2 = fma(S[SH::RT + i], S[SH::RT + i], r2);
          r.out[((size_t)p * (K + 1) + K) * r.ne + e] = 0.5 * r2;
        }
      }
    }
  }
  if (r.mode != MODE_DERIVS) return;
  // ---- block partial: [J2, g(K), H(KP x KP) upper tiles] ---------------------------
  __syncthreads();
  const int PSZ = 1 + K + KP * KP;
  double* PB = smem;
  for (int i = tid; i < PSZ; i += blockDim.x) PB[i] = 0.0;
  __syncthreads();
#pragma unroll
  for (int sl = 0; sl < MAXT; ++sl) {
    const int tile8 = warp + 4 * sl;
    if (tile8 < ntri) {
      int ti = 0, rem = tile8;
      while (rem >= nt8 - ti) { rem -= nt8 - ti; ++ti; }
      const int tj = ti + rem;
      const int row = ti * 8 + (lane >> 2), col = tj * 8 + 2 * (lane & 3);
      PB[1 + K + row * KP + col] = hacc[sl][0];
      PB[1 + K + row * KP + col + 1] = hacc[sl][1];
    }
  }
  __syncthreads();
#pragma unroll
  for (int sl = 0; sl < 2; ++sl) {
    const int pi = tid + sl * DERIV_THREADS;
    if (pi < kx * kx) {
      const int a = pi / kx, b = pi % kx;
      if (a <= b) PB[1 + K + (ku + a) * KP + ku + b] += tacc[sl];
    }
  }
  if (tid < K) PB[1 + tid] = gacc;
  if (tid == 0) PB[0] = jacc;
  __syncthreads();
  double* dst = r.part + ((size_t)p * gridDim.x + blockIdx.x) * PSZ;
  for (int i = tid; i < PSZ; i += blockDim.x) dst[i] = PB[i];
}

__global__ void finalize_derivs_kernel(const double* __restrict__ part, int gx, int K, int KP, int P,
                                       double* __restrict__ out) {
  const int p = blockIdx.y;
  const int PSZ = 1 + K + KP * KP;
  const int OSZ = 1 + K + K * K;
  for (int o = blockIdx.x * blockDim.x + threadIdx.x; o < OSZ; o += gridDim.x * blockDim.x) {
    int src;
    if (o < 1 + K) src = o;
    else {
      int k = (o - 1 - K) / K, l = (o - 1 - K) % K;
      src = 1 + K + min(k, l) * KP + max(k, l);
    }
    double s = 0.0;
    for (int b = 0; b < gx; ++b) s += part[((size_t)p * gx + b) * PSZ + src];
    out[(size_t)p * OSZ + o] = o == 0 ? 0.5 * s : s;
  }
}

}  // namespace strom
