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
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
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

// d N / d x_d for one local coordinate direction d = 2*vertex + component
__device__ __forceinline__ double distortion_grad_dir(const Geo& o, double wsum, double eps, double kappa, int d) {
  const double fro2 = o.G[0][0] * o.G[0][0] + o.G[0][1] * o.G[0][1] + o.G[1][0] * o.G[1][0] + o.G[1][1] * o.G[1][1];
  const double den = o.g >= eps ? o.g : eps, iden = 1.0 / den;  // one reciprocal for ratio and its derivative
  const double ratio = fro2 * iden;
  const int gv = d >> 1, ic = d & 1;
  const double c0 = (gv == 1) - (gv == 0), c1 = (gv == 2) - (gv == 0);
  const double dJ00 = ic == 0 ? c0 : 0.0, dJ01 = ic == 0 ? c1 : 0.0, dJ10 = ic == 1 ? c0 : 0.0, dJ11 = ic == 1 ? c1 : 0.0;
  const double dG00 = dJ00 * o.invr[0][0] + dJ01 * o.invr[1][0], dG01 = dJ00 * o.invr[0][1] + dJ01 * o.invr[1][1];
  const double dG10 = dJ10 * o.invr[0][0] + dJ11 * o.invr[1][0], dG11 = dJ10 * o.invr[0][1] + dJ11 * o.invr[1][1];
  const double dg = dG00 * o.G[1][1] + o.G[0][0] * dG11 - dG01 * o.G[1][0] - o.G[0][1] * dG10;
  const double dfro = 2.0 * (o.G[0][0] * dG00 + o.G[0][1] * dG01 + o.G[1][0] * dG10 + o.G[1][1] * dG11);
  const double dden = o.g >= eps ? dg : 0.0;
  const double dratio = (dfro - ratio * dden) * iden;
  return kappa * wsum * o.detr * 2.0 * ratio * dratio;
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

static __global__ void eta_ref_kernel(int ne, const int* __restrict__ en, const double* __restrict__ nodes, double wsum,
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
  const double l2 = nu[0] * nu[0] + nu[1] * nu[1], il = rsqrt(l2);  // one rsqrt: |nu| and nu / |nu|
  len = l2 * il;
  nh[0] = nu[0] * il; nh[1] = nu[1] * il;
}

// row . w for a basis row of length ku <= 32 with w in registers (compile-time
// indexed, predicated), 16-byte loads of the row (broadcast when the warp shares it)
__device__ __forceinline__ double row_dot(const double* __restrict__ row, const double* wr, int ku) {
  double a0 = 0.0, a1 = 0.0;
  if ((ku & 1) == 0) {
    const double2* r2 = reinterpret_cast<const double2*>(row);
#pragma unroll
    for (int k2 = 0; k2 < 16; ++k2)
      if (2 * k2 < ku) {
        const double2 t = __ldg(r2 + k2);
        a0 = fma(t.x, wr[2 * k2], a0);
        a1 = fma(t.y, wr[2 * k2 + 1], a1);
      }
  } else {
#pragma unroll
    for (int k = 0; k < 32; ++k)
      if (k < ku) a0 = fma(__ldg(row + k), wr[k], a0);
  }
  return a0 + a1;
}

// same with w through an accessor (shared-memory column of the warp's parameter points)
template <class WGet>
__device__ __forceinline__ double row_dot_g(const double* __restrict__ row, WGet WG, int ku) {
  double a0 = 0.0, a1 = 0.0;
  if ((ku & 1) == 0) {
    const double2* r2 = reinterpret_cast<const double2*>(row);
#pragma unroll 4
    for (int k2 = 0; k2 < (ku >> 1); ++k2) {
      const double2 t = __ldg(r2 + k2);
      a0 = fma(t.x, WG(2 * k2), a0);
      a1 = fma(t.y, WG(2 * k2 + 1), a1);
    }
  } else {
    for (int k = 0; k < ku; ++k) a0 = fma(__ldg(row + k), WG(k), a0);
  }
  return a0 + a1;
}

// ============================================================================
// K2: element residual (value path) for one (element, mu); w / tau through the
// accessors WG(k) / TG(a) so one body serves both kernel layouts below
// ============================================================================
template <class LAW, int NB, int NQ, int NS, class WGet, class TGet>
__device__ __forceinline__ void value_unit(const Tabs<NB, NQ, NS, Shape<LAW, NB, NQ, NS>::NF>& T, const Run& r,
                                           const LawArgs& la, int e, int p, WGet WG, TGet TG,
                                           double* R, double& Nd, bool& degenerate) {
  using SH = Shape<LAW, NB, NQ, NS>;
  constexpr int M = SH::M, NU = SH::NU, NF = SH::NF, PD = SH::P;
  double x[6], X[6];
#pragma unroll
  for (int g = 0; g < 3; ++g) {
    int n = r.elem_nodes[3 * e + g];
    X[2 * g] = r.nodes[2 * n];
    X[2 * g + 1] = r.nodes[2 * n + 1];
#pragma unroll
    for (int ic = 0; ic < 2; ++ic) {
      int row = 2 * n + ic;
      double v = r.xref[(size_t)p * r.x_stride + row];
      const double* ps = r.psi + (size_t)row * r.kx;
      for (int a = 0; a < r.kx; ++a) v = fma(__ldg(ps + a), TG(a), v);
      x[2 * g + ic] = v;
    }
  }
  double U[NU];
  {
    const double* ph = r.phi + (size_t)e * NU * r.ku;
#pragma unroll
    for (int i = 0; i < NU; ++i) {
      const double v = r.u0 ? r.u0[(size_t)p * r.u0_stride + (size_t)e * NU + i] : 0.0;
      U[i] = v + row_dot_g(ph + i * r.ku, WG, r.ku);
    }
  }
  Geo o;
  element_geo(x, X, o);
  degenerate = o.g <= 0.0;
#pragma unroll
  for (int i = 0; i < NU; ++i) R[i] = 0.0;
  // volume (dg.py:105-125); rolled loop: keeps the kernel in the instruction cache
#pragma unroll 1
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
    PointVal<LAW>::flux(uq, f, la);
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
          const double v = r.u0 ? r.u0[(size_t)p * r.u0_stride + (size_t)nb * NU + row] : 0.0;
          Un[j][c] = v + row_dot_g(ph + row * r.ku, WG, r.ku);
        }
      }
    }
    double ghost[M];
    if (bc >= 2 && bc != BC_REFLECT && !LAW::GHOST_POS) LAW::ghost(bc - 2, la, nullptr, ghost);
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
      if constexpr (LAW::GHOST_POS) {  // ghost at the deformed face point (vertex part of the trace)
        const int va = f, vb = (f + 1) % 3;
        const double half = NF > 2 ? 0.5 * T.trace[f][s][NF - 1] : 0.0;
        const double la_ = T.trace[f][s][0] + half, lb_ = T.trace[f][s][1] + half;
        const double pos[2] = {la_ * x[2 * va] + lb_ * x[2 * vb], la_ * x[2 * va + 1] + lb_ * x[2 * vb + 1]};
        LAW::ghost(bc - 2, la, pos, ghost);
      }
#pragma unroll
        for (int c = 0; c < M; ++c) uo[c] = ghost[c];
      }
      double Hs[M];
      face_flux_val<LAW>(ui, uo, bc, nu, len, nh, la, Hs);
#pragma unroll
      for (int c = 0; c < M; ++c) {
        const double H = T.ws[s] * Hs[c];
#pragma unroll
        for (int j = 0; j < NF; ++j) R[fnode_of(PD, f, j) * M + c] = fma(T.trace[f][s][j], H, R[fnode_of(PD, f, j) * M + c]);
      }
    }
  }
  Nd = r.kappa * (distortion_eta(o, T.wsum, r.eps, nullptr, nullptr) - r.eta_ref[e]);
}

// one thread per (element, mu): grid (elements / 128, P)
template <class LAW, int NB, int NQ, int NS>
__global__ void __launch_bounds__(128) value_kernel(const __grid_constant__ Params<NB, NQ, NS, Shape<LAW, NB, NQ, NS>::NF> prm) {
  using SH = Shape<LAW, NB, NQ, NS>;
  constexpr int NU = SH::NU;
  const auto& T = prm.t;
  const Run& r = prm.r;
  const int p = blockIdx.y;
  if (r.mask && !r.mask[p]) return;
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
    double R[NU], N;
    bool deg;
    value_unit<LAW, NB, NQ, NS>(T, r, la, e, p, [&](int k) { return __ldg(w + k); }, [&](int a) { return __ldg(tau + a); }, R, N, deg);
    if (deg) flag_degenerate(r, p, e);
    if (r.mode == MODE_RESIDUAL) {
      double* o_ = r.out + ((size_t)p * r.ne + e) * NU;
#pragma unroll
      for (int i = 0; i < NU; ++i) o_[i] = R[i];
    } else {
      double r2 = 0.0;
#pragma unroll
      for (int i = 0; i < NU; ++i) r2 = fma(R[i], R[i], r2);
      contrib = r.mode == MODE_OBJECTIVE ? 0.5 * rho * (r2 + N * N) : r2;
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

// one warp per parameter row: lane-strided partials, fixed-order shuffle tree (deterministic)
struct DynRows {  // device-sized launch of the pass being finalized (Run::dyn_*), count == null: static grid
  const int* count;
  const int* list;
  int target, maxb, ceil_div;
};

static __global__ void sum_partials_kernel(const double* __restrict__ part, int nparts, int P, double* __restrict__ out,
                                    const int* __restrict__ mask, DynRows dyn) {
  // warp per row; device-sized value passes index their partials by the compacted slot
  const int s = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  int p = s;
  if (dyn.count) {
    const int live = *dyn.count;
    if (s >= live) return;
    p = dyn.list[s];
    nparts = dyn_gx(dyn.target, dyn.maxb, 1, (live + 31) / 32);
  } else if (p >= P || (mask && !mask[p])) {
    return;
  }
  double v = 0.0;
  for (int i = lane; i < nparts; i += 32) v += part[(size_t)s * nparts + i];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  if (lane == 0) out[p] = v;
}

// Sum the per-CTA partials of one derivatives pass and expand the upper Gram tiles
// into (J, S|T, H).  Block = 32 consecutive partial entries x 32 warps: warp w reads rows
// b = w, w+32, ... as coalesced 256-byte segments, the 32 warp sums are added in a fixed
// order (deterministic for a fixed grid), and each entry is written to the one or two
// outputs it feeds (H symmetric).
static __global__ void __launch_bounds__(1024) finalize_derivs_kernel(const double* __restrict__ part, int gx, int K,
                                                                      int KP, int P, double* __restrict__ out,
                                                                      const int* __restrict__ mask, DynRows dyn) {
  __shared__ double red[32][33];
  int p = blockIdx.y, prow = blockIdx.y;
  if (dyn.count) {  // row slot -> parameter row; the pass split the grid with the same formula
    const int live = *dyn.count;
    if (prow >= live) return;
    p = dyn.list[prow];
    gx = dyn_gx(dyn.target, dyn.maxb, dyn.ceil_div, live);
  } else if (mask && !mask[p]) {
    return;
  }
  const int PSZ = 1 + K + KP * KP, OSZ = 1 + K + K * K;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int src = blockIdx.x * 32 + lane;
  double s = 0.0;
  if (src < PSZ) {  // four independent sums in flight per warp (fixed order: deterministic per launch shape)
    const double* q = part + (size_t)prow * gx * PSZ + src;
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    int b = w;
    for (; b + 3 * nw < gx; b += 4 * nw) {
      s0 += q[(size_t)b * PSZ];
      s1 += q[(size_t)(b + nw) * PSZ];
      s2 += q[(size_t)(b + 2 * nw) * PSZ];
      s3 += q[(size_t)(b + 3 * nw) * PSZ];
    }
    for (; b < gx; b += nw) s0 += q[(size_t)b * PSZ];
    s = (s0 + s1) + (s2 + s3);
  }
  red[w][lane] = s;
  __syncthreads();
  if (w != 0 || src >= PSZ) return;
  double v = red[0][lane];
  for (int i = 1; i < nw; ++i) v += red[i][lane];
  double* o = out + (size_t)p * OSZ;
  if (src == 0) {
    o[0] = 0.5 * v;
  } else if (src <= K) {
    o[src] = v;
  } else {
    const int d = src - 1 - K, k = d / KP, l = d % KP;
    if (k <= l && l < K) {
      o[1 + K + k * K + l] = v;
      if (k != l) o[1 + K + l * K + k] = v;
    }
  }
}

}  // namespace strom
