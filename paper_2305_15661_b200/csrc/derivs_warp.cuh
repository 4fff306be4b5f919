// K1 / K3 derivatives kernel, warp-synchronous version.
//
// Each warp owns UPW = 32/TPU elements at a time; the TPU lanes of an
// element double as its tangent lanes (lane k <-> reduced state direction
// k).  No block-level barrier inside the element loop: all stages are
// separated by __syncwarp and work on warp-private shared memory.
//   S1  gather: lane k loads column k of Phi_e (coalesced 8*k_u-byte rows)
//       and of the neighbor face-node rows; U_e = U0 + Phi_e w and the
//       neighbor traces are reduced across lanes with shuffle butterflies
//   S2  pointwise physics on the volume / face points (lane = point):
//       B_q = w_q d(f . adj(Jx)_k)/du, face C_in/C_out (LLF linearisation),
//       analytic Jacobians for Euler, forward-mode duals otherwise
//   S3  residual rows (volume / face split) and the mesh-tangent helper Tq
//   S4  state tangents: lane k forms column k of J_e = dR/dU Phi_e + sum_f
//       dR/dU_nf Phi_nf with reference-element tables as constant-bank
//       operands (DFMA) and B_q / C as broadcast shared-memory loads
//   S5  mesh tangents in the 6 local directions, projected on Psi_e
//   S6  rho-weighted Gram of the element Jacobians on DMMA (mma.sync
//       m8n8k4 f64) into warp accumulators, plus S/T/J; or per-element
//       contributions (K3)
#pragma once
#include "element_kernels.cuh"

namespace strom {

constexpr int WTHREADS = 256;

template <class LAW, int NB, int NQ, int NS>
struct WShape {
  static constexpr int M = LAW::M;
  static constexpr int P = NB == 3 ? 1 : 2;
  static constexpr int NF = P + 1;
  static constexpr int NU = NB * M;
  static constexpr int NR = (NU + 3) / 4 * 4;
  static constexpr int NFS = 3 * NS;
  static constexpr int NNB = 3 * NF * M;             // neighbor face-node values
  static constexpr int NQP = NQ % 2 ? NQ : NQ + 1;   // padded point strides (bank spread)
  static constexpr int NFSP = NFS % 2 ? NFS : NFS + 1;
  static constexpr int NUP = NU + 1;
  // meta slots
  static constexpr int MX = 0, MJ = 6, MADJ = 10, MDET = 14, MDETR = 15, MNU = 16, MNLEN = 22, MNHAT = 25,
                       MN = 31, MRHO = 32, DNX = 33, DNP = 40, MINT = 56;  // 8 ints at MINT
  static constexpr int UE = 64;
  static constexpr int UNF = UE + NU;
  static constexpr int RT = UNF + NNB;
  static constexpr int RV = RT + NU;
  static constexpr int RF = RV + NU;
  static constexpr int TQ = RF + NU;                 // [4][NU]
  static constexpr int FXS = 3 * M + 3;              // fields per face point
  static constexpr int FX = TQ + 4 * NU;             // [field][fs] (stride NFSP)
  static constexpr int SW = FX + FXS * NFSP;         // [c][q] (stride NQP)
  static constexpr int SP = SW + (LAW::SRC != SRC_NONE ? M * NQP : 0);  // [c][i][q]
  static constexpr int RB = SP + (LAW::SRC == SRC_POS ? 2 * M * NQP : 0);
  // region B: FQ [c][i][q] + HS [c][fs]  |  dRx [d][NUP]
  static constexpr int FQ = 0;
  static constexpr int HS = 2 * M * NQP;
  static constexpr int RB_A = HS + M * NFSP;
  static constexpr int RB_B = 6 * NUP;
  static constexpr int RBSZ = RB_A > RB_B ? RB_A : RB_B;
  static constexpr int RA = RB + RBSZ;
  // region A: BQ [c][kk][c'][q] + BS [c][c'][q] + CF [side][c][c'][fs]  |  Jt [NR][LDJ]
  static constexpr int BQ = 0;
  static constexpr int BS = 2 * M * M * NQ;
  static constexpr int CF = BS + (LAW::SRC == SRC_U ? M * M * NQ : 0);
  static constexpr int RA_A = CF + 2 * M * M * NFS;
  __host__ __device__ static int unit_stride(int LDJ) {
    int a = RA_A > NR * LDJ ? RA_A : NR * LDJ;
    int s = RA + a;
    return (s + 15) / 16 * 16 + 2;  // 16-byte offset between units
  }
  __host__ __device__ static int warp_stride(int LDJ, int KP, int UPW) {
    int s = UPW * unit_stride(LDJ) + KP * KP + 48;  // + H accumulator + g/J slots
    return (s + 15) / 16 * 16 + 4;
  }
};

// reduce-scatter butterfly over the TPU lanes of a unit: every lane holds
// v[0..V) ; afterwards lane k holds sum over lanes of v[k*V/TPU + j] in v[j]
template <int V, int TPU>
__device__ __forceinline__ void butterfly(double* v, int lane) {
  int L = V;
#pragma unroll
  for (int o = TPU / 2; o >= 1; o >>= 1) {
    const bool up = (lane & o) != 0;
    const int half = L / 2;
#pragma unroll
    for (int j = 0; j < V / 2; ++j) {
      if (j < half) {
        const double send = up ? v[j] : v[j + half];
        const double keep = up ? v[j + half] : v[j];
        v[j] = keep + __shfl_xor_sync(0xffffffffu, send, o);
      }
    }
    L = half;
  }
}

template <class LAW, int NB, int NQ, int NS, int TPU>
__global__ void __launch_bounds__(WTHREADS) derivs_warp_kernel(
    const __grid_constant__ Params<NB, NQ, NS, WShape<LAW, NB, NQ, NS>::NF> prm) {
  using SH = WShape<LAW, NB, NQ, NS>;
  constexpr int M = SH::M, NU = SH::NU, NF = SH::NF, NR = SH::NR, PD = SH::P, NFS = SH::NFS;
  constexpr int NQP = SH::NQP, NFSP = SH::NFSP, NUP = SH::NUP;
  constexpr int UPW = 32 / TPU;
  constexpr int VN = TPU == 16 ? 48 : 64;  // padded neighbor butterfly width
  static_assert(SH::NNB <= VN, "neighbor trace count exceeds butterfly width");
  const auto& T = prm.t;
  const Run& r = prm.r;
  extern __shared__ __align__(16) double smem[];
  __shared__ double s_w[KMAX], s_tau[KMAX];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  const int h = lane / TPU, k = lane % TPU;
  // CTA -> (parameter row, element chunk): grid (gx, P) with a row mask, or a device-sized
  // 1-D grid over the live rows list[0 .. *dyn_count) (graph-resident LM rounds)
  int p, prow_, bx, gxr;
  if (r.dyn_count) {
    const int live = *r.dyn_count;
    gxr = dyn_gx(r.dyn_target, r.dyn_maxb, r.dyn_ceil, live);
    prow_ = blockIdx.x / gxr;
    bx = blockIdx.x - prow_ * gxr;
    if (prow_ >= live) return;
    p = r.list[prow_];
  } else {
    p = prow_ = blockIdx.y;
    bx = blockIdx.x;
    gxr = gridDim.x;
    if (r.mask && !r.mask[p]) return;
  }
  const int ku = r.ku, kx = r.kx, K = r.K, KP = r.KP, LDJ = r.LDJ, STR = r.unit_stride;
  double* const Wb = smem + (size_t)warp * r.gx_warp_stride;
  double* const S = Wb + h * STR;
  int* const SI = reinterpret_cast<int*>(S + SH::MINT);
  double* const HACC = Wb + UPW * STR;
  double* const GW = HACC + KP * KP;

  for (int i = threadIdx.x; i < ku; i += blockDim.x) s_w[i] = r.w[(size_t)p * ku + i];
  for (int i = threadIdx.x; i < kx; i += blockDim.x) s_tau[i] = r.tau[(size_t)p * kx + i];
  for (int i = lane; i < KP * KP; i += 32) HACC[i] = 0.0;
  LawArgs la;
#pragma unroll
  for (int i = 0; i < 8; ++i) la.p[i] = r.lawp[i];
#pragma unroll
  for (int i = 0; i < NMU; ++i) la.mu[i] = i < r.nmu ? r.mu[p * r.nmu + i] : 0.0;
  __syncthreads();

  double gacc0 = 0.0, gacc1 = 0.0, jacc = 0.0;
  const int nunits = r.active ? r.A : r.ne;
  const int ngroups = (nunits + UPW - 1) / UPW;
  const int nt8 = KP / 8, ntri = nt8 * (nt8 + 1) / 2;

  for (int grp = bx * nwarps + warp; grp < ngroups; grp += gxr * nwarps) {
    const int idx = grp * UPW + h;
    const bool valid = idx < nunits;
    const int nvalid = min(UPW, nunits - grp * UPW);
    const int e = valid ? (r.active ? r.active[idx] : idx) : (r.active ? r.active[grp * UPW] : grp * UPW);
    const double rho = valid ? (r.active ? r.rho[idx] : 1.0) : 0.0;
    int nbr[3], fin[3];
#pragma unroll
    for (int f = 0; f < 3; ++f) { nbr[f] = r.nbr[3 * e + f]; fin[f] = r.finfo[3 * e + f]; }
    // ---- S1: coordinates and gathers ------------------------------------------------
    if (k < 6) {
      const int n = r.elem_nodes[3 * e + (k >> 1)];
      const int row = 2 * n + (k & 1);
      double v = r.xref[(size_t)p * r.x_stride + row];
      const double* ps = r.psi + (size_t)row * kx;
      for (int a = 0; a < kx; ++a) v = fma(ps[a], s_tau[a], v);
      S[SH::MX + k] = v;
    }
    if (k == 0) {
      S[SH::MRHO] = rho;
      SI[0] = e;
    }
    {
      const double wk = k < ku ? s_w[k] : 0.0;
      double v[32];
      const double* ph = r.phi + (size_t)e * NU * ku + k;
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] = (i < NU && k < ku) ? __ldg(ph + (size_t)i * ku) * wk : 0.0;
      butterfly<32, TPU>(v, k);
#pragma unroll
      for (int j = 0; j < 32 / TPU; ++j) {
        const int i = k * (32 / TPU) + j;
        if (i < NU) S[SH::UE + i] = v[j] + (r.u0 ? r.u0[(size_t)p * r.u0_stride + (size_t)e * NU + i] : 0.0);
      }
    }
    {
      const double wk = k < ku ? s_w[k] : 0.0;
      double v[VN];
#pragma unroll
      for (int i = 0; i < VN; ++i) v[i] = 0.0;
#pragma unroll
      for (int f = 0; f < 3; ++f) {
        if ((fin[f] >> 3) == 0 && k < ku) {
          const int nf = fin[f] & 3;
          const double* phn = r.phi + (size_t)nbr[f] * NU * ku + k;
#pragma unroll
          for (int j = 0; j < NF; ++j) {
            const int node = j == 0 ? nf : (j == 1 ? (nf + 1) % 3 : 3 + nf * (PD - 1) + (j - 2));
#pragma unroll
            for (int c = 0; c < M; ++c) v[(f * NF + j) * M + c] = __ldg(phn + (size_t)(node * M + c) * ku) * wk;
          }
        }
      }
      butterfly<VN, TPU>(v, k);
#pragma unroll
      for (int j = 0; j < VN / TPU; ++j) {
        const int i = k * (VN / TPU) + j;
        if (i < SH::NNB) {
          const int f = i / (NF * M), jj = (i / M) % NF, c = i % M;
          double off = 0.0;
          if (r.u0 && (fin[f] >> 3) == 0) {
            const int nf = fin[f] & 3;
            const int node = jj == 0 ? nf : (jj == 1 ? (nf + 1) % 3 : 3 + nf * (PD - 1) + (jj - 2));
            off = r.u0[(size_t)p * r.u0_stride + (size_t)nbr[f] * NU + node * M + c];
          }
          S[SH::UNF + i] = v[j] + off;
        }
      }
    }
    __syncwarp();
    // element geometry, normals, distortion (one lane per unit)
    if (k == 0) {
      double X[6];
#pragma unroll
      for (int g = 0; g < 3; ++g) {
        const int n = r.elem_nodes[3 * e + g];
        X[2 * g] = r.nodes[2 * n];
        X[2 * g + 1] = r.nodes[2 * n + 1];
      }
      Geo o;
      element_geo(S + SH::MX, X, o);
      if (valid && o.g <= 0.0) flag_degenerate(r, p, e);
      S[SH::MJ + 0] = o.J[0][0]; S[SH::MJ + 1] = o.J[0][1]; S[SH::MJ + 2] = o.J[1][0]; S[SH::MJ + 3] = o.J[1][1];
      S[SH::MADJ + 0] = o.adj[0][0]; S[SH::MADJ + 1] = o.adj[0][1]; S[SH::MADJ + 2] = o.adj[1][0]; S[SH::MADJ + 3] = o.adj[1][1];
      S[SH::MDET] = o.detJ;
      S[SH::MDETR] = o.detr;
#pragma unroll
      for (int f = 0; f < 3; ++f) face_normal(S + SH::MX, f, S + SH::MNU + 2 * f, S[SH::MNLEN + f], S + SH::MNHAT + 2 * f);
      S[SH::MN] = r.kappa * (distortion_eta(o, T.wsum, r.eps, nullptr, nullptr) - r.eta_ref[e]);
      distortion_grad(o, T.wsum, r.eps, r.kappa, S + SH::DNX);
    }
    __syncwarp();
    // ---- S2: pointwise physics ------------------------------------------------------------
    double* const RA = S + SH::RA;
    double* const RBp = S + SH::RB;
    for (int fs = k; fs < NFS; fs += TPU) {
      const int f = fs / NS, s = fs % NS;
      const int fi = fin[f], bc = fi >> 3;
      const double* nu = S + SH::MNU + 2 * f;
      const double len = S[SH::MNLEN + f];
      const double* nh = S + SH::MNHAT + 2 * f;
      double ui[M], uo[M];
#pragma unroll
      for (int c = 0; c < M; ++c) {
        double v = 0.0;
#pragma unroll
        for (int j = 0; j < NF; ++j) v = fma(T.trace[f][s][j], S[SH::UE + fnode_of(PD, f, j) * M + c], v);
        ui[c] = v;
      }
      if (bc == 0) {
        const int sp = ((fi >> 2) & 1) ? NS - 1 - s : s;
#pragma unroll
        for (int c = 0; c < M; ++c) {
          double v = 0.0;
#pragma unroll
          for (int j = 0; j < NF; ++j) v = fma(T.trace[0][sp][j], S[SH::UNF + (f * NF + j) * M + c], v);
          uo[c] = v;
        }
      } else if (bc == 1) {
#pragma unroll
        for (int c = 0; c < M; ++c) uo[c] = ui[c];
      } else {
        // deformed position of the face point: the vertex part of the trace (the edge-node
        // function splits evenly between the two vertices on a straight face)
        const int va = f, vb = (f + 1) % 3;
        const double half = NF > 2 ? 0.5 * T.trace[f][s][NF - 1] : 0.0;
        const double la_ = T.trace[f][s][0] + half, lb_ = T.trace[f][s][1] + half;
        const double pos[2] = {la_ * S[SH::MX + 2 * va] + lb_ * S[SH::MX + 2 * vb],
                               la_ * S[SH::MX + 2 * va + 1] + lb_ * S[SH::MX + 2 * vb + 1]};
        LAW::ghost(bc - 2, la, pos, uo);
      }
      double fni[M], fno[M], Ai[M][M], Ao[M][M];
      PointOps<LAW>::flux_dir(ui, nu, fni, Ai, la);
      PointOps<LAW>::flux_dir(uo, nu, fno, Ao, la);
      double gi[M], go[M], gni[2], gno[2];
      const double wsi = PointOps<LAW>::wavespeed_grad(ui, nh, gi, gni, la);
      const double wso = PointOps<LAW>::wavespeed_grad(uo, nh, go, gno, la);
      const bool in_wins = wsi >= wso;  // dual.maximum tie -> first argument (dual.py:171)
      const double lam = in_wins ? wsi : wso;
      const double ws = T.ws[s];
      double fi2[M][2], fo2[M][2];
      LAW::flux(ui, fi2, la);
      LAW::flux(uo, fo2, la);
      double* FXp = S + SH::FX;
#pragma unroll
      for (int c = 0; c < M; ++c) {
        const double du = uo[c] - ui[c];
        RBp[SH::HS + c * NFSP + fs] = ws * (0.5 * (fni[c] + fno[c]) - 0.5 * (lam * len) * du);
        FXp[(2 * c + 0) * NFSP + fs] = 0.5 * ws * (fi2[c][0] + fo2[c][0]);
        FXp[(2 * c + 1) * NFSP + fs] = 0.5 * ws * (fi2[c][1] + fo2[c][1]);
        FXp[(2 * M + c) * NFSP + fs] = 0.5 * ws * du;
#pragma unroll
        for (int cp = 0; cp < M; ++cp) {
          const double dl_in = in_wins ? gi[cp] : 0.0;
          const double dl_out = in_wins ? 0.0 : go[cp];
          double cin = 0.5 * Ai[c][cp] + (c == cp ? 0.5 * lam * len : 0.0) - 0.5 * len * du * dl_in;
          double cout = 0.5 * Ao[c][cp] - (c == cp ? 0.5 * lam * len : 0.0) - 0.5 * len * du * dl_out;
          if (bc == 1) { cin += cout; cout = 0.0; }
          if (bc >= 2) cout = 0.0;
          RA[SH::CF + ((0 * M + c) * M + cp) * NFS + fs] = ws * cin;
          RA[SH::CF + ((1 * M + c) * M + cp) * NFS + fs] = ws * cout;
        }
      }
      FXp[(3 * M + 0) * NFSP + fs] = lam;
      FXp[(3 * M + 1) * NFSP + fs] = in_wins ? gni[0] : gno[0];
      FXp[(3 * M + 2) * NFSP + fs] = in_wins ? gni[1] : gno[1];
    }
    for (int q = k; q < NQ; q += TPU) {
      double uq[M];
#pragma unroll
      for (int c = 0; c < M; ++c) {
        double v = 0.0;
#pragma unroll
        for (int n = 0; n < NB; ++n) v = fma(T.phi[q][n], S[SH::UE + n * M + c], v);
        uq[c] = v;
      }
      const double wq = T.wq[q];
      double f2[M][2];
      LAW::flux(uq, f2, la);
#pragma unroll
      for (int c = 0; c < M; ++c) {
        RBp[SH::FQ + (c * 2 + 0) * NQP + q] = wq * f2[c][0];
        RBp[SH::FQ + (c * 2 + 1) * NQP + q] = wq * f2[c][1];
      }
#pragma unroll
      for (int kk = 0; kk < 2; ++kk) {
        const double dir[2] = {S[SH::MADJ + 2 * kk], S[SH::MADJ + 2 * kk + 1]};
        double fn[M], Am[M][M];
        PointOps<LAW>::flux_dir(uq, dir, fn, Am, la);
#pragma unroll
        for (int c = 0; c < M; ++c)
#pragma unroll
          for (int cp = 0; cp < M; ++cp) RA[SH::BQ + ((c * 2 + kk) * M + cp) * NQ + q] = wq * Am[c][cp];
      }
      if (LAW::SRC != SRC_NONE) {
        Dn<M + 2> us[M], ps[2];
#pragma unroll
        for (int c = 0; c < M; ++c) us[c] = seed<M + 2>(uq[c], c);
#pragma unroll
        for (int i = 0; i < 2; ++i)
          ps[i] = seed<M + 2>(T.bary[q][0] * S[SH::MX + i] + T.bary[q][1] * S[SH::MX + 2 + i] + T.bary[q][2] * S[SH::MX + 4 + i], M + i);
        Dn<M + 2> sv[M];
        LAW::source(ps, us, sv, la);
        const double detJ = S[SH::MDET];
#pragma unroll
        for (int c = 0; c < M; ++c) {
          S[SH::SW + c * NQP + q] = wq * sv[c].v;
          if (LAW::SRC == SRC_POS) {
            S[SH::SP + (c * 2 + 0) * NQP + q] = wq * detJ * sv[c].d[M + 0];
            S[SH::SP + (c * 2 + 1) * NQP + q] = wq * detJ * sv[c].d[M + 1];
          }
          if (LAW::SRC == SRC_U) {
#pragma unroll
            for (int cp = 0; cp < M; ++cp) RA[SH::BS + (c * M + cp) * NQ + q] = wq * detJ * sv[c].d[cp];
          }
        }
      }
    }
    __syncwarp();
    // ---- S3: residual rows and Tq ----------------------------------------------------------
    for (int i = k; i < NU; i += TPU) {
      const int n = i / M, c = i % M;
      double tq[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        const double f0 = RBp[SH::FQ + (c * 2 + 0) * NQP + q], f1 = RBp[SH::FQ + (c * 2 + 1) * NQP + q];
        tq[0][0] = fma(T.dphi[q][n][0], f0, tq[0][0]);
        tq[0][1] = fma(T.dphi[q][n][0], f1, tq[0][1]);
        tq[1][0] = fma(T.dphi[q][n][1], f0, tq[1][0]);
        tq[1][1] = fma(T.dphi[q][n][1], f1, tq[1][1]);
      }
      const double* adj = S + SH::MADJ;
      double rv = -(adj[0] * tq[0][0] + adj[1] * tq[0][1] + adj[2] * tq[1][0] + adj[3] * tq[1][1]);
      if (LAW::SRC != SRC_NONE) {
        double sacc = 0.0;
#pragma unroll
        for (int q = 0; q < NQ; ++q) sacc = fma(T.phi[q][n], S[SH::SW + c * NQP + q], sacc);
        rv -= S[SH::MDET] * sacc;
      }
      double rf = 0.0;
#pragma unroll
      for (int f = 0; f < 3; ++f)
#pragma unroll
        for (int j = 0; j < NF; ++j)
          if (fnode_of(PD, f, j) == n)
#pragma unroll
            for (int s = 0; s < NS; ++s) rf = fma(T.trace[f][s][j], RBp[SH::HS + c * NFSP + f * NS + s], rf);
      S[SH::TQ + 0 * NU + i] = tq[0][0];
      S[SH::TQ + 1 * NU + i] = tq[0][1];
      S[SH::TQ + 2 * NU + i] = tq[1][0];
      S[SH::TQ + 3 * NU + i] = tq[1][1];
      S[SH::RV + i] = rv;
      S[SH::RF + i] = rf;
      S[SH::RT + i] = rv + rf;
    }
    __syncwarp();
    // ---- element Jacobian blocks against a bound test space (STROM_ELEMJAC_ENRICHED: the full-space
    // assembly of dg.py:197-326 for every law this kernel serves; the test space may be the trial
    // space itself): the pointwise records of S2 / S3 contracted with the test tabulations,
    // out[e] = [res (NT) | dR/dU_e (NT x NU) | dR/dU_nbr (NT x 3 NU) | dR/dx_e (NT x 6) | N_e | dN_e/dx_e]
    if (r.mode == MODE_ELEMJAC_ENRICHED) {
      const int NBT = r.test_nb, NT = NBT * M;
      const double* __restrict__ tdphi = r.test_tab;            // [NQ][NBT][2]
      const double* __restrict__ ttr = tdphi + NQ * NBT * 2;    // [3][NS][NBT]
      const double* __restrict__ tphi = ttr + 3 * NS * NBT;     // [NQ][NBT]
      double* const eo = r.out + (size_t)e * ((size_t)NT * (1 + 4 * NU + 6) + 7);
      const double* adj = S + SH::MADJ;
      const double* Jm = S + SH::MJ;
      const double detJ = S[SH::MDET];
      const double* FX0 = S + SH::FX;
      if (valid) {
        for (int i = k; i < NT; i += TPU) {  // residual row (n, c) and its six mesh derivatives
          const int n = i / M, c = i % M;
          double t00 = 0.0, t01 = 0.0, t10 = 0.0, t11 = 0.0, sacc = 0.0;
          for (int q = 0; q < NQ; ++q) {
            const double d0 = tdphi[(q * NBT + n) * 2], d1 = tdphi[(q * NBT + n) * 2 + 1];
            const double f0 = RBp[SH::FQ + (c * 2 + 0) * NQP + q], f1 = RBp[SH::FQ + (c * 2 + 1) * NQP + q];
            t00 = fma(d0, f0, t00); t01 = fma(d0, f1, t01); t10 = fma(d1, f0, t10); t11 = fma(d1, f1, t11);
            if (LAW::SRC != SRC_NONE) sacc = fma(tphi[q * NBT + n], S[SH::SW + c * NQP + q], sacc);
          }
          double rv = -(adj[0] * t00 + adj[1] * t01 + adj[2] * t10 + adj[3] * t11);
          if (LAW::SRC != SRC_NONE) rv -= detJ * sacc;
          double rf = 0.0;
          for (int fs = 0; fs < NFS; ++fs) rf = fma(ttr[fs * NBT + n], RBp[SH::HS + c * NFSP + fs], rf);
          eo[i] = rv + rf;
          for (int d = 0; d < 6; ++d) {
            const int gv = d >> 1, ic = d & 1;
            const double c0 = (gv == 1) - (gv == 0), c1 = (gv == 2) - (gv == 0);
            const double dJ00 = ic == 0 ? c0 : 0.0, dJ01 = ic == 0 ? c1 : 0.0, dJ10 = ic == 1 ? c0 : 0.0, dJ11 = ic == 1 ? c1 : 0.0;
            double v = -(dJ11 * t00 - dJ01 * t01 - dJ10 * t10 + dJ00 * t11);
            if (LAW::SRC != SRC_NONE) {
              const double ddet = dJ00 * Jm[3] + Jm[0] * dJ11 - dJ01 * Jm[2] - Jm[1] * dJ10;
              double sv = 0.0;
              for (int q = 0; q < NQ; ++q) {
                double term = ddet * S[SH::SW + c * NQP + q];
                if (LAW::SRC == SRC_POS) term += S[SH::SP + (c * 2 + ic) * NQP + q] * T.bary[q][gv];
                sv = fma(tphi[q * NBT + n], term, sv);
              }
              v -= sv;
            }
            for (int f = 0; f < 3; ++f) {
              const int a = f, b = (f + 1) % 3;
              const double del = (gv == b) - (gv == a);
              if (del == 0.0) continue;
              const double dnu0 = ic == 0 ? 0.0 : del, dnu1 = ic == 0 ? -del : 0.0;
              const double* nh = S + SH::MNHAT + 2 * f;
              const double len = S[SH::MNLEN + f];
              const double dlen = nh[0] * dnu0 + nh[1] * dnu1;
              const double dnh0 = (dnu0 - nh[0] * dlen) / len, dnh1 = (dnu1 - nh[1] * dlen) / len;
              for (int s = 0; s < NS; ++s) {
                const double* FXp = FX0 + f * NS + s;
                const double lam = FXp[(3 * M) * NFSP];
                const double dlam = FXp[(3 * M + 1) * NFSP] * dnh0 + FXp[(3 * M + 2) * NFSP] * dnh1;
                const double coef = dlam * len + lam * dlen;
                const double dH = FXp[(2 * c) * NFSP] * dnu0 + FXp[(2 * c + 1) * NFSP] * dnu1 - FXp[(2 * M + c) * NFSP] * coef;
                v = fma(ttr[(f * NS + s) * NBT + n], dH, v);
              }
            }
            eo[(size_t)NT * (1 + 4 * NU) + i * 6 + d] = v;
          }
        }
        for (int i = k; i < NT * NU; i += TPU) {  // dR/dU_e
          const int row = i / NU, col = i % NU, n = row / M, c = row % M, np_ = col / M, cp = col % M;
          double v = 0.0;
          for (int q = 0; q < NQ; ++q) {
            double g = fma(tdphi[(q * NBT + n) * 2], RA[SH::BQ + ((c * 2 + 0) * M + cp) * NQ + q],
                           tdphi[(q * NBT + n) * 2 + 1] * RA[SH::BQ + ((c * 2 + 1) * M + cp) * NQ + q]);
            if (LAW::SRC == SRC_U) g = fma(tphi[q * NBT + n], RA[SH::BS + (c * M + cp) * NQ + q], g);
            v = fma(-g, T.phi[q][np_], v);
          }
          for (int f = 0; f < 3; ++f)
            for (int j = 0; j < NF; ++j) {
              if (fnode_of(PD, f, j) != np_) continue;
              for (int s = 0; s < NS; ++s)
                v = fma(ttr[(f * NS + s) * NBT + n] * T.trace[f][s][j], RA[SH::CF + (c * M + cp) * NFS + f * NS + s], v);
            }
          eo[NT + i] = v;
        }
        for (int i = k; i < NT * 3 * NU; i += TPU) {  // dR/dU_nbr: the neighbor's face-node columns
          const int row = i / (3 * NU), col = i % (3 * NU), n = row / M, c = row % M;
          const int f = col / NU, node = (col % NU) / M, cp = col % M;
          const int fi = r.finfo[3 * e + f];
          double v = 0.0;
          if ((fi >> 3) == 0) {
            const int nf = fi & 3;
            int jn = -1;
            for (int j = 0; j < NF; ++j) {
              const int nodej = j == 0 ? nf : (j == 1 ? (nf + 1) % 3 : 3 + nf * (PD - 1) + (j - 2));
              if (nodej == node) jn = j;
            }
            if (jn >= 0)
              for (int s = 0; s < NS; ++s) {
                const int sp = ((fi >> 2) & 1) ? NS - 1 - s : s;
                v = fma(ttr[(f * NS + s) * NBT + n] * T.trace[0][sp][jn],
                        RA[SH::CF + M * M * NFS + (c * M + cp) * NFS + f * NS + s], v);
              }
          }
          eo[NT + NT * NU + i] = v;
        }
        if (k < 7) eo[(size_t)NT * (1 + 4 * NU + 6) + k] = k == 0 ? S[SH::MN] : S[SH::DNX + k - 1];
      }
      __syncwarp();
      continue;
    }
    // ---- S4: state tangents (lane k = direction k) ---------------------------------------
    double acc[NU];
#pragma unroll
    for (int i = 0; i < NU; ++i) acc[i] = 0.0;
    {
      // prefetch the next group's basis blocks into L2 while this one computes
      const int ng = grp + gxr * nwarps;
      if (ng < ngroups) {
        const int ni = ng * UPW + h;
        if (ni < nunits) {
          const int ne_ = r.active ? r.active[ni] : ni;
          const char* base = reinterpret_cast<const char*>(r.phi + (size_t)ne_ * NU * ku);
          const int nbytes = NU * ku * 8;
          for (int off = k * 128; off < nbytes; off += TPU * 128) asm volatile("prefetch.global.L2 [%0];" ::"l"(base + off));
        }
      }
    }
    if (k < ku) {
      double pc[NU];
      const double* ph = r.phi + (size_t)e * NU * ku + k;
#pragma unroll
      for (int i = 0; i < NU; ++i) pc[i] = __ldg(ph + (size_t)i * ku);
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
        const double* B = RA + SH::BQ + q;
#pragma unroll
        for (int c = 0; c < M; ++c) {
          double g0 = 0.0, g1 = 0.0;
#pragma unroll
          for (int cp = 0; cp < M; ++cp) {
            g0 = fma(B[((c * 2 + 0) * M + cp) * NQ], du[cp], g0);
            g1 = fma(B[((c * 2 + 1) * M + cp) * NQ], du[cp], g1);
          }
#pragma unroll
          for (int n = 0; n < NB; ++n) acc[n * M + c] = fma(-T.dphi[q][n][0], g0, fma(-T.dphi[q][n][1], g1, acc[n * M + c]));
        }
        if (LAW::SRC == SRC_U) {
          const double* Bs = RA + SH::BS + q;
#pragma unroll
          for (int c = 0; c < M; ++c) {
            double sv = 0.0;
#pragma unroll
            for (int cp = 0; cp < M; ++cp) sv = fma(Bs[(c * M + cp) * NQ], du[cp], sv);
#pragma unroll
            for (int n = 0; n < NB; ++n) acc[n * M + c] = fma(-T.phi[q][n], sv, acc[n * M + c]);
          }
        }
      }
#pragma unroll
      for (int f = 0; f < 3; ++f) {
        const int fi = fin[f], bc = fi >> 3;
        double pn[NF][M];
        if (bc == 0) {
          const int nf = fi & 3;
          const double* phn = r.phi + (size_t)nbr[f] * NU * ku + k;
#pragma unroll
          for (int j = 0; j < NF; ++j) {
            const int node = j == 0 ? nf : (j == 1 ? (nf + 1) % 3 : 3 + nf * (PD - 1) + (j - 2));
#pragma unroll
            for (int c = 0; c < M; ++c) pn[j][c] = __ldg(phn + (size_t)(node * M + c) * ku);
          }
        }
        const bool flip = (fi >> 2) & 1;
#pragma unroll
        for (int s = 0; s < NS; ++s) {
          const int fs = f * NS + s;
          double di[M];
#pragma unroll
          for (int c = 0; c < M; ++c) {
            double v = 0.0;
#pragma unroll
            for (int j = 0; j < NF; ++j) v = fma(T.trace[f][s][j], pc[fnode_of(PD, f, j) * M + c], v);
            di[c] = v;
          }
          const double* Cin = RA + SH::CF + fs;
          const double* Cout = RA + SH::CF + M * M * NFS + fs;
          double dH[M];
#pragma unroll
          for (int c = 0; c < M; ++c) {
            double v = 0.0;
#pragma unroll
            for (int cp = 0; cp < M; ++cp) v = fma(Cin[(c * M + cp) * NFS], di[cp], v);
            dH[c] = v;
          }
          if (bc == 0) {
            double dO[M];
#pragma unroll
            for (int c = 0; c < M; ++c) {
              double v0 = 0.0, v1 = 0.0;
#pragma unroll
              for (int j = 0; j < NF; ++j) {
                v0 = fma(T.trace[0][s][j], pn[j][c], v0);
                v1 = fma(T.trace[0][NS - 1 - s][j], pn[j][c], v1);
              }
              dO[c] = flip ? v1 : v0;
            }
#pragma unroll
            for (int c = 0; c < M; ++c) {
              double v = dH[c];
#pragma unroll
              for (int cp = 0; cp < M; ++cp) v = fma(Cout[(c * M + cp) * NFS], dO[cp], v);
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
    __syncwarp();  // region A (B_q, C) dead from here: becomes Jt
    if (k < ku) {
#pragma unroll
      for (int i = 0; i < NU; ++i) RA[i * LDJ + k] = acc[i];
#pragma unroll
      for (int i = NU; i < NR; ++i) RA[i * LDJ + k] = 0.0;
    }
    // ---- S5: mesh tangents in the 6 local directions ------------------------------------
    for (int d = k; d < 6; d += TPU) {
      const int gv = d >> 1, ic = d & 1;
      const double c0 = (gv == 1) - (gv == 0), c1 = (gv == 2) - (gv == 0);
      const double dJ00 = ic == 0 ? c0 : 0.0, dJ01 = ic == 0 ? c1 : 0.0, dJ10 = ic == 1 ? c0 : 0.0, dJ11 = ic == 1 ? c1 : 0.0;
      const double dadj[4] = {dJ11, -dJ01, -dJ10, dJ00};
      const double* Jm = S + SH::MJ;
      const double ddet = dJ00 * Jm[3] + Jm[0] * dJ11 - dJ01 * Jm[2] - Jm[1] * dJ10;
      double res[NU];
#pragma unroll
      for (int i = 0; i < NU; ++i)
        res[i] = -(dadj[0] * S[SH::TQ + i] + dadj[1] * S[SH::TQ + NU + i] + dadj[2] * S[SH::TQ + 2 * NU + i] +
                   dadj[3] * S[SH::TQ + 3 * NU + i]);
      if (LAW::SRC != SRC_NONE) {
#pragma unroll
        for (int n = 0; n < NB; ++n)
#pragma unroll
          for (int c = 0; c < M; ++c) {
            double v = 0.0;
#pragma unroll
            for (int q = 0; q < NQ; ++q) {
              double term = ddet * S[SH::SW + c * NQP + q];
              if (LAW::SRC == SRC_POS) term += S[SH::SP + (c * 2 + ic) * NQP + q] * T.bary[q][gv];
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
          const double dnu0 = ic == 0 ? 0.0 : del, dnu1 = ic == 0 ? -del : 0.0;
          const double* nh = S + SH::MNHAT + 2 * f;
          const double len = S[SH::MNLEN + f];
          const double dlen = nh[0] * dnu0 + nh[1] * dnu1;
          const double dnh0 = (dnu0 - nh[0] * dlen) / len, dnh1 = (dnu1 - nh[1] * dlen) / len;
#pragma unroll
          for (int s = 0; s < NS; ++s) {
            const int fs = f * NS + s;
            const double* FXp = S + SH::FX + fs;
            const double lam = FXp[(3 * M) * NFSP];
            const double dlam = FXp[(3 * M + 1) * NFSP] * dnh0 + FXp[(3 * M + 2) * NFSP] * dnh1;
            const double coef = dlam * len + lam * dlen;
#pragma unroll
            for (int c = 0; c < M; ++c) {
              const double dH = FXp[(2 * c) * NFSP] * dnu0 + FXp[(2 * c + 1) * NFSP] * dnu1 - FXp[(2 * M + c) * NFSP] * coef;
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
      for (int i = 0; i < NU; ++i) RBp[d * NUP + i] = res[i];
    }
    __syncwarp();
    for (int a = k; a < KP - ku; a += TPU) {
      if (a < kx) {
        double psv[6];
#pragma unroll
        for (int d = 0; d < 6; ++d) {
          const int n = r.elem_nodes[3 * e + (d >> 1)];
          psv[d] = __ldg(r.psi + (size_t)(2 * n + (d & 1)) * kx + a);
        }
#pragma unroll
        for (int i = 0; i < NU; ++i) {
          double v = 0.0;
#pragma unroll
          for (int d = 0; d < 6; ++d) v = fma(RBp[d * NUP + i], psv[d], v);
          RA[i * LDJ + ku + a] = v;
        }
        double dn = 0.0;
#pragma unroll
        for (int d = 0; d < 6; ++d) dn = fma(S[SH::DNX + d], psv[d], dn);
        S[SH::DNP + a] = dn;
#pragma unroll
        for (int i = NU; i < NR; ++i) RA[i * LDJ + ku + a] = 0.0;
      } else {
#pragma unroll
        for (int i = 0; i < NR; ++i) RA[i * LDJ + ku + a] = 0.0;
      }
    }
    __syncwarp();
    // ---- S6 -------------------------------------------------------------------------
    if (r.mode == MODE_DERIVS) {
      for (int t = 0; t < ntri; ++t) {
        int ti = 0, rem = t;
        while (rem >= nt8 - ti) { rem -= nt8 - ti; ++ti; }
        const int tj = ti + rem;
        double c0 = 0.0, c1 = 0.0;
        for (int hh = 0; hh < nvalid; ++hh) {
          const double* Su = Wb + hh * STR;
          const double* Jt = Su + SH::RA;
          const double rr = Su[SH::MRHO];
#pragma unroll
          for (int rs = 0; rs < NR / 4; ++rs) {
            const int row = rs * 4 + (lane & 3);
            dmma(c0, c1, rr * Jt[row * LDJ + ti * 8 + (lane >> 2)], Jt[row * LDJ + tj * 8 + (lane >> 2)]);
          }
        }
        double* Hp = HACC + (ti * 8 + (lane >> 2)) * KP + tj * 8 + 2 * (lane & 3);
        Hp[0] += c0;
        Hp[1] += c1;
      }
      __syncwarp();
      for (int pi = lane; pi < kx * kx; pi += 32) {
        const int a = pi / kx, b = pi % kx;
        if (a <= b) {
          double v = 0.0;
          for (int hh = 0; hh < nvalid; ++hh) {
            const double* Su = Wb + hh * STR;
            v = fma(Su[SH::MRHO] * Su[SH::DNP + a], Su[SH::DNP + b], v);
          }
          HACC[(ku + a) * KP + ku + b] += v;
        }
      }
#pragma unroll
      for (int half = 0; half < 2; ++half) {
        const int j = lane + 32 * half;
        if (j < K) {
          double gsum = 0.0;
          for (int hh = 0; hh < nvalid; ++hh) {
            const double* Su = Wb + hh * STR;
            const double* Jt = Su + SH::RA;
            double v = 0.0;
#pragma unroll
            for (int i = 0; i < NU; ++i) v = fma(Jt[i * LDJ + j], Su[SH::RT + i], v);
            if (j >= ku) v = fma(Su[SH::DNP + j - ku], Su[SH::MN], v);
            gsum = fma(Su[SH::MRHO], v, gsum);
          }
          if (half == 0) gacc0 += gsum; else gacc1 += gsum;
        }
      }
      if (lane == 0) {
        for (int hh = 0; hh < nvalid; ++hh) {
          const double* Su = Wb + hh * STR;
          double r2 = Su[SH::MN] * Su[SH::MN];
#pragma unroll
          for (int i = 0; i < NU; ++i) r2 = fma(Su[SH::RT + i], Su[SH::RT + i], r2);
          jacc = fma(Su[SH::MRHO], r2, jacc);
        }
      }
    } else if (valid) {
      const double* Jt = RA;
      const int extra = r.mode == MODE_CONTRIB_LPROWS ? 1 : 0;
      const int nk = r.mode == MODE_CONTRIB_SPLIT ? 2 * K : K + extra;
      for (int k2 = k; k2 < nk; k2 += TPU) {
        double v = 0.0;
        if (r.mode == MODE_CONTRIB_SPLIT) {
          int kk, part;
          if (k2 < 2 * ku) { kk = k2 % ku; part = k2 / ku; }
          else { kk = ku + (k2 - 2 * ku) % kx; part = (k2 - 2 * ku) / kx; }
          const double* Rp = S + (part == 0 ? SH::RV : SH::RF);
#pragma unroll
          for (int i = 0; i < NU; ++i) v = fma(Jt[i * LDJ + kk], Rp[i], v);
          if (kk >= ku && part == 0) v = fma(S[SH::DNP + kk - ku], S[SH::MN], v);
          r.out[((size_t)p * r.ne + e) * nk + k2] = v;
        } else if (k2 < K) {
#pragma unroll
          for (int i = 0; i < NU; ++i) v = fma(Jt[i * LDJ + k2], S[SH::RT + i], v);
          if (k2 >= ku) v = fma(S[SH::DNP + k2 - ku], S[SH::MN], v);
          if (r.mode == MODE_CONTRIB) r.out[((size_t)p * r.ne + e) * K + k2] = v;
          else r.out[((size_t)p * (K + 1) + k2) * r.ne + e] = v;
        } else {
          double r2 = S[SH::MN] * S[SH::MN];
#pragma unroll
          for (int i = 0; i < NU; ++i) r2 = fma(S[SH::RT + i], S[SH::RT + i], r2);
          r.out[((size_t)p * (K + 1) + K) * r.ne + e] = 0.5 * r2;
        }
      }
    }
    __syncwarp();
  }
  if (r.mode != MODE_DERIVS) return;
  // ---- block partial: fixed-order sum over the block's warps --------------------------
  if (lane < K) GW[lane] = gacc0;
  if (lane + 32 < K) GW[lane + 32] = gacc1;
  if (lane == 0) GW[K] = jacc;
  __syncthreads();
  const int PSZ = 1 + K + KP * KP;
  double* dst = r.part + ((size_t)prow_ * gxr + bx) * PSZ;
  for (int i = threadIdx.x; i < PSZ; i += blockDim.x) {
    double v = 0.0;
    for (int w = 0; w < nwarps; ++w) {
      const double* Wp = smem + (size_t)w * r.gx_warp_stride + UPW * STR;
      const double* GWp = Wp + KP * KP;
      v += i == 0 ? GWp[K] : (i <= K ? GWp[i - 1] : Wp[i - 1 - K]);
    }
    dst[i] = v;
  }
}

}  // namespace strom
