// K1 / K3 derivatives kernel on DMMA for 4-component laws with p = 2 (Euler).
//
// One warp per element.  The reduced Jacobian is formed as a projection of
// the element's local Jacobian instead of propagating k_u tangents:
//   L    = -sum_q Dq^T B_q Pq + sum_f (face-in blocks)        (24 x 24)
//   J_U  = L Phi_e + sum_f E_f Lout_f Phi_nf                  (24 x k_u)
//   J_x  = (dR/dx_e) Psi_e                                    (24 x k_x)
//   H   += rho J^T J   (upper 8x8 tiles)
// with every GEMM on mma.sync.m8n8k4.f64 (DMMA): the Dq^T B_q product is
// fused into the A-fragment loads of the L GEMM (no explicit X matrix), the
// basis rows are read as B fragments straight from global memory (L1/L2
// hits: the gather stage touched them), and the reference-element trace /
// basis tables are per-lane constant registers.  Pointwise physics, residual
// rows, gathers and the Gram are shared with derivs_warp.cuh's design.
#pragma once
#include "derivs_warp.cuh"

namespace strom {

constexpr int MTHREADS = 256;
#ifndef STROM_MMA_MAXNREG_WIDE
#define STROM_MMA_MAXNREG_WIDE 240  // k_u > 16 runs 4 two-warp CTAs/SM (2 warps per SMSP): room for 240
#endif
#ifndef STROM_HREG_WIDE
#define STROM_HREG_WIDE 15  // k_u > 16 (240 registers): register Gram for up to 15 upper tiles (K <= 40)
#endif
#ifndef STROM_MMA_MAXNREG
#define STROM_MMA_MAXNREG 168  // 3 warps per SMSP (12 per SM with 15 KB of smem per warp)
#endif
// Measured and removed in round 2 (DESIGN.md §3 table): buffered three-face out-blocks,
// register prefetch of the projection B fragments, cp.async staging of the next basis block,
// the dR/dx stage in the L-GEMM shadow, L1 / L2 neighbor-row prefetch, flipped J stores, the gradient from Jt
// in shared memory instead of the J fragments, Gram DMMAs accumulating straight into the register Gram.

template <int NQ>
struct MShape {
  static constexpr int M = 4, NB = 6, NU = 24, NF = 3, NS = 4, NFS = 12, NNB = 36, P = 2;
  static constexpr int NQ4 = (NQ + 3) / 4 * 4;
  static constexpr int NQC = NQ4 % 8 == 4 ? NQ4 : NQ4 + 4;  // BQ point stride (== 4 mod 8: conflict-free fragments)
  static constexpr int NQP = NQ % 2 ? NQ : NQ + 1;
  static constexpr int NFSP = 13;
  static constexpr int FXS = 3 * M + 3;
  // per-warp smem layout (doubles)
  static constexpr int MX = 0, MJ = 6, MADJ = 10, MDET = 14, MDETR = 15, MNU = 16, MNLEN = 22, MNHAT = 25, MN = 31,
                       MRHO = 32, DNX = 33, DNP = 40, MINT = 56;
  static constexpr int UE = 64;
  static constexpr int UNF = UE + NU;
  static constexpr int RT = UNF + NNB;
  static constexpr int RV = RT + NU;
  static constexpr int RF = RV + NU;
  static constexpr int TQS = NU + 4;            // Tq row stride (== 12 mod 16: conflict-free fragment stores)
  static constexpr int TQ = RF + NU;            // [4][TQS]
  static constexpr int FD = TQ + 4 * TQS;       // face mesh-response [f][s][c][2]
  static constexpr int RA = FD + 2 * M * NFSP;
  static constexpr int LDX = 12;
  // region A (offsets from RA), by phase:
  //   P/R : BQ [q][c][kk][c'] at 0, FQ [c][i][NQC] and HS [c][NFSP] right after it
  //   L   : L [NU][LDL] at 0 once the L GEMM has read BQ (FQ / HS dead after R)
  //   P/F : CF [fs][side][c][c'] at LA       (read by the face blocks)
  //   P/R : FX [field][NFSP] at LO           (face flux fields, read by the FD stage)
  //   F/J : one face's Lout [12][LDO] at LO  (projected right away)
  //   X/G : DRX [NU][LDX] at max(LA, NU LDJ) (CF, LOUT dead), Jt [NU][LDJ] at 0 (L dead)
  static constexpr int LDL = 28, LDO = 20;  // LDO == 4 mod 16: conflict-free half-warp fragment loads
  static constexpr int NLO = 1;               // out-block buffer (one face at a time)
  // the two sides of BQ / CF sit 12 mod 16 doubles apart, so the 24 point lanes (12 per
  // side) of one store instruction hit 24 distinct banks
  static constexpr int BQS = 16 * NQC + 12, CFS = 16 * NFSP + 12;
  static constexpr int BQ = 0, LL = 0;
  static constexpr int FQ = BQS + 16 * NQC;
  static constexpr int HS = FQ + 2 * M * NQC;
  static constexpr int LA = (HS + M * NFSP > NU * LDL ? HS + M * NFSP : NU * LDL);
  static constexpr int CF = LA;
  static constexpr int LO = LA + CFS + 16 * NFSP;
  static constexpr int FX = LO;
  static_assert(FXS * NFSP <= NLO * 12 * LDO, "FX overlays the Lout buffers");
  __host__ __device__ static constexpr int drx(int LDJ) { return LA > NU * LDJ ? LA : NU * LDJ; }
  __host__ __device__ static constexpr int gtail(int KP) { return KP + 8; }  // gradient (K) + residual norm
  // Gram accumulator: upper 8x8 tiles only, tile (ti <= tj) at tri_tile(ti, tj) * 64
  __host__ __device__ static constexpr int hsize(int KP) { return (KP / 8) * (KP / 8 + 1) / 2 * 64; }
  __host__ __device__ static constexpr int tri_tile(int ti, int tj, int nt8) { return ti * nt8 - ti * (ti - 1) / 2 + (tj - ti); }
  // the element's six Psi rows (gathered once, read by the Jx and distortion stages),
  // row stride == 4 mod 8 (conflict-free B fragments), just below the Gram accumulator
  __host__ __device__ static constexpr int prs(int kx) { return (kx + 3) / 8 * 8 + 4; }
  __host__ __device__ static constexpr int psr(int kx) { return 6 * prs(kx); }
  // Gram accumulator in registers: compile-time K <= 24 (six upper tiles, 12 doubles per lane)
  // k_u > 16 gets the wide register budget (measured per pass: cfg3 -10%, cfg4 -3.5%, cfg5 -6.5%)
  __host__ __device__ static constexpr bool wide(int KUT) { return KUT > 16; }
  __host__ __device__ static constexpr bool hreg(int KUT, int KXT) {
    return KUT > 0 && (KUT + KXT + 7) / 8 * ((KUT + KXT + 7) / 8 + 1) / 2 <= (wide(KUT) ? STROM_HREG_WIDE : 6);
  }
  __host__ __device__ static constexpr int warp_stride(int LDJ, int KP, int kx, bool hreg) {
    const int a = LO + NLO * 12 * LDO, b = drx(LDJ) + NU * LDX;
    const int s = RA + (a > b ? a : b) + (hreg ? 0 : hsize(KP)) + gtail(KP) + psr(kx);
    return (s + 15) / 16 * 16 + 4;
  }
};

// local index of element node n on face f (-1 if not on the face), p = 2
__device__ __forceinline__ int face_local(int f, int n) {
  const int a = f, b = (f + 1) % 3;
  return n == a ? 0 : (n == b ? 1 : (n == 3 + f ? 2 : -1));
}

// Row tiles of the J_U projection GEMMs pair the element nodes as {1,3}, {2,4}, {0,5}:
// every face (nodes {f, f+1, 3+f}) then touches only two of the three 8-row tiles, and
// tile (f+1)%3 holds none of its nodes, so the neighbor projection skips it.
__device__ __forceinline__ int prow(int mt, int lane) {
  const int slot = 2 * mt + (lane >> 4);
  const int node = slot == 0 ? 1 : (slot == 1 ? 3 : (slot == 2 ? 2 : (slot == 3 ? 4 : (slot == 4 ? 0 : 5))));
  return node * 4 + ((lane >> 2) & 3);
}

template <class LAW, int NQ, int KUT = 0, int KXT = 0, int DM = -1>  // KUT/KXT > 0: compile-time reduced dimensions;
                                                                     // DM: 1 derivatives / 0 contributions / -1 runtime
__global__ void __maxnreg__(MShape<NQ>::wide(KUT) ? STROM_MMA_MAXNREG_WIDE : STROM_MMA_MAXNREG) derivs_mma_kernel(const __grid_constant__ Params<6, NQ, 4, 3> prm) {
  using SH = MShape<NQ>;
  constexpr int M = 4, NB = 6, NU = 24, NF = 3, NS = 4, NFS = 12, PD = 2;
  constexpr int NQP = SH::NQP, NFSP = SH::NFSP, LDL = SH::LDL, LDO = SH::LDO, LDX = SH::LDX;
  static_assert(LAW::M == 4, "derivs_mma_kernel is specialised for 4-component laws");
  const auto& T = prm.t;
  const Run& r = prm.r;
  extern __shared__ __align__(16) double smem[];
  __shared__ double s_w[KMAX], s_tau[KMAX];
  __shared__ __align__(16) double s_dphi[NQ * NB * 2];
  __shared__ int s_tile[15];  // upper 8x8 tiles of the Gram (KP <= 40): (ti << 4) | tj
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
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
  constexpr bool CT = KUT > 0;
  const bool DERIVS = DM >= 0 ? DM == 1 : r.mode == MODE_DERIVS;  // compile-time on the specialised path
  // element Jacobian blocks (full-space assembly, dg.py:197-272; generic instantiation only):
  // out[e] = [res (NU) | dR/dU_e (NU x NU) | dR/dU_nbr (NU x 3 NU) | dR/dx_e (NU x 6) | N_e | dN_e/dx_e (6)]
  const bool EJ = DM < 0 && (r.mode == MODE_ELEMJAC || r.mode == MODE_ELEMJAC_ENRICHED);
  // enriched test space (dg.py:275-326): the same pointwise records contracted with the
  // degree p+1 test tabulations, out[e] = [res (NT) | dR/dU_e (NT x NU) | dR/dU_nbr (NT x 3 NU) |
  // dR/dx_e (NT x 6) | N_e | dN_e/dx_e (6)], NT = n_test * M
  const bool EJT = EJ && r.mode == MODE_ELEMJAC_ENRICHED;
  constexpr int EJ_SELF = 24, EJ_NBR = EJ_SELF + 24 * 24, EJ_X = EJ_NBR + 24 * 72, EJ_D = EJ_X + 24 * 6,
                EJ_SZ = EJ_D + 7;
  constexpr int KT = KUT + KXT, KPT = (KT + 7) / 8 * 8;
  const int ku = CT ? KUT : r.ku, kx = CT ? KXT : r.kx, K = CT ? KT : r.K, KP = CT ? KPT : r.KP;
  const int LDJ = CT ? KPT + 4 : r.LDJ;
  // per-warp stride: a compile-time constant on the specialised path (cheap to rematerialise)
  const int WSTR = CT ? SH::warp_stride(KPT + 4, KPT, KXT, SH::hreg(KUT, KXT)) : r.gx_warp_stride;
  double* const S = smem + (size_t)warp * WSTR;
  double* const RA = S + SH::RA;
  const int DRXo = SH::drx(LDJ);
  constexpr bool HREG = SH::hreg(KUT, KXT);
  double* const GW = S + WSTR - 4 - SH::gtail(KP);  // gradient + objective tail
  // warp Gram accumulator (upper 8x8 tiles): registers + region A at the end (HREG), or smem
  double* const HA = HREG ? S + SH::RA : GW - SH::hsize(KP);
  const int PRS = SH::prs(kx);
  double* const PR = (HREG ? GW : HA) - SH::psr(kx);  // Psi rows of the element's vertex coordinates
  constexpr int NT8T = CT ? (KUT + KXT + 7) / 8 : 1, NTRIT = NT8T * (NT8T + 1) / 2;
  double hacc[NTRIT][2];
#pragma unroll
  for (int t = 0; t < NTRIT; ++t) hacc[t][0] = hacc[t][1] = 0.0;

  for (int i = threadIdx.x; i < ku; i += blockDim.x) s_w[i] = r.w[(size_t)p * ku + i];
  for (int i = threadIdx.x; i < kx; i += blockDim.x) s_tau[i] = r.tau[(size_t)p * kx + i];
  for (int i = threadIdx.x; i < NQ * NB * 2; i += blockDim.x) s_dphi[i] = (&T.dphi[0][0][0])[i];
  if (!HREG)
    for (int i = lane; i < SH::hsize(KP); i += 32) HA[i] = 0.0;
  if (threadIdx.x == 0) {
    int t = 0;
    for (int ti = 0; ti < KP / 8; ++ti)
      for (int tj = ti; tj < KP / 8; ++tj) s_tile[t++] = (ti << 4) | tj;
  }
  // enriched mode: the test tabulations ([NQ][NBT][2] gradients, [3][NS][NBT] traces) staged in
  // shared memory (generic instantiation only; up to the degree-3 space, else read from global)
  constexpr int TT_MAX = DM < 0 ? (NQ * 2 + 3 * NS) * 10 : 1;
  __shared__ double s_tt[TT_MAX];
  const double* tt_base = r.test_tab;
  if constexpr (DM < 0) {
    if (EJT && (NQ * 2 + 3 * NS) * r.test_nb <= TT_MAX) {
      for (int i = threadIdx.x; i < (NQ * 2 + 3 * NS) * r.test_nb; i += blockDim.x) s_tt[i] = r.test_tab[i];
      tt_base = s_tt;
    }
  }
  LawArgs la;
#pragma unroll
  for (int i = 0; i < 8; ++i) la.p[i] = r.lawp[i];
#pragma unroll
  for (int i = 0; i < NMU; ++i) la.mu[i] = i < r.nmu ? r.mu[p * r.nmu + i] : 0.0;
  // per-lane constant B fragments of the L GEMM: -Phi[q][n'] at (q = 4ks + lane&3, n' = lane>>2)
  // (negated, so the accumulators come out as L = -sum_q Dq^T B_q Pq directly: exact)
  double phib[SH::NQ4 / 4];
#pragma unroll
  for (int ks = 0; ks < SH::NQ4 / 4; ++ks) {
    const int q = 4 * ks + (lane & 3), np_ = lane >> 2;
    phib[ks] = (q < NQ && np_ < NB) ? -T.phi[q < NQ ? q : 0][np_ < NB ? np_ : 0] : 0.0;
  }
  __syncthreads();

  double gacc0 = 0.0, gacc1 = 0.0, jacc = 0.0;
  // CT path: gradient partials straight from the J accumulators (column layout of the C
  // fragments, reduced over the lane>>2 groups once at the end), distortion part per lane
  double gj[4][2] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}}, gx[2][2] = {{0.0, 0.0}, {0.0, 0.0}}, gd = 0.0;
  const int nunits = r.active ? r.A : r.ne;
  const int nt8 = KP / 8, ntri = nt8 * (nt8 + 1) / 2;
  const int ntu = (ku + 7) / 8;

  // element index block carried in smem: [0] e, [1..3] nodes, [4..6] neighbors, [7..9] face info.
  // Each iteration loads the next unit's block mid-way and stores it after the Jx
  // stage, so the gather's address chain starts from shared memory.
  int* const EI = reinterpret_cast<int*>(S + SH::MINT);
  const int ustride = gxr * nwarps;
  auto index_word = [&](int ue, int l) -> int {
    return l == 0 ? ue : (l < 4 ? __ldg(r.elem_nodes + 3 * ue + l - 1)
                               : (l < 7 ? __ldg(r.nbr + 3 * ue + l - 4) : __ldg(r.finfo + 3 * ue + l - 7)));
  };
  {
    const int idx0 = bx * nwarps + warp;
    if (idx0 < nunits && lane < 10) EI[lane] = index_word(r.active ? __ldg(r.active + idx0) : idx0, lane);
    __syncwarp();
  }
  // per-lane gather roles (CT path): row lane (own row, or neighbor face 0 rows 0..7 for
  // lanes 24..31) and row lane + 32 (neighbor rows 8..35 for lanes 0..27)
  const int g0j = (lane - NU) >> 2;                       // lanes >= NU: face-node slot on face 0
  const int g1i = lane + 32 - NU, g1f = g1i / (NF * M), g1j = (g1i / M) % NF;
  for (int idx = bx * nwarps + warp; idx < nunits; idx += ustride) {
    const int e = EI[0];
    const double rho = r.active ? r.rho[idx] : 1.0;
    const int nidx = idx + ustride;
    const int nact = (r.active && nidx < nunits) ? __ldg(r.active + nidx) : nidx;
    int nbr[3], fin[3];
#pragma unroll
    for (int f = 0; f < 3; ++f) { nbr[f] = EI[4 + f]; fin[f] = EI[7 + f]; }
    // ---- G: coordinates and gathers (lane k = basis column k) --------------------
    // element rows (0..23) and neighbor face-node rows (24..59) land at S[UE + row]:
    // U = U0 + Phi_row . w, one row per lane and round, 16-byte loads of the 8*k_u-byte rows
    auto row_src = [&](int rr, const double*& src, double& v) {
      src = nullptr;
      v = 0.0;
      if (rr < NU) {
        src = r.phi + ((size_t)e * NU + rr) * ku;
        if (r.u0) v = r.u0[(size_t)p * r.u0_stride + (size_t)e * NU + rr];
      } else if (rr < NU + SH::NNB) {
        const int i = rr - NU, f = i / (NF * M), jj = (i / M) % NF, c = i % M;
        if ((fin[f] >> 3) == 0) {
          const int nf = fin[f] & 3;
          const int node = jj == 0 ? nf : (jj == 1 ? (nf + 1) % 3 : 3 + nf);
          src = r.phi + ((size_t)nbr[f] * NU + node * M + c) * ku;
          if (r.u0) v = r.u0[(size_t)p * r.u0_stride + (size_t)nbr[f] * NU + node * M + c];
        }
      }
    };
    double Xr[6], eref = 0.0;
    if constexpr (CT && KUT % 2 == 0) {
      // both rounds' loads (and the coordinate rows) issued before any use: one memory
      // round trip for the whole gather
      constexpr int H = KUT / 2;
      auto nrow = [&](int f, int jj, int c, int& ok) -> int {  // neighbor face-node row (element-major)
        const int fi = EI[7 + f];
        ok = (fi >> 3) == 0;
        const int nf = fi & 3;
        const int node = jj == 0 ? nf : (jj == 1 ? (nf == 2 ? 0 : nf + 1) : 3 + nf);
        return EI[4 + f] * NU + node * M + c;
      };
      int ok0 = 1, ok1 = 0;
      const int row0 = lane < NU ? e * NU + lane : nrow(0, g0j, lane & 3, ok0);
      const int row1 = lane < NU + SH::NNB - 32 ? nrow(g1f, g1j, lane & 3, ok1) : 0;
      const double* src0 = r.phi + (size_t)row0 * KUT;
      const double* src1 = r.phi + (size_t)row1 * KUT;
      double v0 = 0.0, v1 = 0.0;
      if (r.u0) {
        if (ok0) v0 = r.u0[(size_t)p * r.u0_stride + row0];
        if (ok1) v1 = r.u0[(size_t)p * r.u0_stride + row1];
      }
      double2 b0[H], b1[H];
#pragma unroll
      for (int k2 = 0; k2 < H; ++k2) b0[k2] = ok0 ? __ldg(reinterpret_cast<const double2*>(src0) + k2) : make_double2(0.0, 0.0);
#pragma unroll
      for (int k2 = 0; k2 < H; ++k2) b1[k2] = ok1 ? __ldg(reinterpret_cast<const double2*>(src1) + k2) : make_double2(0.0, 0.0);
      const int lx = lane < 6 ? lane : 0;
      const int xrow = 2 * EI[1 + (lx >> 1)] + (lx & 1);
      double xv = r.xref[(size_t)p * r.x_stride + xrow];
      double pv[KXT];
#pragma unroll
      for (int a2 = 0; a2 < KXT; ++a2) pv[a2] = __ldg(r.psi + (size_t)xrow * KXT + a2);
      if (lane < 6)
#pragma unroll
        for (int a2 = 0; a2 < KXT; ++a2) PR[lane * PRS + a2] = pv[a2];
#pragma unroll
      for (int g = 0; g < 3; ++g) {  // reference vertices, loaded with the gather (one round trip)
        const int n = EI[1 + g];
        Xr[2 * g] = r.nodes[2 * n];
        Xr[2 * g + 1] = r.nodes[2 * n + 1];
      }
      eref = lane == 0 ? r.eta_ref[e] : 0.0;
#pragma unroll
      for (int k2 = 0; k2 < H; ++k2) {
        v0 = fma(b0[k2].x, s_w[2 * k2], v0);
        v0 = fma(b0[k2].y, s_w[2 * k2 + 1], v0);
        v1 = fma(b1[k2].x, s_w[2 * k2], v1);
        v1 = fma(b1[k2].y, s_w[2 * k2 + 1], v1);
      }
#pragma unroll
      for (int a2 = 0; a2 < KXT; ++a2) xv = fma(pv[a2], s_tau[a2], xv);
      S[SH::UE + lane] = v0;
      if (lane + 32 < NU + SH::NNB) S[SH::UE + lane + 32] = v1;
      if (lane < 6) S[SH::MX + lane] = xv;
    } else {
      if (lane < 6) {
        const int n = EI[1 + (lane >> 1)];
        const int row = 2 * n + (lane & 1);
        double v = r.xref[(size_t)p * r.x_stride + row];
        const double* ps = r.psi + (size_t)row * kx;
        for (int a2 = 0; a2 < kx; ++a2) {
          const double t = ps[a2];
          PR[lane * PRS + a2] = t;
          v = fma(t, s_tau[a2], v);
        }
        S[SH::MX + lane] = v;
      }
      for (int rr = lane; rr < NU + SH::NNB; rr += 32) {
        const double* src;
        double v;
        row_src(rr, src, v);
        if (src) {
          if ((ku & 1) == 0) {
            const double2* s2 = reinterpret_cast<const double2*>(src);
            for (int k2 = 0; k2 < (ku >> 1); ++k2) {
              const double2 t2 = __ldg(s2 + k2);
              v = fma(t2.x, s_w[2 * k2], v);
              v = fma(t2.y, s_w[2 * k2 + 1], v);
            }
          } else {
            for (int k = 0; k < ku; ++k) v = fma(__ldg(src + k), s_w[k], v);
          }
        }
        S[SH::UE + rr] = v;
      }
#pragma unroll
      for (int g = 0; g < 3; ++g) {
        const int n = EI[1 + g];
        Xr[2 * g] = r.nodes[2 * n];
        Xr[2 * g + 1] = r.nodes[2 * n + 1];
      }
      eref = lane == 0 ? r.eta_ref[e] : 0.0;
    }
    __syncwarp();
    {  // element geometry (all lanes), distortion gradient (lanes 0-5), face normals (lanes 0-2)
      Geo o;
      element_geo(S + SH::MX, Xr, o);
      if (lane < 6) S[SH::DNX + lane] = distortion_grad_dir(o, T.wsum, r.eps, r.kappa, lane);
      if (lane < 3) face_normal(S + SH::MX, lane, S + SH::MNU + 2 * lane, S[SH::MNLEN + lane], S + SH::MNHAT + 2 * lane);
      if (lane == 0) {
        if (o.g <= 0.0) flag_degenerate(r, p, e);
        S[SH::MJ + 0] = o.J[0][0]; S[SH::MJ + 1] = o.J[0][1]; S[SH::MJ + 2] = o.J[1][0]; S[SH::MJ + 3] = o.J[1][1];
        S[SH::MADJ + 0] = o.adj[0][0]; S[SH::MADJ + 1] = o.adj[0][1]; S[SH::MADJ + 2] = o.adj[1][0]; S[SH::MADJ + 3] = o.adj[1][1];
        S[SH::MDET] = o.detJ;
        S[SH::MDETR] = o.detr;
        S[SH::MRHO] = rho;
        S[SH::MN] = r.kappa * (distortion_eta(o, T.wsum, r.eps, nullptr, nullptr) - eref);
      }
    }
    __syncwarp();
    // ---- P: pointwise physics on 24 lanes, one code path: lane = side * 12 + fs evaluates
    // face point fs on side `side` (0 in, 1 out) fused with volume point q = fs along the
    // adj(Jx) row `side`; the two sides of a face point meet through shuffles.
    {
      static_assert(NQ >= NFS, "fused P stage needs n_q >= 12");
      const int l24 = lane < 2 * NFS ? lane : lane - 2 * NFS;  // lanes 24..31 shadow 0..7 (no writes)
      const int side = l24 >= NFS ? 1 : 0, fs = l24 - side * NFS, f = fs / NS, s = fs % NS;
      const int fi = fin[f], bc = fi >> 3;
      const bool nside = side && bc == 0;
      const int sp = (nside && ((fi >> 2) & 1)) ? NS - 1 - s : s;
      const double* nu = S + SH::MNU + 2 * f;
      const double len = S[SH::MNLEN + f];
      const double* nh = S + SH::MNHAT + 2 * f;
      double us[M] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
      for (int j = 0; j < NF; ++j) {  // node values as two 16-byte loads
        const double2* u2 = reinterpret_cast<const double2*>(S + (nside ? SH::UNF + (f * NF + j) * M : SH::UE + fnode_of(PD, f, j) * M));
        const double2 a = u2[0], b = u2[1];
        const double t = T.trace[0][sp][j];
        us[0] = fma(t, a.x, us[0]); us[1] = fma(t, a.y, us[1]); us[2] = fma(t, b.x, us[2]); us[3] = fma(t, b.y, us[3]);
      }
      const bool wall = LAW::WALLS && bc == BC_REFLECT;  // slip wall: exterior = R(nh) u_in
      if (side && bc >= 2) {
        if (wall) reflect_state(us, nh, us);
        else LAW::ghost(bc - 2, la, nullptr, us);  // 4-component laws: constant ghosts
      }
      // A(n) is linear in n: evaluated along sc * nu it comes out already scaled by the face
      // weight and the LLF 1/2 (weight 1 on an extrapolated exterior, whose C_out folds into
      // C_in since u_out == u_in there; 0 for prescribed exteriors, which carry no state
      // tangent; a wall's exterior block is kept and folded into C_in through R after P)
      const double wsq = T.ws[s];
      const double sc = (side == 1 && bc >= 1 && !wall) ? 0.0 : ((side == 0 && bc == 1) ? wsq : 0.5 * wsq);
      const double nus[2] = {sc * nu[0], sc * nu[1]};
      double f2[M][2], A[M][M], g[M], gn[2];
      const double ws = PointOps<LAW>::face_side(us, nus, nh, f2, A, g, gn, la);
      const int q = fs;
      double uq[M] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
      for (int n = 0; n < NB; ++n) {
        const double2* u2 = reinterpret_cast<const double2*>(S + SH::UE + n * M);
        const double2 a = u2[0], b = u2[1];
        const double t = T.phi[q][n];
        uq[0] = fma(t, a.x, uq[0]); uq[1] = fma(t, a.y, uq[1]); uq[2] = fma(t, b.x, uq[2]); uq[3] = fma(t, b.y, uq[3]);
      }
      const double wq = T.wq[q];  // folded into the direction: Aq comes out weighted
      const double dv[2] = {wq * S[SH::MADJ + 2 * side], wq * S[SH::MADJ + 2 * side + 1]};
      double fq[M][2], Aq[M][M];
      PointOps<LAW>::vol_dir(uq, dv, fq, Aq, la);
      const int partner = side ? lane - NFS : (lane + NFS) & 31;
      const double wsp = __shfl_sync(0xffffffffu, ws, partner);
      double up[M], fp[M][2];
#pragma unroll
      for (int c = 0; c < M; ++c) {
        up[c] = __shfl_sync(0xffffffffu, us[c], partner);
        fp[c][0] = __shfl_sync(0xffffffffu, f2[c][0], partner);
        fp[c][1] = __shfl_sync(0xffffffffu, f2[c][1], partner);
      }
      if constexpr (LAW::ROE) {  // Roe (GPU-only extension): the LLF-free part here, D in the Roe pass
        if (lane < 2 * NFS) {
          double* FXp = RA + SH::FX;
          if (side == 0) {
#pragma unroll
            for (int c = 0; c < M; ++c) {
              const double fni = f2[c][0] * nu[0] + f2[c][1] * nu[1], fno = fp[c][0] * nu[0] + fp[c][1] * nu[1];
              RA[SH::HS + c * NFSP + fs] = wsq * (0.5 * (fni + fno));
              FXp[(2 * c + 0) * NFSP + fs] = 0.5 * wsq * (f2[c][0] + fp[c][0]);
              FXp[(2 * c + 1) * NFSP + fs] = 0.5 * wsq * (f2[c][1] + fp[c][1]);
            }
            FXp[(3 * M + 0) * NFSP + fs] = 1.0;  // "lam" = 1, its normal gradient 0: coef = dlen
            FXp[(3 * M + 1) * NFSP + fs] = 0.0;
            FXp[(3 * M + 2) * NFSP + fs] = 0.0;
          }
#pragma unroll
          for (int c = 0; c < M; ++c)
#pragma unroll
            for (int cp = 0; cp < M; ++cp) RA[SH::CF + side * SH::CFS + (c * M + cp) * NFSP + fs] = A[c][cp];
#pragma unroll
          for (int c = 0; c < M; ++c) {
            if (side == 0) {
              RA[SH::FQ + (c * 2 + 0) * SH::NQC + q] = wq * fq[c][0];
              RA[SH::FQ + (c * 2 + 1) * SH::NQC + q] = wq * fq[c][1];
            }
#pragma unroll
            for (int cp = 0; cp < M; ++cp) RA[SH::BQ + side * SH::BQS + (cp * M + c) * SH::NQC + q] = Aq[c][cp];
          }
        }
      } else if (lane < 2 * NFS) {
        const double wsi = side ? wsp : ws, wso = side ? ws : wsp;
        // dual.maximum tie -> first argument (dual.py:171); a wall's ws(R u) equals ws(u): interior
        const bool in_wins = wall || wsi >= wso;
        const bool mine = (side == 0) == in_wins;
        const double lam = in_wins ? wsi : wso;
        double* FXp = RA + SH::FX;
        double du[M];
#pragma unroll
        for (int c = 0; c < M; ++c) du[c] = side ? us[c] - up[c] : up[c] - us[c];
        if (side == 0) {
#pragma unroll
          for (int c = 0; c < M; ++c) {
            const double fni = f2[c][0] * nu[0] + f2[c][1] * nu[1], fno = fp[c][0] * nu[0] + fp[c][1] * nu[1];
            RA[SH::HS + c * NFSP + fs] = wsq * (0.5 * (fni + fno) - 0.5 * (lam * len) * du[c]);
            FXp[(2 * c + 0) * NFSP + fs] = 0.5 * wsq * (f2[c][0] + fp[c][0]);
            FXp[(2 * c + 1) * NFSP + fs] = 0.5 * wsq * (f2[c][1] + fp[c][1]);
            FXp[(2 * M + c) * NFSP + fs] = 0.5 * wsq * du[c];
          }
          FXp[(3 * M + 0) * NFSP + fs] = lam;
        }
        if (mine) {
          FXp[(3 * M + 1) * NFSP + fs] = gn[0];
          FXp[(3 * M + 2) * NFSP + fs] = gn[1];
        }
        // C_side = wsq (A/2 -+ lam len/2 I - len/2 du (d lam/du_side)^T); the extrapolated
        // exterior (du = 0) adds its C_out = A/2 - lam len/2 I into C_in, exterior sides are 0
        const bool ext0 = side == 1 && bc >= 1 && !wall;
        const double dgn = (bc == 1 || ext0) ? 0.0 : (side ? -0.5 : 0.5) * lam * len * wsq;
        const double dsc = ext0 ? 0.0 : -0.5 * len * wsq;
        double gm[M];
#pragma unroll
        for (int cp = 0; cp < M; ++cp) gm[cp] = mine ? g[cp] : 0.0;
#pragma unroll
        for (int c = 0; c < M; ++c) {
          const double dd = dsc * du[c];
#pragma unroll
          for (int cp = 0; cp < M; ++cp)
            RA[SH::CF + side * SH::CFS + (c * M + cp) * NFSP + fs] = fma(dd, gm[cp], A[c][cp]) + (c == cp ? dgn : 0.0);
        }
#pragma unroll
        for (int c = 0; c < M; ++c) {
          if (side == 0) {
            RA[SH::FQ + (c * 2 + 0) * SH::NQC + q] = wq * fq[c][0];
            RA[SH::FQ + (c * 2 + 1) * SH::NQC + q] = wq * fq[c][1];
          }
#pragma unroll
          for (int cp = 0; cp < M; ++cp) RA[SH::BQ + side * SH::BQS + (cp * M + c) * SH::NQC + q] = Aq[c][cp];
        }
      }
    }
    for (int q = NFS + lane; q < NQ; q += 32) {  // remaining volume points (n_q > 12)
      double uq[M];
#pragma unroll
      for (int c = 0; c < M; ++c) {
        double v = 0.0;
#pragma unroll
        for (int n = 0; n < NB; ++n) v = fma(T.phi[q][n], S[SH::UE + n * M + c], v);
        uq[c] = v;
      }
      const double wq = T.wq[q];
      double f2[M][2], A0[M][M], A1[M][M];
      const double d0[2] = {S[SH::MADJ + 0], S[SH::MADJ + 1]}, d1[2] = {S[SH::MADJ + 2], S[SH::MADJ + 3]};
      PointOps<LAW>::vol_point(uq, d0, d1, f2, A0, A1, la);
#pragma unroll
      for (int c = 0; c < M; ++c) {
        RA[SH::FQ + (c * 2 + 0) * SH::NQC + q] = wq * f2[c][0];
        RA[SH::FQ + (c * 2 + 1) * SH::NQC + q] = wq * f2[c][1];
#pragma unroll
        for (int cp = 0; cp < M; ++cp) {
          RA[SH::BQ + (cp * M + c) * SH::NQC + q] = wq * A0[c][cp];
          RA[SH::BQ + SH::BQS + (cp * M + c) * SH::NQC + q] = wq * A1[c][cp];
        }
      }
    }
    __syncwarp();
    if constexpr (LAW::ROE) {  // ---- Roe pass: D = |A_roe(nh)| (u_out - u_in) and its Jacobians
      // outside the P stage (fewer live values): lane = side * 12 + fs recomputes both traces,
      // forward mode along its own state (Dn<4>) and, on side 0, along the face normal (Dn<2>)
      if (lane < 2 * NFS) {
        const int side = lane >= NFS ? 1 : 0, fs = lane - side * NFS, f = fs / NS, s = fs % NS;
        const int fi = fin[f], bc = fi >> 3;
        const bool wall = bc == BC_REFLECT, dz = bc == 1, ext0 = side == 1 && bc >= 1 && !wall;
        const double* nh = S + SH::MNHAT + 2 * f;
        const double len = S[SH::MNLEN + f], wsq = T.ws[s];
        double ui[M] = {0.0, 0.0, 0.0, 0.0}, uo[M] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int j = 0; j < NF; ++j)
#pragma unroll
          for (int c = 0; c < M; ++c) ui[c] = fma(T.trace[0][s][j], S[SH::UE + fnode_of(PD, f, j) * M + c], ui[c]);
        if (bc == 0) {
          const int sp = ((fi >> 2) & 1) ? NS - 1 - s : s;
#pragma unroll
          for (int j = 0; j < NF; ++j)
#pragma unroll
            for (int c = 0; c < M; ++c) uo[c] = fma(T.trace[0][sp][j], S[SH::UNF + (f * NF + j) * M + c], uo[c]);
        } else if (bc == 1) {
#pragma unroll
          for (int c = 0; c < M; ++c) uo[c] = ui[c];
        } else if (wall) {
          reflect_state(ui, nh, uo);
        } else {
          LAW::ghost(bc - 2, la, nullptr, uo);
        }
        if (!dz) {
          // dD/du_side in two passes of two seeded components each (Dn<2>: fewer live values)
          double Dv[M];
#pragma unroll
          for (int half = 0; half < 2; ++half) {
            Dn<2> ua[M], ub[M], nd[2];
#pragma unroll
            for (int c = 0; c < M; ++c) {
              const bool seeded = (c >> 1) == half;
              ua[c] = (side == 0 && seeded) ? seed<2>(ui[c], c & 1) : cst<2>(ui[c]);
              ub[c] = (side == 1 && seeded) ? seed<2>(uo[c], c & 1) : cst<2>(uo[c]);
            }
            nd[0] = cst<2>(nh[0]);
            nd[1] = cst<2>(nh[1]);
            Dn<2> Dd[M];
            roe_diss(ua, ub, nd, la.p[0], la.p[1], Dd);
#pragma unroll
            for (int c = 0; c < M; ++c) Dv[c] = Dd[c].v;
            if (!ext0)
#pragma unroll
              for (int c = 0; c < M; ++c)
#pragma unroll
                for (int k = 0; k < 2; ++k)
                  RA[SH::CF + side * SH::CFS + (c * M + 2 * half + k) * NFSP + fs] -= 0.5 * wsq * len * Dd[c].d[k];
          }
          if (side == 0) {
#pragma unroll
            for (int c = 0; c < M; ++c) {
              RA[SH::HS + c * NFSP + fs] -= wsq * 0.5 * len * Dv[c];
              RA[SH::FX + (2 * M + c) * NFSP + fs] = 0.5 * wsq * Dv[c];  // the FD stage's "du" slot carries D
            }
            // D's own normal dependence: -wsq len / 2 (dD/dnh . dnh) per unit normal perturbation,
            // pre-written into the FD slots (the FD stage adds the flux and |nu| terms)
            Dn<2> ua2[M], ub2[M], nd2[2];
#pragma unroll
            for (int c = 0; c < M; ++c) { ua2[c] = cst<2>(ui[c]); ub2[c] = cst<2>(uo[c]); }
            nd2[0] = seed<2>(nh[0], 0);
            nd2[1] = seed<2>(nh[1], 1);
            Dn<2> Dn2[M];
            roe_diss(ua2, ub2, nd2, la.p[0], la.p[1], Dn2);
            const double il = 1.0 / len;
#pragma unroll
            for (int dir = 0; dir < 2; ++dir) {
              const double dlen = nh[dir];
              const double dn0 = ((dir == 0 ? 1.0 : 0.0) - nh[0] * dlen) * il, dn1 = ((dir == 1 ? 1.0 : 0.0) - nh[1] * dlen) * il;
#pragma unroll
              for (int c = 0; c < M; ++c)
                S[SH::FD + (c * 2 + dir) * NFSP + fs] = -0.5 * wsq * len * (Dn2[c].d[0] * dn0 + Dn2[c].d[1] * dn1);
            }
          }
        } else if (side == 0) {  // extrapolated exterior: D == 0 identically
#pragma unroll
          for (int c = 0; c < M; ++c) {
            RA[SH::FX + (2 * M + c) * NFSP + fs] = 0.0;
            S[SH::FD + (c * 2 + 0) * NFSP + fs] = 0.0;
            S[SH::FD + (c * 2 + 1) * NFSP + fs] = 0.0;
          }
        }
      }
      __syncwarp();
    }
    // ---- slip walls: fold the exterior block into C_in through u_g = R(nh) u_in, and the
    // ghost's normal dependence into the FD slots (warp-uniform: elements without walls skip)
    if (LAW::WALLS && ((fin[0] >> 3) == BC_REFLECT || (fin[1] >> 3) == BC_REFLECT || (fin[2] >> 3) == BC_REFLECT)) {
      if (lane < NFS && (fin[lane / NS] >> 3) == BC_REFLECT) {
        const int fs = lane, f = fs / NS, s = fs % NS;
        const double* nh = S + SH::MNHAT + 2 * f;
        const double len = S[SH::MNLEN + f], il = 1.0 / len;
        double ui[M] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int j = 0; j < NF; ++j)
#pragma unroll
          for (int c = 0; c < M; ++c) ui[c] = fma(T.trace[0][s][j], S[SH::UE + fnode_of(PD, f, j) * M + c], ui[c]);
        double X[M][M];
#pragma unroll
        for (int c = 0; c < M; ++c)
#pragma unroll
          for (int cp = 0; cp < M; ++cp) X[c][cp] = RA[SH::CF + SH::CFS + (c * M + cp) * NFSP + fs];
        const double mn = ui[1] * nh[0] + ui[2] * nh[1];
#pragma unroll
        for (int dir = 0; dir < 2; ++dir) {  // d(R u_in)/dnh . dnh for a unit perturbation of nu
          const double dlen = nh[dir];
          const double dn0 = ((dir == 0 ? 1.0 : 0.0) - nh[0] * dlen) * il, dn1 = ((dir == 1 ? 1.0 : 0.0) - nh[1] * dlen) * il;
          const double dmn = ui[1] * dn0 + ui[2] * dn1;
          const double w1 = -2.0 * (dmn * nh[0] + mn * dn0), w2 = -2.0 * (dmn * nh[1] + mn * dn1);
#pragma unroll
          for (int c = 0; c < M; ++c) {
            const double ex = X[c][1] * w1 + X[c][2] * w2;
            double& slot = S[SH::FD + (c * 2 + dir) * NFSP + fs];
            slot = LAW::ROE ? slot + ex : ex;
          }
        }
        // C_in += X R, R = diag(1, I - 2 nh nh^T, 1)
#pragma unroll
        for (int c = 0; c < M; ++c) {
          const double xn = X[c][1] * nh[0] + X[c][2] * nh[1];
          const double xr[M] = {X[c][0], X[c][1] - 2.0 * xn * nh[0], X[c][2] - 2.0 * xn * nh[1], X[c][3]};
#pragma unroll
          for (int cp = 0; cp < M; ++cp) RA[SH::CF + (c * M + cp) * NFSP + fs] += xr[cp];
        }
      }
      __syncwarp();
    }
    // ---- R: residual rows (volume / face split) and Tq ------------------------------
    // Tq[(n,j)][(c,k)] = sum_q dphi[q][n][j] FQ[(c,k)][q] on DMMA: rows (n,j) in two 8-row
    // tiles, columns (c,k); the lane of row (n,j) holds c = lane&3, k = 0,1
    {
      double tc[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
#pragma unroll
      for (int ks = 0; ks < SH::NQ4 / 4; ++ks) {
        const int q = 4 * ks + (lane & 3);
        const bool qv = q < NQ;
        const double b = qv ? RA[SH::FQ + (lane >> 2) * SH::NQC + q] : 0.0;
#pragma unroll
        for (int mt = 0; mt < 2; ++mt) {
          const int rw = mt * 8 + (lane >> 2);
          const double a = (qv && rw < 2 * NB) ? s_dphi[q * 2 * NB + rw] : 0.0;
          dmma(tc[mt][0], tc[mt][1], a, b);
        }
      }
      const double* adj = S + SH::MADJ;
      const int j = (lane >> 2) & 1, c = lane & 3;
      double rvm[2];
#pragma unroll
      for (int mt = 0; mt < 2; ++mt) {
        const int rw = mt * 8 + (lane >> 2), n = rw >> 1;
        const double pj = adj[2 * j] * tc[mt][0] + adj[2 * j + 1] * tc[mt][1];
        rvm[mt] = -(pj + __shfl_xor_sync(0xffffffffu, pj, 4));  // rows (n,0) + (n,1)
        if (rw < 2 * NB) {
          S[SH::TQ + (2 * j + 0) * SH::TQS + n * M + c] = tc[mt][0];
          S[SH::TQ + (2 * j + 1) * SH::TQS + n * M + c] = tc[mt][1];
          if (j == 0) S[SH::RV + n * M + c] = rvm[mt];
        }
      }
      // row i = (n, c) of the residual: rv from the lane of row (n, 0)
      const int src = (8 * (lane >> 2) + (lane & 3)) & 31;
      const double rv0 = __shfl_sync(0xffffffffu, rvm[0], src), rv1 = __shfl_sync(0xffffffffu, rvm[1], src);
      if (lane < NU) {
        const int i = lane, n = i / M;
        const double rv = n < 4 ? rv0 : rv1;
        double rf = 0.0;
#pragma unroll
        for (int f = 0; f < 3; ++f) {
          const int jf = face_local(f, n);
          if (jf >= 0)
#pragma unroll
            for (int s = 0; s < NS; ++s) rf = fma(T.trace[0][s][jf], RA[SH::HS + c * NFSP + f * NS + s], rf);
        }
        S[SH::RF + i] = rf;
        S[SH::RT + i] = rv + rf;
      }
    }
    // face responses to unit normal-vector perturbations (for the mesh tangents)
    if (lane < NFS) {
      const int fs = lane, f = fs / NS;
      const double* nh = S + SH::MNHAT + 2 * f;
      const double len = S[SH::MNLEN + f];
      const double* FXp = RA + SH::FX + fs;
      const double lam = FXp[(3 * M) * NFSP];
      const bool wallf = LAW::WALLS && (fin[f] >> 3) == BC_REFLECT;
      const double il = 1.0 / len;
#pragma unroll
      for (int dir = 0; dir < 2; ++dir) {  // dnu = e_x or e_y
        const double dnu0 = dir == 0 ? 1.0 : 0.0, dnu1 = dir == 0 ? 0.0 : 1.0;
        const double dlen = nh[0] * dnu0 + nh[1] * dnu1;
        const double dnh0 = (dnu0 - nh[0] * dlen) * il, dnh1 = (dnu1 - nh[1] * dlen) * il;
        const double dlam = FXp[(3 * M + 1) * NFSP] * dnh0 + FXp[(3 * M + 2) * NFSP] * dnh1;
        const double coef = dlam * len + lam * dlen;
#pragma unroll
        for (int c = 0; c < M; ++c) {
          // Roe: D's normal dependence, walls: the ghost's, were pre-written to the slot
          const double pre = (LAW::ROE || wallf) ? S[SH::FD + (c * 2 + dir) * NFSP + fs] : 0.0;
          S[SH::FD + (c * 2 + dir) * NFSP + fs] =
              pre + FXp[(2 * c) * NFSP] * dnu0 + FXp[(2 * c + 1) * NFSP] * dnu1 - FXp[(2 * M + c) * NFSP] * coef;
        }
      }
    }
    if (EJT) {
      __syncwarp();  // FD slots written above
      const int NBT = r.test_nb, NT = NBT * M;
      const double* tdphi = tt_base;               // [NQ][NBT][2]
      const double* ttr = tt_base + NQ * NBT * 2;  // [3][NS][NBT]
      double* const eo = r.out + (size_t)e * (NT * (1 + 4 * NU + 6) + 7);
      const double* adj = S + SH::MADJ;
      for (int i = lane; i < NT; i += 32) {  // residual row (n, c) and its six mesh derivatives
        const int n = i / M, c = i % M;
        double t00 = 0.0, t01 = 0.0, t10 = 0.0, t11 = 0.0;  // t[j][k] = sum_q dphi_t[q][n][j] w_q f[c][k]
        for (int q = 0; q < NQ; ++q) {
          const double d0 = tdphi[(q * NBT + n) * 2], d1 = tdphi[(q * NBT + n) * 2 + 1];
          const double f0 = RA[SH::FQ + (c * 2 + 0) * SH::NQC + q], f1 = RA[SH::FQ + (c * 2 + 1) * SH::NQC + q];
          t00 = fma(d0, f0, t00); t01 = fma(d0, f1, t01); t10 = fma(d1, f0, t10); t11 = fma(d1, f1, t11);
        }
        const double rv = -((adj[0] * t00 + adj[1] * t01) + (adj[2] * t10 + adj[3] * t11));
        double dr[6];
#pragma unroll
        for (int d = 0; d < 6; ++d) {
          const int gv = d >> 1, ic = d & 1;
          const double c0 = (gv == 1) - (gv == 0), c1 = (gv == 2) - (gv == 0);
          dr[d] = ic == 0 ? (c1 * t01 - c0 * t11) : -(c1 * t00 - c0 * t10);
        }
        double rf = 0.0;
#pragma unroll
        for (int f = 0; f < 3; ++f) {
          double rx = 0.0, ry = 0.0;
#pragma unroll
          for (int s = 0; s < NS; ++s) {
            const double tr = ttr[(f * NS + s) * NBT + n];
            rf = fma(tr, RA[SH::HS + c * NFSP + f * NS + s], rf);
            rx = fma(tr, S[SH::FD + (c * 2 + 0) * NFSP + f * NS + s], rx);
            ry = fma(tr, S[SH::FD + (c * 2 + 1) * NFSP + f * NS + s], ry);
          }
          const int a = f, b = (f + 1) % 3;
          dr[2 * b + 1] += rx;  dr[2 * a + 1] -= rx;
          dr[2 * b + 0] -= ry;  dr[2 * a + 0] += ry;
        }
        eo[i] = rv + rf;
#pragma unroll
        for (int d = 0; d < 6; ++d) eo[(size_t)NT * (1 + 4 * NU) + i * 6 + d] = dr[d];
      }
      for (int i = lane; i < NT * NU; i += 32) {  // dR/dU_e
        const int row = i / NU, col = i % NU, n = row / M, c = row % M, np_ = col / M, cp = col % M;
        double v = 0.0;
        for (int q = 0; q < NQ; ++q) {
          const double a = fma(tdphi[(q * NBT + n) * 2], RA[SH::BQ + (cp * M + c) * SH::NQC + q],
                               tdphi[(q * NBT + n) * 2 + 1] * RA[SH::BQ + SH::BQS + (cp * M + c) * SH::NQC + q]);
          v = fma(-a, T.phi[q][np_], v);
        }
        for (int f = 0; f < 3; ++f) {
          const int jp = face_local(f, np_);
          if (jp < 0) continue;
          for (int s = 0; s < NS; ++s)
            v = fma(ttr[(f * NS + s) * NBT + n] * T.trace[0][s][jp], RA[SH::CF + (c * M + cp) * NFSP + f * NS + s], v);
        }
        eo[NT + i] = v;
      }
      // dR/dU_nbr: zero, then the 12 face-node columns of each interior face's neighbor
      for (int i = lane; i < NT * 3 * NU; i += 32) eo[NT + NT * NU + i] = 0.0;
      __syncwarp();
      for (int i = lane; i < NT * 3 * NF * M; i += 32) {
        const int row = i / (3 * NF * M), rem = i % (3 * NF * M), n = row / M, c = row % M;
        const int f = rem / (NF * M), jn = (rem / M) % NF, cp = rem % M;
        const int fi = EI[7 + f];
        if ((fi >> 3) != 0) continue;
        const int nf = fi & 3;
        const int node = jn == 0 ? nf : (jn == 1 ? (nf + 1) % 3 : 3 + nf);
        double v = 0.0;
        for (int s = 0; s < NS; ++s) {
          const int sp = ((fi >> 2) & 1) ? NS - 1 - s : s;
          v = fma(ttr[(f * NS + s) * NBT + n] * T.trace[0][sp][jn],
                  RA[SH::CF + SH::CFS + (c * M + cp) * NFSP + f * NS + s], v);
        }
        eo[NT + NT * NU + (size_t)row * 3 * NU + f * NU + node * M + cp] = v;
      }
      if (lane < 7) eo[(size_t)NT * (1 + 4 * NU + 6) + lane] = lane == 0 ? S[SH::MN] : S[SH::DNX + lane - 1];
      __syncwarp();
      if (nidx < nunits && lane < 10) EI[lane] = index_word(nact, lane);
      __syncwarp();
      continue;
    }
    // (no barrier: the L stage reads only BQ / CF; TQ / FD / R rows are read after later barriers)
    // next unit's index block: loaded here, stored to smem after the Jx stage
    const int wv = (nidx < nunits && lane < 10) ? index_word(nact, lane) : 0;
    // ---- X: local mesh Jacobian dR/dx (24 x 6) -------------------------------------------
    auto x_stage = [&](double* drxb) {
    if (lane < NU) {
      const int i = lane, n = i / M, c = i % M;
      const double t00 = S[SH::TQ + i], t01 = S[SH::TQ + SH::TQS + i], t10 = S[SH::TQ + 2 * SH::TQS + i], t11 = S[SH::TQ + 3 * SH::TQS + i];
      double dr[6];
#pragma unroll
      for (int d = 0; d < 6; ++d) {
        const int gv = d >> 1, ic = d & 1;
        const double c0 = (gv == 1) - (gv == 0), c1 = (gv == 2) - (gv == 0);
        // ic = 0: dadj = [[0,-c1],[0,c0]]; ic = 1: dadj = [[c1,0],[-c0,0]]
        dr[d] = ic == 0 ? (c1 * t01 - c0 * t11) : -(c1 * t00 - c0 * t10);
      }
#pragma unroll
      for (int f = 0; f < 3; ++f) {
        const int j = face_local(f, n);
        if (j < 0) continue;
        double rx = 0.0, ry = 0.0;  // face response to dnu = e_x, e_y
#pragma unroll
        for (int s = 0; s < NS; ++s) {
          rx = fma(T.trace[0][s][j], S[SH::FD + (c * 2 + 0) * NFSP + f * NS + s], rx);
          ry = fma(T.trace[0][s][j], S[SH::FD + (c * 2 + 1) * NFSP + f * NS + s], ry);
        }
        const int a = f, b = (f + 1) % 3;
        // vertex g in {a, b}: del = (g == b) - (g == a); ic = 1 -> dnu = del e_x, ic = 0 -> dnu = -del e_y
        dr[2 * b + 1] += rx;  dr[2 * a + 1] -= rx;
        dr[2 * b + 0] -= ry;  dr[2 * a + 0] += ry;
      }
      {  // three 16-byte pieces (columns 6, 7 are never read: the Jx A fragments are predicated)
        double2* dst = reinterpret_cast<double2*>(drxb + i * LDX);
        dst[0] = make_double2(dr[0], dr[1]);
        dst[1] = make_double2(dr[2], dr[3]);
        dst[2] = make_double2(dr[4], dr[5]);
      }
    }
    };
    // ---- L: volume local Jacobian on DMMA; X = Dq^T B_q fused into the A fragments ------
    {
      double lv[4][3][2];
#pragma unroll
      for (int cp = 0; cp < 4; ++cp)
#pragma unroll
        for (int mt = 0; mt < 3; ++mt) lv[cp][mt][0] = lv[cp][mt][1] = 0.0;
#pragma unroll
      for (int ks = 0; ks < SH::NQ4 / 4; ++ks) {
        const int q = 4 * ks + (lane & 3);
        const bool qv = q < NQ;
        const int qq = qv ? q : 0;
#pragma unroll
        for (int mt = 0; mt < 3; ++mt) {
          const int row = mt * 8 + (lane >> 2), n = row >> 2, c = row & 3;
          const double d0 = qv ? s_dphi[(qq * NB + n) * 2 + 0] : 0.0;
          const double d1 = qv ? s_dphi[(qq * NB + n) * 2 + 1] : 0.0;
          const double* B = RA + SH::BQ + c * SH::NQC + qq;
#pragma unroll
          for (int cp = 0; cp < 4; ++cp) {
            const double a = fma(d0, B[cp * M * SH::NQC], d1 * B[SH::BQS + cp * M * SH::NQC]);
            dmma(lv[cp][mt][0], lv[cp][mt][1], a, phib[ks]);
          }
        }
      }
      __syncwarp();  // BQ / CF reads of other lanes finished before L overwrites region A? (L lives after CF)
      // write L into L[(n,c)][(n',c')], n' = 2(lane&3) + {0,1}: the lane's 8 values are
      // contiguous (columns 8(lane&3) .. +7), written as four 16-byte pieces in an order
      // rotated by (lane&3)>>1 so every quarter-warp store hits 8 distinct bank groups
      if ((lane & 3) < 3) {
        const bool rot = (lane & 2) != 0;
#pragma unroll
        for (int mt = 0; mt < 3; ++mt) {
          double2* dst = reinterpret_cast<double2*>(RA + SH::LL + (mt * 8 + (lane >> 2)) * LDL + 8 * (lane & 3));
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            // piece pc = (t + rot) & 3 holds (h2 = pc >> 1, cp = 2 (pc & 1) + {0, 1})
            const int pa = t, pb = (t + 1) & 3;
            const double xa = lv[2 * (pa & 1)][mt][pa >> 1], ya = lv[2 * (pa & 1) + 1][mt][pa >> 1];
            const double xb = lv[2 * (pb & 1)][mt][pb >> 1], yb = lv[2 * (pb & 1) + 1][mt][pb >> 1];
            dst[rot ? pb : pa] = make_double2(rot ? xb : xa, rot ? yb : ya);
          }
        }
      }
    }
    __syncwarp();
    // face blocks, one face at a time: lanes 0-15 add the in-side block into L, lanes
    // 16-31 form Lout_f in a one-face buffer, then the warp projects it on the
    // neighbor's face-node basis rows straight into the J accumulators
    double ju[4][3][2];  // up to 4 n-tiles (k_u <= 32)
#pragma unroll
    for (int nt = 0; nt < 4; ++nt)
#pragma unroll
      for (int mt = 0; mt < 3; ++mt) ju[nt][mt][0] = ju[nt][mt][1] = 0.0;
    const double* L = RA + SH::LL;
    double* Lo = RA + SH::LO;
    double* const ej = EJ ? r.out + (size_t)e * EJ_SZ : nullptr;
    if (EJ)  // neighbor blocks: zero first (boundary faces and off-face columns stay 0)
      for (int i = lane; i < 24 * 72; i += 32) ej[EJ_NBR + i] = 0.0;
#pragma unroll
    for (int f = 0; f < 3; ++f) {
      {
        const int c = (lane & 15) >> 2, cp = lane & 3, side = lane >> 4;
        double cs[NS];
#pragma unroll
        for (int s = 0; s < NS; ++s) cs[s] = RA[SH::CF + side * SH::CFS + (c * M + cp) * NFSP + f * NS + s];
#pragma unroll
        for (int j = 0; j < NF; ++j)
#pragma unroll
          for (int jp = j; jp < NF; ++jp) {  // t2 is symmetric in (j, j'): one sum per pair
            double v = 0.0;
#pragma unroll
            for (int s = 0; s < NS; ++s) v = fma(T.t2[j][jp][s], cs[s], v);
            if (side == 0) {
              RA[SH::LL + (fnode_of(PD, f, j) * M + c) * LDL + fnode_of(PD, f, jp) * M + cp] += v;
              if (jp != j) RA[SH::LL + (fnode_of(PD, f, jp) * M + c) * LDL + fnode_of(PD, f, j) * M + cp] += v;
            } else {
              Lo[(j * M + c) * LDO + jp * M + cp] = v;
              if (jp != j) Lo[(jp * M + c) * LDO + j * M + cp] = v;
            }
          }
      }
      __syncwarp();
      if (EJ && (fin[f] >> 3) == 0) {  // Lout_f -> dR_e/dU_nbr(f) at the neighbor's face-node columns
        const int nf = fin[f] & 3;
        const bool flip = (fin[f] >> 2) & 1;
        for (int i = lane; i < 144; i += 32) {
          const int row = i / 12, kk = i % 12, j = row / M, c = row % M, ks = kk / M, cp = kk % M;
          const int jn = flip ? (ks == 0 ? 1 : (ks == 1 ? 0 : 2)) : ks;
          const int node = jn == 0 ? nf : (jn == 1 ? (nf + 1) % 3 : 3 + nf);
          ej[EJ_NBR + (fnode_of(PD, f, j) * M + c) * 72 + f * NU + node * M + cp] = Lo[(j * M + c) * LDO + kk];
        }
      }
      if ((fin[f] >> 3) == 0) {
        const int nf = fin[f] & 3;
        const bool flip = (fin[f] >> 2) & 1;
        const double* phn = r.phi + (size_t)nbr[f] * NU * ku;
#pragma unroll
        for (int ks = 0; ks < 3; ++ks) {  // k = (j', c') = 4 ks + lane&3 -> j' = ks
          // neighbor face node j' (flip: the two vertex nodes swap, trace(1-s) = trace(s) with swapped vertices)
          const int jn = flip ? (ks == 0 ? 1 : (ks == 1 ? 0 : 2)) : ks;
          const int node = jn == 0 ? nf : (jn == 1 ? (nf + 1) % 3 : 3 + nf);
          const int brow = node * M + (lane & 3);
          double af[3];
#pragma unroll
          for (int mt = 0; mt < 3; ++mt) {
            const int row = prow(mt, lane), n = row >> 2, c = row & 3;
            const int j = face_local(f, n);
            af[mt] = (mt != (f + 1) % 3 && j >= 0) ? Lo[(j * M + c) * LDO + 4 * ks + (lane & 3)] : 0.0;
          }
#pragma unroll
          for (int nt = 0; nt < 4; ++nt) {
            if (nt < ntu) {
              const int col = nt * 8 + (lane >> 2);
              const double b = col < ku ? __ldg(phn + (size_t)brow * ku + col) : 0.0;
#pragma unroll
              for (int mt = 0; mt < 3; ++mt)
                if (mt != (f + 1) % 3) dmma(ju[nt][mt][0], ju[nt][mt][1], af[mt], b);
            }
          }
        }
      }
      __syncwarp();  // Lout_f consumed before the next face overwrites it
    }
    if (EJ)  // L (volume + face in-blocks) = dR_e/dU_e
      for (int i = lane; i < NU * NU; i += 32) ej[EJ_SELF + i] = L[(i / NU) * LDL + i % NU];
    // ---- J: own-state projection J_U += L Phi_e on DMMA ----------------------------------
    {
      const double* phe = r.phi + (size_t)e * NU * ku;
#pragma unroll
      for (int ks = 0; ks < 6; ++ks) {
        double af[3];
#pragma unroll
        for (int mt = 0; mt < 3; ++mt) af[mt] = L[prow(mt, lane) * LDL + 4 * ks + (lane & 3)];
        const int brow = 4 * ks + (lane & 3);
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) {
          if (nt < ntu) {
            const int col = nt * 8 + (lane >> 2);
            const double b = col < ku ? __ldg(phe + (size_t)brow * ku + col) : 0.0;
#pragma unroll
            for (int mt = 0; mt < 3; ++mt) dmma(ju[nt][mt][0], ju[nt][mt][1], af[mt], b);
          }
        }
      }
    }
    __syncwarp();  // LOUT reads done before DRX overwrites it
    x_stage(RA + DRXo);
    __syncwarp();
    if (EJ) {  // dR_e/dx_e (local coordinates 2 g + i) and the residual
      for (int i = lane; i < NU * 6; i += 32) ej[EJ_X + i] = RA[DRXo + (i / 6) * LDX + i % 6];
      if (lane < NU) ej[lane] = S[SH::RT + lane];
      if (lane < 7) ej[EJ_D + lane] = lane == 0 ? S[SH::MN] : S[SH::DNX + lane - 1];  // distortion.py:64-92
    }
    // ---- write J_U, then J_x = (dR/dx) Psi_e on DMMA, into Jt (region A, phase 3) --------
    double* Jt = RA;
    constexpr bool GFRAG = CT;  // gradient from the J accumulator fragments
    const bool gfrag = GFRAG && DERIVS;
    double rr[3];  // rho * R at the lane's three projection rows
#pragma unroll
    for (int mt = 0; mt < 3; ++mt) rr[mt] = gfrag ? rho * S[SH::RT + prow(mt, lane)] : 0.0;
#pragma unroll
    for (int nt = 0; nt < 4; ++nt)
#pragma unroll
      for (int mt = 0; mt < 3; ++mt)
#pragma unroll
        for (int t = 0; t < 2; ++t) {
          const int h2 = t;
          const int col = nt * 8 + 2 * (lane & 3) + h2;
          const double v = h2 ? ju[nt][mt][1] : ju[nt][mt][0];
          if (nt < ntu && col < ku) Jt[prow(mt, lane) * LDJ + col] = v;
          if (GFRAG && nt < ntu) gj[nt][t] = fma(ju[nt][mt][t], rr[mt], gj[nt][t]);
        }
    {
      double jx[2][3][2];
#pragma unroll
      for (int nt = 0; nt < 2; ++nt)
#pragma unroll
        for (int mt = 0; mt < 3; ++mt) jx[nt][mt][0] = jx[nt][mt][1] = 0.0;
      const int ntx = (kx + 7) / 8;
#pragma unroll
      for (int ks = 0; ks < 2; ++ks) {
        const int d = 4 * ks + (lane & 3);
        double af[3];
#pragma unroll
        for (int mt = 0; mt < 3; ++mt) af[mt] = d < 6 ? (RA + DRXo)[prow(mt, lane) * LDX + d] : 0.0;
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) {
          if (nt < ntx) {
            const int col = nt * 8 + (lane >> 2);
            const double b = (d < 6 && col < kx) ? PR[d * PRS + col] : 0.0;
#pragma unroll
            for (int mt = 0; mt < 3; ++mt) dmma(jx[nt][mt][0], jx[nt][mt][1], af[mt], b);
          }
        }
      }
#pragma unroll
      for (int nt = 0; nt < 2; ++nt)
#pragma unroll
        for (int mt = 0; mt < 3; ++mt)
#pragma unroll
          for (int t = 0; t < 2; ++t) {
            const int h2 = t;
            const int col = nt * 8 + 2 * (lane & 3) + h2;
            const double v = h2 ? jx[nt][mt][1] : jx[nt][mt][0];
            if (col < kx) Jt[prow(mt, lane) * LDJ + ku + col] = v;
            if (GFRAG && nt < ntx) gx[nt][t] = fma(jx[nt][mt][t], rr[mt], gx[nt][t]);
          }
      // Gram padding columns
      for (int col = K + lane; col < KP; col += 32)
#pragma unroll
        for (int i = 0; i < NU; ++i) Jt[i * LDJ + col] = 0.0;
      if (lane < kx) {
        double dn = 0.0;
#pragma unroll
        for (int d = 0; d < 6; ++d) dn = fma(S[SH::DNX + d], PR[d * PRS + lane], dn);
        S[SH::DNP + lane] = dn;
        if (gfrag) gd = fma(rho * dn, S[SH::MN], gd);
      }
    }
    __syncwarp();
    {  // next unit: index block into smem, L2 prefetch of its basis block (3 KB at k_u = 16).
      // (prefetching the neighbor rows, U0, Psi and coordinates too measured 4-9% slower)
      if (nidx < nunits) {
        if (lane < 10) EI[lane] = wv;
        const char* base = reinterpret_cast<const char*>(r.phi + (size_t)nact * NU * ku);
        for (int off = lane * 128; off < NU * ku * 8; off += 32 * 128) asm volatile("prefetch.global.L2 [%0];" ::"l"(base + off));
      }
    }
    // ---- G: Gram and gradient, or per-element contributions --------------------------------
    if (DERIVS) {
      if constexpr (CT) {
        // fragments of J^T per (tile column, k-step), loaded once and shared by the tiles
        constexpr int NT8C = KPT / 8;
        double fr[NT8C][NU / 4];
#pragma unroll
        for (int cc = 0; cc < NT8C; ++cc)
#pragma unroll
          for (int rs = 0; rs < NU / 4; ++rs) fr[cc][rs] = Jt[(rs * 4 + (lane & 3)) * LDJ + cc * 8 + (lane >> 2)];
        constexpr int NTRI = NT8C * (NT8C + 1) / 2;
        double gc[NTRI][2];  // all upper tiles in flight: k-step outer, independent chains inner
#pragma unroll
        for (int t = 0; t < NTRI; ++t) gc[t][0] = gc[t][1] = 0.0;
#pragma unroll
        for (int rs = 0; rs < NU / 4; ++rs)
#pragma unroll
          for (int ti = 0; ti < NT8C; ++ti)
#pragma unroll
            for (int tj = ti; tj < NT8C; ++tj) {
              const int t = SH::tri_tile(ti, tj, NT8C);
              dmma(gc[t][0], gc[t][1], fr[ti][rs], fr[tj][rs]);
            }
#pragma unroll
        for (int ti = 0; ti < NT8C; ++ti)
#pragma unroll
          for (int tj = ti; tj < NT8C; ++tj) {
            const int t = SH::tri_tile(ti, tj, NT8C);
            if constexpr (HREG) {
              hacc[t][0] = fma(rho, gc[t][0], hacc[t][0]);
              hacc[t][1] = fma(rho, gc[t][1], hacc[t][1]);
            } else {
              double2* Hp = reinterpret_cast<double2*>(HA + t * 64 + (lane >> 2) * 8 + 2 * (lane & 3));
              const double2 h = *Hp;
              *Hp = make_double2(fma(rho, gc[t][0], h.x), fma(rho, gc[t][1], h.y));
            }
          }
        if constexpr (HREG) {  // distortion term dN dN^T in the tau-tau block, row <= col
#pragma unroll
          for (int ti = 0; ti < NT8C; ++ti)
#pragma unroll
            for (int tj = ti; tj < NT8C; ++tj)
#pragma unroll
              for (int h = 0; h < 2; ++h) {
                const int row = ti * 8 + (lane >> 2), col = tj * 8 + 2 * (lane & 3) + h;
                if (tj * 8 + 7 >= KUT && row >= KUT && col >= KUT && row < KT && col < KT && row <= col) {
                  const int t = SH::tri_tile(ti, tj, NT8C);
                  hacc[t][h] = fma(rho * S[SH::DNP + row - KUT], S[SH::DNP + col - KUT], hacc[t][h]);
                }
              }
        }
      } else {
        for (int t = 0; t < ntri; ++t) {
          const int ti = s_tile[t] >> 4, tj = s_tile[t] & 15;
          double c0 = 0.0, c1 = 0.0;
          const double* ja = Jt + (lane & 3) * LDJ + ti * 8 + (lane >> 2);
          const double* jb = Jt + (lane & 3) * LDJ + tj * 8 + (lane >> 2);
  #pragma unroll
          for (int rs = 0; rs < NU / 4; ++rs) dmma(c0, c1, ja[rs * 4 * LDJ], jb[rs * 4 * LDJ]);
          double* Hp = HA + t * 64 + (lane >> 2) * 8 + 2 * (lane & 3);
          Hp[0] = fma(rho, c0, Hp[0]);
          Hp[1] = fma(rho, c1, Hp[1]);
        }
      }
      __syncwarp();
      if (!HREG)
      for (int pi = lane; pi < kx * kx; pi += 32) {
        const int a = pi / kx, b = pi % kx;
        const int row = ku + a, col = ku + b;
        if (a <= b) HA[SH::tri_tile(row >> 3, col >> 3, nt8) * 64 + (row & 7) * 8 + (col & 7)] += rho * S[SH::DNP + a] * S[SH::DNP + b];
      }
#pragma unroll
      for (int half = 0; half < 2; ++half) {
        const int j = lane + 32 * half;
        if (!GFRAG && j < K) {
          double v = 0.0;
#pragma unroll
          for (int i = 0; i < NU; ++i) v = fma(Jt[i * LDJ + j], S[SH::RT + i], v);
          if (j >= ku) v = fma(S[SH::DNP + j - ku], S[SH::MN], v);
          if (half == 0) gacc0 = fma(rho, v, gacc0); else gacc1 = fma(rho, v, gacc1);
        }
      }
      {  // per-lane objective partials, reduced across lanes once at the end of the kernel
        const double ri = lane < NU ? S[SH::RT + lane] : (lane == NU ? S[SH::MN] : 0.0);
        jacc = fma(rho * ri, ri, jacc);
      }
    } else if (!EJ) {
      const int extra = r.mode == MODE_CONTRIB_LPROWS ? 1 : 0;
      const int nk = r.mode == MODE_CONTRIB_SPLIT ? 2 * K : K + extra;
      for (int k2 = lane; k2 < nk; k2 += 32) {
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
  if (!DERIVS) return;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) jacc += __shfl_xor_sync(0xffffffffu, jacc, o);
  if constexpr (CT) {
#pragma unroll
    for (int o = 4; o < 32; o <<= 1)
#pragma unroll
      for (int h2 = 0; h2 < 2; ++h2) {
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) gj[nt][h2] += __shfl_xor_sync(0xffffffffu, gj[nt][h2], o);
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) gx[nt][h2] += __shfl_xor_sync(0xffffffffu, gx[nt][h2], o);
      }
    if (lane < 4)
#pragma unroll
      for (int h2 = 0; h2 < 2; ++h2) {
#pragma unroll
        for (int nt = 0; nt < 4; ++nt)
          if (nt * 8 + 2 * lane + h2 < ku) GW[nt * 8 + 2 * lane + h2] = gj[nt][h2];
#pragma unroll
        for (int nt = 0; nt < 2; ++nt)
          if (nt * 8 + 2 * lane + h2 < kx) GW[ku + nt * 8 + 2 * lane + h2] = gx[nt][h2];
      }
    __syncwarp();
    if (lane < kx) GW[ku + lane] += gd;
  } else {
    if (lane < K) GW[lane] = gacc0;
    if (lane + 32 < K) GW[lane + 32] = gacc1;
  }
  if (lane == 0) GW[K] = jacc;
  if constexpr (HREG) {  // the loop is done: region A holds the warp's Gram tiles for the CTA sum
#pragma unroll
    for (int t = 0; t < NTRIT; ++t)
      *reinterpret_cast<double2*>(HA + t * 64 + (lane >> 2) * 8 + 2 * (lane & 3)) = make_double2(hacc[t][0], hacc[t][1]);
  }
  __syncthreads();
  const int PSZ = 1 + K + KP * KP;
  double* dst = r.part + ((size_t)prow_ * gxr + bx) * PSZ;
  for (int i = threadIdx.x; i < PSZ; i += blockDim.x) {
    double v = 0.0;
    for (int w = 0; w < nwarps; ++w) {
      const double* Sw = smem + (size_t)w * WSTR;
      const double* Gw = Sw + WSTR - 4 - SH::gtail(KP);
      const double* Hw = HREG ? Sw + SH::RA : Gw - SH::hsize(KP);
      if (i == 0) v += Gw[K];
      else if (i <= K) v += Gw[i - 1];
      else {
        const int d = i - 1 - K, row = d / KP, col = d % KP;
        if ((row >> 3) <= (col >> 3)) v += Hw[SH::tri_tile(row >> 3, col >> 3, nt8) * 64 + (row & 7) * 8 + (col & 7)];
      }
    }
    dst[i] = v;
  }
}

}  // namespace strom
