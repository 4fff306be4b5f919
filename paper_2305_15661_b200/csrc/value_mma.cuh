// K2 (many parameter points): element residual value path with the state
// reconstruction on DMMA.
//
// One warp per element, lane = parameter point (32 per warp, one point group per
// CTA).  The reconstruction U = U0 + Phi_rows W of the element's rows and of the
// neighbors' face-node rows is a (rows x k_u) x (k_u x 32) GEMM: Phi rows are the
// A fragments (one 8-byte load per lane and k-step, shared by the 32 points), W
// the B fragments (shared memory, per CTA), the result goes through a per-warp
// (rows x 32) shared tile from which each lane reads its own column.  The
// pointwise flux / LLF / quadrature part is value_unit's (element_kernels.cuh),
// one parameter point per lane.  Replaces the per-lane scalar row dots of
// value_mu_kernel (reduced.py:172-184 objective, dg.py:228-240 value assembly).
#pragma once
#include "element_kernels.cuh"

namespace strom {

constexpr int VM_THREADS = 128;
constexpr int VM_NTB_OWN = 4, VM_NTB_F = 4;  // column tiles per reconstruction pass (own rows / face rows)
constexpr int VM_MINB = 3;                    // 3 CTAs of 4 warps per SM at 168 registers (4 CTAs = 128 registers spill: +50%)
constexpr int VM_LDU = 40;  // tile row stride: == 8 mod 16 -> conflict-free double2 C-fragment stores
constexpr int VM_LDW = 36;  // W row stride: == 4 mod 16 -> conflict-free B-fragment loads

template <class LAW, int NB>
struct VShape {
  static constexpr int M = LAW::M, NU = NB * M, P = NB == 3 ? 1 : (NB == 6 ? 2 : 3), NF = P + 1;
  static constexpr int NFR = NF * M;                      // one face's neighbor rows
  static constexpr int MT_OWN = (NU + 7) / 8, MT_F = (NFR + 7) / 8;
  static constexpr int FROW = MT_OWN * 8;                   // first face row of the tile
  static constexpr int TILE = (MT_OWN * 8 + MT_F * 8) * VM_LDU;  // doubles per warp
};

// rows r < nrows of the warp tile <- U0 + Phi[row(r)] . W  for the CTA's 32 points,
// NTB of the four 8-point column tiles per pass (fewer live accumulators; the A
// fragments are re-read from L1 in later passes)
template <int MT, int NTB, int LDB = VM_LDW, class RowOf>
__device__ __forceinline__ void vm_recon_g(const double* __restrict__ basis, int kn, const double* __restrict__ off,
                                           long long off_stride, const double* Ws, double* tile, int nrows,
                                           RowOf row_of, const int* s_prow, int lane) {
  const int ksn = (kn + 3) >> 2;
#pragma unroll
  for (int n0 = 0; n0 < 4; n0 += NTB) {
    double c[MT][NTB][2];
    const double* src[MT];
    bool ok[MT];
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) {
      const int rr = mt * 8 + (lane >> 2);
      ok[mt] = rr < nrows;
      const int row = row_of(ok[mt] ? rr : 0);
      src[mt] = basis + (size_t)row * kn;
#pragma unroll
      for (int nt = 0; nt < NTB; ++nt)
#pragma unroll
        for (int h = 0; h < 2; ++h)
          c[mt][nt][h] = (off && ok[mt]) ? off[(size_t)s_prow[(n0 + nt) * 8 + 2 * (lane & 3) + h] * off_stride + row] : 0.0;
    }
#pragma unroll 2
    for (int ks = 0; ks < ksn; ++ks) {
      const int k = 4 * ks + (lane & 3);
      double a[MT];
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) a[mt] = (ok[mt] && k < kn) ? __ldg(src[mt] + k) : 0.0;
#pragma unroll
      for (int nt = 0; nt < NTB; ++nt) {
        const double b = Ws[k * LDB + (n0 + nt) * 8 + (lane >> 2)];
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) dmma(c[mt][nt][0], c[mt][nt][1], a[mt], b);
      }
    }
#pragma unroll
    for (int mt = 0; mt < MT; ++mt)
#pragma unroll
      for (int nt = 0; nt < NTB; ++nt)
        *reinterpret_cast<double2*>(tile + (mt * 8 + (lane >> 2)) * VM_LDU + (n0 + nt) * 8 + 2 * (lane & 3)) =
            make_double2(c[mt][nt][0], c[mt][nt][1]);
  }
}

template <int MT, int NTB, class RowOf>
__device__ __forceinline__ void vm_recon(const Run& r, const double* Ws, double* tile, int nrows, RowOf row_of,
                                         const int* s_prow, int lane) {
  vm_recon_g<MT, NTB>(r.phi, r.ku, r.u0, r.u0_stride, Ws, tile, nrows, row_of, s_prow, lane);
}

template <class LAW, int NB, int NQ, int NS>
__global__ void __launch_bounds__(VM_THREADS, VM_MINB) value_mma_kernel(const __grid_constant__ Params<NB, NQ, NS, Shape<LAW, NB, NQ, NS>::NF> prm) {
  using VS = VShape<LAW, NB>;
  constexpr int M = VS::M, NU = VS::NU, NF = VS::NF, PD = VS::P, NFR = VS::NFR;
  const auto& T = prm.t;
  const Run& r = prm.r;
  extern __shared__ __align__(16) double vsm[];
  __shared__ __align__(16) double Ws[32 * VM_LDW];  // W[k][point], k_u <= 32 (zero-padded)
  __shared__ __align__(16) double Ts[KXMAX * VM_LDW];  // tau[a][point] (zero-padded rows)
  __shared__ double red[VM_THREADS / 32][32];
  __shared__ int s_prow[32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double* const tile = vsm + warp * VS::TILE;
  // point group = blockIdx.x (fastest: the groups of one element chunk run together and
  // share its basis rows in L2); lane -> parameter row, consecutive or compacted list
  // CTA -> (point group gi, element chunk xi): grid (groups, chunks), or a device-sized 1-D
  // grid over the ceil(*dyn_count / 32) live groups (graph-resident LM rounds)
  int gi = blockIdx.x, xi = blockIdx.y, gxr = gridDim.y, nlist = r.nlist;
  if (r.dyn_count) {
    nlist = *r.dyn_count;
    const int gy = (nlist + 31) / 32;
    if (gy == 0) return;
    gxr = dyn_gx(r.dyn_target, r.dyn_maxb, 1, gy);
    gi = blockIdx.x % gy;
    xi = blockIdx.x / gy;
    if (xi >= gxr) return;
  }
  auto row_of_pt = [&](int l) -> int {
    const int s = gi * 32 + l;
    return r.list ? (s < nlist ? r.list[s] : r.P) : s;
  };
  if (threadIdx.x < 32) {
    const int pr = row_of_pt(threadIdx.x);
    s_prow[threadIdx.x] = pr < r.P ? pr : row_of_pt(0);
  }
  for (int t = threadIdx.x; t < 32 * 32; t += blockDim.x) {
    const int k = t / 32, l = t % 32, pp = row_of_pt(l);
    Ws[k * VM_LDW + l] = (k < r.ku && pp < r.P) ? r.w[(size_t)pp * r.ku + k] : 0.0;
  }
  for (int t = threadIdx.x; t < KXMAX * 32; t += blockDim.x) {
    const int a = t / 32, l = t % 32, pp = row_of_pt(l);
    Ts[a * VM_LDW + l] = (a < r.kx && pp < r.P) ? r.tau[(size_t)pp * r.kx + a] : 0.0;
  }
  __syncthreads();
  const int pr = row_of_pt(lane);
  const bool pv = pr < r.P && (!r.mask || r.mask[pr]);
  const int p = s_prow[lane];  // idle lanes shadow a valid point (no traps, results unused)
  LawArgs la;
#pragma unroll
  for (int i = 0; i < 8; ++i) la.p[i] = r.lawp[i];
#pragma unroll
  for (int i = 0; i < NMU; ++i) la.mu[i] = i < r.nmu ? r.mu[p * r.nmu + i] : 0.0;
  const int nunits = r.active ? r.A : r.ne;
  double acc = 0.0;
  for (int idx = xi * (VM_THREADS / 32) + warp; idx < nunits; idx += gxr * (VM_THREADS / 32)) {
    const int e = r.active ? r.active[idx] : idx;
    const double rho = r.active ? r.rho[idx] : 1.0;
    __syncwarp();  // the previous element's tile reads are done
    // ---- own rows
    vm_recon<VS::MT_OWN, VM_NTB_OWN>(r, Ws, tile, NU, [&](int rr) { return e * NU + rr; }, s_prow, lane);
    __syncwarp();
    const double* U = tile + lane;  // the lane's column of the warp tile: U[i * VM_LDU]
#define VM_U(i) U[(i) * VM_LDU]
    // ---- geometry (value_unit, element_kernels.cuh): the six deformed vertex coordinates
    // x = X_ref + Psi_rows tau of the 32 points as one more DMMA reconstruction through the
    // face rows of the tile (free until the first face), each lane then reads its column
    double x[6], X[6];
    int vn[3];
#pragma unroll
    for (int g = 0; g < 3; ++g) {
      vn[g] = r.elem_nodes[3 * e + g];
      X[2 * g] = r.nodes[2 * vn[g]];
      X[2 * g + 1] = r.nodes[2 * vn[g] + 1];
    }
    vm_recon_g<1, 4>(r.psi, r.kx, r.xref, r.x_stride, Ts, tile + VS::FROW * VM_LDU, 6,
                     [&](int rr) { return 2 * (rr < 2 ? vn[0] : (rr < 4 ? vn[1] : vn[2])) + (rr & 1); }, s_prow, lane);
    __syncwarp();
#pragma unroll
    for (int d = 0; d < 6; ++d) x[d] = tile[(VS::FROW + d) * VM_LDU + lane];
    Geo o;
    element_geo(x, X, o);
    const bool deg = o.g <= 0.0;
    const double N = r.kappa * (distortion_eta(o, T.wsum, r.eps, nullptr, nullptr) - r.eta_ref[e]);
    const double adj00 = o.adj[0][0], adj01 = o.adj[0][1], adj10 = o.adj[1][0], adj11 = o.adj[1][1], detJ = o.detJ;
    double R[NU];
#pragma unroll
    for (int i = 0; i < NU; ++i) R[i] = 0.0;
    // ---- volume (dg.py:105-125); the point loops stay rolled (unrolling spills: neutral to -5%)
#pragma unroll 1
    for (int q = 0; q < NQ; ++q) {
      double uq[M];
#pragma unroll
      for (int c = 0; c < M; ++c) {
        double v = 0.0;
#pragma unroll
        for (int n = 0; n < NB; ++n) v = fma(T.phi[q][n], VM_U(n * M + c), v);
        uq[c] = v;
      }
      double f[M][2];
      PointVal<LAW>::flux(uq, f, la);
#pragma unroll
      for (int c = 0; c < M; ++c) {
        const double F0 = T.wq[q] * (f[c][0] * adj00 + f[c][1] * adj01);
        const double F1 = T.wq[q] * (f[c][0] * adj10 + f[c][1] * adj11);
#pragma unroll
        for (int n = 0; n < NB; ++n) R[n * M + c] = fma(-T.dphi[q][n][1], F1, fma(-T.dphi[q][n][0], F0, R[n * M + c]));
      }
      if (LAW::SRC != SRC_NONE) {
        double pos[2];
#pragma unroll
        for (int i = 0; i < 2; ++i) pos[i] = T.bary[q][0] * x[i] + T.bary[q][1] * x[2 + i] + T.bary[q][2] * x[4 + i];
        double s[M];
        LAW::source(pos, uq, s, la);
#pragma unroll
        for (int c = 0; c < M; ++c) {
          const double sv = T.wq[q] * detJ * s[c];
#pragma unroll
          for (int n = 0; n < NB; ++n) R[n * M + c] -= T.phi[q][n] * sv;
        }
      }
    }
    // ---- faces (dg.py:127-175); neighbor face-node rows reconstructed per face
#pragma unroll
    for (int f = 0; f < 3; ++f) {
      double nu[2], len, nh[2];
      face_normal(x, f, nu, len, nh);
      const int nb = r.nbr[3 * e + f];
      const int fi = r.finfo[3 * e + f];
      const int bc = fi >> 3;
      int flip = 0;
      if (bc == 0) {  // warp-uniform (one element per warp)
        const int nf = fi & 3;
        flip = (fi >> 2) & 1;
        __syncwarp();  // the previous face's reads of the face rows are done
        vm_recon<VS::MT_F, VM_NTB_F>(r, Ws, tile + VS::FROW * VM_LDU, NFR, [&](int rr) {
          const int j = rr / M, c = rr % M;
          const int node = j == 0 ? nf : (j == 1 ? (nf + 1) % 3 : 3 + nf * (PD - 1) + (j - 2));
          return nb * NU + node * M + c;
        }, s_prow, lane);
        __syncwarp();
      }
      double ghost[M];
      if (bc >= 2 && bc != BC_REFLECT && !LAW::GHOST_POS) LAW::ghost(bc - 2, la, nullptr, ghost);
#pragma unroll 1
      for (int s = 0; s < NS; ++s) {
        double ui[M], uo[M];
#pragma unroll
        for (int c = 0; c < M; ++c) {
          double v = 0.0;
#pragma unroll
          for (int j = 0; j < NF; ++j) v = fma(T.trace[f][s][j], VM_U(fnode_of(PD, f, j) * M + c), v);
          ui[c] = v;
        }
        if (bc == 0) {
          const int sp = flip ? NS - 1 - s : s;
#pragma unroll
          for (int c = 0; c < M; ++c) {
            double v = 0.0;
#pragma unroll
            for (int j = 0; j < NF; ++j)
              v = fma(T.trace[0][sp][j], tile[(VS::FROW + j * M + c) * VM_LDU + lane], v);
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
          for (int j = 0; j < NF; ++j)
            R[fnode_of(PD, f, j) * M + c] = fma(T.trace[f][s][j], H, R[fnode_of(PD, f, j) * M + c]);
        }
      }
    }
    if (!pv) continue;
    if (deg) flag_degenerate(r, pr, e);
    if (r.mode == MODE_RESIDUAL) {
      double* o_ = r.out + ((size_t)pr * r.ne + e) * NU;
#pragma unroll
      for (int i = 0; i < NU; ++i) o_[i] = R[i];
    } else {
      double r2 = 0.0;
#pragma unroll
      for (int i = 0; i < NU; ++i) r2 = fma(R[i], R[i], r2);
      acc += r.mode == MODE_OBJECTIVE ? 0.5 * rho * (r2 + N * N) : r2;
    }
  }
  if (r.mode == MODE_RESIDUAL) return;
  red[warp][lane] = acc;
  __syncthreads();
  if (warp == 0 && pv) {
    double v = 0.0;
#pragma unroll
    for (int w = 0; w < VM_THREADS / 32; ++w) v += red[w][lane];
    // device-sized passes: partials by compacted slot (sum_partials_kernel maps slot -> row)
    r.part[(size_t)(r.dyn_count ? gi * 32 + lane : pr) * gxr + xi] = v;
  }
}

}  // namespace strom
