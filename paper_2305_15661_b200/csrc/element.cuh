// Shared definitions for the B200 element kernels (see element_kernels.cu).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include "laws.cuh"

namespace strom {

constexpr int KMAX = 40;      // max k_u + k_x (padded Gram dimension <= 40)
constexpr int KXMAX = 16;     // max k_x
constexpr int NMU = 4;        // max parameters per mu vector
constexpr int DERIV_THREADS = 128;

enum Mode {
  MODE_OBJECTIVE = 0, MODE_DERIVS = 1, MODE_CONTRIB = 2, MODE_CONTRIB_SPLIT = 3,
  MODE_RESIDUAL = 4, MODE_RESNORM2 = 5, MODE_CONTRIB_LPROWS = 6, MODE_ELEMJAC = 7,
  MODE_ELEMJAC_ENRICHED = 8
};

// reference-element constants; lives in the kernel parameter (constant) bank
template <int NB, int NQ, int NS, int NF>
struct Tabs {
  double phi[NQ][NB];
  double dphi[NQ][NB][2];
  double wq[NQ];
  double bary[NQ][3];
  double trace[3][NS][NF];
  double ws[NS];
  double t2[NF][NF][NS];  // trace[0][s][j] * trace[0][s][j'] (face-block products)
  double wsum;
  int fnode[3][NF];
};

struct Run {
  // mesh
  int ne;
  const int* __restrict__ elem_nodes;
  const double* __restrict__ nodes;
  const int* __restrict__ nbr;
  const uint8_t* __restrict__ finfo;
  const double* __restrict__ eta_ref;
  // bases
  const double* __restrict__ phi;
  const double* __restrict__ psi;
  const double* __restrict__ xref;
  const double* __restrict__ u0;
  long long u0_stride, x_stride;  // per-parameter offsets (snapshots): U0 + p*u0_stride, X + p*x_stride
  int ku, kx, K, KP, LDJ;
  // call
  const double* __restrict__ w;
  const double* __restrict__ tau;
  const double* __restrict__ mu;
  int nmu, P;
  const int* __restrict__ active;
  const double* __restrict__ rho;
  int A;
  double* __restrict__ out;
  double* __restrict__ part;
  int* __restrict__ degen;
  int* __restrict__ degen_list;
  int degen_cap;
  int* __restrict__ degen_fill;
  int mode;
  const int* __restrict__ mask;  // per-row enable (batched LM), or null
  const int* __restrict__ list;  // value_mu_kernel: compacted enabled rows (nlist of them), or null
  int nlist;
  // device-sized launch (graph-resident LM rounds): the live row count is read on the device
  // (*dyn_count rows, list[0 .. count)) and the 1-D grid is split over them there (dyn_gx)
  const int* __restrict__ dyn_count;
  int dyn_target, dyn_maxb, dyn_ceil;
  int U;          // units per tile (derivs kernel)
  int ntiles;     // tiles per parameter
  int gx;         // blocks per parameter
  int unit_stride;  // doubles per unit in shared memory
  int gx_warp_stride;  // doubles per warp in shared memory (warp kernel)
  // enriched test space (MODE_ELEMJAC_ENRICHED): [NQ][nbt][2] reference gradients, then
  // [3][NS][nbt] face traces of the degree p+1 nodal basis (geometry.py:162-196)
  const double* __restrict__ test_tab;
  int test_nb;
  double kappa, eps;
  double lawp[8];
};

// CTAs per live row of a device-sized launch: the host formulas of eval_impl.cuh
// (launch_mma_t: one wave, floor; launch_warp: ceil) evaluated with the device count
__device__ __forceinline__ int dyn_gx(int target, int maxb, int ceil_div, int live) {
  live = live > 0 ? live : 1;
  const int g = ceil_div ? (target + live - 1) / live : target / live;
  return g < 1 ? 1 : (g > maxb ? maxb : g);
}

template <int NB, int NQ, int NS, int NF>
struct Params {
  Tabs<NB, NQ, NS, NF> t;
  Run r;
};

}  // namespace strom
