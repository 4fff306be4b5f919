// Internal header shared by the C-ABI translation unit and the per-law kernel units.
#pragma once
#include <cuda_runtime.h>
#include <algorithm>
#include <cstring>
#include <string>
#include <vector>
#include "../../include/strom_b200.h"
#include "element_kernels.cuh"

namespace strom {
struct LmWork {
  int P = 0, K = 0, ku = 0, kx = 0, nmu = 0;
  void* buf = nullptr;
  size_t bytes = 0;
};

inline void lm_free(LmWork& w) {
  if (w.buf) cudaFree(w.buf);
  w = LmWork();
}

}  // namespace strom

namespace strom_host {
using namespace strom;

int fail(int code, const std::string& msg);

#define CK(x)                                                                      \
  do {                                                                             \
    cudaError_t _e = (x);                                                          \
    if (_e != cudaSuccess) return strom_host::fail(-2, std::string(#x ": ") + cudaGetErrorString(_e)); \
  } while (0)

struct EvalArgs {
  int mode;
  const int* mask;
  const double *w, *tau, *mu;
  int P;
  const int* active;
  const double* rho;
  int A;
  double* out;
  int* degen;
  cudaStream_t stream;
  const int* list = nullptr;       // ascending requested rows (compacted); with dyn_count: *dyn_count of them
  const int* dyn_count = nullptr;  // device-sized pass (graph-resident LM rounds): live row count on the device
};

}  // namespace strom_host

using strom_host::EvalArgs;

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
  long long u0_stride = 0, x_stride = 0;
  double* part = nullptr;
  size_t part_cap = 0;
  int* degen_fill = nullptr;
  int* degen_list = nullptr;
  int degen_cap = 0;
  int* degen_scratch = nullptr;
  int degen_scratch_cap = 0;
  std::vector<std::vector<int>> last_degen;
  int num_sms = 148;
  double* test_tab = nullptr;  // enriched test-space tabulation (device, owned), strom_set_test_space
  int test_nb = 0;
  bool has_wall = false;  // slip-wall faces (BC_REFLECT) in the mesh
  double* stage_h = nullptr;  // pinned staging of strom_eval_host
  double* stage_d = nullptr;  // its device twin
  size_t stage_cap = 0;       // doubles
  strom::LmWork lm;
  cudaStream_t lm_stream = nullptr;  // private capture stream of the LM graph
  cudaGraph_t lm_graph = nullptr;    // the last built LM graph, reused while its key matches
  cudaGraphExec_t lm_exec = nullptr;
  std::vector<char> lm_key;
  int lm_graph_builds = 0;
  unsigned long long epoch = 0;      // bumped whenever bases / offsets change (graph key)
  // statistics of the last strom_lm_solve: control rounds, derivative / objective passes
  int lm_rounds = 0, lm_dpasses = 0, lm_opasses = 0;
  double lm_rows[2] = {0, 0};      // rows evaluated by the derivatives / objective passes of the last solve
  double lm_ms[4] = {0, 0, 0, 0};  // device time of the last solve: control rounds, d-only / o-only / d+o pass gaps
  bool prof = false;
  std::vector<cudaEvent_t> ev;
  int nprof = 0;
};

namespace strom_host {
int ensure_part(strom_handle* h, size_t n);
void prof_mark(strom_handle* h, cudaStream_t st, int which);
int eval_linadv(strom_handle* h, const EvalArgs& a);
int eval_linadv_ms(strom_handle* h, const EvalArgs& a);
int eval_burgers_st(strom_handle* h, const EvalArgs& a);
int eval_strip(strom_handle* h, const EvalArgs& a);
int eval_euler(strom_handle* h, const EvalArgs& a);
int eval_euler_roe(strom_handle* h, const EvalArgs& a);
int eval_euler_wall(strom_handle* h, const EvalArgs& a);
}  // namespace strom_host
