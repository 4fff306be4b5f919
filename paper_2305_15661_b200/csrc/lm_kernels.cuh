// K5: batched Levenberg-Marquardt over many parameter points (one CTA per mu).
//
// Device restatement of strom/lm.py:129-271 as a resumable state machine.
// Each round the control kernel advances every mu until it needs an
// evaluation, then posts a request: a derivatives pass at (w, tau) or a
// batch of objective trials at w + alpha_j dw (speculative backtracking:
// alpha_j = 2^-j for the next LM_B values of j; the accepted step is the
// first j that passes Armijo, exactly the sequential loop's choice).  The
// rounds run as a CUDA-graph WHILE loop (lm_capi.inc): the compaction kernel
// decides on the device which batched evaluations a round launches (IF nodes)
// and whether another round follows, so a batch of solves is one graph launch.
// The K x K normal equations [[H_ww, H_wt],[H_wt^T, H_tt + lam I]] dz = -[S;T]
// are solved in-kernel by LDL^T (no pivoting; singular = zero / non-finite
// pivot or non-finite solution, lm.py:111-126).
#pragma once
#include <cmath>
#include <cstdint>

namespace strom {

#ifndef STROM_LM_B
#define STROM_LM_B 4
#endif
#ifndef STROM_LM_THREADS
#define STROM_LM_THREADS 256
#endif
constexpr int LM_B = STROM_LM_B;              // speculative objective trials per round
constexpr int LM_THREADS = STROM_LM_THREADS;  // threads of the per-mu control block

enum LmPhase {
  PH_START = 0, PH_SI_DERIV, PH_SI_BASEJ, PH_SI_LS, PH_MAIN_DERIV, PH_MAIN_ITER_READY, PH_MAIN_LS,
  PH_MAIN_ACCEPT_DERIV, PH_DONE
};
enum LmReason { R_FIRST_ORDER = 0, R_MAX_ITERS = 1, R_LS_FAIL = 2, R_DEGENERATE = 3 };

struct LmCfg {
  double eps1, eps2, lambda0, lambda_inc, lambda_dec, ratio_hi, ratio_lo;
  int max_iters;
  double c1, c2;
  int max_backtracks;
  double lambda_cap, w0_tol;
  int w0_iters, w0_lsq;
};

struct LmState {
  int phase, it, si_cnt, attempts, j0, done, reason, n_done, nhist, have_best, lam_set, si_have_J, evals;
  int ntr;  // trials posted in the current batch (first batch of a line search: nb_first)
  double lam, lam_floor, J, J_si, gdot, J_new, alpha, si_target, nS_prev, nT_prev, J_prev;
  double best_J, best_nS, best_nT;
};

// Device-side round control (one per solve batch)
struct LmCtl {
  int cnt[2][4];      // per round parity: [n_unfinished, n_derivs, n_obj mu, unused]
  int round;          // control rounds run so far
  int waited;         // consecutive rounds a derivatives pass was deferred
  int ran_d, ran_o;   // whether the previous round ran the derivatives / objective pass
  int dcount, ocount; // rows of this round's derivatives / objective passes (dlist / olist)
  int nd, no;         // passes run (statistics)
  int overflow;       // max_rounds reached with unfinished solves
  int ticket;         // control blocks finished this round (the last one ends the round)
  // device-side timing (globaltimer, ns): when block 0 of a control round starts / the round
  // ends; the gaps between a round end and the next round's start are the batched passes
  unsigned long long t_start, t_end;
  unsigned long long ns_ctl, ns_d, ns_o, ns_do;  // control rounds; gaps after rounds that ran d only / o only / both
  unsigned long long rows_d, rows_o;             // rows evaluated by the derivatives / objective passes (statistics)
};

struct LmRun {
  int P, ku, kx, K, nmu;
  int nb_first;      // trials in the first batch of a line search (1..LM_B); later batches LM_B
  int max_rounds;
  LmCtl* ctl;
  LmCfg cfg;
  LmState* st;
  double* w;        // (P, ku) current
  double* tau;      // (P, kx)
  double* dw;       // (P, K) step
  double* best_w;   // (P, K)
  double* S;        // (P, K) current gradient (S;T)
  double* H;        // (P, K*K) current Gauss-Newton matrix
  const double* mu; // (P, nmu)
  const double* dout;  // (P, 1+K+K*K) derivs results
  const int* ddeg;     // (P)
  const double* oout;  // (P*LM_B) objective trial results
  const int* odeg;     // (P*LM_B)
  int* req_d;          // (P) derivs requested
  int* req_o;          // (P*LM_B) objective rows requested
  double* tw;          // (P*LM_B, ku) trial points
  double* ttau;        // (P*LM_B, kx)
  double* tmu;         // (P*LM_B, nmu)
  int* degen_fill;     // the evaluation kernels' degenerate-list fill counter (zeroed per round)
  int* olist;          // (P*LM_B) compacted objective rows requested (ascending)
  int* dlist;          // (P) compacted derivatives rows requested (ascending)
  double* hist;        // (P, max_iters+1, 6) or null
  double* status;      // (P, 8)
};

__device__ __forceinline__ double nrm2(const double* v, int n) {
  double s = 0.0;
  for (int i = 0; i < n; ++i) s = fma(v[i], v[i], s);
  return sqrt(s);
}

// LDL^T solve of the n x n symmetric system in A (row-major, overwritten) for
// x = A^{-1} b; all threads of the block participate.  Returns false when a
// pivot is zero / non-finite or the solution is non-finite.
// tri[q] = (ii << 8) | kk for the row-major lower triangle q = ii (ii + 1) / 2 + kk, kk <= ii
// (the enumeration is the same prefix for every triangle size, so one table serves every step)
constexpr int LM_TRI = KMAX * (KMAX + 1) / 2;

static __device__ bool ldlt_solve(double* A, int n, double* b, double* x, int* flag, const unsigned short* tri) {
  const int t = threadIdx.x, nt = blockDim.x;
  if (t == 0) *flag = 1;
  __syncthreads();
  for (int j = 0; j < n; ++j) {
    const double d = A[j * n + j];
    if (!(d != 0.0) || !isfinite(d)) {
      if (t == 0) *flag = 0;
    }
    __syncthreads();
    if (*flag == 0) return false;
    for (int i = j + 1 + t; i < n; i += nt) A[i * n + j] = A[i * n + j] / d;  // L[i][j]
    __syncthreads();
    // trailing update A[i][k] -= L[i][j] d L[k][j], j < k <= i: one (i, k) entry per thread
    // (per entry the same j-ascending update sequence as the row-wise loop)
    const int m = n - j - 1, cnt = m * (m + 1) / 2;
    for (int q = t; q < cnt; q += nt) {
      const int ii = tri[q] >> 8, kk = tri[q] & 255;  // (ii, kk), 0 <= kk <= ii < m
      const int i = j + 1 + ii, k = j + 1 + kk;
      A[i * n + k] -= (A[i * n + j] * d) * A[k * n + j];
    }
    __syncthreads();
  }
  // L y = b: column sweep (per entry the same k-ascending subtraction order as the row form)
  for (int i = 0; i < n; ++i) {
    const double yi = b[i];
    for (int k = i + 1 + t; k < n; k += nt) b[k] -= A[k * n + i] * yi;
    __syncthreads();
  }
  for (int i = t; i < n; i += nt) x[i] = b[i] / A[i * n + i];
  __syncthreads();
  // L^T x = z: column sweep, x[k] -= L[i][k] x[i] for k < i (i descending)
  for (int i = n - 1; i > 0; --i) {
    const double xi = x[i];
    for (int k = t; k < i; k += nt) x[k] -= A[i * n + k] * xi;
    __syncthreads();
  }
  if (t == 0) {
    bool ok = true;
    for (int i = 0; i < n; ++i) ok = ok && isfinite(x[i]);
    *flag = ok ? 1 : 0;
  }
  __syncthreads();
  return *flag != 0;
}

static __global__ void lm_init_kernel(LmRun R, const double* w0, const double* tau0) {
  const int p = blockIdx.x;
  for (int i = threadIdx.x; i < R.ku; i += blockDim.x) R.w[p * R.ku + i] = w0[p * R.ku + i];
  for (int i = threadIdx.x; i < R.kx; i += blockDim.x) R.tau[p * R.kx + i] = tau0[p * R.kx + i];
  if (threadIdx.x == 0) {
    LmState s;
    memset(&s, 0, sizeof(s));
    s.phase = PH_START;
    s.lam = R.cfg.lambda0;
    s.lam_set = R.cfg.lambda0 >= 0.0;
    R.st[p] = s;
  }
}

// post objective trials at w + alpha_j dw (state init: tau frozen, dz = dw only)
static __device__ void post_trials(const LmRun& R, int p, int j0, bool frozen_tau, int ntr) {
  ntr = min(ntr, LM_B);
  for (int j = 0; j < LM_B; ++j) {
    const int row = p * LM_B + j;
    const bool on = j < ntr;
    R.req_o[row] = on;
    if (!on) continue;
    const double alpha = ldexp(1.0, -(j0 + j));
    for (int i = 0; i < R.ku; ++i) R.tw[row * R.ku + i] = R.w[p * R.ku + i] + alpha * R.dw[p * R.K + i];
    for (int i = 0; i < R.kx; ++i)
      R.ttau[row * R.kx + i] = R.tau[p * R.kx + i] + (frozen_tau ? 0.0 : alpha * R.dw[p * R.K + R.ku + i]);
    for (int i = 0; i < R.nmu; ++i) R.tmu[row * R.nmu + i] = R.mu[p * R.nmu + i];
  }
}

static __device__ void hist_row(const LmRun& R, int p, int it, double J, double nS, double nT, double lam, double alpha) {
  if (!R.hist) return;
  double* h = R.hist + ((size_t)p * (R.cfg.max_iters + 1) + it) * 6;
  h[0] = it; h[1] = J; h[2] = nS; h[3] = nT; h[4] = lam; h[5] = alpha;
}

enum LmAction { ACT_ADVANCE = 0, ACT_SOLVE_SI = 1, ACT_SOLVE_MAIN = 2, ACT_WAIT = 3 };

// the solve's system is filled by all threads of the block right before the solve
// (lm_control_kernel); the state machine only decides which one (ACT_SOLVE_SI / _MAIN)

__device__ __forceinline__ void lm_request_derivs(const LmRun& R, int p, LmState& s, int phase) {
  s.phase = phase;
  R.req_d[p] = 1;
  s.evals++;
}

// escalate after a failed attempt (lm.py:215-225, 237-241); returns the next action
__device__ __forceinline__ int lm_escalate(const LmRun& R, int p, LmState& s, double* A, double* rhs, bool singular) {
  const LmCfg& c = R.cfg;
  s.lam = singular ? fmax(2.0 * s.lam, 1e-12) * 10.0 : fmax(4.0 * s.lam, 1e-12);
  s.attempts += 1;
  if (s.lam > c.lambda_cap || s.attempts >= 60) {
    s.reason = R_LS_FAIL;
    s.phase = PH_DONE;
    return ACT_WAIT;
  }
  return ACT_SOLVE_MAIN;
}

// advance the state machine from the current phase; thread 0 only
static __device__ int lm_advance(const LmRun& R, int p, LmState& s, double* A, double* rhs) {
  const LmCfg& c = R.cfg;
  const int K = R.K, ku = R.ku, kx = R.kx;
  double* Sv = R.S + p * K;
  double* Hm = R.H + (size_t)p * K * K;
  const double* d = R.dout + (size_t)p * (1 + K + K * K);
  switch (s.phase) {
    case PH_START:
      if (c.w0_lsq && ku > 0) {
        s.si_cnt = 0; s.si_have_J = 0;
        lm_request_derivs(R, p, s, PH_SI_DERIV);
      } else {
        lm_request_derivs(R, p, s, PH_MAIN_DERIV);
      }
      return ACT_WAIT;
    case PH_SI_DERIV:
    case PH_MAIN_DERIV:
    case PH_MAIN_ACCEPT_DERIV: {
      if (R.ddeg[p] > 0) {  // derivatives raise DegenerateMappingError out of lm_solve
        s.reason = R_DEGENERATE;
        s.phase = PH_DONE;
        return ACT_WAIT;
      }
      // (S, H) were copied from the derivatives output by the whole block
      const double Jd = d[0];
      if (s.phase == PH_SI_DERIV) {  // lm.py:134-141
        const double nSw = nrm2(Sv, ku);
        if (s.si_cnt == 0 && !s.si_have_J) s.si_target = c.w0_tol * fmax(1.0, nSw);
        if (s.si_cnt >= c.w0_iters || nSw <= s.si_target) {
          lm_request_derivs(R, p, s, PH_MAIN_DERIV);
          return ACT_WAIT;
        }
        return ACT_SOLVE_SI;
      }
      if (s.phase == PH_MAIN_DERIV) {  // lm.py:185
        s.J = Jd;
        s.it = 0;
        s.phase = PH_MAIN_ITER_READY;
        return ACT_ADVANCE;
      }
      // accepted step: gain ratio, curvature, damping update (lm.py:248-264)
      const double pred = -0.5 * s.alpha * s.gdot;
      const double ratio = pred > 0.0 ? (s.J_prev - s.J_new) / pred : 1.0;
      s.J = isfinite(s.J_new) ? s.J_new : Jd;
      double sd = 0.0;
      for (int i = 0; i < K; ++i) sd = fma(Sv[i], R.dw[p * K + i], sd);
      const bool curv_ok = sd >= c.c2 * s.gdot;
      if (s.alpha < 0.25 || ratio < c.ratio_lo) s.lam *= c.lambda_inc;
      else if (s.alpha == 1.0 && ratio > c.ratio_hi && curv_ok) s.lam *= c.lambda_dec;
      s.lam = fmin(fmax(s.lam, s.lam_floor), c.lambda_cap);
      hist_row(R, p, s.it, s.J_prev, s.nS_prev, s.nT_prev, s.lam, s.alpha);
      s.it += 1;
      s.phase = PH_MAIN_ITER_READY;
      return ACT_ADVANCE;
    }
    case PH_SI_BASEJ: {  // J = problem.objective(w, tau) (lm.py:146)
      const int row = p * LM_B;
      s.J_si = R.odeg[row] > 0 ? INFINITY : R.oout[row];
      s.si_have_J = 1;
      s.j0 = 0;
      s.phase = PH_SI_LS;
      s.ntr = R.nb_first;
      post_trials(R, p, 0, true, s.ntr);
      s.evals++;
      return ACT_WAIT;
    }
    case PH_SI_LS: {  // Armijo on the frozen-tau state step (lm.py:147-160)
      double sdw = 0.0;
      for (int i = 0; i < ku; ++i) sdw = fma(Sv[i], R.dw[p * K + i], sdw);
      for (int j = 0; j < s.ntr && s.j0 + j < 30; ++j) {
        const int row = p * LM_B + j;
        const double Jt = R.odeg[row] > 0 ? INFINITY : R.oout[row];
        const double alpha = ldexp(1.0, -(s.j0 + j));
        if (Jt <= s.J_si + 1e-4 * alpha * sdw) {
          for (int i = 0; i < ku; ++i) R.w[p * ku + i] += alpha * R.dw[p * K + i];
          s.J_si = Jt;
          s.si_cnt += 1;
          lm_request_derivs(R, p, s, PH_SI_DERIV);
          return ACT_WAIT;
        }
      }
      if (s.j0 + s.ntr < 30) {
        s.j0 += s.ntr;
        s.ntr = min(LM_B, 30 - s.j0);
        post_trials(R, p, s.j0, true, s.ntr);
        s.evals++;
        return ACT_WAIT;
      }
      lm_request_derivs(R, p, s, PH_MAIN_DERIV);  // not accepted: leave the state init
      return ACT_WAIT;
    }
    case PH_MAIN_ITER_READY: {  // top of the LM iteration (lm.py:187-211)
      if (s.it >= c.max_iters) {
        s.reason = R_MAX_ITERS;
        s.phase = PH_DONE;
        return ACT_WAIT;
      }
      const double nS = nrm2(Sv, ku), nT = nrm2(Sv + ku, kx);
      if (!s.have_best || s.J < s.best_J) {
        s.have_best = 1; s.best_J = s.J; s.best_nS = nS; s.best_nT = nT;
        for (int i = 0; i < ku; ++i) R.best_w[p * K + i] = R.w[p * ku + i];
        for (int i = 0; i < kx; ++i) R.best_w[p * K + ku + i] = R.tau[p * kx + i];
      }
      if (!s.lam_set) {
        if (kx) {
          double tr = 0.0;
          for (int i = 0; i < kx; ++i) tr += Hm[(ku + i) * K + ku + i];
          s.lam = 1e-4 * tr / kx;
        } else {
          s.lam = 0.0;
        }
        s.lam_floor = s.lam > 0.0 ? 1e-10 * s.lam : 0.0;
        s.lam_set = 1;
      }
      hist_row(R, p, s.it, s.J, nS, nT, s.lam, NAN);
      if (nS <= c.eps1 && nT <= c.eps2) {
        hist_row(R, p, s.it, s.J, nS, nT, s.lam, 0.0);
        s.reason = R_FIRST_ORDER;
        s.n_done = s.it;
        s.done = 2;
        s.phase = PH_DONE;
        return ACT_WAIT;
      }
      s.n_done = s.it + 1;
      s.nS_prev = nS; s.nT_prev = nT; s.J_prev = s.J;
      s.attempts = 0;
      return ACT_SOLVE_MAIN;
    }
    case PH_MAIN_LS: {  // Armijo backtracking results (lm.py:226-236)
      for (int j = 0; j < s.ntr && s.j0 + j < c.max_backtracks; ++j) {
        const int row = p * LM_B + j;
        const double Jt = R.odeg[row] > 0 ? INFINITY : R.oout[row];
        const double alpha = ldexp(1.0, -(s.j0 + j));
        if (Jt <= s.J + c.c1 * alpha * s.gdot) {
          s.J_new = Jt;
          s.alpha = alpha;
          for (int i = 0; i < ku; ++i) R.w[p * ku + i] += alpha * R.dw[p * K + i];
          for (int i = 0; i < kx; ++i) R.tau[p * kx + i] += alpha * R.dw[p * K + ku + i];
          lm_request_derivs(R, p, s, PH_MAIN_ACCEPT_DERIV);
          return ACT_WAIT;
        }
      }
      if (s.j0 + s.ntr < c.max_backtracks) {
        s.j0 += s.ntr;
        s.ntr = min(LM_B, c.max_backtracks - s.j0);
        post_trials(R, p, s.j0, false, s.ntr);
        s.evals++;
        return ACT_WAIT;
      }
      return lm_escalate(R, p, s, A, rhs, false);
    }
    case PH_DONE:
    default:
      return ACT_WAIT;
  }
}

// process a finished solve; thread 0 only
static __device__ int lm_after_solve(const LmRun& R, int p, LmState& s, int act, bool ok, const double* x, double* A,
                              double* rhs) {
  const int K = R.K, ku = R.ku, kx = R.kx, nmu = R.nmu;
  if (act == ACT_SOLVE_SI) {
    if (!ok) {  // LinAlgError ends the state init (lm.py:142-143)
      lm_request_derivs(R, p, s, PH_MAIN_DERIV);
      return ACT_WAIT;
    }
    for (int i = 0; i < ku; ++i) R.dw[p * K + i] = x[i];
    if (!s.si_have_J) {
      s.phase = PH_SI_BASEJ;
      const int row = p * LM_B;
      R.req_o[row] = 1;
      for (int i = 0; i < ku; ++i) R.tw[row * ku + i] = R.w[p * ku + i];
      for (int i = 0; i < kx; ++i) R.ttau[row * kx + i] = R.tau[p * kx + i];
      for (int i = 0; i < nmu; ++i) R.tmu[row * nmu + i] = R.mu[p * nmu + i];
    } else {
      s.j0 = 0;
      s.phase = PH_SI_LS;
      s.ntr = R.nb_first;
      post_trials(R, p, 0, true, s.ntr);
    }
    s.evals++;
    return ACT_WAIT;
  }
  // main iteration attempt (lm.py:212-225)
  if (!ok) return lm_escalate(R, p, s, A, rhs, true);
  const double* Sv = R.S + p * K;
  double gd = 0.0;
  for (int i = 0; i < K; ++i) gd = fma(Sv[i], x[i], gd);
  if (!isfinite(gd) || gd >= 0.0) return lm_escalate(R, p, s, A, rhs, false);
  s.gdot = gd;
  for (int i = 0; i < K; ++i) R.dw[p * K + i] = x[i];
  // no backtracking budget: the Armijo loop posts nothing and J_new stays None (lm.py:226-241)
  if (R.cfg.max_backtracks <= 0) return lm_escalate(R, p, s, A, rhs, false);
  s.j0 = 0;
  s.phase = PH_MAIN_LS;
  s.ntr = min(R.nb_first, R.cfg.max_backtracks);
  post_trials(R, p, 0, false, s.ntr);
  s.evals++;
  return ACT_WAIT;
}

// one control round; blockDim = LM_THREADS, dynamic smem (K*K + 2K) doubles
static __device__ void lm_round_end(const LmRun& R, cudaGraphConditionalHandle h_while, cudaGraphConditionalHandle h_d,
                                    cudaGraphConditionalHandle h_o, int graph);
static __device__ void lm_control_body(const LmRun& R, int p, LmState& s, double* A, double* rhs, double* x,
                                       const unsigned short* s_tri, int* counters, int* s_act_p, int* s_flag_p);

static __global__ void __launch_bounds__(LM_THREADS) lm_control_kernel(LmRun R, cudaGraphConditionalHandle h_while,
                                                                       cudaGraphConditionalHandle h_d,
                                                                       cudaGraphConditionalHandle h_o, int graph) {
  extern __shared__ double sm[];
  const int p = blockIdx.x, K = R.K;
  double* A = sm;
  double* rhs = A + K * K;
  double* x = rhs + K;
  __shared__ int s_act, s_flag;
  __shared__ LmState s;
  __shared__ int s_hold;
  __shared__ unsigned short s_tri[LM_TRI];
  for (int q = threadIdx.x; q < K * (K + 1) / 2; q += blockDim.x) {
    int ii = (int)((sqrtf(8.0f * q + 1.0f) - 1.0f) * 0.5f);
    while (ii * (ii + 1) / 2 > q) --ii;
    while ((ii + 1) * (ii + 2) / 2 <= q) ++ii;
    s_tri[q] = (unsigned short)((ii << 8) | (q - ii * (ii + 1) / 2));
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    LmCtl& C = *R.ctl;
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (C.round > 0) {
      const unsigned long long gap = t - C.t_end;
      if (C.ran_d && C.ran_o) C.ns_do += gap;
      else if (C.ran_d) C.ns_d += gap;
      else if (C.ran_o) C.ns_o += gap;
    }
    C.t_start = t;
  }
  const int par = R.ctl->round & 1;
  int* const counters = R.ctl->cnt[par];
  if (blockIdx.x == 0 && threadIdx.x < 4) R.ctl->cnt[par ^ 1][threadIdx.x] = 0;  // next round's set
  if (threadIdx.x == 0) {
    s = R.st[p];
    // a request deferred last round stays posted; the mu waits (no state change)
    const bool wd = s.phase == PH_SI_DERIV || s.phase == PH_MAIN_DERIV || s.phase == PH_MAIN_ACCEPT_DERIV;
    const bool wo = s.phase == PH_SI_BASEJ || s.phase == PH_SI_LS || s.phase == PH_MAIN_LS;
    s_hold = (wd && !R.ctl->ran_d) || (wo && !R.ctl->ran_o);
    if (!s_hold) {
      R.req_d[p] = 0;
      for (int j = 0; j < LM_B; ++j) R.req_o[p * LM_B + j] = 0;
    }
    s_act = ACT_ADVANCE;
  }
  __syncthreads();
  if (s_hold) {
    if (threadIdx.x == 0) {
      atomicAdd(&counters[0], 1);
      if (R.req_d[p]) atomicAdd(&counters[1], 1);
      if (R.req_o[p * LM_B]) atomicAdd(&counters[2], 1);
    }
  } else {
    lm_control_body(R, p, s, A, rhs, x, s_tri, counters, &s_act, &s_flag);
  }
  // the last block to finish ends the round (compaction, pass decisions, graph conditions)
  __shared__ int s_last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    s_last = atomicAdd(&R.ctl->ticket, 1) == (int)gridDim.x - 1;
  }
  __syncthreads();
  if (s_last) {
    __threadfence();
    lm_round_end(R, h_while, h_d, h_o, graph);
  }
}

static __device__ void lm_control_body(const LmRun& R, int p, LmState& s, double* A, double* rhs, double* x,
                                       const unsigned short* s_tri, int* counters, int* s_act_p, int* s_flag_p) {
  const int K = R.K;
  int& s_act = *s_act_p;
  // the mu's vectors live in shared memory for the round: the state machine (thread 0)
  // then works on shared copies; loads / stores of the global arrays are block-parallel
  __shared__ double c_w[32], c_tau[KXMAX], c_dw[KMAX], c_S[KMAX], c_best[KMAX];
  __shared__ double c_tw[LM_B * 32], c_ttau[LM_B * KXMAX], c_tmu[LM_B * NMU];
  const int ku = R.ku, kx = R.kx, nmu = R.nmu, t = threadIdx.x, nt = blockDim.x;
  double* Hm = R.H + (size_t)p * K * K;
  const bool dphase = (s.phase == PH_SI_DERIV || s.phase == PH_MAIN_DERIV || s.phase == PH_MAIN_ACCEPT_DERIV) && R.ddeg[p] == 0;
  if (dphase) {
    const double* d = R.dout + (size_t)p * (1 + K + K * K);  // a finished derivatives pass -> (S, H)
    for (int i = t; i < K; i += nt) c_S[i] = d[1 + i];
    for (int i = t; i < K * K; i += nt) Hm[i] = d[1 + K + i];
  } else {
    for (int i = t; i < K; i += nt) c_S[i] = R.S[p * K + i];
  }
  for (int i = t; i < ku; i += nt) c_w[i] = R.w[p * ku + i];
  for (int i = t; i < kx; i += nt) c_tau[i] = R.tau[p * kx + i];
  for (int i = t; i < K; i += nt) { c_dw[i] = R.dw[p * K + i]; c_best[i] = R.best_w[p * K + i]; }
  LmRun Rl = R;  // per-mu arrays redirected to the shared copies (same indexing)
  Rl.w = c_w - (size_t)p * ku;
  Rl.tau = c_tau - (size_t)p * kx;
  Rl.dw = c_dw - (size_t)p * K;
  Rl.S = c_S - (size_t)p * K;
  Rl.best_w = c_best - (size_t)p * K;
  Rl.tw = c_tw - (size_t)p * LM_B * ku;
  Rl.ttau = c_ttau - (size_t)p * LM_B * kx;
  Rl.tmu = c_tmu - (size_t)p * LM_B * nmu;
  __syncthreads();
  for (int guard = 0; guard < 100000; ++guard) {
    if (t == 0 && s_act == ACT_ADVANCE) s_act = lm_advance(Rl, p, s, A, rhs);
    __syncthreads();
    const int act = s_act;
    if (act == ACT_WAIT) break;
    if (act == ACT_ADVANCE) continue;
    const int n = act == ACT_SOLVE_SI ? ku : K;
    // the system: H_ww (state init, lm.py:141) or [[H_ww, H_wt], [H_wt^T, H_tt + lam I]] (lm.py:116-122)
    const double lam = s.lam;
    for (int i = t; i < n * n; i += nt) {
      const int row = i / n, col = i % n;
      A[i] = Hm[row * K + col] + ((act == ACT_SOLVE_MAIN && row == col && row >= ku) ? lam : 0.0);
    }
    for (int i = t; i < n; i += nt) rhs[i] = -c_S[i];
    __syncthreads();
    const bool ok = ldlt_solve(A, n, rhs, x, s_flag_p, s_tri);
    if (t == 0) s_act = lm_after_solve(Rl, p, s, act, ok, x, A, rhs);
    __syncthreads();
  }
  for (int i = t; i < ku; i += nt) R.w[p * ku + i] = c_w[i];
  for (int i = t; i < kx; i += nt) R.tau[p * kx + i] = c_tau[i];
  for (int i = t; i < K; i += nt) { R.dw[p * K + i] = c_dw[i]; R.S[p * K + i] = c_S[i]; R.best_w[p * K + i] = c_best[i]; }
  for (int j = 0; j < LM_B; ++j) {
    const int row = p * LM_B + j;
    if (!R.req_o[row]) continue;
    for (int i = t; i < ku; i += nt) R.tw[(size_t)row * ku + i] = c_tw[j * ku + i];
    for (int i = t; i < kx; i += nt) R.ttau[(size_t)row * kx + i] = c_ttau[j * kx + i];
    for (int i = t; i < nmu; i += nt) R.tmu[(size_t)row * nmu + i] = c_tmu[j * nmu + i];
  }
  if (t == 0) {
    R.st[p] = s;
    if (s.phase != PH_DONE) atomicAdd(&counters[0], 1);
    if (R.req_d[p]) atomicAdd(&counters[1], 1);
    if (R.req_o[p * LM_B]) atomicAdd(&counters[2], 1);
    // degenerate flags of the evaluations requested now start at zero (read next round)
    if (R.req_d[p]) const_cast<int*>(R.ddeg)[p] = 0;
    for (int j = 0; j < LM_B; ++j)
      if (R.req_o[p * LM_B + j]) const_cast<int*>(R.odeg)[p * LM_B + j] = 0;
  }
}

// ascending compaction of flags[0 .. n) into list (one block, deterministic; the flags were
// written by other blocks of the same launch, so they are read past L1); returns the count to
// every thread
static __device__ int block_compact(const int* flags, int n, int* list, int* wsum) {
  const int t = threadIdx.x, lane = t & 31, wp = t >> 5;
  const int per = (n + blockDim.x - 1) / blockDim.x, lo = t * per;
  int c = 0;
  for (int i = lo; i < lo + per && i < n; ++i) c += __ldcg(flags + i) != 0;  // written by other blocks
  int x = c;  // inclusive warp scan
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) wsum[wp] = x;
  __syncthreads();
  if (wp == 0) {
    int v = lane < (int)(blockDim.x >> 5) ? wsum[lane] : 0;
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, v, o);
      if (lane >= o) v += y;
    }
    wsum[lane] = v;
  }
  __syncthreads();
  int pos = x - c + (wp > 0 ? wsum[wp - 1] : 0);
  for (int i = lo; i < lo + per && i < n; ++i)
    if (__ldcg(flags + i)) list[pos++] = i;
  const int total = wsum[(blockDim.x >> 5) - 1];
  __syncthreads();
  return total;
}

// End of a control round (the last control block to finish): compact the requested derivative / objective rows and
// decide on the device what the round launches.  A derivatives pass waits until every
// unfinished mu asks for one (or no objective trials are pending, or it was deferred
// LM_MAXWAIT rounds in a row): the mu meet at their derivative evaluations, so each K1 pass
// is a full batch (cfg3: 92 -> ~40 passes per batch); deferred requests stay posted and the
// mu waits, so no mu's iterates change.  In graph mode the IF / WHILE conditions are set here.
#ifndef STROM_LM_MAXWAIT
#define STROM_LM_MAXWAIT 3
#endif
constexpr int LM_MAXWAIT = STROM_LM_MAXWAIT;

static __device__ void lm_round_end(const LmRun& R, cudaGraphConditionalHandle h_while, cudaGraphConditionalHandle h_d,
                                    cudaGraphConditionalHandle h_o, int graph) {
  __shared__ int wsum[32];
  LmCtl& C = *R.ctl;
  const int* cnt = C.cnt[C.round & 1];
  const int nobj = block_compact(R.req_o, R.P * LM_B, R.olist, wsum);
  const int nder = block_compact(R.req_d, R.P, R.dlist, wsum);
  if (threadIdx.x != 0) return;
  const int n_active = __ldcg(cnt), n_d = __ldcg(cnt + 1), n_o = __ldcg(cnt + 2);  // atomics of every block
  const bool run_d = n_d > 0 && (n_o == 0 || n_d >= n_active || C.waited >= LM_MAXWAIT);
  const bool run_o = n_o > 0;
  C.waited = (n_d > 0 && !run_d) ? C.waited + 1 : 0;
  C.ran_d = run_d;
  C.ran_o = run_o;
  C.nd += run_d;
  C.no += run_o;
  if (run_d) C.rows_d += nder;
  if (run_o) C.rows_o += nobj;
  C.dcount = nder;
  C.ocount = nobj;
  C.round += 1;
  C.ticket = 0;
  {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    C.ns_ctl += t - C.t_start;
    C.t_end = t;
  }
  const bool more = n_active > 0 && C.round < R.max_rounds;
  if (n_active > 0 && !more) C.overflow = 1;
  *R.degen_fill = 0;
  if (graph) {
    cudaGraphSetConditional(h_d, more && run_d ? 1u : 0u);
    cudaGraphSetConditional(h_o, more && run_o ? 1u : 0u);
    cudaGraphSetConditional(h_while, more ? 1u : 0u);
  }
}

// results: best-iterate fallback (lm.py:266-270) and status rows
static __global__ void lm_finish_kernel(LmRun R) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= R.P) return;
  LmState& s = R.st[p];
  const int K = R.K, ku = R.ku, kx = R.kx;
  double J = s.J;
  double nS = nrm2(R.S + p * K, ku), nT = nrm2(R.S + p * K + ku, kx);
  const bool conv = s.reason == R_FIRST_ORDER;
  if (!conv && s.reason != R_DEGENERATE && s.have_best && s.best_J < J) {
    J = s.best_J; nS = s.best_nS; nT = s.best_nT;
    for (int i = 0; i < ku; ++i) R.w[p * ku + i] = R.best_w[p * K + i];
    for (int i = 0; i < kx; ++i) R.tau[p * kx + i] = R.best_w[p * K + ku + i];
  }
  double* o = R.status + (size_t)p * 8;
  o[0] = conv ? 1.0 : 0.0;
  o[1] = J;
  o[2] = nS;
  o[3] = nT;
  o[4] = conv ? s.n_done : s.n_done;
  o[5] = s.reason;
  o[6] = s.lam;
  o[7] = s.evals;
}

}  // namespace strom
