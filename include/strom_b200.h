/*
 * strom_b200 — C ABI of the B200 (sm_100a) EQP-IFT element core.
 *
 * The reference (`strom`, /root/reference/pkg) is pure Python; its hot-path
 * boundary is the `ReducedOperator` class (strom/reduced.py:116-251) and the
 * Levenberg-Marquardt protocol (strom/lm.py:10-17, 164-271).  Nothing in the
 * reference is an FFI, so every entry point below is the C-level
 * replacement of one Python method; the Python mirror in
 * paper_2305_15661_b200/reduced.py binds them through ctypes
 * (INTEGRATION.md shows the binding).
 *
 * Conventions: all array arguments are DEVICE pointers unless stated
 * otherwise; fp64 state, int32 indices; calls are ordered on `stream`
 * (a cudaStream_t, NULL = legacy default stream); no allocation happens on
 * the evaluation path (workspace is sized by strom_reserve).  Return codes:
 * 0 OK, 1 DEGENERATE (per-parameter degenerate counters are valid),
 * negative = argument or CUDA error (strom_last_error() has the text).
 * A handle is bound to one device and is not thread-safe.
 */
#ifndef STROM_B200_H
#define STROM_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct strom_handle strom_handle;

/* Mesh + discretisation.  Replaces the construction of `Geometry`
 * (strom/geometry.py:29-139) and the index maps of `AssemblyMaps`
 * (strom/meshing.py:166-220): the GPU derives every per-element table from
 * these arrays instead of storing O(ne*nq*nb) tabulations. */
typedef struct {
  int32_t num_elements;
  int32_t num_nodes;
  const int32_t* elem_nodes;  /* (ne, 3) counter-clockwise vertex ids            */
  const double* nodes;        /* (nv, 2) reference node coordinates X             */
  const int32_t* nbr_elem;    /* (ne, 3) neighbor element, -1 on the boundary     */
  const uint8_t* face_info;   /* (ne, 3) nbr_face | flip<<2 | bc_code<<3           */
} strom_mesh_desc;

/* Compiled conservation law (replaces the Python callables of
 * ConservationLawSpec, strom/conslaw.py:32-57). */
typedef struct {
  int32_t law_id;     /* 0 linear-advection, 1 burgers-spacetime, 2 burgers-strip, 3 euler, 4 euler + Roe flux,
                         5 euler on a mesh with slip walls, 6 linear advection with the manufactured solution
                         u = a0 + a1 exp(k1 x + k2 y) (position-dependent source and inflow ghosts) */
  int32_t n_comp;     /* m */
  int32_t n_mu;       /* parameters per mu vector */
  double params[8];   /* law constants (velocity, gamma, boundary states) */
} strom_law_desc;

/* Reference-element tables, host pointers (strom/basis.py, quadrature.py,
 * geometry.py:46-78).  Only straight (q = 1) geometry is supported. */
typedef struct {
  int32_t p, nb, nq, ns, nf;
  const double* phi;    /* (nq, nb)      */
  const double* dphi;   /* (nq, nb, 2)   */
  const double* wq;     /* (nq)          */
  const double* bary;   /* (nq, 3)       */
  const double* trace;  /* (3, ns, nf)   */
  const double* ws;     /* (ns)          */
  const double* s;      /* (ns) face points on [0,1] */
  const int32_t* fnodes;/* (3, nf)       */
} strom_quad_desc;

/* Distortion residual constants (strom/distortion.py:19-26). */
typedef struct { double kappa, eps; } strom_dist_desc;

enum {
  STROM_OBJECTIVE = 0,      /* out[P]: 0.5*sum rho(|R_e|^2+N_e^2)       reduced.py:172-184 */
  STROM_DERIVS = 1,         /* out[P][1+K+K*K]: J,S,T,H (H full, K = ku+kx) reduced.py:209-229 */
  STROM_CONTRIB = 2,        /* out[P][ne][K]: (S_e,T_e)                   reduced.py:244-246 */
  STROM_CONTRIB_SPLIT = 3,  /* out[P][ne][2K]: (Sv,Sf,Tv,Tf)              reduced.py:247-251 */
  STROM_RESIDUAL = 4,       /* out[P][N_u]: global residual vector        dg.py:238-240     */
  STROM_RESNORM2 = 5,       /* out[P]: sum_e |R_e|^2 over the element set (greedy indicator) */
  STROM_CONTRIB_LPROWS = 6, /* out[P][K+1][ne]: S_e,T_e and 0.5(|R_e|^2+N_e^2) as LP rows (config 4) */
  STROM_ELEMJAC = 7,        /* out[ne][24 + 24*24 + 24*72 + 24*6 + 7]: res, dR/dU_e, dR/dU_nbr (3 faces x 24),
                               dR/dx_e, N_e, dN_e/dx_e per element at U = U0, x = x_ref (P = 1;
                               4-component laws, p = 2): dg.py:197-225 and distortion.py:64-92, the
                               blocks assemble_global / assemble_distortion scatter */
  STROM_ELEMJAC_ENRICHED = 8 /* out[ne][NT (1 + 4 n_u + 6) + 7], NT = m n_test, n_u = m n_b: the same blocks with the
                               residual tested against the nodal space bound by strom_set_test_space:
                               res, dR/dU_e (NT x n_u), dR/dU_nbr (NT x 3 n_u), dR/dx_e (NT x 6), N_e, dN_e/dx_e.
                               With the degree p+1 space: what assemble_enriched scatters (dg.py:275-326); with the
                               trial space itself: the STROM_ELEMJAC blocks for every compiled law and degree
                               (scalar laws with sources included, dg.py:197-272).  P = 1. */
};

int strom_create(const strom_mesh_desc* mesh, const strom_law_desc* law, const strom_quad_desc* quad,
                 const strom_dist_desc* dist, int device, strom_handle** out);

/* Bind reduced bases (ReducedBases, strom/reduced.py:30-78).  phi: (N_u, ku)
 * row-major, psi: (N_x, kx) row-major, ref_coords: (N_x) = X of x = X+Psi tau,
 * state_offset: (N_u) or NULL (U = U0 + Phi w; NULL means U0 = 0, the
 * reference's `reconstruct`, reduced.py:81-85).  Pointers are borrowed. */
int strom_set_bases(strom_handle* h, const double* phi, int32_t ku, const double* psi, int32_t kx,
                    const double* ref_coords, const double* state_offset);

/* Per-parameter affine offsets (training snapshots, config 4): evaluation row
 * p uses U0 = state_offset + p*state_stride and X = ref_coords + p*coord_stride
 * (strides in doubles; 0 = shared).  Replaces the offsets of strom_set_bases.
 * There is no reference counterpart (the reference evaluates one snapshot per
 * call, eqp.py:104-106). */
int strom_set_offsets(strom_handle* h, const double* state_offset, int64_t state_stride,
                      const double* ref_coords, int64_t coord_stride);

/* Bind a residual test space (Geometry.test_space, strom/geometry.py:162-196; used by
 * assemble_enriched, dg.py:275-326).  HOST pointers: phi (nq, n_test) values and dphi
 * (nq, n_test, 2) reference gradients of the test basis at the volume points, trace
 * (3, ns, n_test) its values at the face points of each local face (zero off the face).
 * The library keeps its own device copy. */
int strom_set_test_space(strom_handle* h, int32_t n_test, const double* phi, const double* dphi,
                         const double* trace);

/* Size the workspace for up to max_P parameters and max_active elements. */
int strom_reserve(strom_handle* h, int32_t max_P, int32_t max_active);

/* One evaluation pass over P parameter points (batched ReducedOperator
 * call).  w: (P, ku), tau: (P, kx), mu: (P, n_mu); active: (A) ascending
 * element ids, rho: (A) weights — active == NULL means all elements with
 * unit weight (rho is None in the reference, reduced.py:134-141).
 * degen: (P) int32 counters of elements with g <= 0 (dg.py:109-110,134-135),
 * or NULL.  Returns 1 when any counter is non-zero (DegenerateMappingError).
 * `sync` != 0 makes the call blocking so the degenerate verdict is valid. */
int strom_eval(strom_handle* h, int32_t mode, const double* w, const double* tau, const double* mu,
               int32_t P, const int32_t* active, const double* rho, int32_t A, double* out,
               int32_t* degen, void* stream, int32_t sync);

/* The same evaluation through HOST buffers: w (P, ku), tau (P, kx), mu (P, n_mu) and out
 * (out_n doubles, the mode's size) are host pointers; active / rho stay device pointers.
 * Inputs go through a pinned staging buffer owned by the handle with one H2D copy, the
 * result and the per-row degenerate counters (degen_out, host, or NULL) come back with one
 * D2H copy and one stream synchronisation; returns 1 (ids available through
 * strom_degenerate_elements) when an element is degenerate.  This is the single-point
 * public API's path (ReducedOperator.objective / derivatives, reduced.py:172-229). */
int strom_eval_host(strom_handle* h, int32_t mode, const double* w, const double* tau, const double* mu,
                    int32_t P, const int32_t* active, const double* rho, int32_t A, double* out, int64_t out_n,
                    int32_t* degen_out, void* stream);

/* Element ids flagged degenerate by the last eval for parameter p (host
 * buffer `ids`, capacity cap); returns the count written, sorted ascending. */
int strom_degenerate_elements(strom_handle* h, int32_t p, int32_t* ids, int32_t cap);

/* Batched Levenberg-Marquardt over P parameters (lm_solve, strom/lm.py:164-271,
 * with the frozen-tau state init lm.py:129-161).  w, tau: (P, k) in/out,
 * device.  cfg: host pointer to 14 doubles in LmConfig order
 * (eps1, eps2, lambda0 (<0 = None), lambda_inc, lambda_dec, ratio_hi,
 * ratio_lo, max_iters, wolfe_c1, wolfe_c2, max_backtracks, lambda_cap,
 * w0_inner_tol, w0_inner_iters) plus w0_mode (0 keep, 1 lsq) as a 15th.
 * status: (P, 8) doubles out: converged, objective, |S|, |T|, n_iters,
 * reason (0 first-order, 1 max-iters, 2 line-search-failure, 3 degenerate), lambda,
 * evaluation requests.  Returns -3 if the round guard is exhausted.
 * history: (P, max_iters+1, 6) doubles out or NULL. */
int strom_lm_solve(strom_handle* h, double* w, double* tau, const double* mu, int32_t P,
                   const int32_t* active, const double* rho, int32_t A, const double* cfg,
                   double* status, double* history, void* stream);

/* Statistics of the last strom_lm_solve on this handle: out3 = (control rounds,
 * derivative passes, objective passes).  The rounds run device-resident as one
 * CUDA graph (a WHILE node over the control round with IF nodes for the two
 * batched passes), so these counts are read back once per solve batch. */
int strom_lm_stats(strom_handle* h, int32_t* out3);

/* Device-time breakdown of the last strom_lm_solve (ms, from %globaltimer stamps taken by
 * the control kernel): out4 = (control rounds, pass time after rounds that ran only the
 * derivatives pass, only the objective pass, both). */
int strom_lm_timing(strom_handle* h, double* out4);

/* Rows evaluated by the last strom_lm_solve: out2 = (parameter rows summed over the derivatives
 * passes, trial rows summed over the objective passes). */
int strom_lm_rows(strom_handle* h, double* out2);

/* Benchmark probe: while enabled, the dominant kernel of every strom_eval is
 * bracketed by CUDA events recorded on the call's stream (capacity 4096
 * launches).  strom_profile_ms synchronizes on the recorded events and
 * returns the summed kernel time in ms and the launch count. */
int strom_profile(strom_handle* h, int32_t enable);
double strom_profile_ms(strom_handle* h, int32_t* launches);

const char* strom_last_error(void);
void strom_destroy(strom_handle* h);

#ifdef __cplusplus
}
#endif
#endif /* STROM_B200_H */
