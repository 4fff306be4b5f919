// Compiled conservation laws for the B200 element kernels.
//
// Each law is the device restatement of one reference plugin
// (ConservationLawSpec, strom/conslaw.py:32-57): pointwise flux f(u) (m x 2),
// source s(pos, u), LLF wavespeed ws(u, nhat) and the prescribed ghost states.
// Functions are templated on the scalar so the same code yields values
// (T = double) and exact pointwise Jacobians (T = Dn<N>, forward mode with N
// seeded directions) — the pointwise analogue of strom/dual.py, used only on
// per-point quantities; the per-tangent work in the kernels is explicit
// linear algebra on those Jacobians.
#pragma once
#include <cstdint>

namespace strom {

constexpr int BC_REFLECT = 31;  // face-info bc code of a slip wall (laws.py BC_REFLECT); ghosts are 2..30

template <int N>
struct Dn {
  double v;
  double d[N];
};

// ---- scalar helpers overloaded for double and Dn<N> -------------------------
__device__ __forceinline__ double val(double x) { return x; }
template <int N> __device__ __forceinline__ double val(const Dn<N>& x) { return x.v; }

template <int N> __device__ __forceinline__ Dn<N> cst(double c) {
  Dn<N> r; r.v = c;
#pragma unroll
  for (int i = 0; i < N; ++i) r.d[i] = 0.0;
  return r;
}
template <int N> __device__ __forceinline__ Dn<N> seed(double v, int k) {
  Dn<N> r = cst<N>(v); r.d[k] = 1.0; return r;
}
template <int N> __device__ __forceinline__ Dn<N> operator+(const Dn<N>& a, const Dn<N>& b) {
  Dn<N> r; r.v = a.v + b.v;
#pragma unroll
  for (int i = 0; i < N; ++i) r.d[i] = a.d[i] + b.d[i];
  return r;
}
template <int N> __device__ __forceinline__ Dn<N> operator-(const Dn<N>& a, const Dn<N>& b) {
  Dn<N> r; r.v = a.v - b.v;
#pragma unroll
  for (int i = 0; i < N; ++i) r.d[i] = a.d[i] - b.d[i];
  return r;
}
template <int N> __device__ __forceinline__ Dn<N> operator-(const Dn<N>& a) {
  Dn<N> r; r.v = -a.v;
#pragma unroll
  for (int i = 0; i < N; ++i) r.d[i] = -a.d[i];
  return r;
}
template <int N> __device__ __forceinline__ Dn<N> operator*(const Dn<N>& a, const Dn<N>& b) {
  Dn<N> r; r.v = a.v * b.v;
#pragma unroll
  for (int i = 0; i < N; ++i) r.d[i] = a.d[i] * b.v + a.v * b.d[i];
  return r;
}
template <int N> __device__ __forceinline__ Dn<N> operator/(const Dn<N>& a, const Dn<N>& b) {
  Dn<N> r; const double inv = 1.0 / b.v; r.v = a.v * inv;
#pragma unroll
  for (int i = 0; i < N; ++i) r.d[i] = (a.d[i] - r.v * b.d[i]) * inv;
  return r;
}
template <int N> __device__ __forceinline__ Dn<N> operator+(const Dn<N>& a, double c) { Dn<N> r = a; r.v += c; return r; }
template <int N> __device__ __forceinline__ Dn<N> operator+(double c, const Dn<N>& a) { return a + c; }
template <int N> __device__ __forceinline__ Dn<N> operator-(const Dn<N>& a, double c) { Dn<N> r = a; r.v -= c; return r; }
template <int N> __device__ __forceinline__ Dn<N> operator-(double c, const Dn<N>& a) { Dn<N> r = -a; r.v += c; return r; }
template <int N> __device__ __forceinline__ Dn<N> operator*(const Dn<N>& a, double c) {
  Dn<N> r; r.v = a.v * c;
#pragma unroll
  for (int i = 0; i < N; ++i) r.d[i] = a.d[i] * c;
  return r;
}
template <int N> __device__ __forceinline__ Dn<N> operator*(double c, const Dn<N>& a) { return a * c; }
template <int N> __device__ __forceinline__ Dn<N> operator/(const Dn<N>& a, double c) {
  Dn<N> r; r.v = a.v / c;
#pragma unroll
  for (int i = 0; i < N; ++i) r.d[i] = a.d[i] / c;
  return r;
}

__device__ __forceinline__ double dsqrt(double x) { return sqrt(x); }
template <int N> __device__ __forceinline__ Dn<N> dsqrt(const Dn<N>& a) {
  Dn<N> r; r.v = sqrt(a.v); const double h = 0.5 / r.v;
#pragma unroll
  for (int i = 0; i < N; ++i) r.d[i] = h * a.d[i];
  return r;
}
__device__ __forceinline__ double dexp(double x) { return exp(x); }
template <int N> __device__ __forceinline__ Dn<N> dexp(const Dn<N>& a) {
  Dn<N> r; r.v = exp(a.v);
#pragma unroll
  for (int i = 0; i < N; ++i) r.d[i] = r.v * a.d[i];
  return r;
}
// |x| with sign(0) = 0 for the tangent (strom/dual.py:161-163)
__device__ __forceinline__ double dabs(double x) { return fabs(x); }
template <int N> __device__ __forceinline__ Dn<N> dabs(const Dn<N>& a) {
  Dn<N> r; r.v = fabs(a.v); const double sg = a.v > 0.0 ? 1.0 : (a.v < 0.0 ? -1.0 : 0.0);
#pragma unroll
  for (int i = 0; i < N; ++i) r.d[i] = sg * a.d[i];
  return r;
}

enum SrcKind { SRC_NONE = 0, SRC_POS = 1, SRC_U = 2 };

struct LawArgs {
  double p[8];   // law constants
  double mu[4];  // parameter vector of the current unit
};

// ---------------------------------------------------------------------------
// linear advection, conslaw.py:174-253 (no manufactured solution)
struct LinAdv {
  static constexpr bool ANALYTIC = false;
  static constexpr bool ROE = false;
  static constexpr bool WALLS = false;
  static constexpr int M = 1;
  static constexpr int SRC = SRC_NONE;
  static constexpr bool GHOST_POS = false;  // prescribed ghosts depend on the face-point position
  template <class T> __device__ static void flux(const T* u, T (*f)[2], const LawArgs& a) {
    f[0][0] = a.p[0] * u[0];
    f[0][1] = a.p[1] * u[0];
  }
  template <class T> __device__ static void source(const T* pos, const T* u, T* s, const LawArgs& a) {
    s[0] = 0.0 * u[0];
  }
  template <class T> __device__ static T wavespeed(const T* u, const T* n, const LawArgs& a) {
    return dabs(a.p[0] * n[0] + a.p[1] * n[1]) + 0.0 * u[0];
  }
  __device__ static void ghost(int id, const LawArgs& a, const double* pos, double* out) { out[0] = 1.0; }
};

// linear advection with the manufactured solution u(x, y) = a0 + a1 exp(k1 x + k2 y)
// (conslaw.py:174-253 with manufactured = (u_exact, grad_exact)): source c . grad u_exact at the
// deformed position (it enters the x-Jacobian, dg.py:113,121), inflow ghosts u_exact at the
// deformed face points (value only, no x-derivative, dg.py:151-161).
// params: c0, c1, a0, a1, k1, k2
struct LinAdvMS {
  static constexpr bool ANALYTIC = false;
  static constexpr bool ROE = false;
  static constexpr bool WALLS = false;
  static constexpr int M = 1;
  static constexpr int SRC = SRC_POS;
  static constexpr bool GHOST_POS = true;
  template <class T> __device__ static void flux(const T* u, T (*f)[2], const LawArgs& a) {
    f[0][0] = a.p[0] * u[0];
    f[0][1] = a.p[1] * u[0];
  }
  template <class T> __device__ static void source(const T* pos, const T* u, T* s, const LawArgs& a) {
    const T e = a.p[3] * dexp(a.p[4] * pos[0] + a.p[5] * pos[1]);
    s[0] = a.p[0] * (a.p[4] * e) + a.p[1] * (a.p[5] * e) + 0.0 * u[0];
  }
  template <class T> __device__ static T wavespeed(const T* u, const T* n, const LawArgs& a) {
    return dabs(a.p[0] * n[0] + a.p[1] * n[1]) + 0.0 * u[0];
  }
  __device__ static void ghost(int id, const LawArgs& a, const double* pos, double* out) {
    out[0] = a.p[2] + a.p[3] * exp(a.p[4] * pos[0] + a.p[5] * pos[1]);
  }
};

// space-time Burgers, conslaw.py:94-163
struct BurgersST {
  static constexpr bool ANALYTIC = false;
  static constexpr bool ROE = false;
  static constexpr bool WALLS = false;
  static constexpr int M = 1;
  static constexpr int SRC = SRC_POS;
  static constexpr bool GHOST_POS = false;
  template <class T> __device__ static void flux(const T* u, T (*f)[2], const LawArgs& a) {
    f[0][0] = 0.5 * u[0] * u[0];
    f[0][1] = u[0];
  }
  template <class T> __device__ static void source(const T* pos, const T* u, T* s, const LawArgs& a) {
    s[0] = 0.02 * dexp(a.mu[1] * pos[0]);
  }
  template <class T> __device__ static T wavespeed(const T* u, const T* n, const LawArgs& a) {
    T v = u[0] * n[0] + n[1];
    return dsqrt(v * v + 1e-6);
  }
  __device__ static void ghost(int id, const LawArgs& a, const double* pos, double* out) { out[0] = id == 0 ? a.mu[0] : 1.0; }
};

// steady Burgers strip (config 1): (u^2/2)_x = mu u
struct BurgersStrip {
  static constexpr bool ANALYTIC = false;
  static constexpr bool ROE = false;
  static constexpr bool WALLS = false;
  static constexpr int M = 1;
  static constexpr int SRC = SRC_U;
  static constexpr bool GHOST_POS = false;
  template <class T> __device__ static void flux(const T* u, T (*f)[2], const LawArgs& a) {
    f[0][0] = 0.5 * u[0] * u[0];
    f[0][1] = 0.0 * u[0];
  }
  template <class T> __device__ static void source(const T* pos, const T* u, T* s, const LawArgs& a) {
    s[0] = a.mu[0] * u[0];
  }
  template <class T> __device__ static T wavespeed(const T* u, const T* n, const LawArgs& a) {
    T v = u[0] * n[0];
    return dsqrt(v * v + 1e-6);
  }
  __device__ static void ghost(int id, const LawArgs& a, const double* pos, double* out) { out[0] = id == 0 ? a.p[0] : a.p[1]; }
};

// compressible Euler, conservative (rho, rho u, rho v, E); LLF speed |v.n| + c
struct Euler {
  static constexpr bool ANALYTIC = true;
  static constexpr bool ROE = false;    // numerical flux: LLF (the reference's)
  static constexpr bool WALLS = false;  // slip-wall faces compiled in (EulerWall / EulerRoe)
  static constexpr int M = 4;
  static constexpr int SRC = SRC_NONE;
  static constexpr bool GHOST_POS = false;
  // fn = f(u).n and A = d(f.n)/du for a (not necessarily unit) direction n
  __device__ static void flux_dir(const double* u, const double* n, double* fn, double (*A)[4], const LawArgs& a) {
    const double g = a.p[0], gm = g - 1.0;
    const double r = u[0], ir = 1.0 / r, vx = u[1] * ir, vy = u[2] * ir;
    const double p = gm * (u[3] - 0.5 * (u[1] * vx + u[2] * vy));
    const double ke = 0.5 * (vx * vx + vy * vy);
    const double qn = vx * n[0] + vy * n[1];
    const double H = (u[3] + p) * ir;
    fn[0] = r * qn;
    fn[1] = u[1] * qn + p * n[0];
    fn[2] = u[2] * qn + p * n[1];
    fn[3] = (u[3] + p) * qn;
    const double gk = gm * ke;
    A[0][0] = 0.0;                     A[0][1] = n[0];                             A[0][2] = n[1];                             A[0][3] = 0.0;
    A[1][0] = gk * n[0] - vx * qn;     A[1][1] = qn + vx * n[0] - gm * vx * n[0];  A[1][2] = vx * n[1] - gm * vy * n[0];       A[1][3] = gm * n[0];
    A[2][0] = gk * n[1] - vy * qn;     A[2][1] = vy * n[0] - gm * vx * n[1];       A[2][2] = qn + vy * n[1] - gm * vy * n[1];  A[2][3] = gm * n[1];
    A[3][0] = qn * (gk - H);           A[3][1] = H * n[0] - gm * vx * qn;          A[3][2] = H * n[1] - gm * vy * qn;          A[3][3] = g * qn;
  }
  // fused face side: flux components f, A(nu) = d(f.nu)/du, ws(u, nh) and its gradients
  __device__ static double face_side(const double* u, const double* nu, const double* nh, double (*f)[2],
                                     double (*A)[4], double* dwdu, double* dwdn, const LawArgs& a) {
    const double g = a.p[0], gm = g - 1.0;
    const double r = u[0], ir = 1.0 / r, vx = u[1] * ir, vy = u[2] * ir;
    const double p = gm * (u[3] - 0.5 * (u[1] * vx + u[2] * vy));
    const double ke = 0.5 * (vx * vx + vy * vy);
    const double Ep = u[3] + p, H = Ep * ir, gk = gm * ke;
    f[0][0] = u[1];          f[0][1] = u[2];
    f[1][0] = u[1] * vx + p; f[1][1] = u[1] * vy;
    f[2][0] = u[2] * vx;     f[2][1] = u[2] * vy + p;
    f[3][0] = Ep * vx;       f[3][1] = Ep * vy;
    const double qn = vx * nu[0] + vy * nu[1];
    A[0][0] = 0.0;                 A[0][1] = nu[0];                              A[0][2] = nu[1];                              A[0][3] = 0.0;
    A[1][0] = gk * nu[0] - vx * qn; A[1][1] = qn + vx * nu[0] - gm * vx * nu[0]; A[1][2] = vx * nu[1] - gm * vy * nu[0];       A[1][3] = gm * nu[0];
    A[2][0] = gk * nu[1] - vy * qn; A[2][1] = vy * nu[0] - gm * vx * nu[1];       A[2][2] = qn + vy * nu[1] - gm * vy * nu[1]; A[2][3] = gm * nu[1];
    A[3][0] = qn * (gk - H);        A[3][1] = H * nu[0] - gm * vx * qn;           A[3][2] = H * nu[1] - gm * vy * qn;           A[3][3] = g * qn;
    const double qh = vx * nh[0] + vy * nh[1];
    const double c2 = g * p * ir, rc = rsqrt(c2), c = c2 * rc;  // c = sqrt(g p / r), 1/c from one rsqrt
    const double sg = qh > 0.0 ? 1.0 : (qh < 0.0 ? -1.0 : 0.0);
    const double cf = 0.5 * g * ir * rc;  // g / (2 c r)
    dwdu[0] = sg * (-qh * ir) + cf * (gm * ke - p * ir);
    dwdu[1] = sg * nh[0] * ir - cf * gm * vx;
    dwdu[2] = sg * nh[1] * ir - cf * gm * vy;
    dwdu[3] = cf * gm;
    dwdn[0] = sg * vx;
    dwdn[1] = sg * vy;
    return fabs(qh) + c;
  }
  // fused volume point: flux components f and the two directional Jacobians A(d0), A(d1)
  __device__ static void vol_point(const double* u, const double* d0, const double* d1, double (*f)[2],
                                   double (*A0)[4], double (*A1)[4], const LawArgs& a) {
    const double g = a.p[0], gm = g - 1.0;
    const double r = u[0], ir = 1.0 / r, vx = u[1] * ir, vy = u[2] * ir;
    const double p = gm * (u[3] - 0.5 * (u[1] * vx + u[2] * vy));
    const double ke = 0.5 * (vx * vx + vy * vy);
    const double Ep = u[3] + p, H = Ep * ir, gk = gm * ke;
    f[0][0] = u[1];          f[0][1] = u[2];
    f[1][0] = u[1] * vx + p; f[1][1] = u[1] * vy;
    f[2][0] = u[2] * vx;     f[2][1] = u[2] * vy + p;
    f[3][0] = Ep * vx;       f[3][1] = Ep * vy;
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      const double* n = t == 0 ? d0 : d1;
      double (*A)[4] = t == 0 ? A0 : A1;
      const double qn = vx * n[0] + vy * n[1];
      A[0][0] = 0.0;                A[0][1] = n[0];                            A[0][2] = n[1];                            A[0][3] = 0.0;
      A[1][0] = gk * n[0] - vx * qn; A[1][1] = qn + vx * n[0] - gm * vx * n[0]; A[1][2] = vx * n[1] - gm * vy * n[0];     A[1][3] = gm * n[0];
      A[2][0] = gk * n[1] - vy * qn; A[2][1] = vy * n[0] - gm * vx * n[1];      A[2][2] = qn + vy * n[1] - gm * vy * n[1]; A[2][3] = gm * n[1];
      A[3][0] = qn * (gk - H);       A[3][1] = H * n[0] - gm * vx * qn;         A[3][2] = H * n[1] - gm * vy * qn;         A[3][3] = g * qn;
    }
  }
  // volume point along one direction: flux components f and A(n) = d(f.n)/du
  __device__ static void vol_dir(const double* u, const double* n, double (*f)[2], double (*A)[4], const LawArgs& a) {
    const double g = a.p[0], gm = g - 1.0;
    const double r = u[0], ir = 1.0 / r, vx = u[1] * ir, vy = u[2] * ir;
    const double p = gm * (u[3] - 0.5 * (u[1] * vx + u[2] * vy));
    const double ke = 0.5 * (vx * vx + vy * vy);
    const double Ep = u[3] + p, H = Ep * ir, gk = gm * ke;
    f[0][0] = u[1];          f[0][1] = u[2];
    f[1][0] = u[1] * vx + p; f[1][1] = u[1] * vy;
    f[2][0] = u[2] * vx;     f[2][1] = u[2] * vy + p;
    f[3][0] = Ep * vx;       f[3][1] = Ep * vy;
    const double qn = vx * n[0] + vy * n[1];
    A[0][0] = 0.0;                A[0][1] = n[0];                            A[0][2] = n[1];                            A[0][3] = 0.0;
    A[1][0] = gk * n[0] - vx * qn; A[1][1] = qn + vx * n[0] - gm * vx * n[0]; A[1][2] = vx * n[1] - gm * vy * n[0];     A[1][3] = gm * n[0];
    A[2][0] = gk * n[1] - vy * qn; A[2][1] = vy * n[0] - gm * vx * n[1];      A[2][2] = qn + vy * n[1] - gm * vy * n[1]; A[2][3] = gm * n[1];
    A[3][0] = qn * (gk - H);       A[3][1] = H * n[0] - gm * vx * qn;         A[3][2] = H * n[1] - gm * vy * qn;         A[3][3] = g * qn;
  }
  // everything a quadrature point needs, one code path for volume and face points:
  // flux components, A(d0), A(d1), ws(u, nh) with its gradients
  __device__ static double point_full(const double* u, const double* d0, const double* d1, const double* nh,
                                      double (*f)[2], double (*A0)[4], double (*A1)[4], double* dwdu, double* dwdn,
                                      const LawArgs& a) {
    const double g = a.p[0], gm = g - 1.0;
    const double r = u[0], ir = 1.0 / r, vx = u[1] * ir, vy = u[2] * ir;
    const double p = gm * (u[3] - 0.5 * (u[1] * vx + u[2] * vy));
    const double ke = 0.5 * (vx * vx + vy * vy);
    const double Ep = u[3] + p, H = Ep * ir, gk = gm * ke;
    f[0][0] = u[1];          f[0][1] = u[2];
    f[1][0] = u[1] * vx + p; f[1][1] = u[1] * vy;
    f[2][0] = u[2] * vx;     f[2][1] = u[2] * vy + p;
    f[3][0] = Ep * vx;       f[3][1] = Ep * vy;
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      const double* n = t == 0 ? d0 : d1;
      double (*A)[4] = t == 0 ? A0 : A1;
      const double qn = vx * n[0] + vy * n[1];
      A[0][0] = 0.0;                A[0][1] = n[0];                            A[0][2] = n[1];                            A[0][3] = 0.0;
      A[1][0] = gk * n[0] - vx * qn; A[1][1] = qn + vx * n[0] - gm * vx * n[0]; A[1][2] = vx * n[1] - gm * vy * n[0];     A[1][3] = gm * n[0];
      A[2][0] = gk * n[1] - vy * qn; A[2][1] = vy * n[0] - gm * vx * n[1];      A[2][2] = qn + vy * n[1] - gm * vy * n[1]; A[2][3] = gm * n[1];
      A[3][0] = qn * (gk - H);       A[3][1] = H * n[0] - gm * vx * qn;         A[3][2] = H * n[1] - gm * vy * qn;         A[3][3] = g * qn;
    }
    const double qh = vx * nh[0] + vy * nh[1];
    const double c = sqrt(g * p / r);
    const double sg = qh > 0.0 ? 1.0 : (qh < 0.0 ? -1.0 : 0.0);
    const double cf = g / (2.0 * c * r);
    dwdu[0] = sg * (-qh * ir) + cf * (gm * ke - p * ir);
    dwdu[1] = sg * nh[0] * ir - cf * gm * vx;
    dwdu[2] = sg * nh[1] * ir - cf * gm * vy;
    dwdu[3] = cf * gm;
    dwdn[0] = sg * vx;
    dwdn[1] = sg * vy;
    return fabs(qh) + c;
  }
  // ws = |v.nh| + c and its gradients wrt u and nh (sign(0) = 0)
  __device__ static double wavespeed_grad(const double* u, const double* nh, double* dwdu, double* dwdn, const LawArgs& a) {
    const double g = a.p[0], gm = g - 1.0;
    const double r = u[0], ir = 1.0 / r, vx = u[1] * ir, vy = u[2] * ir;
    const double p = gm * (u[3] - 0.5 * (u[1] * vx + u[2] * vy));
    const double ke = 0.5 * (vx * vx + vy * vy);
    const double qn = vx * nh[0] + vy * nh[1];
    const double c = sqrt(g * p / r);
    const double sg = qn > 0.0 ? 1.0 : (qn < 0.0 ? -1.0 : 0.0);
    const double cf = g / (2.0 * c * r);
    dwdu[0] = sg * (-qn * ir) + cf * (gm * ke - p * ir);
    dwdu[1] = sg * nh[0] * ir - cf * gm * vx;
    dwdu[2] = sg * nh[1] * ir - cf * gm * vy;
    dwdu[3] = cf * gm;
    dwdn[0] = sg * vx;
    dwdn[1] = sg * vy;
    return fabs(qn) + c;
  }
  template <class T> __device__ static void flux(const T* u, T (*f)[2], const LawArgs& a) {
    const double g = a.p[0];
    T vx = u[1] / u[0], vy = u[2] / u[0];
    T p = (g - 1.0) * (u[3] - 0.5 * (u[1] * vx + u[2] * vy));
    f[0][0] = u[1];              f[0][1] = u[2];
    f[1][0] = u[1] * vx + p;     f[1][1] = u[1] * vy;
    f[2][0] = u[2] * vx;         f[2][1] = u[2] * vy + p;
    T Ep = u[3] + p;
    f[3][0] = Ep * vx;           f[3][1] = Ep * vy;
  }
  template <class T> __device__ static void source(const T* pos, const T* u, T* s, const LawArgs& a) {
#pragma unroll
    for (int c = 0; c < 4; ++c) s[c] = 0.0 * u[c];
  }
  template <class T> __device__ static T wavespeed(const T* u, const T* n, const LawArgs& a) {
    const double g = a.p[0];
    T vx = u[1] / u[0], vy = u[2] / u[0];
    T p = (g - 1.0) * (u[3] - 0.5 * (u[1] * vx + u[2] * vy));
    T vn = vx * n[0] + vy * n[1];
    return dabs(vn) + dsqrt(g * p / u[0]);
  }
  __device__ static void ghost(int id, const LawArgs& a, const double* pos, double* out) {
    const double g = a.p[0], mach = a.mu[0], p = 1.0 / g;
    out[0] = 1.0; out[1] = mach; out[2] = 0.0; out[3] = p / (g - 1.0) + 0.5 * mach * mach;
  }
};

// Euler with the Roe numerical flux (GPU-only extension; laws.py roe_dissipation):
// H = (f_in + f_out).nu / 2 - |nu| D / 2, D = |A_roe(nh)| (u_out - u_in); p[1] = entropy delta
struct EulerRoe : Euler {
  static constexpr bool ROE = true;
  static constexpr bool WALLS = true;
};

// Euler (LLF) on meshes with slip walls (GPU-only extension): a separate instantiation so the
// wall-free kernels carry none of the wall code
struct EulerWall : Euler {
  static constexpr bool WALLS = true;
};

// slip-wall ghost (bc code BC_REFLECT): momentum mirrored in the face, m - 2 (m . nh) nh
template <class T>
__device__ __forceinline__ void reflect_state(const T* u, const T* nh, T* out) {
  const T mn = u[1] * nh[0] + u[2] * nh[1];
  out[0] = u[0];
  out[1] = u[1] - 2.0 * mn * nh[0];
  out[2] = u[2] - 2.0 * mn * nh[1];
  out[3] = u[3];
}

// Roe matrix dissipation D = |A_roe(nh)| (uR - uL) for 2-D Euler: Roe-averaged state, the three
// wave families, smooth entropy correction |l| -> sqrt(l^2 + (delta c)^2).  Templated on the
// scalar: T = Dn<N> gives its exact Jacobians (K1), T = double its value (K2).  Restates the
// host spec laws.py roe_dissipation, against which the oracle checks it.
template <class T>
__device__ __forceinline__ void roe_diss(const T* uL, const T* uR, const T* nh, double g, double delta, T* D) {
  const double gm = g - 1.0;
  const T sl = dsqrt(uL[0]), sr = dsqrt(uR[0]);
  const T vxl = uL[1] / uL[0], vyl = uL[2] / uL[0], vxr = uR[1] / uR[0], vyr = uR[2] / uR[0];
  const T pl = gm * (uL[3] - 0.5 * (uL[1] * vxl + uL[2] * vyl));
  const T pr = gm * (uR[3] - 0.5 * (uR[1] * vxr + uR[2] * vyr));
  const T hl = (uL[3] + pl) / uL[0], hr = (uR[3] + pr) / uR[0];
  const T den = sl + sr;
  const T ux = (sl * vxl + sr * vxr) / den, uy = (sl * vyl + sr * vyr) / den, ht = (sl * hl + sr * hr) / den;
  const T q2 = ux * ux + uy * uy;
  const T c2 = gm * (ht - 0.5 * q2);
  const T c = dsqrt(c2);
  const T rt = sl * sr;
  const T un = ux * nh[0] + uy * nh[1];
  const T dr = uR[0] - uL[0], dp = pr - pl, dvx = vxr - vxl, dvy = vyr - vyl;
  const T dun = dvx * nh[0] + dvy * nh[1];
  const T a1 = (dp - rt * c * dun) / (2.0 * c2);
  const T a3 = (dp + rt * c * dun) / (2.0 * c2);
  const T a2 = dr - dp / c2;
  const T d2 = (delta * delta) * c2;
  const T l1 = dsqrt((un - c) * (un - c) + d2), l2 = dsqrt(un * un + d2), l3 = dsqrt((un + c) * (un + c) + d2);
  const T w1 = l1 * a1, w3 = l3 * a3;
  D[0] = w1 + l2 * a2 + w3;
  D[1] = w1 * (ux - c * nh[0]) + l2 * (a2 * ux + rt * (dvx - dun * nh[0])) + w3 * (ux + c * nh[0]);
  D[2] = w1 * (uy - c * nh[1]) + l2 * (a2 * uy + rt * (dvy - dun * nh[1])) + w3 * (uy + c * nh[1]);
  D[3] = w1 * (ht - un * c) + l2 * (0.5 * a2 * q2 + rt * (ux * dvx + uy * dvy - un * dun)) + w3 * (ht + un * c);
}

// value-path numerical flux of one face point (K2 / value kernels): uo is the exterior state
// (neighbor trace, extrapolated copy or prescribed ghost; overwritten for a slip wall);
// H[c] = (f_in + f_out).nu / 2 - |nu| (lam (uo - ui) or D) / 2, not yet times the face weight
template <class LAW>
__device__ __forceinline__ void face_flux_val(const double* ui, double* uo, int bc, const double* nu, double len,
                                              const double* nh, const LawArgs& la, double* H);

// ---- value path: flux and LLF wavespeed of one state (K2) --------------------------
// Generic: the law's templated flux / wavespeed.  Euler: one reciprocal of the density
// and one rsqrt for the sound speed instead of five divisions and a sqrt.
template <class LAW>
struct PointVal {
  __device__ static void flux(const double* u, double (*f)[2], const LawArgs& a) { LAW::flux(u, f, a); }
  __device__ static double flux_ws(const double* u, const double* nh, double (*f)[2], const LawArgs& a) {
    LAW::flux(u, f, a);
    return LAW::wavespeed(u, nh, a);
  }
};
template <>
struct PointVal<Euler> {
  __device__ static void flux(const double* u, double (*f)[2], const LawArgs& a) {
    const double g = a.p[0];
    const double ir = 1.0 / u[0], vx = u[1] * ir, vy = u[2] * ir;
    const double p = (g - 1.0) * (u[3] - 0.5 * (u[1] * vx + u[2] * vy)), Ep = u[3] + p;
    f[0][0] = u[1];          f[0][1] = u[2];
    f[1][0] = u[1] * vx + p; f[1][1] = u[1] * vy;
    f[2][0] = u[2] * vx;     f[2][1] = u[2] * vy + p;
    f[3][0] = Ep * vx;       f[3][1] = Ep * vy;
  }
  __device__ static double flux_ws(const double* u, const double* nh, double (*f)[2], const LawArgs& a) {
    const double g = a.p[0];
    const double ir = 1.0 / u[0], vx = u[1] * ir, vy = u[2] * ir;
    const double p = (g - 1.0) * (u[3] - 0.5 * (u[1] * vx + u[2] * vy)), Ep = u[3] + p;
    f[0][0] = u[1];          f[0][1] = u[2];
    f[1][0] = u[1] * vx + p; f[1][1] = u[1] * vy;
    f[2][0] = u[2] * vx;     f[2][1] = u[2] * vy + p;
    f[3][0] = Ep * vx;       f[3][1] = Ep * vy;
    const double c2 = g * p * ir;
    return fabs(vx * nh[0] + vy * nh[1]) + c2 * rsqrt(c2);  // |v.n| + sqrt(g p / rho)
  }
};

template <>
struct PointVal<EulerRoe> : PointVal<Euler> {};
template <>
struct PointVal<EulerWall> : PointVal<Euler> {};

template <class LAW>
__device__ __forceinline__ void face_flux_val(const double* ui, double* uo, int bc, const double* nu, double len,
                                              const double* nh, const LawArgs& la, double* H) {
  constexpr int M = LAW::M;
  if constexpr (M == 4) {
    if (bc == BC_REFLECT) reflect_state(ui, nh, uo);
  }
  double fi_[M][2], fo[M][2];
  const double wi = PointVal<LAW>::flux_ws(ui, nh, fi_, la), wo = PointVal<LAW>::flux_ws(uo, nh, fo, la);
  if constexpr (LAW::ROE) {
    double D[4];
    roe_diss<double>(ui, uo, nh, la.p[0], la.p[1], D);
#pragma unroll
    for (int c = 0; c < M; ++c) {
      const double fn = (fi_[c][0] * nu[0] + fi_[c][1] * nu[1]) + (fo[c][0] * nu[0] + fo[c][1] * nu[1]);
      H[c] = 0.5 * fn - 0.5 * len * D[c];
    }
  } else {
    // dual.maximum tie -> first argument; a slip wall's ws(R u) equals ws(u): the interior one
    const double lam = (bc == BC_REFLECT || wi >= wo) ? wi : wo;
#pragma unroll
    for (int c = 0; c < M; ++c) {
      const double fn = (fi_[c][0] * nu[0] + fi_[c][1] * nu[1]) + (fo[c][0] * nu[0] + fo[c][1] * nu[1]);
      H[c] = 0.5 * fn - 0.5 * (lam * len) * (uo[c] - ui[c]);
    }
  }
}

// ---- point Jacobians: analytic when the law provides them, else forward mode ----
template <class LAW, bool A = LAW::ANALYTIC>
struct PointOps;

template <class LAW>
struct PointOps<LAW, true> {
  __device__ static double face_side(const double* u, const double* nu, const double* nh, double (*f)[2],
                                     double (*Am)[LAW::M], double* dwdu, double* dwdn, const LawArgs& a) {
    return LAW::face_side(u, nu, nh, f, Am, dwdu, dwdn, a);
  }
  __device__ static void vol_point(const double* u, const double* d0, const double* d1, double (*f)[2],
                                   double (*A0)[LAW::M], double (*A1)[LAW::M], const LawArgs& a) {
    LAW::vol_point(u, d0, d1, f, A0, A1, a);
  }
  __device__ static void flux_dir(const double* u, const double* n, double* fn, double (*Am)[LAW::M], const LawArgs& a) {
    LAW::flux_dir(u, n, fn, Am, a);
  }
  __device__ static void vol_dir(const double* u, const double* n, double (*f)[2], double (*Am)[LAW::M], const LawArgs& a) {
    LAW::vol_dir(u, n, f, Am, a);
  }
  __device__ static double wavespeed_grad(const double* u, const double* nh, double* dwdu, double* dwdn, const LawArgs& a) {
    return LAW::wavespeed_grad(u, nh, dwdu, dwdn, a);
  }
};

template <class LAW>
struct PointOps<LAW, false> {
  static constexpr int M = LAW::M;
  __device__ static double face_side(const double* u, const double* nu, const double* nh, double (*f)[2],
                                     double (*Am)[M], double* dwdu, double* dwdn, const LawArgs& a);
  __device__ static void vol_point(const double* u, const double* d0, const double* d1, double (*f)[2],
                                   double (*A0)[M], double (*A1)[M], const LawArgs& a);
  __device__ static void vol_dir(const double* u, const double* n, double (*f)[2], double (*Am)[M], const LawArgs& a) {
    double fn[M];
    LAW::flux(u, f, a);
    flux_dir(u, n, fn, Am, a);
  }
  __device__ static void flux_dir(const double* u, const double* n, double* fn, double (*Am)[M], const LawArgs& a) {
    Dn<M> ud[M];
#pragma unroll
    for (int c = 0; c < M; ++c) ud[c] = seed<M>(u[c], c);
    Dn<M> f[M][2];
    LAW::flux(ud, f, a);
#pragma unroll
    for (int c = 0; c < M; ++c) {
      fn[c] = f[c][0].v * n[0] + f[c][1].v * n[1];
#pragma unroll
      for (int cp = 0; cp < M; ++cp) Am[c][cp] = f[c][0].d[cp] * n[0] + f[c][1].d[cp] * n[1];
    }
  }
  __device__ static double wavespeed_grad(const double* u, const double* nh, double* dwdu, double* dwdn, const LawArgs& a) {
    Dn<M + 2> ud[M], nd[2];
#pragma unroll
    for (int c = 0; c < M; ++c) ud[c] = seed<M + 2>(u[c], c);
    nd[0] = seed<M + 2>(nh[0], M);
    nd[1] = seed<M + 2>(nh[1], M + 1);
    Dn<M + 2> w = LAW::wavespeed(ud, nd, a);
#pragma unroll
    for (int c = 0; c < M; ++c) dwdu[c] = w.d[c];
    dwdn[0] = w.d[M];
    dwdn[1] = w.d[M + 1];
    return w.v;
  }
};

template <class LAW>
__device__ double PointOps<LAW, false>::face_side(const double* u, const double* nu, const double* nh, double (*f)[2],
                                                  double (*Am)[M], double* dwdu, double* dwdn, const LawArgs& a) {
  double fn[M];
  flux_dir(u, nu, fn, Am, a);
  LAW::flux(u, f, a);
  return wavespeed_grad(u, nh, dwdu, dwdn, a);
}

template <class LAW>
__device__ void PointOps<LAW, false>::vol_point(const double* u, const double* d0, const double* d1, double (*f)[2],
                                                double (*A0)[M], double (*A1)[M], const LawArgs& a) {
  double fn[M];
  LAW::flux(u, f, a);
  flux_dir(u, d0, fn, A0, a);
  flux_dir(u, d1, fn, A1, a);
}

}  // namespace strom
