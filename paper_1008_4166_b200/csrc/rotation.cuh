// The 2x2 J-rotation of the inner level, shared by the pivot and Jacobi
// kernels: a branch-free restatement of the reference's _kernels.py:53-92.
#pragma once
#include "common.cuh"

namespace hjb {

// Rotation coefficients with the phase folded in: [x_r, x_s] <-
// [cp x_r + hs x_s, sp x_r + cs x_s], cp = cs*phase, sp = sn*phase,
// hs = hyp*sn -- algebraically _kernels.py:82-92.
template <typename T>
struct RotCoef {
  int code;  // 0 skip, 1 rotate, -1 indefinite pivot
  double cs, hs, num, den, eta, hyp;  // t = num / den (kept off the dependency chain)
  T cp, sp;
};

__device__ __forceinline__ double phase_mul(double a, double s) { return a * s; }
__device__ __forceinline__ cplx phase_mul(cplx a, double s) { return make_double2(a.x * s, a.y * s); }

// _kernels.py:53-81 restated for a short dependency chain.  With q = |a|^2,
// e = 2*eta (e^2 = 4q) and delta = d_s - d_r:
//   trig:       t = sgn(theta)|e| / (|delta| + sqrt(delta^2 + 4q))
//   hyperbolic: t = -e / (s + sqrt(s^2 - 4q)),  s = d_r + d_s
// and cs = den / sqrt(den^2 +- 4q), sn = num / sqrt(den^2 +- 4q).  The chain
// is q -> sqrt -> rsqrt (|a| and the phase come from an independent rsqrt);
// s^2 - 4q and den^2 - 4q are single-rounding FMAs.
template <typename T>
__device__ __forceinline__ RotCoef<T> rot_coef(T a, double dr, double ds, bool same, double otol2) {
  // branch-free: both rotation kinds share den = |x| + sqrt(x^2 +- 4q),
  // r = rsqrt(den^2 +- 4q) with x = d_s - d_r (trig, +) or d_r + d_s (hyp, -)
  RotCoef<T> p;
  const double q = abs2(a);
  const double dd = dr * ds;
  const double q4 = 4.0 * q;
  const double sa = re(a) >= 0.0 ? 1.0 : -1.0;
  // |a| and the phase a/eta: for real a the phase is exactly 1 (a / eta with
  // eta = a, _kernels.py:61-62), so no reciprocal square root is needed
  double ri = 0.0, aa;
  if constexpr (S<T>::cx) {
    ri = rsqrt(q);
    aa = q * ri;
  } else {
    aa = fabs(re(a));
  }
  const double x = same ? ds - dr : dr + ds;
  const double sq4 = same ? q4 : -q4;
  const double disc = fma(x, x, sq4);
  const double den = fabs(x) + sqrt(fmax(disc, 0.0));
  const double r = rsqrt(fma(den, den, sq4));
  const bool pos = x == 0.0 || ((x > 0.0) == (sa > 0.0));
  const double num = same ? (pos ? 2.0 * aa : -2.0 * aa) : -2.0 * sa * aa;
  const bool skip = q <= otol2 * dd;                     // _kernels.py:57
  const bool bad = q >= dd || (!same && disc <= 0.0);   // _kernels.py:59-60, 73-74
  p.code = skip ? 0 : (bad ? -1 : 1);
  p.hyp = same ? -1.0 : 1.0;
  const double cs = den * r, sn = num * r;
  p.cs = cs;
  p.hs = p.hyp * sn;
  if constexpr (S<T>::cx) {
    const T ph = phase_mul(a, sa * ri);
    p.cp = phase_mul(ph, cs);
    p.sp = phase_mul(ph, sn);
  } else {
    p.cp = cs;
    p.sp = sn;
  }
  p.num = num;
  p.den = den;
  p.eta = sa * aa;
  return p;
}

template <typename T>
__device__ __forceinline__ void rot_fold(T &xr, T &xs, const RotCoef<T> &p);
template <>
__device__ __forceinline__ void rot_fold<double>(double &xr, double &xs, const RotCoef<double> &p) {
  const double nr = fma(p.cp, xr, p.hs * xs);
  const double ns = fma(p.sp, xr, p.cs * xs);
  xr = nr;
  xs = ns;
}
template <>
__device__ __forceinline__ void rot_fold<cplx>(cplx &xr, cplx &xs, const RotCoef<cplx> &p) {
  cplx nr, ns;
  nr.x = fma(p.cp.x, xr.x, fma(-p.cp.y, xr.y, p.hs * xs.x));
  nr.y = fma(p.cp.x, xr.y, fma(p.cp.y, xr.x, p.hs * xs.y));
  ns.x = fma(p.sp.x, xr.x, fma(-p.sp.y, xr.y, p.cs * xs.x));
  ns.y = fma(p.sp.x, xr.y, fma(p.sp.y, xr.x, p.cs * xs.y));
  xr = nr;
  xs = ns;
}

}  // namespace hjb
