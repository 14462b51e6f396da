// Dependent-chain latency of the rotation-parameter computation (rot_coef)
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_1008_4166_b200/csrc/common.cuh"
using namespace hjb;
template <typename T> struct RotCoef { int code; double cs, hs, num, den, eta, hyp; T cp, sp; };
__device__ __forceinline__ double phase_mul(double a, double s) { return a * s; }
__device__ __forceinline__ cplx phase_mul(cplx a, double s) { return make_double2(a.x * s, a.y * s); }
template <typename T>
__device__ __forceinline__ RotCoef<T> rot_coef(T a, double dr, double ds, bool same, double otol2) {
  RotCoef<T> p;
  const double q = abs2(a);
  const double dd = dr * ds;
  const double q4 = 4.0 * q;
  const double ri = rsqrt(q);
  const double sa = re(a) >= 0.0 ? 1.0 : -1.0;
  const double aa = q * ri;
  const double x = same ? ds - dr : dr + ds;
  const double sq4 = same ? q4 : -q4;
  const double disc = fma(x, x, sq4);
  const double den = fabs(x) + sqrt(fmax(disc, 0.0));
  const double r = rsqrt(fma(den, den, sq4));
  const bool pos = x == 0.0 || ((x > 0.0) == (sa > 0.0));
  const double num = same ? (pos ? 2.0 * aa : -2.0 * aa) : -2.0 * sa * aa;
  const bool skip = q <= otol2 * dd;
  const bool bad = q >= dd || (!same && disc <= 0.0);
  p.code = skip ? 0 : (bad ? -1 : 1);
  p.hyp = same ? -1.0 : 1.0;
  const double cs = den * r, sn = num * r;
  const T ph = phase_mul(a, sa * ri);
  p.cs = cs; p.hs = p.hyp * sn; p.cp = phase_mul(ph, cs); p.sp = phase_mul(ph, sn);
  p.num = num; p.den = den; p.eta = sa * aa;
  return p;
}
__global__ void chain(double *out, int iters, int same) {
  double a = 0.3 + 1e-3 * threadIdx.x, dr = 2.0, ds = 1.0;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    RotCoef<double> p = rot_coef<double>(a, dr, ds, same, 1e-26);
    a = 0.3 + 1e-3 * p.cs;  // dependence on the output
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = double(t1 - t0) / iters;
  out[1 + threadIdx.x] = a;
}
__global__ void chainc(double *out, int iters, int same) {
  cplx a = make_double2(0.3, 0.1 + 1e-3 * threadIdx.x); double dr = 2.0, ds = 1.0;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    RotCoef<cplx> p = rot_coef<cplx>(a, dr, ds, same, 1e-26);
    a.x = 0.3 + 1e-3 * p.cp.x;
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = double(t1 - t0) / iters;
  out[1 + threadIdx.x] = a.x;
}
int main() {
  double *d; cudaMalloc(&d, 4096 * 8); double h;
  for (int same : {1, 0}) {
    chain<<<1, 32>>>(d, 1000, same); cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("rot_coef<double> %s chain: %.0f cycles\n", same ? "trig" : "hyp", h);
    chainc<<<1, 32>>>(d, 1000, same); cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("rot_coef<cplx>   %s chain: %.0f cycles\n", same ? "trig" : "hyp", h);
  }
  chain<<<1, 256>>>(d, 1000, 1); cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("rot_coef<double> trig, 8 warps: %.0f cycles per iteration\n", h);
  return 0;
}
