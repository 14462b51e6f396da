// Device helpers shared by the hjb200 kernels (sm_100a only).
#pragma once
#include <cuda_runtime.h>
#include <cstdint>

namespace hjb {

using cplx = double2;  // interleaved re/im, as numpy complex128

// ---- scalar traits: double (float64) and double2 (complex128) ----
template <typename T> struct S;
template <> struct S<double> {
  static constexpr bool cx = false;
  __host__ __device__ static inline double zero() { return 0.0; }
  __host__ __device__ static inline double one() { return 1.0; }
};
template <> struct S<cplx> {
  static constexpr bool cx = true;
  __host__ __device__ static inline cplx zero() { return make_double2(0.0, 0.0); }
  __host__ __device__ static inline cplx one() { return make_double2(1.0, 0.0); }
};

__device__ __forceinline__ double re(double a) { return a; }
__device__ __forceinline__ double re(cplx a) { return a.x; }
__device__ __forceinline__ double abs2(double a) { return a * a; }
__device__ __forceinline__ double abs2(cplx a) { return fma(a.x, a.x, a.y * a.y); }
__device__ __forceinline__ double conjv(double a) { return a; }
__device__ __forceinline__ cplx conjv(cplx a) { return make_double2(a.x, -a.y); }
__device__ __forceinline__ double add(double a, double b) { return a + b; }
__device__ __forceinline__ cplx add(cplx a, cplx b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double sub(double a, double b) { return a - b; }
__device__ __forceinline__ cplx sub(cplx a, cplx b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double scale(double a, double s) { return a * s; }
__device__ __forceinline__ cplx scale(cplx a, double s) { return make_double2(a.x * s, a.y * s); }
__device__ __forceinline__ double divr(double a, double s) { return a / s; }
__device__ __forceinline__ cplx divr(cplx a, double s) { return make_double2(a.x / s, a.y / s); }
__device__ __forceinline__ double mul(double a, double b) { return a * b; }
__device__ __forceinline__ cplx mul(cplx a, cplx b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
// acc + conj(a) * b
__device__ __forceinline__ double cfma(double a, double b, double acc) { return fma(a, b, acc); }
__device__ __forceinline__ cplx cfma(cplx a, cplx b, cplx acc) {
  acc.x = fma(a.x, b.x, acc.x);
  acc.x = fma(a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y);
  acc.y = fma(-a.y, b.x, acc.y);
  return acc;
}
// acc - conj(a) * b
__device__ __forceinline__ double cfms(double a, double b, double acc) { return fma(-a, b, acc); }
__device__ __forceinline__ cplx cfms(cplx a, cplx b, cplx acc) {
  acc.x = fma(-a.x, b.x, acc.x);
  acc.x = fma(-a.y, b.y, acc.x);
  acc.y = fma(-a.x, b.y, acc.y);
  acc.y = fma(a.y, b.x, acc.y);
  return acc;
}
__device__ __forceinline__ double shfl_xor(double v, int m) { return __shfl_xor_sync(0xffffffffu, v, m); }
__device__ __forceinline__ cplx shfl_xor(cplx v, int m) {
  return make_double2(__shfl_xor_sync(0xffffffffu, v.x, m), __shfl_xor_sync(0xffffffffu, v.y, m));
}
__device__ __forceinline__ double shfl_down(double v, int d) { return __shfl_down_sync(0xffffffffu, v, d); }
__device__ __forceinline__ cplx shfl_down(cplx v, int d) {
  return make_double2(__shfl_down_sync(0xffffffffu, v.x, d), __shfl_down_sync(0xffffffffu, v.y, d));
}
__device__ __forceinline__ double shfl_up(double v, int d) { return __shfl_up_sync(0xffffffffu, v, d); }
__device__ __forceinline__ cplx shfl_up(cplx v, int d) {
  return make_double2(__shfl_up_sync(0xffffffffu, v.x, d), __shfl_up_sync(0xffffffffu, v.y, d));
}
__device__ __forceinline__ double shfl_idx(double v, int l) { return __shfl_sync(0xffffffffu, v, l); }
__device__ __forceinline__ cplx shfl_idx(cplx v, int l) {
  return make_double2(__shfl_sync(0xffffffffu, v.x, l), __shfl_sync(0xffffffffu, v.y, l));
}
__device__ __forceinline__ bool finite_pos(double d) { return d > 0.0 && d <= 1.79769313486231570e308; }

// ---- FP64 tensor-core tile: D(8x8) += A(8x4, row) * B(4x8, col) ----
// Fragment ownership (PTX ISA, mma.m8n8k4 .f64): A[lane/4][lane%4],
// B[lane%4][lane/4], C/D[lane/4][2*(lane%4) + {0,1}].
__device__ __forceinline__ void dmma(double &d0, double &d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// ---- cp.async staging (LDGSTS) ----
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
// 16-byte copy; bytes < 16 zero-fills the tail (bytes == 0 -> zeros)
__device__ __forceinline__ void cp_async16(void *dst, const void *src, int bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(dst)), "l"(src),
               "r"(bytes));
}
__device__ __forceinline__ void cp_async8(void *dst, const void *src, int bytes) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(smem_u32(dst)), "l"(src),
               "r"(bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// Per-device "function attributes already set" flag: cudaFuncSetAttribute
// applies to the current device only, so a per-process flag would skip the
// attribute on the second device a process uses.
struct DeviceFlags {
  bool set[64] = {};
  bool *here() {
    int d = 0;
    if (cudaGetDevice(&d) != cudaSuccess || d < 0 || d >= 64) return nullptr;
    return &set[d];
  }
};

// one pair-step work item: block column offsets/widths (nj == 0: single block)
struct Item {
  int32_t oi, ni, oj, nj;
};

// per-item pivot statistics, int64 slots (include/hjb200.h hjb_pivot)
enum { ST_NROT = 0, ST_NBIG, ST_MAXT, ST_SWEEPS, ST_STATUS, ST_FR, ST_FS, ST_FALLBACK, ST_N };
enum { PV_OK = 0, PV_INDEFINITE = 1, PV_CHOL = 2 };
// pivot kernel modes: the whole inner level in one kernel (round-1 path), or
// its prologue (structured Cholesky -> R0) and epilogue (W = R0^-1 R_final)
// around the Jacobi kernel
enum { PV_FULL = 0, PV_PROLOGUE = 1, PV_EPILOGUE = 2 };
// factor.cu prologue input: the structured pair factor of the F variants
// (A_ij and the block norms, blocking.py:115-138) or the dense pair Gram of
// the B variants (three Gram items per pair: A_ii, A_jj, A_ij; parallel.py:199-200)
enum { FP_STRUCTURED = 0, FP_DENSE_PAIR = 1 };
// Jacobi kernel modes: sweeps until no rotation (jacobi_diagonalize), one
// cycle over all pairs, one cycle over the cross pairs of the two blocks
enum { JAC_CONVERGE = 0, JAC_ONE_CYCLE = 1, JAC_CROSS = 2 };

}  // namespace hjb
