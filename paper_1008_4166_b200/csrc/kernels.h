// Launch interfaces of the hjb200 kernels (host side).
#pragma once
#include <cuda_runtime.h>
#include <cstdint>

#include "common.cuh"

namespace hjb {

struct GramArgs {
  const void *G;
  int64_t ldg, m;
  const Item *items;
  int count;
  int bmax;
  void *A;          // [count][bmax*bmax] final Gram, column-major ld bmax
  double *D;        // [count][2*bmax] final column norms^2
  void *Apart;      // split-K partial scratch (gram_scratch_bytes), may be null: one split
  size_t part_bytes;
  // set by launch_gram
  int tiles_m, tiles_n;  // tiles per dimension
  int splits;            // K splits (whole K chunks, sizes differ by at most one chunk)
  double *Dpart;
};
// splits_used (optional): the K split count the launch chose
cudaError_t launch_gram(bool cx, GramArgs a, cudaStream_t st, int *splits_used = nullptr);
size_t gram_scratch_bytes(bool cx, int count, int bmax);

struct PivotArgs {
  const void *G;
  int64_t ldg, m;
  const Item *items;
  int count;
  int bmax;
  void *A;            // [count][bmax*bmax] Gram (overwritten with R_ij)
  const double *D;    // [count][2*bmax]
  const int8_t *signs;
  double orth_tol, quad_tol;  // <= 0: defaults of rotations.py:76-80
  int max_sweeps;
  void *W;            // [count][nmax*nmax] accumulated transformation
  int64_t *stats;     // [count][ST_N]
  void *Rout;         // optional [count][nmax*nmax]
  int nmax;
  long long *prof;    // optional per-CTA phase clocks [count*C][8] (debug)
  void *uscr;         // [count][nmax/2][nmax/2+1] factor U of the fast path (L2 scratch)
  void *gchk;         // [count][16][blocks][16] Gram-check partials (L2 scratch), may be null
  int mode;           // PV_FULL: whole pivot; PV_PROLOGUE: R0 -> R0g only; PV_EPILOGUE: W = R0^-1 R_final
  void *R0g;          // [count][nmax*nmax] R0 (prologue output / epilogue input)
  void *dscr;         // [count][nmax] doubles: the Jacobi kernel's Gram-check scratch
  int fp_input;       // factor prologue: FP_STRUCTURED (A[item], D[item]) or FP_DENSE_PAIR
                      // (A[3 item + 0/1/2] = A_ii, A_jj, A_ij of the pair)
};
// cluster: 0 = automatic choice
cudaError_t launch_pivot(bool cx, const PivotArgs &a, int cluster, cudaStream_t st, int *cluster_used);
int pivot_nmax(int bmax);   // NMAX instance for a block width
int pivot_default_cluster(bool cx, int nmax, int count);
int pivot_default_threads(bool cx, int nmax, int cluster);
void pivot_tune(int threads, int cluster);  // 0 = automatic
int pivot_max_active_clusters(bool cx, int nmax, int cluster, int threads);
size_t pivot_check_elems(int nmax);
// the (cluster, threads) launch_pivot picks when not told (honours hjb_tune)
int pivot_choose_cluster(bool cx, int nmax, int count);
int pivot_choose_threads(bool cx, int nmax, int c);  // Gram-check scratch elements per item

// factor.cu: one-CTA-per-pivot prologue (R0) and column-sliced epilogue
// (W = R0^-1 R_final) around the Jacobi kernel
cudaError_t launch_factor_prologue(bool cx, const PivotArgs &a, cudaStream_t st);
cudaError_t launch_factor_epilogue(bool cx, const PivotArgs &a, cudaStream_t st);

cudaError_t launch_plane_rotations(bool cx, int count, const double *arr, const double *ass, const void *ars,
                                   const int8_t *same, double *out, cudaStream_t st);

// Jacobi kernel (jacobi.cu): R0 -> R_final for a batch of pivots.
struct JacobiArgs {
  const Item *items;
  int count;
  int nmax, ld;          // pivot order instance and leading dimension of R0 / Rout
  const void *R0;        // [count][ld*ld] initial factor (pivot kernel prologue)
  void *Rout;            // [count][ld*ld] final factor
  const int8_t *signs;
  double orth_tol, quad_tol;
  int max_sweeps;
  int64_t *stats;        // [count][ST_N]: status/fallback in, counters out
  long long *prof;       // optional per-warp phase clocks [count*C*W][8] (HJB_JAC_PROF builds)
  double *dscr;          // [count][ld] column norms of the final-sweep Gram check (null: no check)
  int mode;              // JAC_CONVERGE (F variants), JAC_ONE_CYCLE / JAC_CROSS (B variants)
};
struct JacShape {
  int c, w, spw;  // cluster size, warps per CTA, pairs per warp (nmax = 2 c w spw)
};
JacShape jacobi_default_shape(bool cx, int nmax, int count);
bool jacobi_shape_for(int nmax, int c, JacShape *out);  // an instantiated shape with cluster size c
cudaError_t launch_jacobi(bool cx, const JacobiArgs &a, JacShape s, cudaStream_t st);
int jacobi_wave_capacity(bool cx, int nmax, JacShape s);  // clusters resident at once (0: unknown)

struct UpdateArgs {
  void *G;
  int64_t ldg, m;
  const Item *items;
  int count;
  int nmax;
  const void *W;
  const int64_t *stats;
};
cudaError_t launch_update(bool cx, const UpdateArgs &a, cudaStream_t st);

cudaError_t launch_extract(bool cx, int64_t m, int64_t n, const void *G, int64_t ldg,
                           const int8_t *signs, double *lam, void *U, int64_t ldu,
                           const int64_t *perm, int *zero_flag, cudaStream_t st);

cudaError_t launch_orth_max(bool cx, const Item *items, int count, int bmax, const void *A,
                            unsigned long long *out, cudaStream_t st);

}  // namespace hjb
