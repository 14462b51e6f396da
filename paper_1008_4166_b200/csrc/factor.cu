// Pivot factor kernels around the Jacobi kernel (round 2).
//
// factor_prologue_kernel: the structured Cholesky of the pair step
// (blocking.py:115-138): R0 = [[sqrt(L_i), A_ij / sqrt(L_i)], [0, chol(S)]],
// S = herm(L_j - R_ij^H R_ij), with the dense fallback of parallel.py:196-198
// (Cholesky of the pair Gram formed from G) when a norm is not positive or
// the Cholesky of S fails; for the F pre-pass (parallel.py:143)
// R0 = chol(herm(B^H B)).  One CTA per pivot: the Schur complement is a
// DMMA product out of shared memory, the b x b Cholesky runs on a register
// tile with one CTA barrier per column.
//
// factor_epilogue_kernel: W = R0^-1 R_final, the accumulated transformation
// of the pivot (the reference accumulates W rotation by rotation,
// rotations.py:209-223; here it is recovered from the initial and final
// factor).  The columns of W are independent, so a pivot is split
// over N / CW CTAs; each CTA keeps its column slice in shared memory and
// runs a blocked back substitution (32-row blocks: DMMA for the off-diagonal
// part with R0 read from L2, warp-shuffle substitution on the diagonal
// block).
//
// Round 1 ran both inside the cluster-wide pivot kernel (pivot.cu,
// PV_PROLOGUE / PV_EPILOGUE), which took 1.86 + 1.82 ms per cfg5r step
// (10 % of the solve); kept there for HJB_FACTOR_V1=1 A/B runs.
#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"

namespace hjb {

namespace {

// conj(a) * b accumulators (Schur complement R_ij^H R_ij)
template <typename T> struct HAcc;
template <> struct HAcc<double> {
  double v[2];
  __device__ __forceinline__ void zero() { v[0] = v[1] = 0.0; }
  __device__ __forceinline__ void mma(double a, double b) { dmma(v[0], v[1], a, b); }
  __device__ __forceinline__ double get(int q) const { return v[q]; }
};
template <> struct HAcc<cplx> {
  double r[2], i[2];
  __device__ __forceinline__ void zero() { r[0] = r[1] = i[0] = i[1] = 0.0; }
  __device__ __forceinline__ void mma(cplx a, cplx b) {
    dmma(r[0], r[1], a.x, b.x);
    dmma(i[0], i[1], a.x, b.y);
    dmma(r[0], r[1], a.y, b.y);
    dmma(i[0], i[1], -a.y, b.x);
  }
  __device__ __forceinline__ cplx get(int q) const { return make_double2(r[q], i[q]); }
};
// a * b accumulators (R0 W)
template <typename T> struct PAcc;
template <> struct PAcc<double> {
  double v[2];
  __device__ __forceinline__ void zero() { v[0] = v[1] = 0.0; }
  __device__ __forceinline__ void mma(double a, double b) { dmma(v[0], v[1], a, b); }
  __device__ __forceinline__ double get(int q) const { return v[q]; }
};
template <> struct PAcc<cplx> {
  double r[2], i[2];
  __device__ __forceinline__ void zero() { r[0] = r[1] = i[0] = i[1] = 0.0; }
  __device__ __forceinline__ void mma(cplx a, cplx b) {
    dmma(r[0], r[1], a.x, b.x);
    dmma(i[0], i[1], a.x, b.y);
    dmma(r[0], r[1], -a.y, b.y);
    dmma(i[0], i[1], a.y, b.x);
  }
  __device__ __forceinline__ cplx get(int q) const { return make_double2(r[q], i[q]); }
};

__device__ __forceinline__ int pk(int i, int l) { return l * (l + 1) / 2 + i; }  // packed upper triangle, i <= l

template <typename T, int B>
struct ProCfg {
  static constexpr int NT = B >= 128 ? 512 : (B >= 64 ? 256 : 128);
  static constexpr int NW = NT / 32;
  static constexpr int KC = 32, KCP = KC + 4;
  static constexpr int PK = B * (B + 1) / 2;
  static constexpr size_t OFF_S = 0;                                   // packed S / U
  static constexpr size_t OFF_X = OFF_S + size_t(PK) * sizeof(T);      // staged R_ij chunk [B][KCP]
  static constexpr size_t OFF_ROW = OFF_X + size_t(B) * KCP * sizeof(T);  // Cholesky row buffers [2][B]
  static constexpr size_t OFF_LAM = OFF_ROW + 2 * size_t(B) * sizeof(T);  // lam [2B], sqrt(lam_i) [B], pivots [B]
  static constexpr size_t SMEM = OFF_LAM + 4 * size_t(B) * sizeof(double);
};

// Right-looking Cholesky of the n x n matrix whose upper triangle is packed
// in Sp (shared memory), on a register tile: thread (ti, tl) of a TI x TL
// grid holds rows ti + TI x, columns tl + TL y.  The rows stay unscaled
// (U[i][l] -= conj(U[k][i]) U[k][l] / U[k][k]); row k + 1 is published
// through a double buffer, so a step costs one CTA barrier.  On success the
// factor R[k][l] = U[k][l] / sqrt(U[k][k]) overwrites Sp.  Returns false
// (uniformly) on a non-positive or non-finite pivot (blocking.py:106-112).
template <typename T, int B, int NT>
__device__ bool chol_tile(T *Sp, int n, T *rowb, double *piv) {
  constexpr int TI = 16, TL = NT / TI, XI = B / TI, YL = (B + TL - 1) / TL;
  const int tid = threadIdx.x, ti = tid % TI, tl = tid / TI;
  T u[XI][YL];
#pragma unroll
  for (int x = 0; x < XI; ++x)
#pragma unroll
    for (int y = 0; y < YL; ++y) {
      if (TI * x >= TL * (y + 1)) continue;  // tile position below the diagonal for every thread
      const int i = ti + TI * x, l = tl + TL * y;
      u[x][y] = (i <= l && l < n) ? Sp[pk(i, l)] : S<T>::zero();
    }
  auto publish = [&](int k) {
    if (k < n && ti == k % TI) {
      const int xk = k / TI;
#pragma unroll
      for (int x = 0; x < XI; ++x) {
        if (x != xk) continue;
#pragma unroll
        for (int y = 0; y < YL; ++y) {
          if (TI * x >= TL * (y + 1)) continue;
          const int l = tl + TL * y;
          if (l >= k && l < n) rowb[(k & 1) * B + l] = u[x][y];
        }
      }
    }
  };
  publish(0);
  __syncthreads();
  bool ok = true;
  for (int k = 0; k < n; ++k) {
    const T *rk = rowb + (k & 1) * B;
    const double dk = re(rk[k]);
    if (!finite_pos(dk)) {
      ok = false;
      break;
    }
    if (tid == 0) piv[k] = dk;
    const double inv = 1.0 / dk;
    T ri[XI], rl[YL];
#pragma unroll
    for (int x = 0; x < XI; ++x) ri[x] = scale(rk[min(ti + TI * x, B - 1)], inv);
#pragma unroll
    for (int y = 0; y < YL; ++y) rl[y] = rk[min(tl + TL * y, B - 1)];
#pragma unroll
    for (int x = 0; x < XI; ++x) {
      const int i = ti + TI * x;
      if (i <= k) continue;  // finished rows
#pragma unroll
      for (int y = 0; y < YL; ++y) {
        if (TI * x >= TL * (y + 1)) continue;
        const int l = tl + TL * y;
        if (l >= i && l < n) u[x][y] = cfms(ri[x], rl[y], u[x][y]);
      }
    }
    publish(k + 1);
    __syncthreads();
  }
  if (!ok) return false;
#pragma unroll
  for (int x = 0; x < XI; ++x)
#pragma unroll
    for (int y = 0; y < YL; ++y) {
      if (TI * x >= TL * (y + 1)) continue;
      const int i = ti + TI * x, l = tl + TL * y;
      if (i <= l && l < n) {
        const double rd = sqrt(piv[i]);
        Sp[pk(i, l)] = i == l ? scale(S<T>::one(), rd) : divr(u[x][y], rd);
      }
    }
  __syncthreads();
  return true;
}

template <typename T, int B>
__global__ void __launch_bounds__(ProCfg<T, B>::NT, 1) factor_prologue_kernel(PivotArgs a) {
  using Cfg = ProCfg<T, B>;
  constexpr int NT = Cfg::NT, NW = Cfg::NW, KC = Cfg::KC, KCP = Cfg::KCP;
  extern __shared__ __align__(16) unsigned char smem[];
  T *Sp = reinterpret_cast<T *>(smem + Cfg::OFF_S);
  T *Xs = reinterpret_cast<T *>(smem + Cfg::OFF_X);
  T *rowk = reinterpret_cast<T *>(smem + Cfg::OFF_ROW);
  double *lam = reinterpret_cast<double *>(smem + Cfg::OFF_LAM);  // [2B]
  double *sq = lam + 2 * B;                                       // sqrt(lam_i) [B]
  double *piv = sq + B;                                           // Cholesky pivots [B]
  __shared__ int s_ok;

  const int item_id = blockIdx.x;
  const Item it = a.items[item_id];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const bool dense = it.nj == 0;
  const int ni = it.ni, nj = it.nj, N = ni + nj;
  const int bmax = a.bmax, ld = a.nmax;
  const T *A = reinterpret_cast<const T *>(a.A) + int64_t(item_id) * bmax * bmax;
  T *R0 = reinterpret_cast<T *>(a.R0g) + int64_t(item_id) * ld * ld;
  const int nu = dense ? ni : nj;  // order of the Cholesky block

  if (tid == 0) s_ok = 1;
  for (int c = tid; c < 2 * B; c += NT) {
    double v = 1.0;
    if (!dense && c < B && c < ni) v = a.D[int64_t(item_id) * 2 * bmax + c];
    if (!dense && c >= B && c - B < nj) v = a.D[int64_t(item_id) * 2 * bmax + bmax + (c - B)];
    lam[c] = v;
  }
  // R0 is zero outside the pieces written below (strict lower triangle,
  // padding up to nmax): store-only, overlaps with everything that follows
  for (int e = tid; e < ld * ld; e += NT) R0[e] = S<T>::zero();
  __syncthreads();
  int status = PV_OK, fallback = 0;
  bool structured = false;
  if (!dense) {
    // structured_cholesky needs positive norms (blocking.py:125-126)
    int ok = 1;
    for (int c = tid; c < 2 * B; c += NT) ok &= finite_pos(lam[c]);
    ok = __syncthreads_and(ok);
    if (ok) {
      for (int c = tid; c < B; c += NT) sq[c] = sqrt(lam[c]);
      // S = diag(L_j) - R_ij^H R_ij on the upper triangle
      for (int e = tid; e < Cfg::PK; e += NT) Sp[e] = S<T>::zero();
      __syncthreads();
      for (int c = tid; c < nj; c += NT) Sp[pk(c, c)] = scale(S<T>::one(), lam[B + c]);
      constexpr int TJ = B / 32, NTILE = (B / 16) * TJ;  // 16 x 32 tiles
      for (int h0 = 0; h0 < ni; h0 += KC) {
        __syncthreads();
        // stage R_ij = A_ij / sqrt(L_i) (rows h0 .. h0 + KC) and write it to
        // its place in R0 on the way (the top-right block)
#pragma unroll 4
        for (int e = tid; e < B * KC; e += NT) {
          const int k = e % KC, l = e / KC;
          const int h = h0 + k;
          T v = S<T>::zero();
          if (h < ni && l < nj) {
            v = divr(A[h + int64_t(l) * bmax], sq[h]);
            R0[h + int64_t(ni + l) * ld] = v;
          }
          Xs[l * KCP + k] = v;
        }
        __syncthreads();
        for (int t = warp; t < NTILE; t += NW) {
          const int ti = t / TJ, tj = t % TJ;
          if (16 * ti >= 32 * (tj + 1) || 16 * ti >= nj || 32 * tj >= nj) continue;  // below the diagonal / empty
          HAcc<T> acc[2][4];
#pragma unroll
          for (int mi = 0; mi < 2; ++mi)
#pragma unroll
            for (int nn = 0; nn < 4; ++nn) acc[mi][nn].zero();
#pragma unroll 2
          for (int kk = 0; kk < KC; kk += 4) {
            T fa[2], fb[4];
#pragma unroll
            for (int mi = 0; mi < 2; ++mi) fa[mi] = Xs[((ti * 2 + mi) * 8 + (lane >> 2)) * KCP + kk + (lane & 3)];
#pragma unroll
            for (int nn = 0; nn < 4; ++nn) fb[nn] = Xs[((tj * 4 + nn) * 8 + (lane >> 2)) * KCP + kk + (lane & 3)];
#pragma unroll
            for (int mi = 0; mi < 2; ++mi)
#pragma unroll
              for (int nn = 0; nn < 4; ++nn) acc[mi][nn].mma(fa[mi], fb[nn]);
          }
#pragma unroll
          for (int mi = 0; mi < 2; ++mi)
#pragma unroll
            for (int nn = 0; nn < 4; ++nn)
#pragma unroll
              for (int q = 0; q < 2; ++q) {
                const int i = (ti * 2 + mi) * 8 + (lane >> 2);
                const int l = (tj * 4 + nn) * 8 + 2 * (lane & 3) + q;
                if (i <= l && l < nj) Sp[pk(i, l)] = sub(Sp[pk(i, l)], acc[mi][nn].get(q));
              }
        }
      }
      __syncthreads();
      for (int c = tid; c < nj; c += NT) Sp[pk(c, c)] = scale(S<T>::one(), re(Sp[pk(c, c)]));  // Hermitian diagonal
      __syncthreads();
      structured = chol_tile<T, B, NT>(Sp, nj, rowk, piv);
    }
    if (!structured) fallback = 1;  // parallel.py:196-198
  } else {
    // pre-pass: herm(B^H B) (core.py:54-55)
    for (int e = tid; e < ni * ni; e += NT) {
      const int i = e % ni, l = e / ni;
      if (i > l) continue;
      Sp[pk(i, l)] = i == l ? scale(S<T>::one(), re(A[i + int64_t(i) * bmax]))
                            : scale(add(A[i + int64_t(l) * bmax], conjv(A[l + int64_t(i) * bmax])), 0.5);
    }
    __syncthreads();
    if (!chol_tile<T, B, NT>(Sp, ni, rowk, piv)) status = PV_CHOL;
  }
  __syncthreads();

  if (fallback) {
    // dense fallback: R0 = chol(gram([G_i G_j])) formed from G itself
    // (parallel.py:196-198), factored in place in the global R0 slab.  Rare
    // (0 of ~20k pivots on the BASELINE configs): one CTA, plain loops.
    const T *G = reinterpret_cast<const T *>(a.G);
    auto colptr = [&](int c) -> const T * { return G + int64_t(c < ni ? it.oi + c : it.oj + (c - ni)) * a.ldg; };
    for (int e = tid; e < ld * ld; e += NT) R0[e] = S<T>::zero();
    __syncthreads();
    for (int e = warp; e < N * N; e += NW) {  // one warp per entry of the upper triangle
      const int g = e % N, l = e / N;
      if (g > l) continue;
      const T *xg = colptr(g), *xl = colptr(l);
      T s = S<T>::zero();
      for (int64_t r = lane; r < a.m; r += 32) s = cfma(xg[r], xl[r], s);
#pragma unroll
      for (int dist = 16; dist >= 1; dist >>= 1) s = add(s, shfl_xor(s, dist));
      if (lane == 0) R0[g + int64_t(l) * ld] = g == l ? scale(S<T>::one(), re(s)) : s;
    }
    __syncthreads();
    for (int k = 0; k < N && status == PV_OK; ++k) {
      const double d = re(R0[k + int64_t(k) * ld]);
      if (!finite_pos(d)) {
        status = PV_CHOL;
        break;
      }
      const double rkk = sqrt(d);
      __syncthreads();
      for (int l = k + tid; l < N; l += NT)
        R0[k + int64_t(l) * ld] = l == k ? scale(S<T>::one(), rkk) : divr(R0[k + int64_t(l) * ld], rkk);
      __syncthreads();
      for (int l = k + 1 + warp; l < N; l += NW) {
        const T ul = R0[k + int64_t(l) * ld];
        for (int i = k + 1 + lane; i <= l; i += 32)
          R0[i + int64_t(l) * ld] = cfms(R0[k + int64_t(i) * ld], ul, R0[i + int64_t(l) * ld]);
      }
      __syncthreads();
    }
  } else if (status == PV_OK) {
    // the rest of R0 (zero filled above, R_ij written while staging): the
    // diagonal sqrt(L_i) block and the Cholesky factor of the second block
    const int nt = dense ? 0 : ni;
    for (int g = tid; g < nt; g += NT) R0[g + int64_t(g) * ld] = scale(S<T>::one(), sq[g]);
    const int nu2 = N - nt;
    for (int e = tid; e < nu2 * nu2; e += NT) {
      const int g = e % nu2, c = e / nu2;
      if (g <= c) R0[(nt + g) + int64_t(nt + c) * ld] = Sp[pk(g, c)];
    }
  }
  if (tid == 0) {
    int64_t *st = a.stats + int64_t(item_id) * ST_N;
    st[ST_NROT] = 0;
    st[ST_NBIG] = 0;
    st[ST_MAXT] = 0;
    st[ST_SWEEPS] = 0;
    st[ST_STATUS] = status;
    st[ST_FR] = -1;
    st[ST_FS] = -1;
    st[ST_FALLBACK] = fallback;
  }
  (void)nu;
}

// ------------------------------------------------------------------ dense pair (B variants)
// R0 = chol(gram([G_i G_j])) (parallel.py:199-200) by blocks:
//   R_ii = chol(herm(A_ii)),  X = R_ii^-H A_ij,  R_jj = chol(herm(A_jj) - X^H X).
// A_ii, A_jj, A_ij are items 3t, 3t+1, 3t+2 of the Gram launch.  The forward
// substitution runs on 32-column slices of A_ij in shared memory (32-row
// blocks: DMMA for the part above the diagonal block, warp-shuffle
// substitution inside it); X goes to the top-right block of R0 in global
// memory and is staged back in K chunks for the Schur complement.
template <typename T, int B>
__global__ void __launch_bounds__(ProCfg<T, B>::NT, 1) factor_dense_pair_kernel(PivotArgs a) {
  using Cfg = ProCfg<T, B>;
  constexpr int NT = Cfg::NT, NW = Cfg::NW, KC = Cfg::KC, KCP = Cfg::KCP;
  constexpr int SW = 32;                // slice width (columns of A_ij)
  constexpr int CPW = SW / NW;          // columns per warp in the substitution
  constexpr int LDS_ = B + 4;           // slice leading dimension
  static_assert(SW * LDS_ <= B * KCP, "the slice buffer aliases the chunk staging buffer");
  extern __shared__ __align__(16) unsigned char smem[];
  T *Sp = reinterpret_cast<T *>(smem + Cfg::OFF_S);
  T *Xs = reinterpret_cast<T *>(smem + Cfg::OFF_X);
  T *rowk = reinterpret_cast<T *>(smem + Cfg::OFF_ROW);
  double *piv = reinterpret_cast<double *>(smem + Cfg::OFF_LAM) + 3 * B;

  const int item_id = blockIdx.x;
  const Item it = a.items[item_id];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int ni = it.ni, nj = it.nj, N = ni + nj;
  const int bmax = a.bmax, ld = a.nmax;
  const int64_t asz = int64_t(bmax) * bmax;
  const T *Aii = reinterpret_cast<const T *>(a.A) + (int64_t(item_id) * 3 + 0) * asz;
  const T *Ajj = reinterpret_cast<const T *>(a.A) + (int64_t(item_id) * 3 + 1) * asz;
  const T *Aij = reinterpret_cast<const T *>(a.A) + (int64_t(item_id) * 3 + 2) * asz;
  T *R0 = reinterpret_cast<T *>(a.R0g) + int64_t(item_id) * ld * ld;
  int status = PV_OK;

  auto load_herm = [&](const T *A, int n) {
    for (int e = tid; e < n * n; e += NT) {
      const int i = e % n, l = e / n;
      if (i > l) continue;
      Sp[pk(i, l)] = i == l ? scale(S<T>::one(), re(A[i + int64_t(i) * bmax]))
                            : scale(add(A[i + int64_t(l) * bmax], conjv(A[l + int64_t(i) * bmax])), 0.5);
    }
  };
  for (int e = tid; e < ld * ld; e += NT) R0[e] = S<T>::zero();
  load_herm(Aii, ni);
  __syncthreads();
  if (!chol_tile<T, B, NT>(Sp, ni, rowk, piv)) status = PV_CHOL;
  if (status == PV_OK) {
    for (int e = tid; e < ni * ni; e += NT) {
      const int g = e % ni, c = e / ni;
      if (g <= c) R0[g + int64_t(c) * ld] = Sp[pk(g, c)];
    }
    // ---- X = R_ii^-H A_ij, slice by slice ----
    T *Xl = Xs;  // [SW][LDS_]
    const int nblk = (ni + 31) / 32;
    for (int c0 = 0; c0 < nj; c0 += SW) {
      __syncthreads();
      for (int e = tid; e < SW * B; e += NT) {
        const int r = e % B, c = e / B;
        Xl[c * LDS_ + r] = (r < ni && c0 + c < nj) ? Aij[r + int64_t(c0 + c) * bmax] : S<T>::zero();
      }
      __syncthreads();
      for (int I = 0; I < nblk; ++I) {
        const int r0 = 32 * I;
        if (I > 0) {
          // T_I -= (R_ii^H)[I rows, h] X[h, :], h < r0: 32 x SW output, 16 fragments over the warps
          for (int f = warp; f < 16; f += NW) {
            const int mi = f >> 2, nn = f & 3;
            HAcc<T> acc;
            acc.zero();
            const int row = r0 + mi * 8 + (lane >> 2);
            const T *bp = Xl + (nn * 8 + (lane >> 2)) * LDS_ + (lane & 3);
            for (int h = 0; h < r0; h += 4) {
              const int hh = h + (lane & 3);
              const T fa = row < ni ? Sp[pk(hh, row)] : S<T>::zero();  // R_ii[h][row], h < row
              acc.mma(fa, bp[h]);
            }
#pragma unroll
            for (int q = 0; q < 2; ++q) {
              T *pp = Xl + (nn * 8 + 2 * (lane & 3) + q) * LDS_ + r0 + mi * 8 + (lane >> 2);
              *pp = sub(*pp, acc.get(q));
            }
          }
          __syncthreads();
        }
        // forward substitution inside the diagonal block: lane s holds row r0 + s
        {
          const int row = r0 + lane;
          T rr[32];
#pragma unroll
          for (int r = 0; r < 32; ++r)
            rr[r] = (r < lane && row < ni) ? conjv(Sp[pk(r0 + r, row)]) : S<T>::zero();
          const double rinv = row < ni ? 1.0 / re(Sp[pk(row, row)]) : 0.0;
          T t[CPW];
#pragma unroll
          for (int j = 0; j < CPW; ++j) t[j] = Xl[(warp * CPW + j) * LDS_ + row];
#pragma unroll
          for (int r = 0; r < 32; ++r) {
#pragma unroll
            for (int j = 0; j < CPW; ++j) {
              const T xr = shfl_idx(scale(t[j], rinv), r);
              if (lane == r) t[j] = xr;
              if (lane > r) t[j] = sub(t[j], mul(rr[r], xr));
            }
          }
#pragma unroll
          for (int j = 0; j < CPW; ++j) Xl[(warp * CPW + j) * LDS_ + row] = t[j];
        }
        __syncthreads();
      }
      for (int e = tid; e < SW * ni; e += NT) {
        const int r = e % ni, c = e / ni;
        if (c0 + c < nj) R0[r + int64_t(ni + c0 + c) * ld] = Xl[c * LDS_ + r];
      }
    }
    __syncthreads();
    // ---- S = herm(A_jj) - X^H X, R_jj = chol(S) ----
    load_herm(Ajj, nj);
    constexpr int TJ = B / 32, NTILE = (B / 16) * TJ;
    for (int h0 = 0; h0 < ni; h0 += KC) {
      __syncthreads();
      for (int e = tid; e < B * KC; e += NT) {
        const int k = e % KC, l = e / KC;
        const int h = h0 + k;
        Xs[l * KCP + k] = (h < ni && l < nj) ? R0[h + int64_t(ni + l) * ld] : S<T>::zero();
      }
      __syncthreads();
      for (int t = warp; t < NTILE; t += NW) {
        const int ti = t / TJ, tj = t % TJ;
        if (16 * ti >= 32 * (tj + 1) || 16 * ti >= nj || 32 * tj >= nj) continue;
        HAcc<T> acc[2][4];
#pragma unroll
        for (int mi = 0; mi < 2; ++mi)
#pragma unroll
          for (int nn = 0; nn < 4; ++nn) acc[mi][nn].zero();
#pragma unroll 2
        for (int kk = 0; kk < KC; kk += 4) {
          T fa[2], fb[4];
#pragma unroll
          for (int mi = 0; mi < 2; ++mi) fa[mi] = Xs[((ti * 2 + mi) * 8 + (lane >> 2)) * KCP + kk + (lane & 3)];
#pragma unroll
          for (int nn = 0; nn < 4; ++nn) fb[nn] = Xs[((tj * 4 + nn) * 8 + (lane >> 2)) * KCP + kk + (lane & 3)];
#pragma unroll
          for (int mi = 0; mi < 2; ++mi)
#pragma unroll
            for (int nn = 0; nn < 4; ++nn) acc[mi][nn].mma(fa[mi], fb[nn]);
        }
#pragma unroll
        for (int mi = 0; mi < 2; ++mi)
#pragma unroll
          for (int nn = 0; nn < 4; ++nn)
#pragma unroll
            for (int q = 0; q < 2; ++q) {
              const int i = (ti * 2 + mi) * 8 + (lane >> 2);
              const int l = (tj * 4 + nn) * 8 + 2 * (lane & 3) + q;
              if (i <= l && l < nj) Sp[pk(i, l)] = sub(Sp[pk(i, l)], acc[mi][nn].get(q));
            }
      }
    }
    __syncthreads();
    for (int c = tid; c < nj; c += NT) Sp[pk(c, c)] = scale(S<T>::one(), re(Sp[pk(c, c)]));
    __syncthreads();
    if (!chol_tile<T, B, NT>(Sp, nj, rowk, piv)) {
      status = PV_CHOL;
    } else {
      for (int e = tid; e < nj * nj; e += NT) {
        const int g = e % nj, c = e / nj;
        if (g <= c) R0[(ni + g) + int64_t(ni + c) * ld] = Sp[pk(g, c)];
      }
    }
  }
  if (tid == 0) {
    int64_t *st = a.stats + int64_t(item_id) * ST_N;
    st[ST_NROT] = 0;
    st[ST_NBIG] = 0;
    st[ST_MAXT] = 0;
    st[ST_SWEEPS] = 0;
    st[ST_STATUS] = status;
    st[ST_FR] = -1;
    st[ST_FS] = -1;
    st[ST_FALLBACK] = 1;  // R0 is a general upper-triangular factor for the epilogue
  }
  (void)N;
}

// ------------------------------------------------------------------ epilogue

template <typename T>
struct EpiCfg {
  static constexpr int NT = 256, NW = 8;
  static constexpr int CW = S<T>::cx ? 16 : 32;  // columns of W per CTA
  static constexpr int CPW = CW / NW;            // columns per warp in the substitution
  static constexpr int NF = CW / 16;             // 8-column DMMA fragments per warp (4 row groups x 2 column groups of warps)
};

template <typename T>
__global__ void __launch_bounds__(256) factor_epilogue_kernel(PivotArgs a) {
  using Cfg = EpiCfg<T>;
  constexpr int NT = Cfg::NT, CW = Cfg::CW, CPW = Cfg::CPW, NF = Cfg::NF;
  extern __shared__ __align__(16) unsigned char smem[];
  T *Fs = reinterpret_cast<T *>(smem);  // [CW][LDF]: column slice of R_final, then of W

  const int item_id = blockIdx.y;
  const int64_t *sv = a.stats + int64_t(item_id) * ST_N;
  // nothing to do for a failed pivot or one that applied no rotation (the update skips it)
  if (__ldcg(sv + ST_STATUS) != PV_OK || __ldcg(sv + ST_NROT) == 0) return;
  const Item it = a.items[item_id];
  const int ni = it.ni, nj = it.nj, N = ni + nj;
  const int c0 = blockIdx.x * CW;
  if (c0 >= N) return;
  const bool structured = nj > 0 && __ldcg(sv + ST_FALLBACK) == 0;
  const int ld = a.nmax, LDF = ld + 4;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const T *R0 = reinterpret_cast<const T *>(a.R0g) + int64_t(item_id) * ld * ld;
  T *F = reinterpret_cast<T *>(a.W) + int64_t(item_id) * ld * ld;
  T *Rout = a.Rout ? reinterpret_cast<T *>(a.Rout) + int64_t(item_id) * ld * ld : nullptr;

  for (int e = tid; e < CW * ld; e += NT) {
    const int r = e % ld, c = e / ld;
    T v = S<T>::zero();
    if (r < N && c0 + c < N) {
      v = __ldcg(F + r + int64_t(c0 + c) * ld);
      if (Rout) Rout[r + int64_t(c0 + c) * ld] = v;  // R_final for the optional output
    }
    Fs[c * LDF + r] = v;
  }
  __syncthreads();

  const int nblk = (N + 31) / 32;
  const int kend = min(ld, (N + 3) & ~3);
  for (int I = nblk - 1; I >= 0; --I) {
    const int r0 = 32 * I;
    // ---- T_I = F_I - R0[I, k] W[k, :] over the rows below the block ----
    // the diagonal block's row of this lane and its reciprocal pivot: loaded
    // first so that their L2 latency overlaps the DMMA part
    const int row = r0 + lane;
    T rr[32];
#pragma unroll
    for (int r = 0; r < 32; ++r)
      rr[r] = (r > lane && row < N && r0 + r < N) ? __ldcg(R0 + row + int64_t(r0 + r) * ld) : S<T>::zero();
    const double rdiag = row < N ? re(__ldcg(R0 + row + int64_t(row) * ld)) : 1.0;
    int kstart = r0 + 32;
    if (structured && r0 + 32 <= ni) kstart = max(kstart, ni & ~3);  // the sqrt(L_i) block is diagonal
    if (kstart < kend) {
      const int mi = warp >> 1, nb = (warp & 1) * NF;
      PAcc<T> acc[NF];
#pragma unroll
      for (int f = 0; f < NF; ++f) acc[f].zero();
      const T *ap = R0 + (r0 + mi * 8 + (lane >> 2)) + int64_t(lane & 3) * ld;
      const T *bp = Fs + ((nb * 8) + (lane >> 2)) * LDF + (lane & 3);
#pragma unroll 8
      for (int k = kstart; k < kend; k += 4) {
        const T fa = __ldcg(ap + int64_t(k) * ld);
#pragma unroll
        for (int f = 0; f < NF; ++f) acc[f].mma(fa, bp[f * 8 * LDF + k]);
      }
#pragma unroll
      for (int f = 0; f < NF; ++f)
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          T *p = Fs + ((nb + f) * 8 + 2 * (lane & 3) + q) * LDF + r0 + mi * 8 + (lane >> 2);
          *p = sub(*p, acc[f].get(q));
        }
    }
    __syncthreads();
    // ---- W_I = R0[I, I]^-1 T_I: lane s holds row r0 + s; each solved row is
    // broadcast by a shuffle (the diagonal of a Cholesky factor is real) ----
    {
      const double rinv = row < N ? 1.0 / rdiag : 0.0;
      T t[CPW];
#pragma unroll
      for (int j = 0; j < CPW; ++j) t[j] = Fs[(warp * CPW + j) * LDF + row];
#pragma unroll
      for (int r = 31; r >= 0; --r) {
#pragma unroll
        for (int j = 0; j < CPW; ++j) {
          const T wr = shfl_idx(scale(t[j], rinv), r);
          if (lane == r) t[j] = wr;
          if (lane < r) t[j] = sub(t[j], mul(rr[r], wr));
        }
      }
#pragma unroll
      for (int j = 0; j < CPW; ++j) Fs[(warp * CPW + j) * LDF + row] = t[j];
    }
    __syncthreads();
  }
  for (int e = tid; e < CW * ld; e += NT) {
    const int r = e % ld, c = e / ld;
    if (r < N && c0 + c < N) F[r + int64_t(c0 + c) * ld] = Fs[c * LDF + r];
  }
}

template <typename T, int B>
cudaError_t launch_prologue_t(const PivotArgs &a, cudaStream_t st) {
  using Cfg = ProCfg<T, B>;
  auto k = a.fp_input == FP_DENSE_PAIR ? factor_dense_pair_kernel<T, B> : factor_prologue_kernel<T, B>;
  static DeviceFlags attr_flags[2];
  bool *attr = attr_flags[a.fp_input == FP_DENSE_PAIR].here();
  if (!attr) return cudaErrorInvalidDevice;
  if (!*attr) {
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(Cfg::SMEM));
    if (e != cudaSuccess) return e;
    *attr = true;
  }
  k<<<unsigned(a.count), Cfg::NT, Cfg::SMEM, st>>>(a);
  return cudaGetLastError();
}

template <typename T>
cudaError_t launch_epilogue_t(const PivotArgs &a, cudaStream_t st) {
  using Cfg = EpiCfg<T>;
  auto k = factor_epilogue_kernel<T>;
  const size_t smem = size_t(Cfg::CW) * (a.nmax + 4) * sizeof(T);
  static DeviceFlags attr_flags;
  bool *attr = attr_flags.here();
  if (!attr) return cudaErrorInvalidDevice;
  if (!*attr) {
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         int(size_t(Cfg::CW) * (256 + 4) * sizeof(T)));
    if (e != cudaSuccess) return e;
    *attr = true;
  }
  dim3 grid(unsigned((a.nmax + Cfg::CW - 1) / Cfg::CW), unsigned(a.count));
  k<<<grid, Cfg::NT, smem, st>>>(a);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_factor_prologue(bool cx, const PivotArgs &a, cudaStream_t st) {
  if (a.count == 0) return cudaSuccess;
  switch (a.nmax) {
    case 32: return cx ? launch_prologue_t<cplx, 32>(a, st) : launch_prologue_t<double, 32>(a, st);  // b <= 16: the 32-wide instance
    case 64: return cx ? launch_prologue_t<cplx, 32>(a, st) : launch_prologue_t<double, 32>(a, st);
    case 128: return cx ? launch_prologue_t<cplx, 64>(a, st) : launch_prologue_t<double, 64>(a, st);
    case 256: return cx ? launch_prologue_t<cplx, 128>(a, st) : launch_prologue_t<double, 128>(a, st);
  }
  return cudaErrorInvalidConfiguration;
}

cudaError_t launch_factor_epilogue(bool cx, const PivotArgs &a, cudaStream_t st) {
  if (a.count == 0) return cudaSuccess;
  if (a.nmax > 256) return cudaErrorInvalidConfiguration;
  return cx ? launch_epilogue_t<cplx>(a, st) : launch_epilogue_t<double>(a, st);
}

}  // namespace hjb
