// Block-pivot kernel: the inner level of the 2F step.
//
// For each work item (a block pair (i, j), or a single block in the F
// pre-pass) one thread-block cluster of C CTAs
//   1. builds the upper-triangular factor R of the pivot Gram by the
//      structured Cholesky R = [[sqrt(L_i), L_i^-1/2 A_ij], [0, chol(S)]],
//      S = L_j - R_ij^H R_ij (reference blocking.py:115-138), or by a dense
//      Cholesky of the block Gram for the pre-pass (parallel.py:143); on a
//      Cholesky failure it falls back to the dense Cholesky of the pair Gram
//      computed from G (parallel.py:196-198);
//   2. diagonalises R by one-sided J-Jacobi sweeps until a sweep applies no
//      rotation (rotations.py:203-223), with the 2x2 trigonometric /
//      hyperbolic rotations of _kernels.py:53-98, accumulating W on chip;
//   3. writes W (for the block update) and the rotation counters.
//
// Inner pair order: a circle-method tournament (N/2 disjoint pairs per
// round, N-1 rounds per sweep) instead of the reference's sequential
// column-cyclic order (_kernels.py:41-52) -- the parallel order a CTA can
// execute; see DESIGN.md for the parity consequences.
//
// On-chip layout: R and W (N x N) are split by rows across the C CTAs of
// the cluster, each CTA holding an RPC-row slab of both in shared memory
// (column-major, padded stride).  A pair's dot product is a CTA-partial
// (warp-shuffle reduction over the TPP lanes that own the pair) combined
// across the cluster through distributed shared memory in a fixed tree, so
// every CTA derives bit-identical rotation parameters and applies them to
// its own rows.  One cluster barrier per round.
#include <cooperative_groups.h>

#include <cfloat>
#include <climits>

#include "common.cuh"
#include "kernels.h"

namespace cg = cooperative_groups;

namespace hjb {

constexpr double kEps = 2.220446049250313e-16;

template <typename T, int NMAX, int C, int NT>
struct PivCfg {
  static constexpr int RPC = NMAX / C;   // rows of R/W per CTA
  static constexpr int RS = RPC + 1;     // padded column stride (elements)
  static constexpr int P2 = NMAX / 2;    // pair slots per round
  static constexpr int TPP = NT / P2;    // threads per pair slot
  static constexpr int RPT = RPC / TPP;  // rows per thread
  static constexpr int OPT = RPC * NMAX / NT;  // Cholesky outputs per thread
  static constexpr int HC = 16;                // R_ij rows staged per chunk
  static_assert(TPP >= 1 && TPP <= 32 && (TPP & (TPP - 1)) == 0, "threads per pair");
  static_assert(RPT >= 1 && RPC % TPP == 0, "rows per thread");
  static_assert(OPT >= 1 && (RPC * NMAX) % NT == 0, "outputs per thread");
  static_assert(HC * NMAX <= NMAX * RS, "scratch fits in the W slab");
  // shared-memory carve-up (bytes, 16-aligned)
  static constexpr size_t OFF_R = 0;
  static constexpr size_t OFF_W = OFF_R + size_t(NMAX) * RS * sizeof(T);
  static constexpr size_t OFF_PART = OFF_W + size_t(NMAX) * RS * sizeof(T);
  static constexpr size_t OFF_ROW = OFF_PART + 2 * size_t(P2) * sizeof(T);
  static constexpr size_t OFF_NPART = OFF_ROW + 2 * size_t(NMAX) * sizeof(T);
  static constexpr size_t OFF_D = OFF_NPART + NMAX * sizeof(double);
  static constexpr size_t OFF_LAM = OFF_D + NMAX * sizeof(double);
  static constexpr size_t OFF_J = OFF_LAM + NMAX * sizeof(double);
  static constexpr size_t SMEM = OFF_J + NMAX * sizeof(int);
};

template <int C>
__device__ __forceinline__ void cluster_sync() {
  if constexpr (C > 1)
    cg::this_cluster().sync();
  else
    __syncthreads();
}

template <int C, typename P>
__device__ __forceinline__ P *remote(P *p, int rank) {
  if constexpr (C > 1)
    return cg::this_cluster().map_shared_rank(p, rank);
  else
    return p;
}

template <typename T>
struct RotParams {
  int code;  // 0 skip, 1 rotate, -1 indefinite pivot
  double cs, sn, t, eta, hyp;
  T phase;
};

__device__ __forceinline__ double absv(double a) { return fabs(a); }
__device__ __forceinline__ double absv(cplx a) { return hypot(a.x, a.y); }

// _kernels.py:53-81 for one pair (a = g_r^H g_s, dr/ds = cached Gram diagonal)
template <typename T>
__device__ __forceinline__ RotParams<T> rot_params(T a, double dr, double ds, bool same, double otol) {
  RotParams<T> p;
  p.code = 0;
  p.cs = 1.0; p.sn = 0.0; p.t = 0.0; p.eta = 0.0; p.hyp = 0.0;
  p.phase = S<T>::one();
  const double aa = absv(a);
  if (aa <= otol * sqrt(dr * ds)) return p;
  if (aa * aa >= dr * ds) { p.code = -1; return p; }
  const double eta = re(a) >= 0.0 ? aa : -aa;
  p.phase = divr(a, eta);
  double t, h;
  if (same) {
    p.hyp = -1.0;
    const double theta = (ds - dr) / (2.0 * eta);
    const double sg = theta >= 0.0 ? 1.0 : -1.0;
    t = sg / (fabs(theta) + sqrt(theta * theta + 1.0));
    h = sqrt(1.0 + t * t);
  } else {
    p.hyp = 1.0;
    const double theta = -(dr + ds) / (2.0 * eta);
    const double disc = theta * theta - 1.0;
    if (disc <= 0.0) { p.code = -1; return p; }
    const double sg = theta >= 0.0 ? 1.0 : -1.0;
    t = sg / (fabs(theta) + sqrt(disc));
    h = sqrt(1.0 - t * t);
  }
  p.cs = 1.0 / h;
  p.sn = p.cs * t;
  p.t = t;
  p.eta = eta;
  p.code = 1;
  return p;
}

// [x_r, x_s] <- [cs*(phase x_r) + hyp*sn*x_s, sn*(phase x_r) + cs*x_s]  (_kernels.py:82-92)
template <typename T>
__device__ __forceinline__ void rot_apply(T &xr, T &xs, const RotParams<T> &p) {
  const T f = mul(p.phase, xr);
  const double hs = p.hyp * p.sn;
  const T nr = add(scale(f, p.cs), scale(xs, hs));
  const T ns = add(scale(f, p.sn), scale(xs, p.cs));
  xr = nr;
  xs = ns;
}
template <>
__device__ __forceinline__ void rot_apply<double>(double &xr, double &xs, const RotParams<double> &p) {
  const double f = p.phase * xr;
  const double nr = p.cs * f + (p.hyp * p.sn) * xs;
  const double ns = p.sn * f + p.cs * xs;
  xr = nr;
  xs = ns;
}

template <typename T, int NMAX, int C, int NT>
__global__ void __launch_bounds__(NT, 1) pivot_kernel(PivotArgs a) {
  using Cfg = PivCfg<T, NMAX, C, NT>;
  constexpr int RPC = Cfg::RPC, RS = Cfg::RS, TPP = Cfg::TPP, RPT = Cfg::RPT, OPT = Cfg::OPT;
  constexpr int HC = Cfg::HC;
  extern __shared__ __align__(16) unsigned char smem[];
  T *Rs = reinterpret_cast<T *>(smem + Cfg::OFF_R);
  T *Ws = reinterpret_cast<T *>(smem + Cfg::OFF_W);
  T *part = reinterpret_cast<T *>(smem + Cfg::OFF_PART);
  T *rowbuf = reinterpret_cast<T *>(smem + Cfg::OFF_ROW);
  double *npart = reinterpret_cast<double *>(smem + Cfg::OFF_NPART);
  double *Dv = reinterpret_cast<double *>(smem + Cfg::OFF_D);
  double *lam = reinterpret_cast<double *>(smem + Cfg::OFF_LAM);
  int *Jv = reinterpret_cast<int *>(smem + Cfg::OFF_J);
  __shared__ int s_flag[2];
  __shared__ int s_cnt[2];
  __shared__ int s_big;
  __shared__ int s_fail;
  __shared__ unsigned long long s_maxt;

  int crank = 0;
  if constexpr (C > 1) crank = int(cg::this_cluster().block_rank());
  const int item_id = blockIdx.x / C;
  const Item it = a.items[item_id];
  const int tid = threadIdx.x;
  const bool dense = it.nj == 0;
  const int ni = it.ni, nj = it.nj, N = ni + nj;
  const int row0 = crank * RPC;
  const int bmax = a.bmax;
  T *A = reinterpret_cast<T *>(a.A) + int64_t(item_id) * bmax * bmax;
  const T *G = reinterpret_cast<const T *>(a.G);
  auto colptr = [&](int c) -> const T * {
    return G + int64_t(c < ni ? it.oi + c : it.oj + (c - ni)) * a.ldg;
  };

  for (int c = tid; c < NMAX; c += NT) {
    Jv[c] = c < ni ? a.signs[it.oi + c] : (c < N ? a.signs[it.oj + (c - ni)] : 1);
    lam[c] = (!dense && c < N) ? a.D[int64_t(item_id) * 2 * bmax + (c < ni ? c : bmax + (c - ni))] : 1.0;
  }
  for (int e = tid; e < NMAX * RS; e += NT) {
    Rs[e] = S<T>::zero();
    Ws[e] = S<T>::zero();
  }
  if (tid == 0) { s_fail = INT_MAX; s_maxt = 0ull; s_big = 0; s_cnt[0] = s_cnt[1] = 0; }
  __syncthreads();

  // ------------------------------------------------------------------ R
  int status = PV_OK;
  int fallback = 0;
  int k0 = 0;
  bool need_dense = dense;
  if (!dense) {
    int ok = 1;
    for (int c = tid; c < N; c += NT) ok &= (lam[c] > 0.0);
    ok = __syncthreads_and(ok);
    if (!ok) {
      need_dense = true;  // structured_cholesky raises (blocking.py:125-126)
      fallback = 1;
    } else {
      // rows g < ni: R_ii = sqrt(L_i), R_ij = A_ij / sqrt(L_i); R_ij also
      // written back over A for the Schur complement of the other CTAs
      for (int e = tid; e < RPC * (nj + 1); e += NT) {
        const int gl = e % RPC, l = e / RPC;
        const int g = row0 + gl;
        if (g >= ni) continue;
        const double rg = sqrt(lam[g]);
        if (l == nj) {
          Rs[gl + g * RS] = scale(S<T>::one(), rg);
        } else {
          const T v = divr(A[g + int64_t(l) * bmax], rg);
          Rs[gl + (ni + l) * RS] = v;
          A[g + int64_t(l) * bmax] = v;
        }
      }
      __threadfence();
      cluster_sync<C>();
      // rows g in [ni, N): S[k][l] = L_j[k] d_kl - sum_h conj(Rij[h][k]) Rij[h][l], l >= k
      T acc[OPT];
#pragma unroll
      for (int o = 0; o < OPT; ++o) acc[o] = S<T>::zero();
      T *scr = Ws;  // scratch: HC x NMAX staging of R_ij rows
      for (int h0 = 0; h0 < ni; h0 += HC) {
        const int hc = min(HC, ni - h0);
        for (int e = tid; e < HC * nj; e += NT) {
          const int h = e % HC, l = e / HC;
          scr[h * NMAX + l] = h < hc ? A[(h0 + h) + int64_t(l) * bmax] : S<T>::zero();
        }
        __syncthreads();
#pragma unroll
        for (int o = 0; o < OPT; ++o) {
          const int idx = tid + o * NT;
          const int gl = idx % RPC, l = idx / RPC;
          const int k = row0 + gl - ni;
          if (k < 0 || row0 + gl >= N || l < k || l >= nj) continue;
          T s = acc[o];
          for (int h = 0; h < hc; ++h) s = cfma(scr[h * NMAX + k], scr[h * NMAX + l], s);
          acc[o] = s;
        }
        __syncthreads();
      }
#pragma unroll
      for (int o = 0; o < OPT; ++o) {
        const int idx = tid + o * NT;
        const int gl = idx % RPC, l = idx / RPC;
        const int k = row0 + gl - ni;
        if (k < 0 || row0 + gl >= N || l < k || l >= nj) continue;
        T v = sub(l == k ? scale(S<T>::one(), lam[ni + k]) : S<T>::zero(), acc[o]);
        if (l == k) v = scale(S<T>::one(), re(v));  // exactly Hermitian diagonal
        Rs[gl + (ni + l) * RS] = v;
      }
      __syncthreads();
      k0 = ni;
    }
  } else {
    // pre-pass: R = chol(herm(B^H B)) (parallel.py:143, core.py:54-55)
    for (int e = tid; e < RPC * NMAX; e += NT) {
      const int gl = e % RPC, l = e / RPC;
      const int g = row0 + gl;
      if (g >= N || l < g || l >= N) continue;
      T v;
      if (l == g)
        v = scale(S<T>::one(), re(A[g + int64_t(g) * bmax]));
      else
        v = scale(add(A[g + int64_t(l) * bmax], conjv(A[l + int64_t(g) * bmax])), 0.5);
      Rs[gl + l * RS] = v;
    }
    __syncthreads();
    need_dense = false;
    k0 = 0;
  }

  // distributed right-looking Cholesky of rows [k0, N) of the slab, upper
  auto cholesky = [&](int kstart) -> bool {
    for (int k = kstart; k < N; ++k) {
      const int owner = k / RPC, lk = k % RPC, buf = k & 1;
      if (crank == owner) {
        const double d = re(Rs[lk + k * RS]);
        const bool ok = finite_pos(d);
        const double rkk = ok ? sqrt(d) : 1.0;
        __syncthreads();
        for (int l = k + tid; l < N; l += NT) {
          const T v = (l == k) ? scale(S<T>::one(), rkk) : divr(Rs[lk + l * RS], rkk);
          Rs[lk + l * RS] = v;
#pragma unroll 1
          for (int q = 0; q < C; ++q) remote<C>(rowbuf, q)[buf * NMAX + l] = v;
        }
        if (tid == 0) {
#pragma unroll 1
          for (int q = 0; q < C; ++q) remote<C>(s_flag, q)[buf] = ok ? 1 : 0;
        }
      }
      cluster_sync<C>();
      if (!s_flag[buf]) return false;
      const T *row = rowbuf + buf * NMAX;
      for (int e = tid; e < RPC * NMAX; e += NT) {
        const int gl = e % RPC, l = e / RPC;
        const int g = row0 + gl;
        if (g <= k || g >= N || l < g || l >= N) continue;
        Rs[gl + l * RS] = cfms(row[g], row[l], Rs[gl + l * RS]);
      }
      __syncthreads();
    }
    return true;
  };

  if (!need_dense) {
    if (!cholesky(k0)) {
      if (dense) {
        status = PV_CHOL;
      } else {
        need_dense = true;
        fallback = 1;
      }
    }
  }
  if (need_dense && status == PV_OK) {
    // dense fallback: chol(gram([G_i G_j])) from G itself (parallel.py:196-198)
    for (int e = tid; e < NMAX * RS; e += NT) Rs[e] = S<T>::zero();
    __syncthreads();
    for (int e = tid; e < RPC * NMAX; e += NT) {
      const int gl = e % RPC, l = e / RPC;
      const int g = row0 + gl;
      if (g >= N || l < g || l >= N) continue;
      const T *xg = colptr(g);
      const T *xl = colptr(l);
      T s = S<T>::zero();
      for (int64_t r = 0; r < a.m; ++r) s = cfma(xg[r], xl[r], s);
      if (l == g) s = scale(S<T>::one(), re(s));
      Rs[gl + l * RS] = s;
    }
    __syncthreads();
    if (!cholesky(0)) status = PV_CHOL;
  }

  // ------------------------------------------------------------------ Jacobi
  for (int e = tid; e < NMAX * RS; e += NT) Ws[e] = S<T>::zero();
  __syncthreads();
  for (int gl = tid; gl < RPC; gl += NT) {
    const int g = row0 + gl;
    if (g < N) Ws[gl + g * RS] = S<T>::one();
  }
  const double otol = a.orth_tol > 0.0 ? a.orth_tol : sqrt(double(N)) * kEps;
  const double qtol = a.quad_tol > 0.0 ? a.quad_tol : double(N) * kEps;
  const int ne = N + (N & 1);
  const int rounds = ne - 1;
  const int slot = tid / TPP, lane_in = tid % TPP;
  long long nrot_total = 0;
  int sweeps = 0;
  int gr = 0;  // global round counter (partial-buffer parity)
  __syncthreads();

  if (status == PV_OK) {
    for (int sw = 0; sw < a.max_sweeps; ++sw) {
      ++sweeps;
      // D = colnorms^2(R) (rotations.py:217), reduced over the cluster
      for (int c = tid; c < NMAX; c += NT) {
        double s = 0.0;
        for (int gl = 0; gl < RPC; ++gl) s += abs2(Rs[gl + c * RS]);
        npart[c] = s;
      }
      cluster_sync<C>();
      for (int c = tid; c < NMAX; c += NT) {
        double s = 0.0;
#pragma unroll 1
        for (int q = 0; q < C; ++q) s += remote<C>(npart, q)[c];
        Dv[c] = s;
      }
      if (tid == 0) s_cnt[(sw + 1) & 1] = 0;
      __syncthreads();

      for (int rnd = 0; rnd < rounds; ++rnd, ++gr) {
        int pa, pb;
        if (slot == 0) {
          pa = ne - 1;
          pb = rnd;
        } else {
          pa = (rnd + slot) % (ne - 1);
          pb = (rnd - slot + ne - 1) % (ne - 1);
        }
        const int r = min(pa, pb), s = max(pa, pb);
        const bool active = (slot < ne / 2) && (s < N);
        const int rr = active ? r : 0, ss = active ? s : 1;
        T xr[RPT], xs[RPT];
        T dot = S<T>::zero();
#pragma unroll
        for (int u = 0; u < RPT; ++u) {
          const int row = lane_in + u * TPP;
          xr[u] = Rs[rr * RS + row];
          xs[u] = Rs[ss * RS + row];
          dot = cfma(xr[u], xs[u], dot);
        }
#pragma unroll
        for (int o = 1; o < TPP; o <<= 1) dot = add(dot, shfl_xor(dot, o));
        if constexpr (C > 1) {
          const int buf = gr & 1;
          if (lane_in == 0) part[buf * Cfg::P2 + slot] = dot;
          cluster_sync<C>();
          T acc = S<T>::zero();
#pragma unroll 1
          for (int q = lane_in; q < C; q += TPP) acc = add(acc, remote<C>(part, q)[buf * Cfg::P2 + slot]);
#pragma unroll
          for (int o = 1; o < TPP; o <<= 1) acc = add(acc, shfl_xor(acc, o));
          dot = acc;
        }
        if (active) {
          const double dr = Dv[rr], ds = Dv[ss];
          const RotParams<T> p = rot_params<T>(dot, dr, ds, Jv[rr] == Jv[ss], otol);
          if (p.code == 1) {
#pragma unroll
            for (int u = 0; u < RPT; ++u) {
              const int row = lane_in + u * TPP;
              rot_apply<T>(xr[u], xs[u], p);
              Rs[rr * RS + row] = xr[u];
              Rs[ss * RS + row] = xs[u];
              T wr = Ws[rr * RS + row], ws = Ws[ss * RS + row];
              rot_apply<T>(wr, ws, p);
              Ws[rr * RS + row] = wr;
              Ws[ss * RS + row] = ws;
            }
            if (lane_in == 0) {
              Dv[rr] = dr + p.hyp * p.t * p.eta;
              Dv[ss] = ds + p.t * p.eta;
              atomicAdd(&s_cnt[sw & 1], 1);
              const double at = fabs(p.t);
              if (at > qtol) atomicAdd(&s_big, 1);
              atomicMax(&s_maxt, static_cast<unsigned long long>(__double_as_longlong(at)));
            }
          } else if (p.code < 0 && lane_in == 0) {
            atomicMin(&s_fail, r * 4096 + s);
          }
        }
        __syncthreads();
        if (s_fail != INT_MAX) break;
      }
      if (s_fail != INT_MAX) {
        status = PV_INDEFINITE;
        break;
      }
      const int cnt = s_cnt[sw & 1];
      nrot_total += cnt;
      if (cnt == 0) break;
    }
  }

  // ------------------------------------------------------------------ out
  const int nmax = a.nmax;
  T *Wout = reinterpret_cast<T *>(a.W) + int64_t(item_id) * nmax * nmax;
  for (int e = tid; e < RPC * N; e += NT) {
    const int gl = e % RPC, c = e / RPC;
    const int g = row0 + gl;
    if (g < N) Wout[g + int64_t(c) * nmax] = Ws[gl + c * RS];
  }
  if (a.Rout) {
    T *Rout = reinterpret_cast<T *>(a.Rout) + int64_t(item_id) * nmax * nmax;
    for (int e = tid; e < RPC * N; e += NT) {
      const int gl = e % RPC, c = e / RPC;
      const int g = row0 + gl;
      if (g < N) Rout[g + int64_t(c) * nmax] = Rs[gl + c * RS];
    }
  }
  if (crank == 0 && tid == 0) {
    int64_t *st = a.stats + int64_t(item_id) * ST_N;
    st[ST_NROT] = nrot_total;
    st[ST_NBIG] = s_big;
    st[ST_MAXT] = static_cast<int64_t>(s_maxt);
    st[ST_SWEEPS] = sweeps;
    st[ST_STATUS] = status;
    st[ST_FR] = status == PV_INDEFINITE ? s_fail / 4096 : -1;
    st[ST_FS] = status == PV_INDEFINITE ? s_fail % 4096 : -1;
    st[ST_FALLBACK] = fallback;
  }
  // keep every CTA's shared memory alive until remote readers are done
  if constexpr (C > 1) cg::this_cluster().sync();
}

template <typename T, int NMAX, int C, int NT>
static cudaError_t launch_pivot_t(const PivotArgs &a, cudaStream_t st) {
  using Cfg = PivCfg<T, NMAX, C, NT>;
  auto k = pivot_kernel<T, NMAX, C, NT>;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(Cfg::SMEM));
    if (e != cudaSuccess) return e;
    if (C > 8) {
      e = cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      if (e != cudaSuccess) return e;
    }
    attr = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(a.count * C);
  cfg.blockDim = dim3(NT);
  cfg.dynamicSmemBytes = Cfg::SMEM;
  cfg.stream = st;
  cudaLaunchAttribute attrs[1];
  attrs[0].id = cudaLaunchAttributeClusterDimension;
  attrs[0].val.clusterDim.x = C;
  attrs[0].val.clusterDim.y = 1;
  attrs[0].val.clusterDim.z = 1;
  cfg.attrs = attrs;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k, a);
}

int pivot_nmax(int bmax) {
  const int n = 2 * bmax;
  if (n <= 32) return 32;
  if (n <= 64) return 64;
  if (n <= 128) return 128;
  if (n <= 256) return 256;
  return -1;
}

int pivot_default_cluster(bool cx, int nmax) {
  // R and W slabs <= ~140 KB of shared memory per CTA
  const size_t bytes = 2ull * nmax * nmax * (cx ? 16 : 8);
  int c = 1;
  while (bytes / c > 140 * 1024) c *= 2;
  return c;
}

template <typename T, int NMAX, int C>
static cudaError_t launch_if_valid(const PivotArgs &a, cudaStream_t st) {
  if constexpr (NMAX / C >= 16 && NMAX / C >= 256 / (NMAX / 2) ) {
    if constexpr (PivCfg<T, NMAX, C, 256>::SMEM <= 227 * 1024) return launch_pivot_t<T, NMAX, C, 256>(a, st);
  }
  return cudaErrorInvalidConfiguration;
}

template <typename T, int NMAX>
static cudaError_t dispatch_c(const PivotArgs &a, int c, cudaStream_t st) {
  switch (c) {
    case 1: return launch_if_valid<T, NMAX, 1>(a, st);
    case 2: return launch_if_valid<T, NMAX, 2>(a, st);
    case 4: return launch_if_valid<T, NMAX, 4>(a, st);
    case 8: return launch_if_valid<T, NMAX, 8>(a, st);
    case 16: return launch_if_valid<T, NMAX, 16>(a, st);
  }
  return cudaErrorInvalidConfiguration;
}

cudaError_t launch_pivot(bool cx, const PivotArgs &a, int cluster, cudaStream_t st, int *cluster_used) {
  const int c = cluster > 0 ? cluster : pivot_default_cluster(cx, a.nmax);
  if (cluster_used) *cluster_used = c;
  if (cx) {
    switch (a.nmax) {
      case 32: return dispatch_c<cplx, 32>(a, c, st);
      case 64: return dispatch_c<cplx, 64>(a, c, st);
      case 128: return dispatch_c<cplx, 128>(a, c, st);
      case 256: return dispatch_c<cplx, 256>(a, c, st);
    }
  } else {
    switch (a.nmax) {
      case 32: return dispatch_c<double, 32>(a, c, st);
      case 64: return dispatch_c<double, 64>(a, c, st);
      case 128: return dispatch_c<double, 128>(a, c, st);
      case 256: return dispatch_c<double, 256>(a, c, st);
    }
  }
  return cudaErrorInvalidValue;
}

}  // namespace hjb
