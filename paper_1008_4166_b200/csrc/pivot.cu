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

#include <algorithm>
#include <cfloat>
#include <climits>

#include "common.cuh"
#include "kernels.h"

namespace cg = cooperative_groups;

// per-round phase clocks (tools/pivot_bench.py); off in production builds
#ifndef HJB_ROUND_PROFILE
#define HJB_ROUND_PROFILE 0
#endif
#if HJB_ROUND_PROFILE
#define RCLK() clock64()
#else
#define RCLK() 0LL
#endif

namespace hjb {

constexpr double kEps = 2.220446049250313e-16;
static int g_tune_threads = 0, g_tune_cluster = 0;  // hjb_tune overrides (0 = auto)

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
  static constexpr int NWARP = NT / 32;
  static constexpr int SPW = 32 / TPP;                       // pair slots per warp
  static constexpr int XBUF = 2 * NWARP * RPC;               // [parity][warp][row]
  static constexpr int SCR0 = HC * NMAX > XBUF ? HC * NMAX : XBUF;
  static constexpr int SCR = SCR0 > NMAX * RS ? SCR0 : NMAX * RS;   // also the R_final / W slab
  // shared-memory carve-up (bytes, 16-aligned)
  static constexpr size_t OFF_R = 0;
  static constexpr size_t OFF_W = OFF_R + size_t(NMAX) * RS * sizeof(T);  // scratch
  static constexpr size_t OFF_PART = OFF_W + size_t(SCR) * sizeof(T);
  static constexpr size_t PART = (2 * C * P2 > RPC) ? 2 * C * P2 : RPC;  // also W-block scratch (column chunks)
  static constexpr size_t OFF_ROW = OFF_PART + PART * sizeof(T);
  static constexpr size_t OFF_NPART = OFF_ROW + 2 * size_t(NMAX) * sizeof(T);
  static constexpr size_t OFF_D = OFF_NPART + NMAX * sizeof(double);
  static constexpr size_t OFF_LAM = OFF_D + NMAX * sizeof(double);
  static constexpr size_t OFF_J = OFF_LAM + NMAX * sizeof(double);
  static constexpr size_t SMEM = OFF_J + NMAX * sizeof(int);
};

// cluster-scope barrier with release/acquire semantics only (cg's sync()
// adds a gpu-scope MEMBAR that the DSMEM exchanges here do not need)
template <int C>
__device__ __forceinline__ void cluster_sync() {
  if constexpr (C > 1) {
    asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
    asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
  } else {
    __syncthreads();
  }
}

template <int C, typename P>
__device__ __forceinline__ P *remote(P *p, int rank) {
  if constexpr (C > 1)
    return cg::this_cluster().map_shared_rank(p, rank);
  else
    return p;
}

// ---- cluster partial-dot exchange: st.async into peer smem + mbarrier ----
__device__ __forceinline__ void mbar_init(uint64_t *bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_arm(uint64_t *bar, unsigned tx) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(tx)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "HJB_WAIT_%=:\n"
      " mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra HJB_WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ uint32_t mapa_u32(uint32_t addr, int rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
__device__ __forceinline__ void st_async(uint32_t raddr, double v, uint32_t rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];\n" ::"r"(raddr),
               "l"(__double_as_longlong(v)), "r"(rbar)
               : "memory");
}
__device__ __forceinline__ void st_async(uint32_t raddr, cplx v, uint32_t rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.b64 [%0], {%1, %2}, [%3];\n" ::"r"(raddr),
               "l"(__double_as_longlong(v.x)), "l"(__double_as_longlong(v.y)), "r"(rbar)
               : "memory");
}

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
  const bool skip = q <= otol2 * dd;                     // _kernels.py:57
  const bool bad = q >= dd || (!same && disc <= 0.0);   // _kernels.py:59-60, 73-74
  p.code = skip ? 0 : (bad ? -1 : 1);
  p.hyp = same ? -1.0 : 1.0;
  const double cs = den * r, sn = num * r;
  const T ph = phase_mul(a, sa * ri);
  p.cs = cs;
  p.hs = p.hyp * sn;
  p.cp = phase_mul(ph, cs);
  p.sp = phase_mul(ph, sn);
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
  __shared__ uint64_t s_mbar[2];
  __shared__ int cib[NMAX / 2], cjb[NMAX / 2], k_on[NMAX / 2];
  __shared__ double k_cs[NMAX / 2], k_hs[NMAX / 2];
  __shared__ T k_cp[NMAX / 2], k_sp[NMAX / 2];

  int crank = 0;
  if constexpr (C > 1) crank = int(cg::this_cluster().block_rank());
  const long long t_start = clock64();
  long long t_chol = 0, t_jac = 0, t_rij = 0, t_s = 0;
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
  for (int e = tid; e < NMAX * RS; e += NT) Rs[e] = S<T>::zero();
  if (tid == 0) { s_fail = INT_MAX; s_maxt = 0ull; s_big = 0; s_cnt[0] = s_cnt[1] = 0; s_flag[0] = 1; }
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
      t_rij = clock64();
      // rows g in [ni, N): S[k][l] = L_j[k] d_kl - sum_h conj(Rij[h][k]) Rij[h][l], l >= k
      T acc[OPT];
#pragma unroll
      for (int o = 0; o < OPT; ++o) acc[o] = S<T>::zero();
      T *scr = Ws;  // scratch: HC x NMAX staging of R_ij rows
      for (int h0 = 0; h0 < ni; h0 += HC) {
        const int hc = min(HC, ni - h0);
        for (int e = tid; e < HC * nj; e += NT) {
          const int h = e % HC, l = e / HC;
          scr[h * NMAX + l] = h < hc ? __ldcg(A + (h0 + h) + int64_t(l) * bmax) : S<T>::zero();
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
      t_s = clock64();
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
  // distributed right-looking Cholesky of rows [kstart, N) of the slab,
  // blocked by CTA: the owner of a row block factors it locally (CTA
  // barriers only), the cluster synchronises once per block, and every later
  // CTA copies the finished block (DSMEM) and applies the rank-RPC update
  auto cholesky = [&](int kstart) -> bool {
    for (int K = 0; K < C; ++K) {
      const int kb0 = max(kstart, K * RPC), kb1 = min(N, (K + 1) * RPC);
      if (kb0 >= kb1) continue;
      if (crank == K) {
        for (int k = kb0; k < kb1; ++k) {
          const int lk = k - row0;
          const double d = re(Rs[lk + k * RS]);
          const bool ok = finite_pos(d);
          __syncthreads();
          if (!ok) {
            if (tid == 0) s_flag[0] = 0;
            break;
          }
          const double rkk = sqrt(d);
          for (int l = k + tid; l < N; l += NT)
            Rs[lk + l * RS] = (l == k) ? scale(S<T>::one(), rkk) : divr(Rs[lk + l * RS], rkk);
          __syncthreads();
          for (int e = tid; e < RPC * NMAX; e += NT) {
            const int gl = e % RPC, l = e / RPC;
            const int g = row0 + gl;
            if (g <= k || g >= kb1 || l < g || l >= N) continue;
            Rs[gl + l * RS] = cfms(Rs[lk + g * RS], Rs[lk + l * RS], Rs[gl + l * RS]);
          }
          __syncthreads();
        }
      }
      cluster_sync<C>();
      if (!remote<C>(s_flag, K)[0]) return false;
      if (crank > K) {
        const T *RK = remote<C>(Rs, K);
        T *Bl = Ws;  // scratch: (kb1-kb0) x NMAX rows of the finished block
        const int nb = kb1 - kb0;
        for (int e = tid; e < nb * NMAX; e += NT) {
          const int kk = e % nb, l = e / nb;
          Bl[kk * NMAX + l] = (l >= kb0 && l < N) ? RK[(kb0 + kk - K * RPC) + l * RS] : S<T>::zero();
        }
        __syncthreads();
        for (int e = tid; e < RPC * NMAX; e += NT) {
          const int gl = e % RPC, l = e / RPC;
          const int g = row0 + gl;
          if (g >= N || l < g || l >= N) continue;
          T acc = Rs[gl + l * RS];
          for (int kk = 0; kk < nb; ++kk) acc = cfms(Bl[kk * NMAX + g], Bl[kk * NMAX + l], acc);
          Rs[gl + l * RS] = acc;
        }
        __syncthreads();
      }
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
    cluster_sync<C>();  // every CTA is done reading the failed attempt's flag
    if (tid == 0) s_flag[0] = 1;
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

  t_chol = clock64();
  // ------------------------------------------------------------------ Jacobi
  // Register-resident columns.  Pair slot q (TPP lanes) holds the RPC-row
  // slab of two columns of R in registers; lane l owns rows l, l+TPP, ...
  // After each round the slot keeps one column and passes the other to its
  // ring neighbour, exactly as the reference's modulus stepper passes block
  // columns between workers (strategies.py:58-92, applied with nbl = N): a
  // warp shuffle inside a warp, shared memory across warps.  W is not
  // accumulated rotation by rotation: the initial factor R0 stays in shared
  // memory and W = R0^-1 R_final is formed once at the end.
  const double otol = a.orth_tol > 0.0 ? a.orth_tol : sqrt(double(N)) * kEps;
  const double otol2 = otol * otol;
  const double qtol = a.quad_tol > 0.0 ? a.quad_tol : double(N) * kEps;
  const int ne = N + (N & 1);
  const int pr = ne / 2;  // ring slots in use
  const int slot = tid / TPP, lane_in = tid % TPP;
  constexpr int SPW = Cfg::SPW;
  const bool in_ring = slot < pr;
  const int wslot = slot % SPW, warp = slot / SPW;
  int ip = slot + 1, jp = ne - slot, ib = ip, jb = jp;  // strategies.py:58-66
  long long nrot_total = 0;
  int sweeps = 0;
  int gr = 0;  // global round counter (buffer parities)
  int my_big = 0, my_cnt = 0;
  double my_maxt = 0.0;
  long long ph[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  int pd_on = 0, pd_ci = 0, pd_cj = 0;
  double pd_dr = 0, pd_ds = 0, pd_num = 0, pd_den = 1, pd_eta = 0, pd_hyp = 0;
  auto finish_d = [&]() {
    const double t = pd_num / pd_den;
    Dv[pd_ci] = pd_dr + pd_hyp * t * pd_eta;
    Dv[pd_cj] = pd_ds + t * pd_eta;
    ++my_cnt;
    const double at = fabs(t);
    my_big += at > qtol;
    my_maxt = fmax(my_maxt, at);
    pd_on = 0;
  };
  T *xbuf = Ws;
  constexpr unsigned TX = (C - 1) * Cfg::P2 * sizeof(T);  // bytes pushed into each CTA per round
  if constexpr (C > 1) {
    if (tid == 0) {
      for (int b = 0; b < 2; ++b) mbar_init(&s_mbar[b], 1);
      fence_mbar_init();
      for (int b = 0; b < 2; ++b) mbar_arm(&s_mbar[b], TX);
    }
  }
  if (in_ring && lane_in == 0) {
    cib[slot] = ib - 1;
    cjb[slot] = jb - 1;
  }
  T X[RPT], Y[RPT];
#pragma unroll
  for (int u = 0; u < RPT; ++u) {
    const int row = lane_in + u * TPP;
    const int ci = in_ring ? ib - 1 : 0, cj = in_ring ? jb - 1 : 1;
    X[u] = Rs[ci * RS + row];
    Y[u] = Rs[cj * RS + row];
  }
  cluster_sync<C>();

  if (status == PV_OK) {
    for (int sw = 0; sw < a.max_sweeps; ++sw) {
      ++sweeps;
      const bool odd = (sw & 1) == 0;  // reference sweeps count from 1; odd send to q-1
      // D = colnorms^2(R) (rotations.py:217), from the registers, reduced over the cluster
      {
        double nx0 = 0.0, nx1 = 0.0, ny0 = 0.0, ny1 = 0.0;
#pragma unroll
        for (int u = 0; u < RPT; ++u) {
          if (u & 1) { nx1 += abs2(X[u]); ny1 += abs2(Y[u]); }
          else { nx0 += abs2(X[u]); ny0 += abs2(Y[u]); }
        }
        double nx = nx0 + nx1, ny = ny0 + ny1;
#pragma unroll
        for (int o = 1; o < TPP; o <<= 1) {
          nx += __shfl_xor_sync(0xffffffffu, nx, o);
          ny += __shfl_xor_sync(0xffffffffu, ny, o);
        }
        if (in_ring && lane_in == 0) {
          npart[ib - 1] = nx;
          npart[jb - 1] = ny;
        }
        cluster_sync<C>();
        if (in_ring && lane_in < 2) {
          const int col = lane_in == 0 ? ib - 1 : jb - 1;
          double sacc = 0.0;
#pragma unroll 1
          for (int q = 0; q < C; ++q) sacc += remote<C>(npart, q)[col];
          Dv[col] = sacc;
        }
      }
      if (tid == 0) s_cnt[(sw + 1) & 1] = 0;
      __syncthreads();

      for (int rnd = 0; rnd < ne; ++rnd, ++gr) {
        const long long c0 = RCLK();
        if (pd_on) finish_d();
        // (1) slab phase: CTA-partial of g_i^H g_j for this slot's pair
        T d0 = S<T>::zero(), d1 = S<T>::zero();
#pragma unroll
        for (int u = 0; u < RPT; ++u) {
          if (u & 1)
            d1 = cfma(X[u], Y[u], d1);
          else
            d0 = cfma(X[u], Y[u], d0);
        }
        T dot = add(d0, d1);
#pragma unroll
        for (int o = 1; o < TPP; o <<= 1) dot = add(dot, shfl_xor(dot, o));
        const int buf = gr & 1;
        {
          T *mine = part + (buf * C + crank) * Cfg::P2 + slot;
          if constexpr (C > 1) {
            const uint32_t la = smem_u32(mine), lb = smem_u32(&s_mbar[buf]);
#pragma unroll 1
            for (int q = lane_in; q < C; q += TPP) {
              if (q == crank)
                *mine = dot;
              else
                st_async(mapa_u32(la, q), dot, mapa_u32(lb, q));
            }
          } else {
            if (lane_in == 0) *mine = dot;
          }
        }
        const long long c1 = RCLK();
        long long c2 = c1, c3 = c1, c4 = c1;
        __syncthreads();
        // (2) pair phase: one thread per pair sums the cluster partials in
        // fixed rank order (bit-identical in every CTA), derives the rotation
        // once and publishes its coefficients
        if (tid < pr) {
          const int q = tid;
          const int ci = cib[q], cj = cjb[q];
          if constexpr (C > 1) mbar_wait(&s_mbar[buf], (gr >> 1) & 1);
          c2 = RCLK();
          T acc = part[(buf * C) * Cfg::P2 + q];
#pragma unroll 1
          for (int r = 1; r < C; ++r) acc = add(acc, part[(buf * C + r) * Cfg::P2 + q]);
          c3 = RCLK();
          int on = 0;
          if (ci < N && cj < N) {
            const double dr = Dv[ci], ds = Dv[cj];
            const RotCoef<T> p = rot_coef<T>(acc, dr, ds, Jv[ci] == Jv[cj], otol2);
            on = p.code == 1;
            k_cs[q] = p.cs;
            k_hs[q] = p.hs;
            k_cp[q] = p.cp;
            k_sp[q] = p.sp;
            if (p.code < 0) atomicMin(&s_fail, ci * 4096 + cj);
            // the D update (_kernels.py:80-81) is finished at the start of
            // the next round, off the critical path
            pd_on = on;
            pd_ci = ci;
            pd_cj = cj;
            pd_dr = dr;
            pd_ds = ds;
            pd_num = p.num;
            pd_den = p.den;
            pd_eta = p.eta;
            pd_hyp = p.hyp;
          }
          k_on[q] = on;
          c4 = RCLK();
        }
        __syncthreads();
        if constexpr (C > 1) {
          // this round's buffer is consumed: re-arm it for round gr+2 before
          // the end-of-round barrier, i.e. before this CTA pushes round gr+1
          // (no peer can push round gr+2 into it earlier)
          if (tid == NT - 1) mbar_arm(&s_mbar[buf], TX);
        }
        const long long c5 = RCLK();
        // (3) slab phase: apply, then the ring step
        if (in_ring && k_on[slot]) {
          RotCoef<T> p;
          p.cs = k_cs[slot];
          p.hs = k_hs[slot];
          p.cp = k_cp[slot];
          p.sp = k_sp[slot];
#pragma unroll
          for (int u = 0; u < RPT; ++u) rot_fold<T>(X[u], Y[u], p);
        }
        // ---- ring step: strategies.py:75-92 (nbl = ne) ----
        const bool send_i = ip + jp > ne;
        if (send_i) {
          ++ip;
          if (ip == jp) {
            ip -= pr;
            jp = ip;
          }
          ib = ip;
        } else {
          ++jp;
          jb = jp;
        }
        // odd sweeps: receive from slot+1, send to slot-1 (strategies.py:69-72)
        const int par = gr & 1;
        const bool via_smem = odd ? (wslot == SPW - 1 || slot == pr - 1) : (wslot == 0 || slot == 0);
        const bool writer = in_ring && (odd ? (wslot == 0) : (wslot == SPW - 1 || slot == pr - 1));
        const int src = odd ? (slot + 1 == pr ? 0 : slot + 1) : (slot == 0 ? pr - 1 : slot - 1);
        T *xw = xbuf + (size_t(par) * Cfg::NWARP + warp) * RPC;
        const T *xr = xbuf + (size_t(par) * Cfg::NWARP + src / SPW) * RPC;
        const int lane = threadIdx.x & 31;
        const int src_lane = odd ? min(lane + TPP, 31) : max(lane - TPP, 0);
#pragma unroll
        for (int u = 0; u < RPT; ++u) {
          const T v = send_i ? X[u] : Y[u];
          if (writer) xw[lane_in + u * TPP] = v;
          const T nv = shfl_idx(v, src_lane);
          if (send_i)
            X[u] = nv;
          else
            Y[u] = nv;
        }
        if (in_ring && lane_in == 0) {
          cib[slot] = ib - 1;
          cjb[slot] = jb - 1;
        }
        const long long c6 = RCLK();
        __syncthreads();
        const long long c7 = RCLK();
        if (in_ring && via_smem) {
#pragma unroll
          for (int u = 0; u < RPT; ++u) {
            const T nv = xr[lane_in + u * TPP];
            if (send_i)
              X[u] = nv;
            else
              Y[u] = nv;
          }
        }
        const long long c8 = RCLK();
        if (HJB_ROUND_PROFILE && a.prof) {
          ph[0] += c1 - c0; ph[1] += c2 - c1; ph[2] += c3 - c2; ph[3] += c4 - c3;
          ph[4] += c5 - c4; ph[5] += c6 - c5; ph[6] += c7 - c6; ph[7] += c8 - c7;
        }
        if (s_fail != INT_MAX) break;
      }
      if (pd_on) finish_d();
      if (my_cnt) atomicAdd(&s_cnt[sw & 1], my_cnt);
      nrot_total += 0;
      my_cnt = 0;
      __syncthreads();
      if (s_fail != INT_MAX) {
        status = PV_INDEFINITE;
        break;
      }
      const int cnt = s_cnt[sw & 1];
      nrot_total += cnt;
      if (cnt == 0) break;
    }
  }
  t_jac = clock64();

  // ------------------------------------------------------------------ W = R0^-1 R
  // R_final columns -> shared slab Fs (by column); back substitution by row
  // blocks from the last CTA of the cluster to the first.
  T *Fs = Ws;  // RPC x NMAX slab (scratch region is large enough)
  __syncthreads();
#pragma unroll
  for (int u = 0; u < RPT; ++u) {
    if (!in_ring) break;
    const int row = lane_in + u * TPP;
    Fs[(ib - 1) * RS + row] = X[u];
    Fs[(jb - 1) * RS + row] = Y[u];
  }
  if (my_big) atomicAdd(&s_big, my_big);
  if (my_maxt > 0.0) atomicMax(&s_maxt, static_cast<unsigned long long>(__double_as_longlong(my_maxt)));
  __syncthreads();
  for (int k = C - 1; k >= 0; --k) {
    if (crank == k) {
      // local rows, last to first; columns of W are independent, so each
      // thread back-substitutes whole columns (no barrier inside the block)
      for (int gl = tid; gl < RPC; gl += NT) {
        const int g = row0 + gl;
        npart[gl] = g < N ? 1.0 / re(Rs[g * RS + gl]) : 0.0;  // reciprocal diagonal
      }
      __syncthreads();
      for (int c = tid; c < N; c += NT) {
        T col[RPC];
#pragma unroll
        for (int gl = 0; gl < RPC; ++gl) col[gl] = Fs[c * RS + gl];
#pragma unroll
        for (int gl = RPC - 1; gl >= 0; --gl) {
          if (row0 + gl >= N) continue;
          const T w = scale(col[gl], npart[gl]);
          col[gl] = w;
#pragma unroll
          for (int gl2 = 0; gl2 < gl; ++gl2) col[gl2] = sub(col[gl2], mul(Rs[(row0 + gl) * RS + gl2], w));
        }
#pragma unroll
        for (int gl = 0; gl < RPC; ++gl) Fs[c * RS + gl] = col[gl];
      }
      __syncthreads();
    }
    cluster_sync<C>();
    if (crank < k) {
      // T[rows of this CTA] -= R0[these rows, block k] W[block k, :]; the
      // block of W is first copied from CTA k (DSMEM) into local scratch
      const T *Wk = remote<C>(Fs, k);
      T *Wl = part;  // scratch: PART elements, processed in column chunks
      constexpr int CW = int(Cfg::PART) / RPC;
      const int rk0 = k * RPC;
      const int jn = min(RPC, N - rk0);
      for (int c0 = 0; c0 < N; c0 += CW) {
        const int cw = min(CW, N - c0);
        for (int e = tid; e < RPC * cw; e += NT) {
          const int j = e % RPC, cc = e / RPC;
          Wl[j * CW + cc] = Wk[(c0 + cc) * RS + j];
        }
        __syncthreads();
        for (int e = tid; e < RPC * cw; e += NT) {
          const int gl = e % RPC, cc = e / RPC;
          if (row0 + gl >= N) continue;
          T acc = Fs[(c0 + cc) * RS + gl];
          for (int j = 0; j < jn; ++j) acc = sub(acc, mul(Rs[(rk0 + j) * RS + gl], Wl[j * CW + cc]));
          Fs[(c0 + cc) * RS + gl] = acc;
        }
        __syncthreads();
      }
    }
    cluster_sync<C>();
  }

  // ------------------------------------------------------------------ out
  {
    const int nmax = a.nmax;
    T *Wout = reinterpret_cast<T *>(a.W) + int64_t(item_id) * nmax * nmax;
    T *Rout = a.Rout ? reinterpret_cast<T *>(a.Rout) + int64_t(item_id) * nmax * nmax : nullptr;
    for (int e = tid; e < RPC * N; e += NT) {
      const int gl = e % RPC, c = e / RPC;
      const int g = row0 + gl;
      if (g < N) Wout[g + int64_t(c) * nmax] = Fs[c * RS + gl];
    }
    if (Rout) {
      // R_final = R0 W (rows of this CTA), recomputed for the optional output
      for (int e = tid; e < RPC * N; e += NT) {
        const int gl = e % RPC, c = e / RPC;
        const int g = row0 + gl;
        if (g >= N) continue;
        T acc = S<T>::zero();
        for (int j = g; j < N; ++j) {
          const T *Wj = remote<C>(Fs, j / RPC);
          acc = add(acc, mul(Rs[j * RS + gl], Wj[c * RS + (j % RPC)]));
        }
        Rout[g + int64_t(c) * nmax] = acc;
      }
    }
  }
  __syncthreads();
  if (a.prof && tid == 0) {
    long long *pf = a.prof + int64_t(blockIdx.x) * 8;
    pf[0] = t_chol - t_start;
    pf[1] = t_jac - t_chol;
    pf[2] = clock64() - t_jac;
    pf[3] = gr;
    pf[4] = sweeps;
    pf[5] = fallback;
    pf[6] = t_rij ? t_rij - t_start : 0;
    pf[7] = t_s ? t_s - t_start : 0;
    long long *pp = a.prof + int64_t(gridDim.x) * 8 + int64_t(blockIdx.x) * 8;
    for (int i = 0; i < 8; ++i) pp[i] = ph[i];
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
  cluster_sync<C>();
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

static size_t pivot_smem(bool cx, int nmax, int c) {
  const size_t w = cx ? 16 : 8;
  const size_t rs = nmax / c + 1;
  const size_t slab = nmax * rs;
  return (slab + std::max<size_t>(slab, 16 * nmax)) * w + 2 * c * (nmax / 2) * w + 2 * nmax * w +
         3 * nmax * 8 + nmax * 4;
}

int pivot_default_cluster(bool cx, int nmax, int count) {
  // smallest cluster whose shared-memory slabs fit
  int cmin = 1;
  while (cmin < 16 && pivot_smem(cx, nmax, cmin) > 200 * 1024) cmin *= 2;
  // largest cluster (rows per CTA >= 16) whose whole batch is co-resident in
  // one wave (cudaOccupancyMaxActiveClusters: e.g. 33 clusters of 4 but only
  // 15 of 8 on a 148-SM B200); if none, the batch needs several waves anyway
  // and the smallest cluster has the least exchange overhead
  static int cache[2][5][5];
  const int ni = nmax == 32 ? 0 : nmax == 64 ? 1 : nmax == 128 ? 2 : 3;
  int best = cmin;
  for (int c = cmin; c <= 16; c *= 2) {
    if (nmax / c < 16 && c > cmin) break;
    const int ci = c == 1 ? 0 : c == 2 ? 1 : c == 4 ? 2 : c == 8 ? 3 : 4;
    const int nt = pivot_default_threads(cx, nmax, c);
    int &occ = cache[cx][ni][ci];
    if (occ == 0) occ = pivot_max_active_clusters(cx, nmax, c, nt);
    if (occ >= count && (count * c <= 148 || c == cmin)) best = c;  // one wave, one CTA per SM
  }
  return best;
}

static int g_query_clusters = 0;  // when set, launch_pivot only reports max active clusters

template <typename T, int NMAX, int C, int NT>
static cudaError_t query_clusters(int *out) {
  using Cfg = PivCfg<T, NMAX, C, NT>;
  auto k = pivot_kernel<T, NMAX, C, NT>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(Cfg::SMEM));
  if (e != cudaSuccess) return e;
  if (C > 8) {
    e = cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(C * 64);
  cfg.blockDim = dim3(NT);
  cfg.dynamicSmemBytes = Cfg::SMEM;
  cudaLaunchAttribute attrs[1];
  attrs[0].id = cudaLaunchAttributeClusterDimension;
  attrs[0].val.clusterDim.x = C;
  attrs[0].val.clusterDim.y = 1;
  attrs[0].val.clusterDim.z = 1;
  cfg.attrs = attrs;
  cfg.numAttrs = 1;
  return cudaOccupancyMaxActiveClusters(out, k, &cfg);
}

template <typename T, int NMAX, int C, int NT>
static cudaError_t launch_if_valid(const PivotArgs &a, cudaStream_t st) {
  constexpr int P2 = NMAX / 2, RPC = NMAX / C;
  if constexpr (RPC >= 4 && NT >= P2 && NT / P2 <= 32 && NT / P2 <= RPC && NT <= RPC * NMAX) {
    if constexpr (PivCfg<T, NMAX, C, NT>::SMEM <= 227 * 1024) {
      if (g_query_clusters) return query_clusters<T, NMAX, C, NT>(&g_query_clusters);
      return launch_pivot_t<T, NMAX, C, NT>(a, st);
    }
  }
  return cudaErrorInvalidConfiguration;
}

int pivot_max_active_clusters(bool cx, int nmax, int c, int nt) {
  g_query_clusters = 1;
  PivotArgs a{};
  a.nmax = nmax;
  const int saved_t = g_tune_threads, saved_c = g_tune_cluster;
  g_tune_threads = nt;
  g_tune_cluster = c;
  cudaError_t e = launch_pivot(cx, a, c, nullptr, nullptr);
  g_tune_threads = saved_t;
  g_tune_cluster = saved_c;
  const int r = g_query_clusters;
  g_query_clusters = 0;
  return e == cudaSuccess ? r : -int(e);
}

template <typename T, int NMAX, int C>
static cudaError_t dispatch_nt(const PivotArgs &a, int nt, cudaStream_t st) {
  switch (nt) {
    case 256: return launch_if_valid<T, NMAX, C, 256>(a, st);
    case 512: return launch_if_valid<T, NMAX, C, 512>(a, st);
    case 1024: return launch_if_valid<T, NMAX, C, 1024>(a, st);
  }
  return cudaErrorInvalidConfiguration;
}

template <typename T, int NMAX>
static cudaError_t dispatch_c(const PivotArgs &a, int c, int nt, cudaStream_t st) {
  switch (c) {
    case 1: return dispatch_nt<T, NMAX, 1>(a, nt, st);
    case 2: return dispatch_nt<T, NMAX, 2>(a, nt, st);
    case 4: return dispatch_nt<T, NMAX, 4>(a, nt, st);
    case 8: return dispatch_nt<T, NMAX, 8>(a, nt, st);
    case 16: return dispatch_nt<T, NMAX, 16>(a, nt, st);
  }
  return cudaErrorInvalidConfiguration;
}

void pivot_tune(int threads, int cluster) {
  g_tune_threads = threads;
  g_tune_cluster = cluster;
}

int pivot_default_threads(bool cx, int nmax, int c) {
  // smallest CTA whose register-resident slab (4 arrays x RPT rows) stays
  // within ~4 complex / 8 real rows per thread
  const int p2 = nmax / 2, rpc = nmax / c, cap = 8;
  for (int nt = 256; nt <= 1024; nt *= 2) {
    const int tpp = nt / p2;
    if (tpp < 1 || tpp > 32 || tpp > rpc) continue;
    if (rpc / tpp <= cap) return nt;
  }
  return 1024;
}

cudaError_t launch_pivot(bool cx, const PivotArgs &a, int cluster, cudaStream_t st, int *cluster_used) {
  int c = cluster > 0 ? cluster : (g_tune_cluster > 0 ? g_tune_cluster : pivot_default_cluster(cx, a.nmax, a.count));
  const int nt = g_tune_threads > 0 ? g_tune_threads : pivot_default_threads(cx, a.nmax, c);
  if (cluster_used) *cluster_used = c;
  if (cx) {
    switch (a.nmax) {
      case 32: return dispatch_c<cplx, 32>(a, c, nt, st);
      case 64: return dispatch_c<cplx, 64>(a, c, nt, st);
      case 128: return dispatch_c<cplx, 128>(a, c, nt, st);
      case 256: return dispatch_c<cplx, 256>(a, c, nt, st);
    }
  } else {
    switch (a.nmax) {
      case 32: return dispatch_c<double, 32>(a, c, nt, st);
      case 64: return dispatch_c<double, 64>(a, c, nt, st);
      case 128: return dispatch_c<double, 128>(a, c, nt, st);
      case 256: return dispatch_c<double, 256>(a, c, nt, st);
    }
  }
  return cudaErrorInvalidValue;
}

}  // namespace hjb
