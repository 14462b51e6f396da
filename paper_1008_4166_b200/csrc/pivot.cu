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
#include <type_traits>
#include <cfloat>
#include <climits>

#include "common.cuh"
#include "kernels.h"
#include "rotation.cuh"

namespace cg = cooperative_groups;

// per-round phase clocks (tools/pivot_bench.py); off in production builds
// a sweep whose largest |t| is below HJB_CHK_SCALE * sqrt(orth_tol) is
// followed by the one-shot Gram check instead of a ring sweep
#ifndef HJB_CHK_SCALE
#define HJB_CHK_SCALE 2.0
#endif
#ifndef HJB_WBLOCK
#define HJB_WBLOCK 1
#endif
#ifndef HJB_ABL_WARPRING
#define HJB_ABL_WARPRING 0
#endif
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
// This file builds as TWO translation units to halve the wall time of the
// library build: pivot.cu itself (the float64 instantiations and every
// non-template function) and pivot_c128.cu, which defines HJB_PIVOT_CPLX_TU
// and includes this file (the complex128 instantiations only).
#ifndef HJB_PIVOT_CPLX_TU
static int g_tune_threads = 0, g_tune_cluster = 0;  // hjb_tune overrides (0 = auto)
#endif

template <typename T, int NMAX, int C, int NT>
struct PivCfg {
  static constexpr int RPC = NMAX / C;   // rows of R/W per CTA
  static constexpr int RS = RPC + 1;     // padded column stride (elements)
  static constexpr int P2 = NMAX / 2;    // pair slots per round
  static constexpr int TPP = NT / P2;    // threads per pair slot
  static constexpr int RPT = RPC / TPP;  // rows per thread
  static constexpr int OPT = RPC * NMAX / NT;  // Cholesky outputs per thread (distributed path)
  static constexpr int HC = 16;                // R_ij rows staged per chunk
  static_assert(TPP >= 1 && TPP <= 32 && (TPP & (TPP - 1)) == 0, "threads per pair");
  static_assert(RPT >= 1 && RPC % TPP == 0, "rows per thread");
  static_assert(OPT >= 1 && (RPC * NMAX) % NT == 0, "outputs per thread");
  static constexpr int NWARP = NT / 32;
  static constexpr int SPW = 32 / TPP;                       // pair slots per warp
  static constexpr int XBUF = 2 * NWARP * RPC;               // ring pass buffers [parity][warp][row]
  // fast path: the whole b x b factor U (Schur complement / block Gram
  // Cholesky) is kept in every CTA; register tile of the Cholesky
  static constexpr int UB = NMAX / 2;                        // largest block width
  static constexpr int UL = UB + 1;                          // U column stride
  static constexpr int TI = UB < 16 ? UB : 16;               // Cholesky thread grid TI x TL
  static constexpr int TL = NT / TI;
  static constexpr int XI = UB / TI;                         // rows per thread
  static constexpr int YL = (UB + TL - 1) / TL;              // columns per thread
  static constexpr int RV = (UB + 31) / 32;                  // back-substitution rows per lane
  static constexpr int SCR0 = HC * NMAX;
  static constexpr int SCR1 = SCR0 > NMAX * RS ? SCR0 : NMAX * RS;  // also the R_final / W slab
  static constexpr bool FAST_OK = NMAX <= 128 && XI * YL <= 32;
  static constexpr int SCR = SCR1;
  // U staged on chip for the back substitution (the contiguous Rs|Ws region)
  static constexpr bool U_SMEM = UB * UL <= NMAX * RS + SCR;
  // shared-memory carve-up (bytes, 16-aligned)
  static constexpr size_t OFF_R = 0;
  static constexpr size_t OFF_W = OFF_R + size_t(NMAX) * RS * sizeof(T);  // scratch / U
  static constexpr size_t OFF_X = OFF_W + size_t(SCR) * sizeof(T);        // ring buffers
  static constexpr size_t OFF_XD = OFF_X + size_t(XBUF) * sizeof(T);      // their D values
  static constexpr size_t OFF_PART = OFF_XD + 2 * NWARP * sizeof(double);
  static constexpr size_t PART = (2 * C * P2 > RPC) ? 2 * C * P2 : RPC;  // also W-block scratch (column chunks)
  static constexpr size_t OFF_ROW = OFF_PART + PART * sizeof(T);         // Cholesky row buffers [2][UB]
  static constexpr size_t OFF_NPART = OFF_ROW + 2 * size_t(UB) * sizeof(T);
  // [2][C][P2] column-norm pairs (complex: they fit the dot-partial buffer)
  static constexpr size_t NPART = (!S<T>::cx && 4 * C * P2 > NMAX) ? 4 * C * P2 : NMAX;
  static constexpr size_t OFF_LAM = OFF_NPART + NPART * sizeof(double);
  static constexpr size_t OFF_J = OFF_LAM + NMAX * sizeof(double);
  static constexpr size_t SMEM = OFF_J + NMAX * sizeof(int);
  static constexpr bool FAST = FAST_OK && SMEM <= 227 * 1024;
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
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t *bar, unsigned tx) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(tx)
               : "memory");
}
// wait for the phase with the given parity.  CTA-scope acquire: the data
// guarded here is this CTA's shared memory, written by its own warps or by
// the peers' st.async (whose bytes complete_tx on this barrier) -- a
// cluster-scope acquire would add an L1 invalidation (CCTL.IVALL) per wait
__device__ __forceinline__ void mbar_wait_cta(uint64_t *bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "HJB_WAITC_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra HJB_WAITC_%=;\n}\n" ::"r"(smem_u32(bar)),
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

// predicated shared-memory store (no branch, so the surrounding shuffles stay
// in one basic block)
__device__ __forceinline__ void st_shared_if(bool p, double *dst, double v) {
  asm volatile("{\n .reg .pred q;\n setp.ne.b32 q, %0, 0;\n @q st.shared.f64 [%1], %2;\n}\n" ::"r"(int(p)),
               "r"(smem_u32(dst)), "d"(v)
               : "memory");
}
__device__ __forceinline__ void st_shared_if(bool p, cplx *dst, cplx v) {
  asm volatile("{\n .reg .pred q;\n setp.ne.b32 q, %0, 0;\n @q st.shared.v2.f64 [%1], {%2, %3};\n}\n" ::"r"(int(p)),
               "r"(smem_u32(dst)), "d"(v.x), "d"(v.y)
               : "memory");
}

// compute_plane_rotation (rotations.py:128-155) for a batch of 2x2 Gram
// pivots [[a_rr, a_rs], [conj(a_rs), a_ss]] through the pivot kernel's own
// rot_coef (no skip threshold: only a_rs == 0 is the identity).  out[k] =
// (code, cs, sn, t, eta, phase_re, phase_im, hyp); code 0 identity, 1
// rotation, -1 not positive definite (rotations.py:134-135, 147-148).
template <typename T>
__global__ void plane_rotation_kernel(int count, const double *arr, const double *ass, const T *ars,
                                      const int8_t *same, double *out) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= count) return;
  const double dr = arr[k], ds = ass[k];
  const T a = ars[k];
  double *o = out + int64_t(k) * 8;
  if (!(dr > 0.0) || !(ds > 0.0)) {
    o[0] = -1.0;
    return;
  }
  const RotCoef<T> p = rot_coef<T>(a, dr, ds, same[k] != 0, 0.0);
  const double q = abs2(a);
  const double ri = q > 0.0 ? rsqrt(q) : 0.0;
  const double sa = re(a) >= 0.0 ? 1.0 : -1.0;
  T ph = phase_mul(a, sa * ri);
  if constexpr (!S<T>::cx) ph = 1.0;  // a / eta is exactly 1 for real a (_kernels.py:61-62)
  o[0] = p.code;
  o[1] = p.code == 1 ? p.cs : 1.0;
  o[2] = p.code == 1 ? p.hs * p.hyp : 0.0;  // sn (hs = hyp * sn)
  o[3] = p.code == 1 ? p.num / p.den : 0.0;
  o[4] = p.code == 1 ? p.eta : 0.0;
  o[5] = p.code == 1 ? re(ph) : 1.0;
  if constexpr (S<T>::cx) o[6] = p.code == 1 ? ph.y : 0.0;
  else o[6] = 0.0;
  o[7] = p.hyp;
}

#ifndef HJB_PIVOT_CPLX_TU
cudaError_t launch_plane_rotations(bool cx, int count, const double *arr, const double *ass, const void *ars,
                                   const int8_t *same, double *out, cudaStream_t st) {
  if (count <= 0) return cudaSuccess;
  const int nb = (count + 127) / 128;
  if (cx)
    plane_rotation_kernel<cplx><<<nb, 128, 0, st>>>(count, arr, ass, static_cast<const cplx *>(ars), same, out);
  else
    plane_rotation_kernel<double><<<nb, 128, 0, st>>>(count, arr, ass, static_cast<const double *>(ars), same, out);
  return cudaGetLastError();
}
#endif  // !HJB_PIVOT_CPLX_TU

template <typename T, int NMAX, int C, int NT>
__global__ void __launch_bounds__(NT, 1) pivot_kernel(PivotArgs a) {
  using Cfg = PivCfg<T, NMAX, C, NT>;
  constexpr int RPC = Cfg::RPC, RS = Cfg::RS, TPP = Cfg::TPP, RPT = Cfg::RPT, OPT = Cfg::OPT;
  constexpr int HC = Cfg::HC;
  extern __shared__ __align__(16) unsigned char smem[];
  T *Rs = reinterpret_cast<T *>(smem + Cfg::OFF_R);
  T *Ws = reinterpret_cast<T *>(smem + Cfg::OFF_W);
  T *part = reinterpret_cast<T *>(smem + Cfg::OFF_PART);
  double *npart = reinterpret_cast<double *>(smem + Cfg::OFF_NPART);
  double *lam = reinterpret_cast<double *>(smem + Cfg::OFF_LAM);
  int *Jv = reinterpret_cast<int *>(smem + Cfg::OFF_J);
  __shared__ int s_flag[2];
  __shared__ int s_cnt[2];
  __shared__ int s_big;
  __shared__ int s_fail;
  __shared__ unsigned long long s_maxt;
  __shared__ unsigned long long s_swt[2];  // per-sweep max |t| (double bits)
  __shared__ uint64_t s_mbar[2];
  __shared__ uint64_t s_pbar[NT / 32];
  __shared__ int s_wbid[HJB_WBLOCK ? NMAX : 1];  // block-step exchange: column ids

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
  if (tid == 0) {
    s_fail = INT_MAX; s_maxt = 0ull; s_big = 0; s_cnt[0] = s_cnt[1] = 0; s_flag[0] = 1; s_flag[1] = 0;
    s_swt[0] = s_swt[1] = 0ull;
  }
  __syncthreads();

  // ------------------------------------------------------------------ R
  int status = PV_OK;
  int fallback = 0;
  int k0 = 0;
  bool need_dense = dense;
  // Fast path (NMAX <= 128): every CTA of the cluster redundantly forms the
  // whole b x b matrix U_in -- the Schur complement S = L_j - R_ij^H R_ij of
  // the structured Cholesky (blocking.py:131-134), or herm(B^H B) for the
  // pre-pass (parallel.py:143, core.py:54-55) -- and factors it in a
  // register tile (one CTA barrier per column, no cluster traffic).  The
  // factor is kept in an L2 scratch (written by CTA 0) for the back
  // substitution W = R0^-1 R_final.
  bool fast = false;
  const int nt = dense ? 0 : ni;  // rows of R0 with the diagonal sqrt(L_i) block
  const int nu = dense ? N : nj;  // order of U
  const int mode = a.mode;
  T *R0g = a.R0g ? reinterpret_cast<T *>(a.R0g) + int64_t(item_id) * a.nmax * a.nmax : nullptr;
  if (mode == PV_EPILOGUE) {
    // W = R0^-1 R_final after the Jacobi kernel: R_final is in W, R0 in R0g
    // (the U factor of the fast path in the L2 scratch); nothing to do for a
    // failed pivot or one that applied no rotation (the update skips it)
    const int64_t *sv = a.stats + int64_t(item_id) * ST_N;
    status = int(__ldcg(sv + ST_STATUS));
    fallback = int(__ldcg(sv + ST_FALLBACK));
    if (status != PV_OK || __ldcg(sv + ST_NROT) == 0) return;  // uniform over the cluster
    fast = Cfg::FAST && !fallback;
    if (!fast) {
      for (int e = tid; e < RPC * NMAX; e += NT) {
        const int gl = e % RPC, c = e / RPC;
        Rs[gl + c * RS] = __ldcg(R0g + (row0 + gl) + int64_t(c) * a.nmax);
      }
      __syncthreads();
    }
  } else {
  if constexpr (Cfg::FAST) {
    int ok = 1;
    if (!dense) {
      for (int c = tid; c < N; c += NT) ok &= (lam[c] > 0.0);
      ok = __syncthreads_and(ok);
    }
    if (!ok) {
      need_dense = true;  // structured_cholesky raises (blocking.py:125-126)
      fallback = 1;
    } else {
      constexpr int TI = Cfg::TI, TL = Cfg::TL, XI = Cfg::XI, YL = Cfg::YL, UL = Cfg::UL;
      const int ti = tid % TI, tl = tid / TI;
      T u[XI][YL];
      if (!dense) {
        // S[i][l] = L_j[i] d_il - sum_h conj(Rij[h][i]) Rij[h][l], Rij = A / sqrt(L_i)
#pragma unroll
        for (int x = 0; x < XI; ++x)
#pragma unroll
          for (int y = 0; y < YL; ++y) u[x][y] = S<T>::zero();
        T *scr = Ws;  // staging: HC x NMAX rows of R_ij
        for (int h0 = 0; h0 < ni; h0 += HC) {
          const int hc = min(HC, ni - h0);
          for (int e = tid; e < HC * nj; e += NT) {
            const int h = e % HC, l = e / HC;
            scr[h * NMAX + l] = h < hc ? divr(A[(h0 + h) + int64_t(l) * bmax], sqrt(lam[h0 + h])) : S<T>::zero();
          }
          __syncthreads();
          for (int h = 0; h < hc; ++h) {
            T ri[XI], rl[YL];
#pragma unroll
            for (int x = 0; x < XI; ++x) ri[x] = scr[h * NMAX + ti + TI * x];
#pragma unroll
            for (int y = 0; y < YL; ++y) rl[y] = scr[h * NMAX + min(tl + TL * y, NMAX - 1)];
#pragma unroll
            for (int x = 0; x < XI; ++x)
#pragma unroll
              for (int y = 0; y < YL; ++y) u[x][y] = cfma(ri[x], rl[y], u[x][y]);
          }
          __syncthreads();
        }
#pragma unroll
        for (int x = 0; x < XI; ++x)
#pragma unroll
          for (int y = 0; y < YL; ++y) {
            const int i = ti + TI * x, l = tl + TL * y;
            T v = sub(i == l && i < nj ? scale(S<T>::one(), lam[ni + i]) : S<T>::zero(), u[x][y]);
            if (i == l) v = scale(S<T>::one(), re(v));  // exactly Hermitian diagonal
            u[x][y] = v;
          }
      } else {
#pragma unroll
        for (int x = 0; x < XI; ++x)
#pragma unroll
          for (int y = 0; y < YL; ++y) {
            const int i = ti + TI * x, l = tl + TL * y;
            T v = S<T>::zero();
            if (i <= l && l < N) {
              if (i == l)
                v = scale(S<T>::one(), re(A[i + int64_t(i) * bmax]));
              else
                v = scale(add(A[i + int64_t(l) * bmax], conjv(A[l + int64_t(i) * bmax])), 0.5);
            }
            u[x][y] = v;
          }
      }
      // right-looking Cholesky on the unscaled rows: U[i][l] -= conj(U[k][i])
      // U[k][l] / U[k][k]; row k+1 is published through a double buffer
      T *rowb = reinterpret_cast<T *>(smem + Cfg::OFF_ROW);  // [2][UB]
      double *piv = npart;                                    // pivots U[k][k]
      auto publish = [&](int k) {
        if (k < nu && ti == k % TI) {
          const int x = k / TI;
#pragma unroll
          for (int xx = 0; xx < XI; ++xx) {
            if (xx != x) continue;
#pragma unroll
            for (int y = 0; y < YL; ++y) {
              const int l = tl + TL * y;
              if (l >= k && l < nu) rowb[(k & 1) * Cfg::UB + l] = u[xx][y];
            }
          }
        }
      };
      publish(0);
      __syncthreads();
      int chol_ok = 1;
      for (int k = 0; k < nu; ++k) {
        const T *rk = rowb + (k & 1) * Cfg::UB;
        const double dk = re(rk[k]);
        if (!finite_pos(dk)) {
          chol_ok = 0;
          break;
        }
        if (tid == 0) piv[k] = dk;
        const double inv = 1.0 / dk;
        T ri[XI], rl[YL];
#pragma unroll
        for (int x = 0; x < XI; ++x) ri[x] = scale(rk[min(ti + TI * x, Cfg::UB - 1)], inv);
#pragma unroll
        for (int y = 0; y < YL; ++y) rl[y] = rk[min(tl + TL * y, Cfg::UB - 1)];
#pragma unroll
        for (int x = 0; x < XI; ++x) {
          if (ti + TI * x <= k) continue;  // finished rows (whole warps skip late in the factorisation)
#pragma unroll
          for (int y = 0; y < YL; ++y) {
            const int i = ti + TI * x, l = tl + TL * y;
            if (l >= i && l < nu) u[x][y] = cfms(ri[x], rl[y], u[x][y]);
          }
        }
        publish(k + 1);
        __syncthreads();
      }
      if (chol_ok) {
        // final factor R[k][k] = sqrt(d_k), R[k][l] = U[k][l] / sqrt(d_k):
        // CTA 0 keeps it in the L2 scratch for the back substitution, every
        // CTA writes its own rows into the R0 slab
        T *Ug = reinterpret_cast<T *>(a.uscr) + int64_t(item_id) * Cfg::UB * UL;
        for (int e = tid; e < NMAX * RS; e += NT) Rs[e] = S<T>::zero();
        __syncthreads();
#pragma unroll
        for (int x = 0; x < XI; ++x)
#pragma unroll
          for (int y = 0; y < YL; ++y) {
            const int i = ti + TI * x, l = tl + TL * y;
            if (l >= Cfg::UB) continue;
            T v = S<T>::zero();
            if (i <= l && l < nu) {
              const double rd = sqrt(piv[i]);
              v = i == l ? scale(S<T>::one(), rd) : divr(u[x][y], rd);
            }
            if (crank == 0) Ug[i + l * UL] = v;
            const int g = nt + i;
            if (g >= row0 && g < row0 + RPC && i <= l && l < nu) Rs[(g - row0) + (nt + l) * RS] = v;
          }
        // rows of the diagonal block: [sqrt(L_i), A / sqrt(L_i)]
        for (int e = tid; e < RPC * NMAX; e += NT) {
          const int gl = e % RPC, c = e / RPC;
          const int g = row0 + gl;
          if (g >= nt || c >= N || c < g) continue;
          Rs[gl + c * RS] = c == g ? scale(S<T>::one(), sqrt(lam[g]))
                                   : (c < nt ? S<T>::zero() : divr(A[g + int64_t(c - nt) * bmax], sqrt(lam[g])));
        }
        __threadfence();
        __syncthreads();
        fast = true;
        need_dense = false;
      } else if (dense) {
        status = PV_CHOL;
      } else {
        need_dense = true;  // parallel.py:196-198
        fallback = 1;
      }
    }
  } else
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

  if (!need_dense && !fast) {
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
  }  // mode != PV_EPILOGUE

  if (mode == PV_PROLOGUE) {
    // R0 (whole N x N, zero padded) -> global for the Jacobi kernel; status
    // and fallback for it and the epilogue
    if (status == PV_OK)
      for (int e = tid; e < RPC * a.nmax; e += NT) {
        const int gl = e % RPC, c = e / RPC;
        const int g = row0 + gl;
        if (g < a.nmax) R0g[g + int64_t(c) * a.nmax] = c < NMAX ? Rs[gl + c * RS] : S<T>::zero();
      }
    if (crank == 0 && tid == 0) {
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
    cluster_sync<C>();  // peers' shared memory stays alive until every remote read is done
    return;
  }

  t_chol = clock64();
  // ------------------------------------------------------------------ Jacobi
  // Register-resident columns.  Pair slot q (TPP lanes of one warp) holds the
  // RPC-row slab of its two columns of R in registers (lane l owns rows l,
  // l+TPP, ...) together with their D values (the D cache of
  // rotations.py:217 / _kernels.py:80-81 travels with its column).  After
  // each round the slot keeps one column and passes the other to its ring
  // neighbour, exactly as the reference's modulus stepper passes block
  // columns between workers (strategies.py:58-92 with nbl = N): a warp
  // shuffle inside a warp, shared memory + a per-warp mbarrier across warps.
  //
  // One round, without any CTA-wide barrier:
  //   dot partial over the lane's rows -> shuffle reduction over the TPP
  //   lanes -> st.async of the CTA partial into every cluster peer (local
  //   store for this CTA) -> per-warp arrive on the round's mbarrier (which
  //   also waits for the peers' bytes) -> every lane sums the C partials in
  //   rank order (bit-identical in all CTAs) and derives the rotation itself
  //   -> apply -> ring step.
  // Every CTA computes every pair's rotation, so the sweep's rotation count
  // (the convergence test, parallel.py:239-244) is known in each CTA without
  // a cluster exchange.  W is not accumulated per rotation: W = R0^-1 R_final
  // is formed once at the end.
  const double otol = a.orth_tol > 0.0 ? a.orth_tol : sqrt(double(N)) * kEps;
  const double otol2 = otol * otol;
  const double qtol = a.quad_tol > 0.0 ? a.quad_tol : double(N) * kEps;
  // HJB_WBLOCK: warp-block inner order (oracle WBlockState) over all NMAX
  // column positions (ids >= N are zero padding that never rotates)
  constexpr bool WB = HJB_WBLOCK;
  const int ne = WB ? NMAX : N + (N & 1);
  const int pr = ne / 2;  // ring slots in use
  const int slot = tid / TPP, lane_in = tid % TPP;
  constexpr int SPW = Cfg::SPW, NWARP = Cfg::NWARP;
  const int warp = tid >> 5, lane = tid & 31;
  const bool in_ring = slot < pr;
  const int wslot = slot % SPW;
  int ip = slot + 1, jp = ne - slot, ib = ip, jb = jp;  // strategies.py:58-66
  int cX = ib - 1, cY = jb - 1;  // column ids held in X / Y (travel with the data under WB)
  long long nrot_total = 0;
  int sweeps = 0;
  int gr = 0;  // exchange counter (mbarrier phases / buffer parities)
  int pg = 0;  // ring-pass counter (pass-buffer parities)
  int my_big = 0, my_cnt = 0, my_fail = INT_MAX;
  double my_maxt = 0.0, my_swt = 0.0;
  // max |t| = num/den kept as a fraction (compared by cross-multiplication,
  // divided once per sweep) so no division sits before the apply loop
  double mt_n = 0.0, mt_d = 1.0, sw_n = 0.0, sw_d = 1.0;
  long long ph[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  T *xbuf = reinterpret_cast<T *>(smem + Cfg::OFF_X);             // [2][NWARP][RPC]
  double *xd = reinterpret_cast<double *>(smem + Cfg::OFF_XD);     // [2][NWARP]
  constexpr unsigned TX = (C - 1) * Cfg::P2 * sizeof(T);          // dot partials pushed into each CTA
  constexpr unsigned TXN = (C - 1) * Cfg::P2 * 16;                // column-norm partials
  if (tid == 0) {
    for (int b = 0; b < 2; ++b) mbar_init(&s_mbar[b], NWARP);
    for (int w = 0; w < NWARP; ++w) mbar_init(&s_pbar[w], TPP);
    fence_mbar_init();
  }
  T X[RPT], Y[RPT];
#pragma unroll
  for (int u = 0; u < RPT; ++u) {
    const int row = lane_in + u * TPP;
    const int ci = in_ring ? cX : 0, cj = in_ring ? cY : 1;
    X[u] = Rs[ci * RS + row];
    Y[u] = Rs[cj * RS + row];
  }
  double dX = 0.0, dY = 0.0;
  int sX = 1, sY = 1;  // J signs of the two columns
  cluster_sync<C>();   // barriers initialised in every CTA before any push

  // push this slot's CTA partial v (sizeof(V) bytes) to every CTA of the
  // cluster (plain store into this CTA), then arrive on the exchange barrier
  auto push = [&](auto *base, auto v, unsigned tx) {
    const int buf = gr & 1;
    auto *mine = base + (buf * C + crank) * Cfg::P2 + slot;
    if constexpr (C > 1) {
      const uint32_t la = smem_u32(mine), lb = smem_u32(&s_mbar[buf]);
#pragma unroll
      for (int q0 = 0; q0 < C; q0 += TPP) {
        const int q = q0 + lane_in;
        if (q < C) {
          if (q == crank)
            *mine = v;
          else
            st_async(mapa_u32(la, q), v, mapa_u32(lb, q));
        }
      }
    } else {
      if (lane_in == 0) *mine = v;
    }
    __syncwarp();
    if (lane == 0) {
      if (warp == 0)
        mbar_arrive_tx(&s_mbar[buf], tx);
      else
        mbar_arrive(&s_mbar[buf]);
    }
  };

  // dot partial of this lane's rows for its slot's current pair
  auto dot_part = [&]() {
    T d[4] = {S<T>::zero(), S<T>::zero(), S<T>::zero(), S<T>::zero()};
#pragma unroll
    for (int u = 0; u < RPT; ++u) d[u & 3] = cfma(X[u], Y[u], d[u & 3]);
    return add(add(d[0], d[2]), add(d[1], d[3]));
  };
  T dn = dot_part();
  double prev_swt = 1.0;
  const double chk_thr = HJB_CHK_SCALE * sqrt(otol);
  // Gram of the current columns (partials of this CTA's rows, 4 x 4 column
  // blocks) -> L2 scratch; CTA r checks the blocks b = r mod C against the
  // skip test; cluster-wide OR of the failures
  auto gram_check = [&]() -> bool {
    constexpr int NB = NMAX / 4, NBLK = NB * (NB + 1) / 2;
    __syncthreads();
    if (in_ring) {
#pragma unroll
      for (int u = 0; u < RPT; ++u) {
        const int row = lane_in + u * TPP;
        if (cX < N) Ws[cX * RS + row] = X[u];
        if (cY < N) Ws[cY * RS + row] = Y[u];
      }
    }
    __syncthreads();
    T *gs = reinterpret_cast<T *>(a.gchk) + int64_t(item_id) * 16 * NBLK * 16;
    for (int blk = tid; blk < NBLK; blk += NT) {
      int R = 0, rem = blk;
      while (rem >= NB - R) {
        rem -= NB - R;
        ++R;
      }
      const int Sb = R + rem;
      T acc[4][4];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = S<T>::zero();
      if (4 * R < N && 4 * Sb < N) {
        for (int row = 0; row < RPC; ++row) {
          T x[4], y[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            x[i] = Ws[(4 * R + i) * RS + row];
            y[i] = Ws[(4 * Sb + i) * RS + row];
          }
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[i][j] = cfma(x[i], y[j], acc[i][j]);
        }
      }
      T *dst = gs + (int64_t(crank) * NBLK + blk) * 16;
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dst[i * 4 + j] = acc[i][j];
    }
    __threadfence();
    cluster_sync<C>();
    // fresh column norms (diagonal blocks), summed in rank order
    double *Dc = npart;
    for (int c = tid; c < N; c += NT) {
      const int R = c >> 2, blk = R * NB - R * (R - 1) / 2;  // diagonal block (R, R)
      double d = 0.0;
      for (int q = 0; q < C; ++q) d += re(__ldcg(gs + (int64_t(q) * NBLK + blk) * 16 + (c & 3) * 5));
      Dc[c] = d;
    }
    __syncthreads();
    int bad = 0;
    for (int e = tid; e < NBLK * 16; e += NT) {
      const int blk = e >> 4, ij = e & 15;
      if (blk % C != crank) continue;
      int R = 0, rem = blk;
      while (rem >= NB - R) {
        rem -= NB - R;
        ++R;
      }
      const int r = 4 * R + (ij >> 2), sc = 4 * (R + rem) + (ij & 3);
      if (r >= sc || sc >= N) continue;
      T m = S<T>::zero();
      for (int q = 0; q < C; ++q) m = add(m, __ldcg(gs + (int64_t(q) * NBLK + blk) * 16 + ij));
      if (!(abs2(m) <= otol2 * (Dc[r] * Dc[sc]))) bad = 1;
    }
    bad = __syncthreads_or(bad);
    if (tid == 0 && bad)
      for (int q = 0; q < C; ++q) remote<C>(s_flag, q)[1] = 1;
    cluster_sync<C>();
    const bool ok = s_flag[1] == 0;
    __syncthreads();
    if (tid == 0) s_flag[1] = 0;
    return ok;
  };
  if (status == PV_OK && mode == PV_FULL) {
    for (int sw = 0; sw < a.max_sweeps; ++sw) {
      ++sweeps;
      // A sweep after one whose rotations were all tiny is almost surely the
      // final zero-rotation sweep (rotations.py:220-222): check all its pairs
      // at once on the Gram matrix of the current columns.  If every pair
      // passes the skip test of _kernels.py:57 (with D = colnorms^2 at the
      // sweep start, rotations.py:217) the sweep applies no rotation -- the
      // same outcome as running it; otherwise run it.
      {
        // (pre-pass blocks after the first outer sweep are already
        // diagonal: check them before their first inner sweep too)
        const long long cg0 = RCLK();
        const bool gc_try = a.gchk && ((sw > 0 && prev_swt <= chk_thr) || (sw == 0 && dense));
        const bool gc_ok = gc_try && gram_check();
        if (HJB_ROUND_PROFILE && a.prof) ph[7] += RCLK() - cg0;
        if (gc_ok) break;
      }
      const bool odd = (sw & 1) == 0;  // reference sweeps count from 1; odd send to q-1
      const int src = odd ? (slot + 1 == pr ? 0 : slot + 1) : (slot == 0 ? pr - 1 : slot - 1);
      const int srcw = src / SPW;
#if HJB_ABL_WARPRING  // timing ablation only (wrong ordering): the ring wraps inside each warp
      const bool via_smem = false, writer = false;
      const int src_lane = (odd ? (wslot + 1) % SPW : (wslot + SPW - 1) % SPW) * TPP + lane_in;
#else
      // WB: every column move stays inside the warp (slot q receives from q+1 mod SPW)
      const bool via_smem = !WB && in_ring && (odd ? (wslot == SPW - 1 || slot == pr - 1) : (wslot == 0 || slot == 0));
      const bool writer = !WB && in_ring && (odd ? (wslot == 0) : (wslot == SPW - 1 || slot == pr - 1));
      const int src_lane = WB ? ((wslot + 1) % SPW) * TPP + lane_in : (odd ? min(lane + TPP, 31) : max(lane - TPP, 0));
#endif
      // ---- D = colnorms^2(R) (rotations.py:217): cluster-reduced norms ----
      {
        double nx = 0.0, ny = 0.0, nx1 = 0.0, ny1 = 0.0;
#pragma unroll
        for (int u = 0; u < RPT; ++u) {
          if (u & 1) { nx1 += abs2(X[u]); ny1 += abs2(Y[u]); }
          else { nx += abs2(X[u]); ny += abs2(Y[u]); }
        }
        nx += nx1;
        ny += ny1;
#pragma unroll
        for (int o = 1; o < TPP; o <<= 1) {
          nx += __shfl_xor_sync(0xffffffffu, nx, o);
          ny += __shfl_xor_sync(0xffffffffu, ny, o);
        }
        const int buf = gr & 1;
        double2 *nbuf = S<T>::cx ? reinterpret_cast<double2 *>(part) : reinterpret_cast<double2 *>(npart);
        push(nbuf, make_double2(nx, ny), TXN);
        mbar_wait_cta(&s_mbar[buf], (gr >> 1) & 1);
        const double2 *np0 = nbuf + (buf * C) * Cfg::P2 + slot;
        double2 nn = np0[0];
#pragma unroll
        for (int r = 1; r < C; ++r) {
          const double2 v = np0[r * Cfg::P2];
          nn.x += v.x;
          nn.y += v.y;
        }
        dX = nn.x;
        dY = nn.y;
        ++gr;
      }
      sX = Jv[min(cX, NMAX - 1)];
      sY = Jv[min(cY, NMAX - 1)];
      int lip = wslot + 1, ljp = 2 * SPW - wslot;  // WB phase A: warp-local modulus stepper

      for (int rnd = 0; rnd < ne; ++rnd, ++gr, ++pg) {
        if constexpr (WB) {
          // phase B block step t (circle method over M = 2 NWARP blocks of
          // SPW columns; warp i holds pair i): all columns move through
          // shared memory at the step start, never inside a round
          const int rb = rnd - 2 * SPW;
          if (rb >= 0 && rb % SPW == 0) {
            const long long cx0 = RCLK();
            constexpr int M = 2 * NWARP;
            const int t = 1 + rb / SPW;
            auto bpair = [&](int tt, int &bx, int &by) {
              if (warp == 0) { bx = M - 1; by = tt; }
              else { bx = (tt + warp) % (M - 1); by = (tt - warp + (M - 1)) % (M - 1); }
            };
            int bx, by;
            bpair(t - 1, bx, by);
            T *xb = Ws;  // [M * SPW positions][RS]; the padding row carries D
            __syncthreads();
            {
              const int px = bx * SPW + wslot, py = by * SPW + wslot;
#pragma unroll
              for (int u = 0; u < RPT; ++u) {
                xb[px * RS + lane_in + u * TPP] = X[u];
                xb[py * RS + lane_in + u * TPP] = Y[u];
              }
              if (lane_in == 0) {
                xb[px * RS + RPC] = scale(S<T>::one(), dX);
                xb[py * RS + RPC] = scale(S<T>::one(), dY);
                s_wbid[px] = cX;
                s_wbid[py] = cY;
              }
            }
            __syncthreads();
            bpair(t, bx, by);
            {
              const int px = bx * SPW + wslot, py = by * SPW + wslot;
#pragma unroll
              for (int u = 0; u < RPT; ++u) {
                X[u] = xb[px * RS + lane_in + u * TPP];
                Y[u] = xb[py * RS + lane_in + u * TPP];
              }
              dX = re(xb[px * RS + RPC]);
              dY = re(xb[py * RS + RPC]);
              cX = s_wbid[px];
              cY = s_wbid[py];
            }
            sX = Jv[min(cX, NMAX - 1)];
            sY = Jv[min(cY, NMAX - 1)];
            dn = dot_part();
            if (HJB_ROUND_PROFILE && a.prof) ph[6] += RCLK() - cx0;
          }
        }
        const long long c0 = RCLK();
        // (1) CTA partial of g_i^H g_j (computed at the end of the previous
        // round), reduced over the slot's TPP lanes, pushed to the cluster
        T dot = dn;
#pragma unroll
        for (int o = 1; o < TPP; o <<= 1) dot = add(dot, shfl_xor(dot, o));
        push(part, dot, TX);
        const long long c1 = RCLK();
        // (2) every lane sums the cluster partials in fixed rank order
        // (bit-identical in every CTA) and derives its slot's rotation
        // (_kernels.py:53-81)
        const int buf = gr & 1;
        mbar_wait_cta(&s_mbar[buf], (gr >> 1) & 1);
        const long long c2 = RCLK();
        // pairwise tree over the C partials (same fixed order in every CTA)
        T pv[C];
#pragma unroll
        for (int r = 0; r < C; ++r) pv[r] = part[(buf * C + r) * Cfg::P2 + slot];
#pragma unroll
        for (int h = 1; h < C; h <<= 1)
#pragma unroll
          for (int r = 0; r + h < C; r += 2 * h) pv[r] = add(pv[r], pv[r + h]);
        const T acc = pv[0];
        const int ci = cX, cj = cY;
        // skip test first (_kernels.py:57); the rotation parameters are only
        // derived in warps where some pair is not yet orthogonal
        bool rot = in_ring && ci < N && cj < N && !(abs2(acc) <= otol2 * (dX * dY));
        const bool any_rot = __any_sync(0xffffffffu, rot);
        RotCoef<T> p;
        p.cp = S<T>::one();
        p.sp = S<T>::zero();
        p.hs = 0.0;
        p.cs = 1.0;
        const long long c3 = RCLK();
        // D update (_kernels.py:80-81) te = t eta, t = num/den: its division
        // is done after the apply loop (dX/dY are not needed before)
        double te_n = 0.0, te_d = 1.0, te_h = 0.0;
        if (any_rot) {
          if (rot) {
            const RotCoef<T> q = rot_coef<T>(acc, dX, dY, sX == sY, otol2);
            if (q.code == 1) {
              p = q;
              te_n = q.num * q.eta;
              te_d = q.den;
              te_h = q.hyp;
              if (lane_in == 0) {
                ++my_cnt;
                const double an = fabs(q.num);
                my_big += an > qtol * q.den;  // |t| > quad_tol
                if (an * mt_d > mt_n * q.den) { mt_n = an; mt_d = q.den; }
                if (an * sw_d > sw_n * q.den) { sw_n = an; sw_d = q.den; }
              }
            } else {
              rot = false;
              if (q.code < 0) my_fail = min(my_fail, ci * 4096 + cj);
            }
          }
        }
        const long long c4 = RCLK();
        // (3) fused per row: apply the rotation, ring step (strategies.py:75-92
        // with nbl = ne: the slot keeps one column and receives the one its
        // neighbour sends; odd sweeps receive from slot+1, strategies.py:69-72)
        // and the next round's dot partial
        bool send_i;
        if constexpr (WB) {
          // phase A: the modulus stepper inside the warp (nbl = 2 SPW);
          // phase B: the Y column moves every round
          send_i = false;
          if (rnd < 2 * SPW) {
            send_i = lip + ljp > 2 * SPW;
            if (send_i) {
              ++lip;
              if (lip == ljp) {
                lip -= SPW;
                ljp = lip;
              }
            } else {
              ++ljp;
            }
          }
        } else {
          send_i = ip + jp > ne;
          if (in_ring) {
            if (send_i) {
              ++ip;
              if (ip == jp) {
                ip -= pr;
                jp = ip;
              }
              ib = ip;
              cX = ib - 1;
            } else {
              ++jp;
              jb = jp;
              cY = jb - 1;
            }
          }
        }
        const int par = pg & 1;
        T *xw = xbuf + (size_t(par) * NWARP + warp) * RPC;
        const bool all_i = __all_sync(0xffffffffu, send_i || !in_ring);
        const bool all_j = __all_sync(0xffffffffu, !send_i || !in_ring);
        // one straight-line body per (rotation, moving register) case so the
        // rows software-pipeline: apply -> shuffle -> next dot partial
        T e[4] = {S<T>::zero(), S<T>::zero(), S<T>::zero(), S<T>::zero()};
        auto fused = [&](auto rot_c, auto mode_c) {
          constexpr bool ROT = decltype(rot_c)::value;
          constexpr int MODE = decltype(mode_c)::value;  // 0: X moves, 1: Y moves, 2: per lane
#pragma unroll
          for (int u = 0; u < RPT; ++u) {
            if constexpr (ROT) rot_fold<T>(X[u], Y[u], p);
            const T v = MODE == 0 ? X[u] : (MODE == 1 ? Y[u] : (send_i ? X[u] : Y[u]));
            st_shared_if(writer, xw + lane_in + u * TPP, v);
            const T nv = shfl_idx(v, src_lane);
            if constexpr (MODE == 0) X[u] = nv;
            else if constexpr (MODE == 1) Y[u] = nv;
            else { if (send_i) X[u] = nv; else Y[u] = nv; }
            e[u & 3] = cfma(X[u], Y[u], e[u & 3]);
          }
          if constexpr (ROT) {
            const double te = te_n / te_d;
            dX = fma(te_h, te, dX);
            dY = dY + te;
          }
          // the moving column's D value (and id) follow it
          const double dv = MODE == 0 ? dX : (MODE == 1 ? dY : (send_i ? dX : dY));
          if (writer && lane_in == 0) xd[par * NWARP + warp] = dv;
          const double nd = __shfl_sync(0xffffffffu, dv, src_lane);
          if (MODE == 0 || (MODE == 2 && send_i)) dX = nd; else dY = nd;
          if constexpr (WB) {
            const int cv = MODE == 0 ? cX : (MODE == 1 ? cY : (send_i ? cX : cY));
            const int nc = __shfl_sync(0xffffffffu, cv, src_lane);
            if (MODE == 0 || (MODE == 2 && send_i)) cX = nc; else cY = nc;
          }
        };
        using B1 = std::integral_constant<bool, true>;
        using B0 = std::integral_constant<bool, false>;
        using M0 = std::integral_constant<int, 0>;
        using M1 = std::integral_constant<int, 1>;
        using M2 = std::integral_constant<int, 2>;
        __syncwarp();
        if (any_rot) {
          if (all_i) fused(B1{}, M0{}); else if (all_j) fused(B1{}, M1{}); else fused(B1{}, M2{});
        } else {
          if (all_i) fused(B0{}, M0{}); else if (all_j) fused(B0{}, M1{}); else fused(B0{}, M2{});
        }
        dn = add(add(e[0], e[2]), add(e[1], e[3]));
        if (writer) mbar_arrive(&s_pbar[warp]);
        const long long c5 = RCLK();
        if (via_smem) {
          // the warp-edge slot receives through shared memory and redoes its
          // dot partial
          const T *xr = xbuf + (size_t(par) * NWARP + srcw) * RPC;
          mbar_wait_cta(&s_pbar[srcw], par);
          const double nd = xd[par * NWARP + srcw];
          if (send_i) {
            dX = nd;
#pragma unroll
            for (int u = 0; u < RPT; ++u) X[u] = xr[lane_in + u * TPP];
          } else {
            dY = nd;
#pragma unroll
            for (int u = 0; u < RPT; ++u) Y[u] = xr[lane_in + u * TPP];
          }
          dn = dot_part();
        }
        // J signs of the slot's (possibly new) columns (static per column)
        sX = Jv[min(cX, NMAX - 1)];
        sY = Jv[min(cY, NMAX - 1)];
        __syncwarp();
        const long long c6 = RCLK();
        if (HJB_ROUND_PROFILE && a.prof) {
          ph[0] += c1 - c0; ph[1] += c2 - c1; ph[2] += c3 - c2; ph[3] += c4 - c3;
          ph[4] += c5 - c4; ph[5] += c6 - c5;
        }
      }
      // sweep end: the rotation count and failures are the same in every
      // CTA (every CTA derived every rotation), so a CTA barrier suffices
      if (tid == 0) {
        s_cnt[(sw + 1) & 1] = 0;
        s_swt[(sw + 1) & 1] = 0ull;
      }
      my_swt = sw_n / sw_d;
      if (my_swt > 0.0) atomicMax(&s_swt[sw & 1], static_cast<unsigned long long>(__double_as_longlong(my_swt)));
      my_swt = 0.0;
      sw_n = 0.0;
      sw_d = 1.0;
      const int wc = __reduce_add_sync(0xffffffffu, my_cnt);
      const int wf = __reduce_min_sync(0xffffffffu, my_fail);
      if (lane == 0) {
        if (wc) atomicAdd(&s_cnt[sw & 1], wc);
        if (wf != INT_MAX) atomicMin(&s_fail, wf);
      }
      my_cnt = 0;
      __syncthreads();
      if (s_fail != INT_MAX) {
        status = PV_INDEFINITE;
        break;
      }
      const int cnt = s_cnt[sw & 1];
      nrot_total += cnt;
      if (cnt == 0) break;
      prev_swt = __longlong_as_double(static_cast<long long>(s_swt[sw & 1]));
    }
  }
  t_jac = clock64();

  // ------------------------------------------------------------------ W = R0^-1 R
  if (my_big) atomicAdd(&s_big, my_big);
  my_maxt = mt_n / mt_d;
  if (my_maxt > 0.0) atomicMax(&s_maxt, static_cast<unsigned long long>(__double_as_longlong(my_maxt)));
  const int nmax = a.nmax;
  T *Wout = reinterpret_cast<T *>(a.W) + int64_t(item_id) * nmax * nmax;
  T *Rout = a.Rout ? reinterpret_cast<T *>(a.Rout) + int64_t(item_id) * nmax * nmax : nullptr;
  if constexpr (Cfg::FAST) {
    if (fast) {
      // R0 = [[diag(s), A/s], [0, U]] (s = sqrt(L_i)), so W = R0^-1 R_final is
      //   W_b = U^-1 F_b,   W_t = F_t / s - (A W_b) / s^2.
      // R_final goes through the W buffer (L2); CTA r then owns the columns
      // [r RPC, (r+1) RPC): one warp per column group back-substitutes with
      // its lanes holding rows (shuffle broadcast of each solved row).
      constexpr int UL = Cfg::UL, RV = Cfg::RV;
      constexpr int CW = (RPC + NWARP - 1) / NWARP;
      const T *Ug = reinterpret_cast<const T *>(a.uscr) + int64_t(item_id) * Cfg::UB * UL;  // L2
      if constexpr (Cfg::U_SMEM) {
        for (int e = tid; e < Cfg::UB * UL; e += NT) Rs[e] = __ldcg(Ug + e);
      }
      const T *U = Cfg::U_SMEM ? Rs : Ug;
      if (mode == PV_EPILOGUE && Rout) {  // R_final (from the Jacobi kernel) for the optional output
        for (int e = tid; e < RPC * N; e += NT) {
          const int gl = e % RPC, c = e / RPC;
          const int g = row0 + gl;
          if (g < N) Rout[g + int64_t(c) * nmax] = __ldcg(Wout + g + int64_t(c) * nmax);
        }
      }
      if (mode == PV_FULL && in_ring) {
#pragma unroll
        for (int u = 0; u < RPT; ++u) {
          const int g = row0 + lane_in + u * TPP;
          if (g >= N) continue;
          if (cX < N) Wout[g + int64_t(cX) * nmax] = X[u];
          if (cY < N) Wout[g + int64_t(cY) * nmax] = Y[u];
          if (Rout) {
            if (cX < N) Rout[g + int64_t(cX) * nmax] = X[u];
            if (cY < N) Rout[g + int64_t(cY) * nmax] = Y[u];
          }
        }
      }
      double *rdg = npart;  // 1 / U[k][k]
      for (int k = tid; k < nu; k += NT) rdg[k] = 1.0 / re(__ldcg(Ug + k + k * UL));
      __threadfence();
      cluster_sync<C>();
      const int c0 = crank * RPC, c1 = min(N, c0 + RPC);
      const int cw0 = c0 + warp * CW;
      T f[CW][RV];
#pragma unroll
      for (int cc = 0; cc < CW; ++cc)
#pragma unroll
        for (int v = 0; v < RV; ++v) {
          const int c = cw0 + cc, i = lane + 32 * v;
          f[cc][v] = (c < c1 && i < nu) ? __ldcg(Wout + (nt + i) + int64_t(c) * nmax) : S<T>::zero();
        }
      if (cw0 < c1) {
        for (int k = nu - 1; k >= 0; --k) {
          const int ow = k & 31, vk = k >> 5;
          const double rk = rdg[k];
          T wk[CW];
#pragma unroll
          for (int cc = 0; cc < CW; ++cc) {
            T fk = f[cc][0];
#pragma unroll
            for (int v = 1; v < RV; ++v)
              if (v == vk) fk = f[cc][v];
            wk[cc] = scale(shfl_idx(fk, ow), rk);
          }
#pragma unroll
          for (int v = 0; v < RV; ++v) {
            const int i = lane + 32 * v;
            if (i < k) {
              const T uik = Cfg::U_SMEM ? U[i + k * UL] : __ldcg(U + i + k * UL);
#pragma unroll
              for (int cc = 0; cc < CW; ++cc) f[cc][v] = sub(f[cc][v], mul(uik, wk[cc]));
            } else if (i == k) {
#pragma unroll
              for (int cc = 0; cc < CW; ++cc) f[cc][v] = wk[cc];
            }
          }
        }
      }
#pragma unroll
      for (int cc = 0; cc < CW; ++cc)
#pragma unroll
        for (int v = 0; v < RV; ++v) {
          const int c = cw0 + cc, i = lane + 32 * v;
          if (c < c1 && i < nu) Wout[(nt + i) + int64_t(c) * nmax] = f[cc][v];
        }
      if (nt > 0) {
        // W_t = F_t / s - (A W_b) / s^2 for this CTA's columns
        T *Wb = Rs;  // [nu][RPC] staging (column stride UL)
        __syncthreads();
#pragma unroll
        for (int cc = 0; cc < CW; ++cc)
#pragma unroll
          for (int v = 0; v < RV; ++v) {
            const int c = cw0 + cc, i = lane + 32 * v;
            if (c < c1 && i < nu) Wb[i + (c - c0) * UL] = f[cc][v];
          }
        __syncthreads();
        const int ncol = max(0, c1 - c0);
        for (int e = tid; e < nt * ncol; e += NT) {
          const int h = e % nt, cl = e / nt;
          T acc0 = S<T>::zero(), acc1 = S<T>::zero();
          int l = 0;
          for (; l + 1 < nu; l += 2) {
            acc0 = add(acc0, mul(A[h + int64_t(l) * bmax], Wb[l + cl * UL]));
            acc1 = add(acc1, mul(A[h + int64_t(l + 1) * bmax], Wb[(l + 1) + cl * UL]));
          }
          if (l < nu) acc0 = add(acc0, mul(A[h + int64_t(l) * bmax], Wb[l + cl * UL]));
          const double lh = lam[h];
          const T fv = __ldcg(Wout + h + int64_t(c0 + cl) * nmax);
          Wout[h + int64_t(c0 + cl) * nmax] = sub(divr(fv, sqrt(lh)), divr(add(acc0, acc1), lh));
        }
      }
    }
  }
  if (!fast) {
    T *Fs = Ws;  // RPC x NMAX slab (scratch region is large enough)
    __syncthreads();
    if (mode == PV_EPILOGUE) {  // R_final rows of this CTA from the Jacobi kernel's output
      for (int e = tid; e < RPC * NMAX; e += NT) {
        const int gl = e % RPC, c = e / RPC;
        const int g = row0 + gl;
        Fs[c * RS + gl] = (g < N && c < N) ? __ldcg(Wout + g + int64_t(c) * nmax) : S<T>::zero();
      }
    }
  #pragma unroll
    for (int u = 0; u < RPT; ++u) {
      if (!in_ring || mode != PV_FULL) break;
      const int row = lane_in + u * TPP;
      Fs[cX * RS + row] = X[u];
      Fs[cY * RS + row] = Y[u];
    }
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

    {
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
  if (crank == 0 && tid == 0 && mode == PV_FULL) {
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
  static DeviceFlags attr_flags;
  bool *attr = attr_flags.here();
  if (!attr) return cudaErrorInvalidDevice;
  if (!*attr) {
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(Cfg::SMEM));
    if (e != cudaSuccess) return e;
    if (C > 8) {
      e = cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      if (e != cudaSuccess) return e;
    }
    *attr = true;
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

#ifndef HJB_PIVOT_CPLX_TU
size_t pivot_check_elems(int nmax) {
  const size_t nb = nmax / 4;
  return 16 * (nb * (nb + 1) / 2) * 16;  // up to 16 CTAs per cluster
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
  const size_t ub = nmax / 2;
  const size_t scr = std::max<size_t>(slab, 16 * nmax);
  (void)ub;
  return (slab + scr) * w + 2 * c * (nmax / 2) * w + 2 * nmax * w + 3 * nmax * 8 + nmax * 4;
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

#endif  // !HJB_PIVOT_CPLX_TU

// when set, launch_pivot only reports max active clusters
#ifdef HJB_PIVOT_CPLX_TU
extern int g_query_clusters;
#else
int g_query_clusters = 0;
#endif

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

// The instantiated (NMAX, C, NT) table.  Build with -DHJB_PIVOT_DEV to
// compile only the configurations of the BASELINE bench workloads (fast
// iteration on the kernel).
template <typename T, int NMAX, int C, int NT>
constexpr bool pivot_allowed() {
#ifdef HJB_PIVOT_DEV
  return (S<T>::cx && NMAX == 128 && (C == 4 || C == 8 || C == 16)) || (NMAX == 64 && NT == 256) ||
         (!S<T>::cx && NMAX == 128 && NT == 256 && (C == 2 || C == 4));
#else
  if (NMAX == 32) return C <= 2 && NT <= 256;
  if (NMAX == 64) return C <= 4 && NT <= 256;
  if (NMAX == 128) return C >= 2 && C <= 8;
  return C >= 4;
#endif
}

template <typename T, int NMAX, int C, int NT>
static cudaError_t launch_if_valid(const PivotArgs &a, cudaStream_t st) {
  constexpr int P2 = NMAX / 2, RPC = NMAX / C;
  if constexpr (pivot_allowed<T, NMAX, C, NT>() && RPC >= 4 && NT >= P2 && NT / P2 <= 32 && NT / P2 <= RPC &&
                NT <= RPC * NMAX) {
    if constexpr (PivCfg<T, NMAX, C, NT>::SMEM <= 227 * 1024) {
      if (g_query_clusters) return query_clusters<T, NMAX, C, NT>(&g_query_clusters);
      return launch_pivot_t<T, NMAX, C, NT>(a, st);
    }
  }
  return cudaErrorInvalidConfiguration;
}

#ifndef HJB_PIVOT_CPLX_TU
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
#endif  // !HJB_PIVOT_CPLX_TU

template <typename T, int NMAX, int C>
static cudaError_t dispatch_nt(const PivotArgs &a, int nt, cudaStream_t st) {
  switch (nt) {
    case 128: return launch_if_valid<T, NMAX, C, 128>(a, st);
    case 256: return launch_if_valid<T, NMAX, C, 256>(a, st);
    case 512: return launch_if_valid<T, NMAX, C, 512>(a, st);
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

#ifdef HJB_PIVOT_CPLX_TU
cudaError_t launch_pivot_cplx(const PivotArgs &a, int c, int nt, cudaStream_t st) {
  switch (a.nmax) {
    case 32: return dispatch_c<cplx, 32>(a, c, nt, st);
    case 64: return dispatch_c<cplx, 64>(a, c, nt, st);
    case 128: return dispatch_c<cplx, 128>(a, c, nt, st);
    case 256: return dispatch_c<cplx, 256>(a, c, nt, st);
  }
  return cudaErrorInvalidValue;
}
#else
cudaError_t launch_pivot_cplx(const PivotArgs &a, int c, int nt, cudaStream_t st);  // pivot_c128.cu

void pivot_tune(int threads, int cluster) {
  g_tune_threads = threads;
  g_tune_cluster = cluster;
}

int pivot_default_threads(bool cx, int nmax, int c) {
  // smallest CTA whose register-resident slab (4 arrays x RPT rows) stays
  // within ~4 complex / 8 real rows per thread
  const int p2 = nmax / 2, rpc = nmax / c, cap = 8;
  for (int nt = 128; nt <= 512; nt *= 2) {
    const int tpp = nt / p2;
    if (tpp < 1 || tpp > 32 || tpp > rpc) continue;
    if (rpc / tpp <= cap) return nt;
  }
  return 512;
}

int pivot_choose_cluster(bool cx, int nmax, int count) {
  return g_tune_cluster > 0 ? g_tune_cluster : pivot_default_cluster(cx, nmax, count);
}

int pivot_choose_threads(bool cx, int nmax, int c) {
  return g_tune_threads > 0 ? g_tune_threads : pivot_default_threads(cx, nmax, c);
}

cudaError_t launch_pivot(bool cx, const PivotArgs &a, int cluster, cudaStream_t st, int *cluster_used) {
  int c = cluster > 0 ? cluster : (g_tune_cluster > 0 ? g_tune_cluster : pivot_default_cluster(cx, a.nmax, a.count));
  const int nt = g_tune_threads > 0 ? g_tune_threads : pivot_default_threads(cx, a.nmax, c);
  if (cluster_used) *cluster_used = c;
  if (cx) return launch_pivot_cplx(a, c, nt, st);
  switch (a.nmax) {
    case 32: return dispatch_c<double, 32>(a, c, nt, st);
    case 64: return dispatch_c<double, 64>(a, c, nt, st);
    case 128: return dispatch_c<double, 128>(a, c, nt, st);
    case 256: return dispatch_c<double, 256>(a, c, nt, st);
  }
  return cudaErrorInvalidValue;
}
#endif  // HJB_PIVOT_CPLX_TU

}  // namespace hjb
