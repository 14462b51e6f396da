// Jacobi kernel: the inner level of the 2F step (rotations.py:203-223) as a
// ring of rings.
//
// The pivot factor R (N x N, from the structured Cholesky of the pivot
// kernel's prologue) is diagonalised by one-sided J-Jacobi sweeps until a
// sweep applies no rotation.  One thread-block cluster of C CTAs per pivot;
// every warp of the cluster is a RING WORKER of the reference's own parallel
// ordering (strategies.py:58-136, round-robin) applied to 2*Q column
// SUB-BLOCKS of SPW columns (Q = C * W workers):
//
//   * a warp holds two sub-blocks (its i and j sub-block, 2*SPW columns) in
//     registers; lane l holds rows l, l+32, ... of all of them, so a pair's
//     dot product is a butterfly reduction over the warp and NO column data
//     moves inside a step;
//   * step 0 of an inner sweep pairs every two of the warp's own columns
//     (2*SPW - 1 rounds of SPW disjoint pairs, circle method); every later
//     step pairs the i sub-block with the j sub-block (SPW rounds);
//   * after every step the worker's stepper (round_robin_step,
//     strategies.py:95-136) sends one sub-block to ring neighbour q-1 (odd
//     inner sweeps) or q+1 (even, strategies.py:69-72) and receives one:
//     st.async into the neighbour's inbox (shared memory of its CTA, DSMEM
//     across CTAs) completing on the neighbour's mbarrier; a second mbarrier
//     per link returns the empty slot.  Warps are coupled only to their ring
//     neighbours -- there is no CTA or cluster barrier inside a sweep;
//   * the D cache (rotations.py:217, _kernels.py:80-81) travels with its
//     column; one cluster reduction of the rotation count per inner sweep is
//     the convergence test (rotations.py:220-222).
//
// Per sweep: (2Q - 1) steps, N - 1 rounds -- every pair of columns meets once
// (the order is replayed exactly by the oracle, RingOfRings).  Input R0 and
// output R_final live in global memory ([count][ld*ld], column-major); the
// pivot kernel forms R0 before and W = R0^-1 R_final after.
#include <cooperative_groups.h>

#include <cfloat>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <type_traits>
#include <utility>

#include "common.cuh"
#include "kernels.h"
#include "rotation.cuh"

namespace cg = cooperative_groups;

// per-warp phase clocks (tools/jac_bench.py); compiled out unless
// -DHJB_JAC_PROF=1 (a separate profiling build of the library)
#ifndef HJB_JAC_PROF
#define HJB_JAC_PROF 0
#endif
#ifndef HJB_JAC_MINB_SMALL  // resident CTAs per SM for 4-warp CTAs of pivots of order <= 128
#define HJB_JAC_MINB_SMALL 3
#endif
#ifndef HJB_JAC_FUSE  // 1: gather-first + fused next-round dots (slower on B200: register pressure)
#define HJB_JAC_FUSE 0
#endif
#if HJB_JAC_PROF
#define JCLK() clock64()
#else
#define JCLK() 0LL
#endif

namespace hjb {

namespace {

constexpr double kEpsJ = 2.220446049250313e-16;

template <int N, typename F, int... I>
__device__ __forceinline__ void sfor_impl(F &&f, std::integer_sequence<int, I...>) {
  (f(std::integral_constant<int, I>{}), ...);
}
// static for: f(integral_constant<0>) ... f(integral_constant<N-1>)
template <int N, typename F>
__device__ __forceinline__ void sfor(F &&f) {
  sfor_impl<N>(static_cast<F &&>(f), std::make_integer_sequence<int, N>{});
}

constexpr int ilog2(int x) { return x <= 1 ? 0 : 1 + ilog2(x / 2); }

// Phase-A pairing of the warp's 2*SPW local slots (circle method): round r,
// pair k -> (slot a, slot b), a < b.
template <int SPW>
struct PhaseA {
  static constexpr int M = 2 * SPW;
  __host__ __device__ static constexpr int x(int r, int k) { return k == 0 ? M - 1 : (r + k) % (M - 1); }
  __host__ __device__ static constexpr int y(int r, int k) { return k == 0 ? r : (r - k + (M - 1)) % (M - 1); }
  __host__ __device__ static constexpr int a(int r, int k) { return x(r, k) < y(r, k) ? x(r, k) : y(r, k); }
  __host__ __device__ static constexpr int b(int r, int k) { return x(r, k) < y(r, k) ? y(r, k) : x(r, k); }
};

// mbarrier / DSMEM helpers
__device__ __forceinline__ void jb_init(uint64_t *bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void jb_arrive_expect(uint64_t *bar, unsigned tx) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(tx)
               : "memory");
}
// wait for completion of the phase with the given parity (acquire at cluster
// scope: the data or the empty slot was produced by another CTA)
__device__ __forceinline__ void jb_wait(uint64_t *bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "JB_WAIT_%=:\n"
      " mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra JB_WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void jb_wait_cta(uint64_t *bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "JB_WAITC_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra JB_WAITC_%=;\n}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void jb_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ uint32_t jb_mapa(uint32_t addr, int rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
__device__ __forceinline__ void jb_arrive_remote(uint32_t rbar) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];\n" ::"r"(rbar) : "memory");
}
__device__ __forceinline__ void jb_st_async(uint32_t raddr, double v, uint32_t rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];\n" ::"r"(raddr),
               "l"(__double_as_longlong(v)), "r"(rbar)
               : "memory");
}
__device__ __forceinline__ void jb_st_async(uint32_t raddr, cplx v, uint32_t rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.b64 [%0], {%1, %2}, [%3];\n" ::"r"(raddr),
               "l"(__double_as_longlong(v.x)), "l"(__double_as_longlong(v.y)), "r"(rbar)
               : "memory");
}
template <int C>
__device__ __forceinline__ void jb_cluster_sync() {
  if constexpr (C > 1) {
    asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
    asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
  } else {
    __syncthreads();
  }
}

// round_robin_step of strategies.py:95-136 on one worker's state
struct Stepper {
  int ip, jp, ib, jb;  // 1-based, as the reference
  __device__ __forceinline__ void init(int q, int nbl) {
    ip = q + 1;
    jp = nbl - q;
    ib = ip;
    jb = jp;
  }
  // returns the sent block; ib/jb become the new layout
  __device__ __forceinline__ int step(int nbl) {
    int snd;
    if (ip + jp > nbl) {
      if (jp < nbl) {
        snd = ib;
        ip += 1;
        if (ip < jp) {
          ib = ip;
        } else {
          ip = jp;
          ib = jb;
          jp = nbl;
          jb = nbl;
        }
      } else if (ip > nbl / 2) {
        snd = ib;
        ip = ip - nbl / 2 + 1;
        ib = ip;
      } else {
        snd = jb;
        jp = ip + 1;
        jb = jp;
      }
    } else {
      snd = jb;
      jp += 1;
      jb = jp;
    }
    return snd;
  }
};

}  // namespace

template <typename T, int N, int C, int W, int SPW>
struct JacCfg {
  static constexpr int NT = 32 * W;
  static constexpr int CPW = 2 * SPW;           // columns per warp
  static constexpr int RPL = N / 32;             // rows per lane
  static constexpr int Q = C * W;                // ring workers
  static constexpr int NBL = 2 * Q;              // sub-blocks
  static constexpr int LS = ilog2(SPW);
  static constexpr int GS = 32 >> LS;             // lanes per pair group after the reduce-scatter
  static constexpr int MSG = SPW * N + SPW;      // inbox message: SPW columns + their D values (elements)
  static constexpr unsigned MSG_BYTES = MSG * sizeof(T);
  static_assert(N == 2 * C * W * SPW, "N = 2 C W SPW");
  static_assert(N % 32 == 0 && (SPW & (SPW - 1)) == 0 && SPW <= 8, "shape");
  // shared memory: inbox [W][2][MSG] T, full/empty barriers [W][2], J [N]
  static constexpr size_t OFF_IN = 0;
  static constexpr size_t OFF_BAR = OFF_IN + size_t(W) * 2 * MSG * sizeof(T);
  static constexpr size_t OFF_J = OFF_BAR + size_t(W) * 4 * sizeof(uint64_t);
  static constexpr size_t SMEM = OFF_J + N * sizeof(int);
};

template <typename T, int N, int C, int W, int SPW, int MINB>
__global__ void __launch_bounds__(32 * W, MINB) jacobi_kernel(JacobiArgs a) {
  using Cfg = JacCfg<T, N, C, W, SPW>;
  constexpr int RPL = Cfg::RPL, CPW = Cfg::CPW, Q = Cfg::Q, NBL = Cfg::NBL, LS = Cfg::LS, GS = Cfg::GS;
  constexpr int MSG = Cfg::MSG;
  extern __shared__ __align__(16) unsigned char smem[];
  T *inbox = reinterpret_cast<T *>(smem + Cfg::OFF_IN);         // [W][2][MSG]
  uint64_t *bars = reinterpret_cast<uint64_t *>(smem + Cfg::OFF_BAR);  // [W][full 2, empty 2]
  int *Jv = reinterpret_cast<int *>(smem + Cfg::OFF_J);
  __shared__ int s_cnt[2], s_big[2], s_fail[2], s_chk[2];
  __shared__ unsigned long long s_maxt, s_swt[2];

  int crank = 0;
  if constexpr (C > 1) crank = int(cg::this_cluster().block_rank());
  const int item_id = blockIdx.x / C;
  const Item it = a.items[item_id];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int q = crank * W + warp;  // ring worker
  const int ni = it.ni, nj = it.nj, Nq = ni + nj;
  int64_t *st = a.stats + int64_t(item_id) * ST_N;
  // the prologue failed (DefinitenessError): nothing to diagonalise
  if (__ldcg(st + ST_STATUS) != PV_OK) return;  // uniform over the cluster
  const int ld = a.ld;
  const T *R0 = reinterpret_cast<const T *>(a.R0) + int64_t(item_id) * ld * ld;
  T *Rf = reinterpret_cast<T *>(a.Rout) + int64_t(item_id) * ld * ld;

  for (int c = tid; c < N; c += Cfg::NT)
    Jv[c] = c < ni ? a.signs[it.oi + c] : (c < Nq ? a.signs[it.oj + (c - ni)] : 1);
  if (tid < 2 * W) {
    // full[dir] of warp w: the receiver's own arrival (+ expect_tx when the
    // sender is in another CTA, + the sender's arrival when it is local);
    // dir 0 receives from q+1 (remote for the last warp), dir 1 from q-1
    // (remote for warp 0); empty[dir]: the receiver's arrival
    const int w = tid >> 1, dr = tid & 1;
    const bool remote = C > 1 && (dr == 0 ? w == W - 1 : w == 0);
    jb_init(&bars[w * 4 + dr], remote ? 1 : 2);
    jb_init(&bars[w * 4 + 2 + dr], 1);
  }
  if (tid == 0) {
    s_cnt[0] = s_cnt[1] = 0;
    s_big[0] = s_big[1] = 0;
    s_fail[0] = s_fail[1] = INT_MAX;
    s_chk[0] = s_chk[1] = 0;
    s_swt[0] = s_swt[1] = 0ull;
    s_maxt = 0ull;
  }
  if (tid == 0) asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");

  // ---- this worker's two sub-blocks, rows lane + 32u ----
  Stepper sp;
  sp.init(q, NBL);
  T V[RPL][CPW];
  double D[CPW] = {};
  auto col_of = [&](int slot) { return (slot < SPW ? (sp.ib - 1) * SPW + slot : (sp.jb - 1) * SPW + slot - SPW); };
#pragma unroll
  for (int c = 0; c < CPW; ++c) {
    const int col = col_of(c);
#pragma unroll
    for (int u = 0; u < RPL; ++u) V[u][c] = __ldcg(R0 + (lane + 32 * u) + int64_t(col) * ld);
  }
  jb_cluster_sync<C>();  // Jv, barriers initialised in every CTA

  const double otol = a.orth_tol > 0.0 ? a.orth_tol : sqrt(double(Nq)) * kEpsJ;
  const double otol2 = otol * otol;
  const double qtol = a.quad_tol > 0.0 ? a.quad_tol : double(Nq) * kEpsJ;
  int my_cnt = 0, my_big = 0, my_fail = INT_MAX;
  double my_maxt = 0.0, my_swt = 0.0, prev_swt = 1.0;
  long long nrot_total = 0, big_total = 0;
  int sweeps = 0, status = PV_OK;
  long long pf[8] = {0, 0, 0, 0, 0, 0, 0, 0};  // round, empty wait, send, full wait, receive, sweep end, rounds, t0
  pf[7] = JCLK();

  // per-slot column state: J sign and "real column" flag (ids >= Nq are padding)
  // JAC_CROSS (the B variants' annihilation pass, parallel.py:170-174 /
  // _kernels.py:41-52 with diag_bl = False): only pairs with one column in
  // each block rotate; the sweep still visits every pair of columns
  const bool cross = a.mode == JAC_CROSS;
  int sg[CPW];
  bool live[CPW], side[CPW];
  auto refresh_slot = [&](int c) {
    const int col = col_of(c);
    sg[c] = Jv[col];
    live[c] = col < Nq;
    side[c] = col >= ni;
  };
  sfor<CPW>([&](auto c) { refresh_slot(c); });

  // -------------------------------------------------------------- one round
  // The round's SPW pairs (slot A(k), slot B(k)); A plays r, B plays s.  The
  // dot partials are reduce-scattered over the warp (lane group kk owns pair
  // kk), each group derives its pair's rotation, the parameters of all pairs
  // are gathered by shuffles, and the rotations are applied row by row fused
  // with the next round's dot partials (HJB_JAC_FUSE; when the next pairing is
  // in the same step, NEXT).
  T dp[SPW];
  auto dots = [&](auto pa, auto pb) {
    sfor<SPW>([&](auto k) {
      constexpr int A = decltype(pa(k))::value, B = decltype(pb(k))::value;
      T d0 = S<T>::zero(), d1 = S<T>::zero();
#pragma unroll
      for (int u = 0; u < RPL; u += 2) {
        d0 = cfma(V[u][A], V[u][B], d0);
        if (u + 1 < RPL) d1 = cfma(V[u + 1][A], V[u + 1][B], d1);
      }
      dp[k] = add(d0, d1);
    });
  };
  auto round = [&](auto pa, auto pb, auto na, auto nb, auto has_next) {
    constexpr bool NEXT = HJB_JAC_FUSE && decltype(has_next)::value;
    const long long r0 = JCLK();
    // butterfly reduce-scatter: lane keeps pair kk = lane >> (5 - LS)
#pragma unroll
    for (int j = 0; j < LS; ++j) {
      const int dist = 16 >> j;
      const bool hi = lane & dist;
      const int half = SPW >> (j + 1);
#pragma unroll
      for (int x = 0; x < half; ++x) {
        const T snd = hi ? dp[x] : dp[x + half];
        const T keep = hi ? dp[x + half] : dp[x];
        dp[x] = add(keep, shfl_xor(snd, dist));
      }
    }
    T acc = dp[0];
#pragma unroll
    for (int dist = 16 >> LS; dist >= 1; dist >>= 1) acc = add(acc, shfl_xor(acc, dist));
    const int kk = lane >> (5 - LS);
    double dr = 0.0, ds = 0.0;
    int sr = 1, ss = 1, ar = 0, as = 0;
    bool lv = false;
    sfor<SPW>([&](auto k) {
      constexpr int A = decltype(pa(k))::value, B = decltype(pb(k))::value;
      if (kk == k) {
        dr = D[A];
        ds = D[B];
        sr = sg[A];
        ss = sg[B];
        lv = live[A] && live[B] && (!cross || side[A] != side[B]);
        ar = A;
        as = B;
      }
    });
    bool rot = lv && !(abs2(acc) <= otol2 * (dr * ds));  // _kernels.py:57
    RotCoef<T> p;
    p.cp = S<T>::one();
    p.sp = S<T>::zero();
    p.hs = 0.0;
    p.cs = 1.0;
    double te_n = 0.0, te_h = 0.0;
    const bool any = __any_sync(0xffffffffu, rot);
    if (any && rot) {
      const RotCoef<T> r = rot_coef<T>(acc, dr, ds, sr == ss, otol2);
      if (r.code == 1) {
        p = r;
        te_n = r.num * r.eta / r.den;  // t * eta (_kernels.py:80-81)
        te_h = r.hyp;
        if ((lane & (GS - 1)) == 0) {
          ++my_cnt;
          my_big += fabs(r.num) > qtol * r.den;  // |t| > quad_tol
          my_maxt = fmax(my_maxt, fabs(r.num) / r.den);
          my_swt = fmax(my_swt, fabs(r.num) / r.den);
        }
      } else {
        rot = false;
        if (r.code < 0 && (lane & (GS - 1)) == 0) {
          const int cr = col_of(ar), cs = col_of(as);
          my_fail = min(my_fail, min(cr, cs) * 4096 + max(cr, cs));
        }
      }
    }
#if HJB_JAC_FUSE
    // gather every pair's parameters (first lane of its group), then one
    // fused pass over the rows
    RotCoef<T> pk[SPW];
    bool rk[SPW];
    if (any) {
      sfor<SPW>([&](auto k) {
        constexpr int A = decltype(pa(k))::value, B = decltype(pb(k))::value;
        const int src = k * GS;
        rk[k] = __shfl_sync(0xffffffffu, rot, src);
        pk[k].cp = shfl_idx(p.cp, src);
        pk[k].sp = shfl_idx(p.sp, src);
        pk[k].hs = __shfl_sync(0xffffffffu, p.hs, src);
        pk[k].cs = __shfl_sync(0xffffffffu, p.cs, src);
        const double te = __shfl_sync(0xffffffffu, te_n, src);
        const double th = __shfl_sync(0xffffffffu, te_h, src);
        if (rk[k]) {
          D[A] = fma(th, te, D[A]);
          D[B] = D[B] + te;
        }
      });
    }
    if constexpr (NEXT) sfor<SPW>([&](auto k) { dp[k] = S<T>::zero(); });
#pragma unroll
    for (int u = 0; u < RPL; ++u) {
      if (any) {
        sfor<SPW>([&](auto k) {
          constexpr int A = decltype(pa(k))::value, B = decltype(pb(k))::value;
          if (rk[k]) rot_fold<T>(V[u][A], V[u][B], pk[k]);
        });
      }
      if constexpr (NEXT) {
        sfor<SPW>([&](auto k) {
          constexpr int A = decltype(na(k))::value, B = decltype(nb(k))::value;
          dp[k] = cfma(V[u][A], V[u][B], dp[k]);
        });
      }
    }
#else
    if (any) {
      sfor<SPW>([&](auto k) {
        constexpr int A = decltype(pa(k))::value, B = decltype(pb(k))::value;
        const int src = k * GS;
        const bool rk = __shfl_sync(0xffffffffu, rot, src);
        if (rk) {
          RotCoef<T> pk;
          pk.cp = shfl_idx(p.cp, src);
          pk.sp = shfl_idx(p.sp, src);
          pk.hs = __shfl_sync(0xffffffffu, p.hs, src);
          pk.cs = __shfl_sync(0xffffffffu, p.cs, src);
          const double te = __shfl_sync(0xffffffffu, te_n, src);
          const double th = __shfl_sync(0xffffffffu, te_h, src);
#pragma unroll
          for (int u = 0; u < RPL; ++u) rot_fold<T>(V[u][A], V[u][B], pk);
          D[A] = fma(th, te, D[A]);
          D[B] = D[B] + te;
        }
      });
    }
#endif
    if constexpr (!NEXT) {
      if constexpr (decltype(has_next)::value) dots(na, nb);
    }
    if (HJB_JAC_PROF) {
      pf[0] += JCLK() - r0;
      pf[6] += 1;
    }
  };
  using BT = std::integral_constant<bool, true>;
  using BF = std::integral_constant<bool, false>;

  // phase A: all pairs of the warp's 2 SPW columns; phase B: i x j
  auto phase_a = [&]() {
    dots([](auto k) { return std::integral_constant<int, PhaseA<SPW>::a(0, decltype(k)::value)>{}; },
         [](auto k) { return std::integral_constant<int, PhaseA<SPW>::b(0, decltype(k)::value)>{}; });
    sfor<CPW - 1>([&](auto r) {
      constexpr int R = decltype(r)::value;
      constexpr int R1 = R + 1 < CPW - 1 ? R + 1 : R;
      auto pa = [](auto k) { return std::integral_constant<int, PhaseA<SPW>::a(R, decltype(k)::value)>{}; };
      auto pb = [](auto k) { return std::integral_constant<int, PhaseA<SPW>::b(R, decltype(k)::value)>{}; };
      auto na = [](auto k) { return std::integral_constant<int, PhaseA<SPW>::a(R1, decltype(k)::value)>{}; };
      auto nb = [](auto k) { return std::integral_constant<int, PhaseA<SPW>::b(R1, decltype(k)::value)>{}; };
      if constexpr (R + 1 < CPW - 1) round(pa, pb, na, nb, BT{});
      else round(pa, pb, na, nb, BF{});
    });
  };
  auto phase_b = [&]() {
    dots([](auto k) { return std::integral_constant<int, decltype(k)::value>{}; },
         [](auto k) { return std::integral_constant<int, SPW + decltype(k)::value>{}; });
    sfor<SPW>([&](auto r) {
      constexpr int R = decltype(r)::value;
      auto pa = [](auto k) { return std::integral_constant<int, decltype(k)::value>{}; };
      auto pb = [](auto k) { return std::integral_constant<int, SPW + (decltype(k)::value + R) % SPW>{}; };
      auto nb = [](auto k) { return std::integral_constant<int, SPW + (decltype(k)::value + R + 1) % SPW>{}; };
      if constexpr (R + 1 < SPW) round(pa, pb, pa, nb, BT{});
      else round(pa, pb, pa, nb, BF{});
    });
  };

  // ---------------------------------------------------------- the exchange
  // strategies.py:69-72: odd sweeps send to q-1 and receive from q+1.  Links
  // inside a CTA use plain shared-memory stores and a counted arrival; the
  // two links that cross a CTA boundary use st.async into the neighbour's
  // shared memory (DSMEM) completing on its barrier's transaction count.
  int g_dn = 0, g_up = 0;  // messages per direction (equal in every worker)
  auto exchange = [&](int nsweep) {
    const int old_i = sp.ib, old_j = sp.jb;
    const int snd = sp.step(NBL);
    const bool send_i = snd == old_i;
    const bool swap = send_i && sp.ib == old_j;  // j moved into the i slots, receive into j
    const int d = (nsweep & 1) ? 0 : 1;
    const int dst = (nsweep & 1) ? (q + Q - 1) % Q : (q + 1) % Q;
    const int srcw = (nsweep & 1) ? (q + 1) % Q : (q + Q - 1) % Q;
    const int dc = dst / W, dw = dst % W, sc = srcw / W, sw = srcw % W;
    const bool rsend = C > 1 && dc != crank, rrecv = C > 1 && sc != crank;
    const int g = d == 0 ? g_dn++ : g_up++;
    uint64_t *full = &bars[warp * 4 + d];
    uint64_t *empty = &bars[warp * 4 + 2 + d];
    // send: wait until the receiver has consumed this link's previous message
    const long long x0 = JCLK();
    if (g > 0) {
      if (rsend) jb_wait(empty, (g - 1) & 1);
      else jb_wait_cta(empty, (g - 1) & 1);
    }
    const long long x1 = JCLK();
    T *box_out = inbox + (size_t(dw) * 2 + d) * MSG;
    auto send = [&](auto base) {
      constexpr int B0 = decltype(base)::value;
      double dv = 0.0;
      sfor<SPW>([&](auto k) {
        if (lane == decltype(k)::value) dv = D[B0 + decltype(k)::value];
      });
      if (rsend) {
        const uint32_t rbox = jb_mapa(smem_u32(box_out), dc);
        const uint32_t rbar = jb_mapa(smem_u32(&bars[dw * 4 + d]), dc);
        sfor<SPW>([&](auto k) {
          constexpr int K = decltype(k)::value;
#pragma unroll
          for (int u = 0; u < RPL; ++u)
            jb_st_async(rbox + uint32_t((K * N + lane + 32 * u) * sizeof(T)), V[u][B0 + K], rbar);
        });
        if (lane < SPW) jb_st_async(rbox + uint32_t((SPW * N + lane) * sizeof(T)), scale(S<T>::one(), dv), rbar);
      } else {
        sfor<SPW>([&](auto k) {
          constexpr int K = decltype(k)::value;
#pragma unroll
          for (int u = 0; u < RPL; ++u) box_out[K * N + lane + 32 * u] = V[u][B0 + K];
        });
        if (lane < SPW) box_out[SPW * N + lane] = scale(S<T>::one(), dv);
        __syncwarp();
        if (lane == 0) jb_arrive(&bars[dw * 4 + d]);
      }
    };
    if (send_i) send(std::integral_constant<int, 0>{});
    else send(std::integral_constant<int, SPW>{});
    // receive into the vacated slots
    if (swap) {
      sfor<SPW>([&](auto k) {
        constexpr int K = decltype(k)::value;
#pragma unroll
        for (int u = 0; u < RPL; ++u) V[u][K] = V[u][SPW + K];
        D[K] = D[SPW + K];
      });
    }
    if (lane == 0) {
      if (rrecv) jb_arrive_expect(full, Cfg::MSG_BYTES);
      else jb_arrive(full);
    }
    const long long x2 = JCLK();
    jb_wait_cta(full, g & 1);
    const long long x3 = JCLK();
    const T *box = inbox + (size_t(warp) * 2 + d) * MSG;
    auto recv = [&](auto base) {
      constexpr int B0 = decltype(base)::value;
      sfor<SPW>([&](auto k) {
        constexpr int K = decltype(k)::value;
#pragma unroll
        for (int u = 0; u < RPL; ++u) V[u][B0 + K] = box[K * N + lane + 32 * u];
        D[B0 + K] = re(box[SPW * N + K]);
      });
    };
    if (send_i && !swap) recv(std::integral_constant<int, 0>{});
    else recv(std::integral_constant<int, SPW>{});
    __syncwarp();
    if (lane == 0) {
      if (rrecv) jb_arrive_remote(jb_mapa(smem_u32(&bars[sw * 4 + 2 + d]), sc));
      else jb_arrive(&bars[sw * 4 + 2 + d]);
    }
    sfor<CPW>([&](auto c) { refresh_slot(c); });
    if (HJB_JAC_PROF) {
      const long long x4 = JCLK();
      pf[1] += x1 - x0;
      pf[2] += x2 - x1;
      pf[3] += x3 - x2;
      pf[4] += x4 - x3;
    }
  };

  // ---------------------------------------------------------- inner sweeps
  // Final-sweep Gram check: after a sweep whose largest |t| is below
  // 2 sqrt(orth_tol) the next sweep is almost surely the zero-rotation sweep
  // that ends the loop (rotations.py:220-222).  Instead of running its N - 1
  // rounds, every warp tests its columns against all later columns with the
  // skip test of _kernels.py:57 (D = colnorms^2 at the sweep start,
  // rotations.py:217); if every pair passes, the sweep applies no rotation --
  // the outcome of running it -- and counts as a sweep; otherwise it runs.
  // Pre-pass blocks (diagonal after the first outer sweep) are checked before
  // their first sweep.
  const double chk_thr = 2.0 * sqrt(otol);
  double *dsc = (a.dscr && a.mode == JAC_CONVERGE) ? a.dscr + int64_t(item_id) * ld : nullptr;
  auto gram_check = [&](int slot) -> bool {
#pragma unroll
    for (int c = 0; c < CPW; ++c) {
      const int col = col_of(c);
#pragma unroll
      for (int u = 0; u < RPL; ++u) Rf[(lane + 32 * u) + int64_t(col) * ld] = V[u][c];
      if (lane == 0) dsc[col] = D[c];
    }
    jb_cluster_sync<C>();
    bool bad = false;
    // lane group g = lane >> (5 - LC) ends up with the complete dot product
    // of local column g (butterfly reduce-scatter over the CPW partials,
    // then a reduction inside the group): 2 CPW - 2 + (5 - LC) shuffles per
    // column instead of 5 CPW
    constexpr int LC = ilog2(CPW);
    const int gc = lane >> (5 - LC);
    double dmine = 0.0;
    int cmine = 0;
    bool lmine = false;
    sfor<CPW>([&](auto cc) {
      constexpr int c = decltype(cc)::value;
      if (gc == c) {
        dmine = D[c];
        cmine = col_of(c);
        lmine = live[c];
      }
    });
    for (int oc = 0; oc < Nq; ++oc) {
      T x[RPL];
#pragma unroll
      for (int u = 0; u < RPL; ++u) x[u] = __ldcg(Rf + (lane + 32 * u) + int64_t(oc) * ld);
      const double dother = __ldcg(dsc + oc);
      T dd[CPW];
      sfor<CPW>([&](auto cc) {
        constexpr int c = decltype(cc)::value;
        T d0 = S<T>::zero(), d1 = S<T>::zero();
#pragma unroll
        for (int u = 0; u < RPL; u += 2) {
          d0 = cfma(V[u][c], x[u], d0);
          if (u + 1 < RPL) d1 = cfma(V[u + 1][c], x[u + 1], d1);
        }
        dd[c] = add(d0, d1);
      });
#pragma unroll
      for (int j = 0; j < LC; ++j) {
        const int dist = 16 >> j;
        const bool hi = lane & dist;
        const int half = CPW >> (j + 1);
#pragma unroll
        for (int xx = 0; xx < half; ++xx) {
          const T snd = hi ? dd[xx] : dd[xx + half];
          const T keep = hi ? dd[xx + half] : dd[xx];
          dd[xx] = add(keep, shfl_xor(snd, dist));
        }
      }
      T acc = dd[0];
#pragma unroll
      for (int dist = 16 >> LC; dist >= 1; dist >>= 1) acc = add(acc, shfl_xor(acc, dist));
      // every pair once: the owner of the lower column checks it
      if (lmine && oc > cmine) bad |= !(abs2(acc) <= otol2 * (dmine * dother));
    }
    bad = __any_sync(0xffffffffu, bad);
    if (bad && lane == 0) atomicOr(&s_chk[slot], 1);
    jb_cluster_sync<C>();
    int any_bad = 0;
#pragma unroll
    for (int r = 0; r < C; ++r)
      any_bad |= C > 1 ? *cg::this_cluster().map_shared_rank(&s_chk[slot], r) : s_chk[slot];
    return any_bad == 0;
  };

  for (int sw = 0; sw < a.max_sweeps; ++sw) {
    const int nsweep = sw + 1;  // the reference counts sweeps from 1
    ++sweeps;
    // D = colnorms^2(R) (rotations.py:217): butterfly all-reduce per column
    {
#pragma unroll
      for (int c = 0; c < CPW; ++c) {
        double s0 = 0.0, s1 = 0.0;
#pragma unroll
        for (int u = 0; u < RPL; u += 2) {
          s0 += abs2(V[u][c]);
          if (u + 1 < RPL) s1 += abs2(V[u + 1][c]);
        }
        D[c] = s0 + s1;
      }
#pragma unroll
      for (int dist = 16; dist >= 1; dist >>= 1)
#pragma unroll
        for (int c = 0; c < CPW; ++c) D[c] += __shfl_xor_sync(0xffffffffu, D[c], dist);
    }
    if (dsc && ((sw > 0 && prev_swt <= chk_thr) || (sw == 0 && nj == 0))) {
      const long long g0 = JCLK();
      const bool ok = gram_check(sw & 1);
      if (HJB_JAC_PROF) pf[5] += JCLK() - g0;
      if (ok) break;  // the zero-rotation sweep, counted
    }
    phase_a();
    for (int s = 1; s < NBL - 1; ++s) {
      exchange(nsweep);
      phase_b();
    }
    // ---- sweep end: cluster-wide rotation count (parallel.py:239-244 at the
    // inner level, rotations.py:220-222) ----
    const long long e0 = JCLK();
    const int par = sw & 1;
    {
      const int wc = __reduce_add_sync(0xffffffffu, my_cnt);
      const int wb = __reduce_add_sync(0xffffffffu, my_big);
      const int wf = __reduce_min_sync(0xffffffffu, my_fail);
      if (lane == 0) {
        if (wc) atomicAdd(&s_cnt[par], wc);
        if (wb) atomicAdd(&s_big[par], wb);
        if (wf != INT_MAX) atomicMin(&s_fail[par], wf);
      }
      my_cnt = my_big = 0;
      double wt = my_swt;
#pragma unroll
      for (int dist = 16; dist >= 1; dist >>= 1) wt = fmax(wt, __shfl_xor_sync(0xffffffffu, wt, dist));
      if (lane == 0 && wt > 0.0) atomicMax(&s_swt[par], static_cast<unsigned long long>(__double_as_longlong(wt)));
      my_swt = 0.0;
    }
    jb_cluster_sync<C>();
    long long tot = 0;
    unsigned long long swt = 0ull;
    int big = 0, fl = INT_MAX;
#pragma unroll
    for (int r = 0; r < C; ++r) {
      const int *pc = C > 1 ? cg::this_cluster().map_shared_rank(&s_cnt[par], r) : &s_cnt[par];
      const int *pb = C > 1 ? cg::this_cluster().map_shared_rank(&s_big[par], r) : &s_big[par];
      const int *pf = C > 1 ? cg::this_cluster().map_shared_rank(&s_fail[par], r) : &s_fail[par];
      const unsigned long long *pt = C > 1 ? cg::this_cluster().map_shared_rank(&s_swt[par], r) : &s_swt[par];
      tot += *pc;
      big += *pb;
      fl = min(fl, *pf);
      swt = max(swt, *pt);
    }
    prev_swt = __longlong_as_double(static_cast<long long>(swt));
    if (tid == 0) {  // reset the other parity for the next sweep (read only after the next cluster sync)
      s_cnt[par ^ 1] = 0;
      s_big[par ^ 1] = 0;
      s_fail[par ^ 1] = INT_MAX;
      s_chk[par ^ 1] = 0;
      s_swt[par ^ 1] = 0ull;
    }
    big_total += big;
    nrot_total += tot;
    if (HJB_JAC_PROF) pf[5] += JCLK() - e0;
    if (fl != INT_MAX) {
      status = PV_INDEFINITE;
      my_fail = fl;
      break;
    }
    // one cycle only for the B variants (tol.with_max_sweeps(1), parallel.py:162-174)
    if (tot == 0 || sw + 1 == a.max_sweeps || a.mode != JAC_CONVERGE) break;
    exchange(nsweep);  // the sweep's last exchange (parallel.py:234-237)
  }
  // max |t| over the cluster
  if (my_maxt > 0.0) atomicMax(&s_maxt, static_cast<unsigned long long>(__double_as_longlong(my_maxt)));
  // ---- R_final -> global (column ids travel with the sub-blocks) ----
#pragma unroll
  for (int c = 0; c < CPW; ++c) {
    const int col = col_of(c);
#pragma unroll
    for (int u = 0; u < RPL; ++u) Rf[(lane + 32 * u) + int64_t(col) * ld] = V[u][c];
  }
  jb_cluster_sync<C>();
  if (tid == 0) {
    unsigned long long mt = s_maxt;
#pragma unroll
    for (int r = 0; r < C; ++r) {
      const unsigned long long *pm = C > 1 ? cg::this_cluster().map_shared_rank(&s_maxt, r) : &s_maxt;
      mt = max(mt, *pm);
    }
    if (crank == 0) {
      st[ST_NROT] = nrot_total;
      st[ST_NBIG] = big_total;
      st[ST_MAXT] = static_cast<int64_t>(mt);
      st[ST_SWEEPS] = sweeps;
      st[ST_STATUS] = status;
      st[ST_FR] = status == PV_INDEFINITE ? my_fail / 4096 : -1;
      st[ST_FS] = status == PV_INDEFINITE ? my_fail % 4096 : -1;
    }
  }
  if (HJB_JAC_PROF && a.prof && lane == 0) {
    long long *o = a.prof + (int64_t(blockIdx.x) * W + warp) * 8;
    pf[7] = JCLK() - pf[7];
    for (int k = 0; k < 8; ++k) o[k] = pf[k];
  }
  jb_cluster_sync<C>();  // peers' shared memory stays alive until read
}

// ------------------------------------------------------------------ launch

template <typename T, int N, int C, int W, int SPW>
static cudaError_t launch_jacobi_t(const JacobiArgs &a, cudaStream_t st) {
  using Cfg = JacCfg<T, N, C, W, SPW>;
  // two CTAs per SM for 4-warp CTAs (255 registers per thread either way)
  constexpr int MINB = Cfg::NT <= 128 ? (N <= 128 ? HJB_JAC_MINB_SMALL : 2) : 1;
  auto k = jacobi_kernel<T, N, C, W, SPW, MINB>;
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
  cfg.blockDim = dim3(Cfg::NT);
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

// instantiated shapes: (N, C, W, SPW) with N = 2 C W SPW
#define HJB_JAC_SHAPES(X)                                                                              \
  X(32, 1, 4, 4) X(32, 2, 4, 2) X(64, 2, 4, 4) X(64, 4, 4, 2) X(128, 4, 8, 2) X(128, 8, 4, 2)         \
  X(128, 4, 4, 4) X(256, 8, 8, 2) X(256, 4, 8, 4) X(256, 16, 4, 2)

JacShape jacobi_default_shape(bool cx, int nmax, int count) {
  static int ov_c = -1, ov_w = 0, ov_s = 0;
  if (ov_c < 0) {  // experiments: HJB_JAC_SHAPE="C,W,SPW"
    ov_c = 0;
    if (const char *e = std::getenv("HJB_JAC_SHAPE")) sscanf(e, "%d,%d,%d", &ov_c, &ov_w, &ov_s);
  }
  if (ov_c > 0 && 2 * ov_c * ov_w * ov_s == nmax) return JacShape{ov_c, ov_w, ov_s};
  (void)count;
  // measured on B200 (tools/jac_bench.py, profiles/r2_jacobi_shapes.jsonl)
  switch (nmax) {
    case 32: return JacShape{1, 4, 4};
    case 64: return JacShape{4, 4, 2};
    case 128: return JacShape{8, 4, 2};
    case 256: return cx ? JacShape{16, 4, 2} : JacShape{4, 8, 4};
  }
  return JacShape{0, 0, 0};
}

bool jacobi_shape_for(int nmax, int c, JacShape *out) {
#define HJB_JAC_FIND(N_, C_, W_, S_)          \
  if (nmax == N_ && c == C_) {                \
    *out = JacShape{C_, W_, S_};              \
    return true;                              \
  }
  HJB_JAC_SHAPES(HJB_JAC_FIND)
#undef HJB_JAC_FIND
  return false;
}

// register-resident columns per lane (RPL x 2 SPW elements) that fit without
// spilling: 64 doubles
template <typename T, int N, int SPW>
constexpr bool jac_shape_ok() {
  return (N / 32) * 2 * SPW * int(sizeof(T) / 8) <= 64;
}

template <typename T>
static cudaError_t dispatch_jacobi(const JacobiArgs &a, JacShape s, cudaStream_t st) {
#define HJB_JAC_CASE(N_, C_, W_, S_)                                              \
  if constexpr (jac_shape_ok<T, N_, S_>())                                         \
    if (a.nmax == N_ && s.c == C_ && s.w == W_ && s.spw == S_) return launch_jacobi_t<T, N_, C_, W_, S_>(a, st);
  HJB_JAC_SHAPES(HJB_JAC_CASE)
#undef HJB_JAC_CASE
  return cudaErrorInvalidConfiguration;
}

cudaError_t launch_jacobi(bool cx, const JacobiArgs &a, JacShape s, cudaStream_t st) {
  if (a.count == 0) return cudaSuccess;
  return cx ? dispatch_jacobi<cplx>(a, s, st) : dispatch_jacobi<double>(a, s, st);
}

// Pivots (clusters) of this shape that are resident on the GPU at once: one
// "wave" of the Jacobi launch (cudaOccupancyMaxActiveClusters, cached).
template <typename T, int N, int C, int W, int SPW>
static int query_jacobi_t() {
  using Cfg = JacCfg<T, N, C, W, SPW>;
  constexpr int MINB = Cfg::NT <= 128 ? (N <= 128 ? HJB_JAC_MINB_SMALL : 2) : 1;
  auto k = jacobi_kernel<T, N, C, W, SPW, MINB>;
  if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(Cfg::SMEM)) != cudaSuccess) return 0;
  if (C > 8 && cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess) return 0;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(C * 256);
  cfg.blockDim = dim3(Cfg::NT);
  cfg.dynamicSmemBytes = Cfg::SMEM;
  cudaLaunchAttribute attrs[1];
  attrs[0].id = cudaLaunchAttributeClusterDimension;
  attrs[0].val.clusterDim.x = C;
  attrs[0].val.clusterDim.y = 1;
  attrs[0].val.clusterDim.z = 1;
  cfg.attrs = attrs;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, k, &cfg) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

template <typename T>
static int query_jacobi(int nmax, JacShape s) {
#define HJB_JAC_Q(N_, C_, W_, S_)                  \
  if constexpr (jac_shape_ok<T, N_, S_>())          \
    if (nmax == N_ && s.c == C_ && s.w == W_ && s.spw == S_) return query_jacobi_t<T, N_, C_, W_, S_>();
  HJB_JAC_SHAPES(HJB_JAC_Q)
#undef HJB_JAC_Q
  return 0;
}

int jacobi_wave_capacity(bool cx, int nmax, JacShape s) {
  static int cache[64][2][4][5];  // [device][type][nmax][log2 cluster]
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 0;
  const int ni = nmax == 32 ? 0 : nmax == 64 ? 1 : nmax == 128 ? 2 : 3;
  int ci = 0;
  while ((1 << ci) < s.c && ci < 4) ++ci;
  int &v = cache[dev][cx][ni][ci];
  if (v == 0) {
    v = cx ? query_jacobi<cplx>(nmax, s) : query_jacobi<double>(nmax, s);
    if (v <= 0) v = -1;
  }
  return v > 0 ? v : 0;
}

}  // namespace hjb
