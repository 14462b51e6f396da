// Block-column update [G_i G_j] <- [G_i G_j] W on FP64 tensor cores (DMMA).
//
// Replaces parallel.py:203-207 (Gq @ sub.W, only when the pivot rotated) and
// the pre-pass update B <- B W (parallel.py:145-146).  One CTA owns MT full
// rows of the pair (all N output columns), so the update is done in place:
// every CTA reads all of its rows before it writes them back, and no other
// CTA touches those rows.  X (rows of the pair) and W are streamed through
// shared memory in K chunks with cp.async and multiplied with
// mma.sync.m8n8k4.f64.  Items whose pivot applied no rotation exit at once.
#include "common.cuh"
#include "kernels.h"

#ifndef HJB_UPD_R256_MT  // rows per CTA of the N_max = 256 update (real / complex)
#define HJB_UPD_R256_MT 32
#endif
#ifndef HJB_UPD_C256_MT
#define HJB_UPD_C256_MT 16
#endif

namespace hjb {

template <typename T, int NMAX, int MT, int KW>
struct UpdCfg {
  static constexpr int NT = 256;
  static constexpr int NW = NMAX / 8;          // output columns per warp
  static constexpr int NI = NW / 8;            // 8-wide MMA tiles per warp (N)
  static constexpr int MI = MT / 8;            // 8-high MMA tiles (M)
  static constexpr int MTP = MT + (S<T>::cx ? 2 : 4);
  static constexpr int KWP = KW + 4;
  static constexpr int XS = KW * MTP;          // X stage elements ([k][row])
  static constexpr int WSZ = NMAX * KWP;       // W stage elements ([col][k])
  static constexpr int STAGE = XS + WSZ;
  static constexpr size_t SMEM = 2 * size_t(STAGE) * sizeof(T);
  // N_max = 256: short row tiles (32 real / 16 complex rows) with 2 CTAs per
  // SM, so 16 warps keep DMMA chains in flight: 1 CTA of 8 warps with 64/32
  // rows ran the tensor pipe at ~65 % (tools/upd_bench.py: cfg5r shape 24.2 ->
  // 29.5 TFLOP/s, cfg5c shape 25.6 -> 31.4 TFLOP/s)
  static constexpr int MINB = (2 * SMEM <= 227 * 1024) ? 2 : 1;  // (an explicit 1 lets ptxas take >128 registers)
  static_assert(NI >= 1, "at least one MMA tile per warp");
};

template <typename T> struct UpdAcc;
template <> struct UpdAcc<double> {
  double v[2];
  __device__ void zero() { v[0] = v[1] = 0.0; }
  __device__ void mma(double a, double b) { dmma(v[0], v[1], a, b); }
  __device__ double get(int q) const { return v[q]; }
};
template <> struct UpdAcc<cplx> {
  double r[2], i[2];
  __device__ void zero() { r[0] = r[1] = i[0] = i[1] = 0.0; }
  __device__ void mma(cplx a, cplx b) {
    // a b = (ar br - ai bi) + i (ar bi + ai br)
    dmma(r[0], r[1], a.x, b.x);
    dmma(r[0], r[1], -a.y, b.y);
    dmma(i[0], i[1], a.x, b.y);
    dmma(i[0], i[1], a.y, b.x);
  }
  __device__ cplx get(int q) const { return make_double2(r[q], i[q]); }
};

template <typename T, int NMAX, int MT, int KW, int VEC>
__global__ void __launch_bounds__(256, (UpdCfg<T, NMAX, MT, KW>::MINB)) update_kernel(UpdateArgs a) {
  using Cfg = UpdCfg<T, NMAX, MT, KW>;
  constexpr int NT = Cfg::NT, NW = Cfg::NW, NI = Cfg::NI, MI = Cfg::MI;
  constexpr int MTP = Cfg::MTP, KWP = Cfg::KWP;
  constexpr int EPP = VEC / int(sizeof(T));
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T *smem = reinterpret_cast<T *>(smem_raw);

  const int item_id = blockIdx.y;
  if (a.stats[int64_t(item_id) * ST_N + ST_NROT] == 0) return;  // parallel.py:203
  const Item it = a.items[item_id];
  const int ni = it.ni, N = it.ni + it.nj;
  const int64_t r0 = int64_t(blockIdx.x) * MT;
  T *G = reinterpret_cast<T *>(a.G);
  const T *W = reinterpret_cast<const T *>(a.W) + int64_t(item_id) * a.nmax * a.nmax;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nchunks = (N + KW - 1) / KW;
  auto gcol = [&](int c) -> int64_t { return c < ni ? it.oi + c : it.oj + (c - ni); };

  auto load_stage = [&](int stage, int chunk) {
    T *Xs = smem + stage * Cfg::STAGE;
    T *Wsm = Xs + Cfg::XS;
    const int kb = chunk * KW;
    constexpr int XP = MT / EPP;  // pieces per staged X column
    for (int pc = tid; pc < KW * XP; pc += NT) {
      const int k = pc / XP, w = pc % XP;
      const int64_t row = r0 + int64_t(w) * EPP;
      int64_t valid = (kb + k < N) ? min(int64_t(EPP), a.m - row) : 0;
      if (valid < 0) valid = 0;
      const T *src = valid > 0 ? G + gcol(kb + k) * a.ldg + row : G;
      T *dst = Xs + k * MTP + w * EPP;
      if (VEC == 16) cp_async16(dst, src, int(valid * sizeof(T)));
      else cp_async8(dst, src, int(valid * sizeof(T)));
    }
    constexpr int WP = KW / (16 / int(sizeof(T)));  // W pieces per staged column (16 B)
    for (int pc = tid; pc < NMAX * WP; pc += NT) {
      const int c = pc / WP, w = pc % WP;
      const int k = kb + w * (16 / int(sizeof(T)));
      int valid = (c < N) ? min(16 / int(sizeof(T)), N - k) : 0;
      if (valid < 0) valid = 0;
      const T *src = valid > 0 ? W + k + int64_t(c) * a.nmax : W;
      cp_async16(Wsm + c * KWP + w * (16 / int(sizeof(T))), src, valid * int(sizeof(T)));
    }
  };

  // Full tiles (every BASELINE config: N == NMAX, whole row tiles, K chunks
  // inside one block): the per-thread source offsets are loop invariant, so a
  // stage costs one address add per 16-byte piece instead of the div/mod and
  // bounds arithmetic above
  constexpr int XP = MT / EPP, XPT = (KW * XP + NT - 1) / NT;
  constexpr int EW = 16 / int(sizeof(T)), WP = KW / EW, WPT = (NMAX * WP + NT - 1) / NT;
  const bool full = VEC == 16 && N == NMAX && r0 + MT <= a.m && ni % KW == 0;
  int64_t xoff[XPT];
  int xdst[XPT], woff[WPT], wdst[WPT];
#pragma unroll
  for (int i = 0; i < XPT; ++i) {
    const int pc = tid + i * NT, k = pc / XP, w = pc % XP;
    xoff[i] = int64_t(k) * a.ldg + r0 + int64_t(w) * EPP;
    xdst[i] = k * MTP + w * EPP;
  }
#pragma unroll
  for (int i = 0; i < WPT; ++i) {
    const int pc = tid + i * NT, c = pc / WP, w = pc % WP;
    woff[i] = w * EW + c * a.nmax;
    wdst[i] = c * KWP + w * EW;
  }
  auto load_stage_full = [&](int stage, int chunk) {
    T *Xs = smem + stage * Cfg::STAGE;
    T *Wsm = Xs + Cfg::XS;
    const int kb = chunk * KW;
    const T *gsrc = G + int64_t(kb < ni ? it.oi + kb : it.oj + (kb - ni)) * a.ldg;
    const T *wsrc = W + kb;
#pragma unroll
    for (int i = 0; i < XPT; ++i)
      if ((KW * XP) % NT == 0 || tid + i * NT < KW * XP) cp_async16(Xs + xdst[i], gsrc + xoff[i], 16);
#pragma unroll
    for (int i = 0; i < WPT; ++i)
      if ((NMAX * WP) % NT == 0 || tid + i * NT < NMAX * WP) cp_async16(Wsm + wdst[i], wsrc + woff[i], 16);
  };
  auto stage_in = [&](int stage, int chunk) {
    if (full) load_stage_full(stage, chunk);
    else load_stage(stage, chunk);
  };

  UpdAcc<T> acc[MI][NI];
#pragma unroll
  for (int mi = 0; mi < MI; ++mi)
#pragma unroll
    for (int nn = 0; nn < NI; ++nn) acc[mi][nn].zero();

  stage_in(0, 0);
  cp_async_commit();
  for (int c = 0; c < nchunks; ++c) {
    if (c + 1 < nchunks) stage_in((c + 1) & 1, c + 1);
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    const T *Xs = smem + (c & 1) * Cfg::STAGE;
    const T *Wsm = Xs + Cfg::XS;
#pragma unroll
    for (int kk = 0; kk < KW; kk += 4) {
      T fb[NI];
#pragma unroll
      for (int nn = 0; nn < NI; ++nn) fb[nn] = Wsm[(warp * NW + nn * 8 + (lane >> 2)) * KWP + kk + (lane & 3)];
#pragma unroll
      for (int mi = 0; mi < MI; ++mi) {
        const T fa = Xs[(kk + (lane & 3)) * MTP + mi * 8 + (lane >> 2)];
#pragma unroll
        for (int nn = 0; nn < NI; ++nn) acc[mi][nn].mma(fa, fb[nn]);
      }
    }
    __syncthreads();
  }
  cp_async_wait<0>();
  __syncthreads();
  // in-place write-back of this CTA's rows
#pragma unroll
  for (int mi = 0; mi < MI; ++mi) {
    const int64_t row = r0 + mi * 8 + (lane >> 2);
    if (row >= a.m) continue;
#pragma unroll
    for (int nn = 0; nn < NI; ++nn)
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int col = warp * NW + nn * 8 + 2 * (lane & 3) + q;
        if (col < N) G[gcol(col) * a.ldg + row] = acc[mi][nn].get(q);
      }
  }
}

template <typename T, int NMAX, int MT, int KW, int VEC>
static cudaError_t launch_update_t(const UpdateArgs &a, cudaStream_t st) {
  using Cfg = UpdCfg<T, NMAX, MT, KW>;
  auto k = update_kernel<T, NMAX, MT, KW, VEC>;
  static DeviceFlags attr_flags;
  bool *attr = attr_flags.here();
  if (!attr) return cudaErrorInvalidDevice;
  if (!*attr) {
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(Cfg::SMEM));
    if (e != cudaSuccess) return e;
    *attr = true;
  }
  dim3 grid(unsigned((a.m + MT - 1) / MT), a.count);
  k<<<grid, Cfg::NT, Cfg::SMEM, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_update(bool cx, const UpdateArgs &a, cudaStream_t st) {
  if (cx) {
    switch (a.nmax) {
      case 32:  // W keeps ld = nmax; columns >= N are zero-filled
      case 64: return launch_update_t<cplx, 64, 64, 8, 16>(a, st);
      case 128: return launch_update_t<cplx, 128, 32, 8, 16>(a, st);
      case 256: return launch_update_t<cplx, 256, HJB_UPD_C256_MT, 8, 16>(a, st);
    }
  } else {
    const bool v16 = a.ldg % 2 == 0;
    switch (a.nmax) {
      case 32:
      case 64: return v16 ? launch_update_t<double, 64, 128, 16, 16>(a, st) : launch_update_t<double, 64, 128, 16, 8>(a, st);
      case 128: return v16 ? launch_update_t<double, 128, 64, 16, 16>(a, st) : launch_update_t<double, 128, 64, 16, 8>(a, st);
      case 256: return v16 ? launch_update_t<double, 256, HJB_UPD_R256_MT, 16, 16>(a, st)
                           : launch_update_t<double, 256, HJB_UPD_R256_MT, 16, 8>(a, st);
    }
  }
  return cudaErrorInvalidValue;
}

// ---------------------------------------------------------------- extract
// rotations.py:226-251: lam_k = j_k ||g_k||^2, u_k = g_k / ||g_k||, then an
// optional column permutation (U[:, o] <- U[:, perm[o]]).
template <typename T>
__global__ void __launch_bounds__(256) extract_kernel(int64_t m, int64_t n, const T *G, int64_t ldg,
                                                     const int8_t *signs, double *lam, T *U,
                                                     int64_t ldu, const int64_t *perm, int *zero_flag) {
  const int64_t o = blockIdx.x;
  const int64_t c = perm ? perm[o] : o;
  const T *g = G + c * ldg;
  __shared__ double red[256];
  double s = 0.0;
  for (int64_t r = threadIdx.x; r < m; r += blockDim.x) s += abs2(g[r]);
  red[threadIdx.x] = s;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  const double n2 = red[0];
  if (n2 == 0.0) {
    if (threadIdx.x == 0) atomicExch(zero_flag, 1);
    return;
  }
  const double nrm = sqrt(n2);
  if (threadIdx.x == 0) lam[o] = double(signs[c]) * n2;
  T *u = U + o * ldu;
  for (int64_t r = threadIdx.x; r < m; r += blockDim.x) u[r] = divr(g[r], nrm);
}

cudaError_t launch_extract(bool cx, int64_t m, int64_t n, const void *G, int64_t ldg,
                           const int8_t *signs, double *lam, void *U, int64_t ldu,
                           const int64_t *perm, int *zero_flag, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  if (cx)
    extract_kernel<cplx><<<unsigned(n), 256, 0, st>>>(m, n, reinterpret_cast<const cplx *>(G), ldg, signs,
                                                       lam, reinterpret_cast<cplx *>(U), ldu, perm, zero_flag);
  else
    extract_kernel<double><<<unsigned(n), 256, 0, st>>>(m, n, reinterpret_cast<const double *>(G), ldg,
                                                         signs, lam, reinterpret_cast<double *>(U), ldu, perm,
                                                         zero_flag);
  return cudaGetLastError();
}


// ---------------------------------------------------------------- orthogonality
// solve.py:108-110: max |U^H U - I|.  A holds the Gram tiles of a batch of
// block pairs (gram_kernel, items with oi <= oj); each CTA folds one tile and
// the maximum goes to *out as the bit pattern of a non-negative double
// (ordered like unsigned integers, so atomicMax is exact; a NaN wins).
template <typename T>
__global__ void __launch_bounds__(256) orth_max_kernel(const Item *items, int bmax, const T *A,
                                                      unsigned long long *out) {
  const Item it = items[blockIdx.x];
  const T *a = A + size_t(blockIdx.x) * bmax * bmax;
  double v = 0.0;
  for (int e = threadIdx.x; e < it.ni * it.nj; e += blockDim.x) {
    const int r = e % it.ni, c = e / it.ni;
    T x = a[size_t(c) * bmax + r];
    double d;
    if constexpr (sizeof(T) == 16) {
      if (it.oi + r == it.oj + c) x.x -= 1.0;
      d = sqrt(abs2(x));
    } else {
      if (it.oi + r == it.oj + c) x -= 1.0;
      d = fabs(x);
    }
    v = (d > v || d != d) ? d : v;
  }
  __shared__ double red[256];
  red[threadIdx.x] = v;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w) {
      const double o = red[threadIdx.x + w];
      if (o > red[threadIdx.x] || o != o) red[threadIdx.x] = o;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) atomicMax(out, static_cast<unsigned long long>(__double_as_longlong(red[0])));
}

cudaError_t launch_orth_max(bool cx, const Item *items, int count, int bmax, const void *A,
                            unsigned long long *out, cudaStream_t st) {
  if (count == 0) return cudaSuccess;
  if (cx)
    orth_max_kernel<cplx><<<unsigned(count), 256, 0, st>>>(items, bmax, reinterpret_cast<const cplx *>(A), out);
  else
    orth_max_kernel<double><<<unsigned(count), 256, 0, st>>>(items, bmax, reinterpret_cast<const double *>(A),
                                                            out);
  return cudaGetLastError();
}

}  // namespace hjb
