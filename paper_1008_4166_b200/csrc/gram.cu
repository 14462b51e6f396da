// Batched long-K Gram of block-column pairs on FP64 tensor cores (DMMA).
//
// Replaces the per-pair Gram A_ij = G_i^H G_j of the reference's 2F step
// (pkg/src/hjacobi/parallel.py:193 -> core.py:42-56) and the diagonal-block
// Gram of the F pre-pass (parallel.py:143), and fuses the column-norm
// refresh D = colnorms^2 (parallel.py:208-209 / core.py:59-61) into the same
// pass over the data.
//
// Layout: G column-major (ld = ldg); block column = contiguous m x b slab.
// One CTA computes a TM x TN tile of one item's Gram over one K split;
// operands are staged through shared memory with a cp.async pipeline and fed
// to mma.sync.m8n8k4.f64 (SASS DMMA).  The number of K splits is chosen so
// that items x tiles x splits fills a whole number of waves of the GPU
// (148 SMs x resident CTAs): round 1's fixed tiling left cfg5r with 1.15
// waves (512 CTAs on 444 slots).  With more than one split every CTA writes
// its partial tile to an L2-resident scratch and gram_reduce_kernel adds the
// partials in split order (deterministic).
//
// gram_ffma_kernel is the CUDA-core (DFMA) variant of the same contraction,
// kept for the DMMA-vs-DFMA measurement the north star asks for
// (HJB_GRAM_FFMA=1; tools/gram_bench.py).
#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"

namespace hjb {

// WM x WN warps per CTA tile; each warp owns MI x NI 8x8 DMMA fragments
template <typename T, int WM, int WN, int MI, int NI, int KC, int STAGES>
struct GramCfg {
  static constexpr int TM = WM * MI * 8;       // X columns (rows of A) per tile
  static constexpr int TN = WN * NI * 8;       // Y columns per tile
  static constexpr int NT = 32 * WM * WN;
  static constexpr int KCP = KC + 4;           // elements per staged column (bank-conflict-free fragments)
  static constexpr int STAGE_ELEMS = (TM + TN) * KCP;
  static constexpr size_t SMEM = size_t(STAGES) * STAGE_ELEMS * sizeof(T);
};

// (X^H Y) fragment products: real a*b; complex conj(a)*b on 4 DMMAs, two
// accumulator pairs per fragment.
template <typename T> struct GramAcc;
template <> struct GramAcc<double> {
  double v[2];
  __device__ __forceinline__ void zero() { v[0] = v[1] = 0.0; }
  __device__ __forceinline__ void mma(double a, double b) { dmma(v[0], v[1], a, b); }
  __device__ __forceinline__ double get(int q) const { return v[q]; }
};
template <> struct GramAcc<cplx> {
  // conj(a) b = (ar br + ai bi) + i (ar bi - ai br)
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

// rows [k0, k1) of split `split` out of `splits`: whole K chunks, sizes differ by at most one chunk
__device__ __forceinline__ void split_range(int64_t m, int kc, int splits, int split, int64_t *k0, int64_t *k1) {
  const int64_t chunks = (m + kc - 1) / kc;
  *k0 = (chunks * split / splits) * kc;
  *k1 = min(m, (chunks * (split + 1) / splits) * kc);
}

template <typename T, int WM, int WN, int MI, int NI, int KC, int STAGES, int VEC, int MINB>
__global__ void __launch_bounds__(GramCfg<T, WM, WN, MI, NI, KC, STAGES>::NT, MINB) gram_kernel(GramArgs a) {
  using Cfg = GramCfg<T, WM, WN, MI, NI, KC, STAGES>;
  constexpr int TM = Cfg::TM, TN = Cfg::TN, NT = Cfg::NT, KCP = Cfg::KCP;
  constexpr int EPP = VEC / int(sizeof(T));       // elements per cp.async piece
  constexpr int PPC = KC / EPP;                   // pieces per staged column
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T *smem = reinterpret_cast<T *>(smem_raw);

  // blockIdx.x = split * (tm * tn) + tile: the tiles of one item and K range
  // are neighbours in launch order (shared operand rows hit in L2)
  const int ntile = a.tiles_m * a.tiles_n;
  const int split = blockIdx.x / ntile, tile_id = blockIdx.x % ntile;
  const int ti = tile_id / a.tiles_n, tj = tile_id % a.tiles_n;
  const int item_id = blockIdx.y;
  const Item it = a.items[item_id];
  const bool dense = it.nj == 0;
  const int nX = it.ni, nY = dense ? it.ni : it.nj;
  const int oX = it.oi + ti * TM, oY = (dense ? it.oi : it.oj) + tj * TN;
  const int cX = min(TM, nX - ti * TM), cY = min(TN, nY - tj * TN);  // may be <= 0
  int64_t k0, k1;
  split_range(a.m, KC, a.splits, split, &k0, &k1);
  const int nchunks = k1 > k0 ? int((k1 - k0 + KC - 1) / KC) : 0;
  const T *G = reinterpret_cast<const T *>(a.G);

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp / WN, wn = warp % WN;

  auto load_stage = [&](int stage, int chunk) {
    T *Xs = smem + stage * Cfg::STAGE_ELEMS;
    const int64_t kb = k0 + int64_t(chunk) * KC;
    for (int pc = tid; pc < (TM + TN) * PPC; pc += NT) {
      const int col = pc / PPC, within = pc % PPC;  // col < TM: X, else Y
      const bool y = col >= TM;
      const int lc = y ? col - TM : col;
      const int64_t row = kb + within * EPP;
      int64_t valid = (lc < (y ? cY : cX)) ? min(int64_t(EPP), k1 - row) : 0;
      if (valid < 0) valid = 0;
      const T *src = valid > 0 ? G + int64_t((y ? oY : oX) + lc) * a.ldg + row : G;
      T *dst = Xs + col * KCP + within * EPP;
      if (VEC == 16)
        cp_async16(dst, src, int(valid * sizeof(T)));
      else
        cp_async8(dst, src, int(valid * sizeof(T)));
    }
  };

  // Full tiles and whole K chunks (every BASELINE config): thread t stages
  // pieces t, t + NT, ... whose column advances by NT / PPC per piece, so a
  // stage is two base pointers plus compile-time strides -- no per-piece
  // div/mod or bounds arithmetic
  constexpr int CS = NT / PPC;  // column stride between a thread's pieces
  constexpr bool FAST_OK = VEC == 16 && NT % PPC == 0 && TM % CS == 0 && TN % CS == 0;
  const bool fast_cols = FAST_OK && cX == TM && cY == TN;
  const int col0 = tid / PPC, within0 = tid % PPC;
  const T *xsrc0 = G + int64_t(oX + col0) * a.ldg + within0 * EPP;
  const T *ysrc0 = G + int64_t(oY + col0) * a.ldg + within0 * EPP;
  const int64_t sstride = int64_t(CS) * a.ldg;
  auto load_stage_fast = [&](int stage, int chunk) {
    T *Xs = smem + stage * Cfg::STAGE_ELEMS + col0 * KCP + within0 * EPP;
    const int64_t kb = k0 + int64_t(chunk) * KC;
    if constexpr (FAST_OK) {
#pragma unroll
      for (int i = 0; i < TM / CS; ++i) cp_async16(Xs + i * CS * KCP, xsrc0 + i * sstride + kb, 16);
#pragma unroll
      for (int i = 0; i < TN / CS; ++i) cp_async16(Xs + (TM + i * CS) * KCP, ysrc0 + i * sstride + kb, 16);
    }
  };
  auto stage_in = [&](int stage, int chunk) {
    if (fast_cols && k0 + int64_t(chunk + 1) * KC <= k1) load_stage_fast(stage, chunk);
    else load_stage(stage, chunk);
  };

  GramAcc<T> acc[MI][NI];
#pragma unroll
  for (int mi = 0; mi < MI; ++mi)
#pragma unroll
    for (int ni = 0; ni < NI; ++ni) acc[mi][ni].zero();
  double dx[MI], dy[NI];
#pragma unroll
  for (int mi = 0; mi < MI; ++mi) dx[mi] = 0.0;
#pragma unroll
  for (int ni = 0; ni < NI; ++ni) dy[ni] = 0.0;
  const bool do_dx = !dense && tj == 0 && wn == 0;
  const bool do_dy = !dense && ti == 0 && wm == 0;

#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < nchunks) stage_in(s, s);
    cp_async_commit();
  }
  for (int c = 0; c < nchunks; ++c) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    {
      const int nxt = c + STAGES - 1;
      if (nxt < nchunks) stage_in(nxt % STAGES, nxt);
      cp_async_commit();
    }
    const T *Xs = smem + (c % STAGES) * Cfg::STAGE_ELEMS;
    const T *Ys = Xs + TM * KCP;
#pragma unroll
    for (int kk = 0; kk < KC; kk += 4) {
      T fa[MI], fb[NI];
#pragma unroll
      for (int mi = 0; mi < MI; ++mi) fa[mi] = Xs[((wm * MI + mi) * 8 + (lane >> 2)) * KCP + kk + (lane & 3)];
#pragma unroll
      for (int ni = 0; ni < NI; ++ni) fb[ni] = Ys[((wn * NI + ni) * 8 + (lane >> 2)) * KCP + kk + (lane & 3)];
#pragma unroll
      for (int mi = 0; mi < MI; ++mi)
#pragma unroll
        for (int ni = 0; ni < NI; ++ni) acc[mi][ni].mma(fa[mi], fb[ni]);
      if (do_dx) {
#pragma unroll
        for (int mi = 0; mi < MI; ++mi) dx[mi] += abs2(fa[mi]);
      }
      if (do_dy) {
#pragma unroll
        for (int ni = 0; ni < NI; ++ni) dy[ni] += abs2(fb[ni]);
      }
    }
  }
  cp_async_wait<0>();

  // column norms: reduce the 4 lanes holding the same column
#pragma unroll
  for (int mi = 0; mi < MI; ++mi) {
    dx[mi] += __shfl_xor_sync(0xffffffffu, dx[mi], 1);
    dx[mi] += __shfl_xor_sync(0xffffffffu, dx[mi], 2);
  }
#pragma unroll
  for (int ni = 0; ni < NI; ++ni) {
    dy[ni] += __shfl_xor_sync(0xffffffffu, dy[ni], 1);
    dy[ni] += __shfl_xor_sync(0xffffffffu, dy[ni], 2);
  }
  // final result (one split) or this split's partial
  const int bmax = a.bmax;
  const int64_t asz = int64_t(bmax) * bmax;
  const int64_t slot = a.splits == 1 ? int64_t(item_id) : int64_t(item_id) * a.splits + split;
  T *Af = reinterpret_cast<T *>(a.splits == 1 ? a.A : a.Apart) + slot * asz;
  double *Df = (a.splits == 1 ? a.D : a.Dpart) + slot * 2 * bmax;
#pragma unroll
  for (int mi = 0; mi < MI; ++mi)
#pragma unroll
    for (int ni = 0; ni < NI; ++ni)
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int r = ti * TM + (wm * MI + mi) * 8 + (lane >> 2);
        const int cc = tj * TN + (wn * NI + ni) * 8 + 2 * (lane & 3) + q;
        if (r < bmax && cc < bmax) Af[r + int64_t(cc) * bmax] = acc[mi][ni].get(q);
      }
  if ((lane & 3) == 0) {
#pragma unroll
    for (int mi = 0; mi < MI; ++mi) {
      const int r = ti * TM + (wm * MI + mi) * 8 + (lane >> 2);
      if (do_dx && r < bmax) Df[r] = dx[mi];
    }
#pragma unroll
    for (int ni = 0; ni < NI; ++ni) {
      const int cc = tj * TN + (wn * NI + ni) * 8 + (lane >> 2);
      if (do_dy && cc < bmax) Df[bmax + cc] = dy[ni];
    }
  }
}

// A[item] = sum over splits (in split order) of the partial tiles; same for
// the column norms of pair items
template <typename T>
__global__ void __launch_bounds__(256) gram_reduce_kernel(GramArgs a) {
  const int item_id = blockIdx.y;
  const int bmax = a.bmax;
  const int64_t asz = int64_t(bmax) * bmax;
  const int64_t e = int64_t(blockIdx.x) * 256 + threadIdx.x;
  if (e < asz) {
    const T *p = reinterpret_cast<const T *>(a.Apart) + int64_t(item_id) * a.splits * asz + e;
    T v = __ldcg(p);
    for (int s = 1; s < a.splits; ++s) v = add(v, __ldcg(p + s * asz));
    reinterpret_cast<T *>(a.A)[int64_t(item_id) * asz + e] = v;
  } else if (e < asz + 2 * bmax && a.items[item_id].nj != 0) {
    const int64_t d = e - asz;
    const double *p = a.Dpart + int64_t(item_id) * a.splits * 2 * bmax + d;
    double v = __ldcg(p);
    for (int s = 1; s < a.splits; ++s) v += __ldcg(p + s * 2 * bmax);
    a.D[int64_t(item_id) * 2 * bmax + d] = v;
  }
}

// ------------------------------------------------------------------ DFMA variant
// CUDA-core FP64 version of the same tile product: 128 x 128 tile, 256
// threads, 8 x 8 outputs per thread (rows tx + 16 i, columns ty + 16 j), operands
// staged [column][k] exactly like the DMMA kernel.  Real only: it exists for
// the DMMA-vs-DFMA comparison, not as a product path.
template <int KC, int VEC>
__global__ void __launch_bounds__(256, 1) gram_ffma_kernel(GramArgs a) {
  constexpr int TM = 128, TN = 128, NT = 256, KCP = KC + 2, STAGES = 2;
  constexpr int STAGE_ELEMS = (TM + TN) * KCP;
  constexpr int EPP = VEC / 8, PPC = KC / EPP;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double *smem = reinterpret_cast<double *>(smem_raw);
  const int ntile = a.tiles_m * a.tiles_n;
  const int split = blockIdx.x / ntile, tile_id = blockIdx.x % ntile;
  const int ti = tile_id / a.tiles_n, tj = tile_id % a.tiles_n;
  const int item_id = blockIdx.y;
  const Item it = a.items[item_id];
  const bool dense = it.nj == 0;
  const int nX = it.ni, nY = dense ? it.ni : it.nj;
  const int oX = it.oi + ti * TM, oY = (dense ? it.oi : it.oj) + tj * TN;
  const int cX = min(TM, nX - ti * TM), cY = min(TN, nY - tj * TN);
  int64_t k0, k1;
  split_range(a.m, KC, a.splits, split, &k0, &k1);
  const int nchunks = k1 > k0 ? int((k1 - k0 + KC - 1) / KC) : 0;
  const double *G = reinterpret_cast<const double *>(a.G);
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;

  auto load_stage = [&](int stage, int chunk) {
    double *Xs = smem + stage * STAGE_ELEMS;
    const int64_t kb = k0 + int64_t(chunk) * KC;
    for (int pc = tid; pc < (TM + TN) * PPC; pc += NT) {
      const int col = pc / PPC, within = pc % PPC;
      const bool y = col >= TM;
      const int lc = y ? col - TM : col;
      const int64_t row = kb + within * EPP;
      int64_t valid = (lc < (y ? cY : cX)) ? min(int64_t(EPP), k1 - row) : 0;
      if (valid < 0) valid = 0;
      const double *src = valid > 0 ? G + int64_t((y ? oY : oX) + lc) * a.ldg + row : G;
      double *dst = Xs + col * KCP + within * EPP;
      if (VEC == 16)
        cp_async16(dst, src, int(valid * 8));
      else
        cp_async8(dst, src, int(valid * 8));
    }
  };
  double acc[8][8];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j] = 0.0;
  double dx[8] = {0, 0, 0, 0, 0, 0, 0, 0}, dy[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  const bool do_dx = !dense && tj == 0 && ty == 0;
  const bool do_dy = !dense && ti == 0 && tx == 0;
  load_stage(0, 0);
  cp_async_commit();
  for (int c = 0; c < nchunks; ++c) {
    if (c + 1 < nchunks) load_stage((c + 1) & 1, c + 1);
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    const double *Xs = smem + (c & 1) * STAGE_ELEMS;
    const double *Ys = Xs + TM * KCP;
#pragma unroll
    for (int kk = 0; kk < KC; kk += 2) {
      double2 fa[8], fb[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) fa[i] = *reinterpret_cast<const double2 *>(Xs + (tx + 16 * i) * KCP + kk);
#pragma unroll
      for (int j = 0; j < 8; ++j) fb[j] = *reinterpret_cast<const double2 *>(Ys + (ty + 16 * j) * KCP + kk);
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = fma(fa[i].y, fb[j].y, fma(fa[i].x, fb[j].x, acc[i][j]));
      if (do_dx) {
#pragma unroll
        for (int i = 0; i < 8; ++i) dx[i] = fma(fa[i].y, fa[i].y, fma(fa[i].x, fa[i].x, dx[i]));
      }
      if (do_dy) {
#pragma unroll
        for (int j = 0; j < 8; ++j) dy[j] = fma(fb[j].y, fb[j].y, fma(fb[j].x, fb[j].x, dy[j]));
      }
    }
    __syncthreads();
  }
  cp_async_wait<0>();
  const int bmax = a.bmax;
  const int64_t asz = int64_t(bmax) * bmax;
  const int64_t slot = a.splits == 1 ? int64_t(item_id) : int64_t(item_id) * a.splits + split;
  double *Af = reinterpret_cast<double *>(a.splits == 1 ? a.A : a.Apart) + slot * asz;
  double *Df = (a.splits == 1 ? a.D : a.Dpart) + slot * 2 * bmax;
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int r = ti * TM + tx + 16 * i, cc = tj * TN + ty + 16 * j;
      if (r < bmax && cc < bmax) Af[r + int64_t(cc) * bmax] = acc[i][j];
    }
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int r = ti * TM + tx + 16 * i, cc = tj * TN + ty + 16 * i;
    if (do_dx && r < bmax) Df[r] = dx[i];
    if (do_dy && cc < bmax) Df[bmax + cc] = dy[i];
  }
}

// ------------------------------------------------------------------ launch

namespace {

int env_int(const char *name, int dflt) {
  const char *e = std::getenv(name);
  return e ? std::atoi(e) : dflt;
}

// K splits: the smallest S whose grid (units * S CTAs on `slots` resident
// CTAs) wastes less than 3 % of the last wave -- or the best fill found --
// with at least `min_chunks` K chunks per split and a partial scratch that fits
int plan_splits(int64_t units, int slots, int64_t chunks, int min_chunks, int64_t max_by_scratch) {
  static const int forced = env_int("HJB_GRAM_SPLITS", 0);  // experiments only
  int64_t smax = std::min<int64_t>(64, std::max<int64_t>(1, chunks / min_chunks));
  smax = std::max<int64_t>(1, std::min(smax, max_by_scratch));
  if (forced > 0) return int(std::min<int64_t>(forced, smax));
  int best = 1;
  double best_eff = 0.0;
  for (int s = 1; s <= smax; ++s) {
    const int64_t ctas = units * s;
    const int64_t waves = (ctas + slots - 1) / slots;
    const double eff = double(ctas) / double(waves * slots);
    if (eff > best_eff + 1e-9) {
      best_eff = eff;
      best = s;
    }
    if (eff >= 0.97) return s;
  }
  return best;
}

template <typename T, int WM, int WN, int MI, int NI, int KC, int STAGES, int VEC, int MINB>
cudaError_t launch_gram_t(GramArgs a, cudaStream_t st, int *splits_used) {
  using Cfg = GramCfg<T, WM, WN, MI, NI, KC, STAGES>;
  auto k = gram_kernel<T, WM, WN, MI, NI, KC, STAGES, VEC, MINB>;
  static DeviceFlags attr_flags;
  static int slots_dev[64];
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  bool *attr = attr_flags.here();
  if (!attr) return cudaErrorInvalidDevice;
  if (!*attr) {
    e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(Cfg::SMEM));
    if (e != cudaSuccess) return e;
    int per_sm = 0, sms = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, Cfg::NT, Cfg::SMEM);
    if (e != cudaSuccess) return e;
    e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (e != cudaSuccess) return e;
    slots_dev[dev] = std::max(1, per_sm) * std::max(1, sms);
    *attr = true;
  }
  a.tiles_m = (a.bmax + Cfg::TM - 1) / Cfg::TM;
  a.tiles_n = (a.bmax + Cfg::TN - 1) / Cfg::TN;
  const int64_t units = int64_t(a.count) * a.tiles_m * a.tiles_n;
  const int64_t chunks = (a.m + KC - 1) / KC;
  const size_t per_slot = (size_t(a.bmax) * a.bmax * sizeof(T) + 2 * size_t(a.bmax) * sizeof(double)) * a.count;
  const int64_t by_scratch = a.Apart ? int64_t(a.part_bytes / std::max<size_t>(per_slot, 1)) : 1;
  a.splits = plan_splits(units, slots_dev[dev], chunks, 4, by_scratch);
  if (a.splits > 1) {
    // scratch: [count][splits] partial tiles, then [count][splits] norm partials
    a.Dpart = reinterpret_cast<double *>(static_cast<char *>(a.Apart) +
                                         size_t(a.count) * a.splits * a.bmax * a.bmax * sizeof(T));
  }
  if (splits_used) *splits_used = a.splits;
  dim3 grid(unsigned(a.tiles_m * a.tiles_n * a.splits), unsigned(a.count));
  k<<<grid, Cfg::NT, Cfg::SMEM, st>>>(a);
  e = cudaGetLastError();
  if (e != cudaSuccess || a.splits == 1) return e;
  const int64_t elems = int64_t(a.bmax) * a.bmax + 2 * a.bmax;
  gram_reduce_kernel<T><<<dim3(unsigned((elems + 255) / 256), unsigned(a.count)), 256, 0, st>>>(a);
  return cudaGetLastError();
}

template <int KC, int VEC>
cudaError_t launch_gram_ffma(GramArgs a, cudaStream_t st, int *splits_used) {
  constexpr size_t SMEM = 2 * size_t(256) * (KC + 2) * sizeof(double);
  auto k = gram_ffma_kernel<KC, VEC>;
  static DeviceFlags attr_flags;
  bool *attr = attr_flags.here();
  if (!attr) return cudaErrorInvalidDevice;
  if (!*attr) {
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(SMEM));
    if (e != cudaSuccess) return e;
    *attr = true;
  }
  a.tiles_m = (a.bmax + 127) / 128;
  a.tiles_n = a.tiles_m;
  const int64_t units = int64_t(a.count) * a.tiles_m * a.tiles_n;
  const size_t per_slot = (size_t(a.bmax) * a.bmax * 8 + 2 * size_t(a.bmax) * 8) * a.count;
  const int64_t by_scratch = a.Apart ? int64_t(a.part_bytes / std::max<size_t>(per_slot, 1)) : 1;
  a.splits = plan_splits(units, 148, (a.m + KC - 1) / KC, 4, by_scratch);
  if (a.splits > 1)
    a.Dpart = reinterpret_cast<double *>(static_cast<char *>(a.Apart) + size_t(a.count) * a.splits * a.bmax * a.bmax * 8);
  if (splits_used) *splits_used = a.splits;
  k<<<dim3(unsigned(a.tiles_m * a.tiles_n * a.splits), unsigned(a.count)), 256, SMEM, st>>>(a);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess || a.splits == 1) return e;
  const int64_t elems = int64_t(a.bmax) * a.bmax + 2 * a.bmax;
  gram_reduce_kernel<double><<<dim3(unsigned((elems + 255) / 256), unsigned(a.count)), 256, 0, st>>>(a);
  return cudaGetLastError();
}

}  // namespace

size_t gram_scratch_bytes(bool cx, int count, int bmax) {
  // room for up to 16 splits of every item (plan_splits takes fewer when the scratch is smaller)
  const size_t w = cx ? 16 : 8;
  return size_t(count) * 16 * (size_t(bmax) * bmax * w + 2 * size_t(bmax) * sizeof(double));
}

cudaError_t launch_gram(bool cx, GramArgs a, cudaStream_t st, int *splits_used) {
  if (a.count == 0) return cudaSuccess;
  static const int variant = env_int("HJB_GRAM_CFG", 0);  // experiments: tile shape override
  static const int ffma = env_int("HJB_GRAM_FFMA", 0);
  const bool v16 = cx || (a.ldg % 2 == 0);
  if (cx) {
    if (a.bmax <= 32) return launch_gram_t<cplx, 1, 2, 4, 2, 16, 2, 16, 4>(a, st, splits_used);
    switch (variant) {
      case 1: return launch_gram_t<cplx, 2, 2, 4, 4, 16, 2, 16, 2>(a, st, splits_used);   // 64 x 64, 4 warps of 32 x 32
      case 2: return launch_gram_t<cplx, 4, 4, 4, 2, 16, 2, 16, 1>(a, st, splits_used);   // 128 x 64, 16 warps
      case 3: return launch_gram_t<cplx, 2, 4, 4, 2, 16, 3, 16, 2>(a, st, splits_used);   // 64 x 64, 8 warps, 3 stages
      case 4: return launch_gram_t<cplx, 4, 2, 4, 4, 16, 2, 16, 1>(a, st, splits_used);   // 128 x 64, 8 warps of 32 x 32
      default: return launch_gram_t<cplx, 2, 4, 4, 2, 16, 2, 16, 2>(a, st, splits_used);  // 64 x 64, 8 warps
    }
  }
  if (ffma && a.bmax > 32)
    return v16 ? launch_gram_ffma<16, 16>(a, st, splits_used) : launch_gram_ffma<16, 8>(a, st, splits_used);
#define HJB_GRAM_R(WM, WN, MI, NI, KC, ST, MB)                                       \
  (v16 ? launch_gram_t<double, WM, WN, MI, NI, KC, ST, 16, MB>(a, st, splits_used)  \
       : launch_gram_t<double, WM, WN, MI, NI, KC, ST, 8, MB>(a, st, splits_used))
  if (a.bmax <= 32) return HJB_GRAM_R(1, 2, 4, 2, 32, 2, 4);
  // measured on B200 (tools/gram_bench.py, profiles/r2_gram_variants.jsonl):
  // cfg5r 27.1 / 25.4 / 26.5 / 25.6 / 25.7 / 20.7 TFLOP/s for the default / 1 .. 5
  switch (variant) {
    case 1: return HJB_GRAM_R(2, 4, 4, 2, 32, 2, 3);   // 64 x 64, 8 warps of 32 x 16 (round 1's shape)
    case 2: return HJB_GRAM_R(4, 2, 4, 4, 32, 2, 2);   // 128 x 64, 8 warps of 32 x 32
    case 3: return HJB_GRAM_R(2, 4, 4, 2, 32, 3, 2);   // 64 x 64, 8 warps, 3 stages
    case 4: return HJB_GRAM_R(4, 4, 4, 4, 32, 2, 1);   // 128 x 128, 16 warps of 32 x 32
    case 5: return HJB_GRAM_R(4, 2, 4, 4, 16, 4, 2);   // 128 x 64, K chunk 16, 4 stages
    case 6: return HJB_GRAM_R(2, 2, 4, 8, 32, 2, 2);   // 64 x 128, 4 warps of 32 x 64
    default: return HJB_GRAM_R(2, 2, 4, 4, 32, 2, 3);  // 64 x 64, 4 warps of 32 x 32
  }
#undef HJB_GRAM_R
}

}  // namespace hjb
