// Batched long-K Gram of block-column pairs on FP64 tensor cores (DMMA).
//
// Replaces the per-pair Gram A_ij = G_i^H G_j of the reference's 2F step
// (pkg/src/hjacobi/parallel.py:193 -> core.py:42-56) and the diagonal-block
// Gram of the F pre-pass (parallel.py:143), and fuses the column-norm
// refresh D = colnorms^2 (parallel.py:208-209 / core.py:59-61) into the same
// pass over the data.
//
// Layout: G column-major (ld = ldg); block column = contiguous m x b slab.
// One CTA computes a TILE x TILE tile of one item's Gram over one K split;
// operands are staged through shared memory with a cp.async pipeline and fed
// to mma.sync.m8n8k4.f64 (SASS DMMA).  The K splits of one tile form a
// thread-block cluster: every CTA parks its partial tile in shared memory and
// after one cluster barrier reduces a 1/CL slice of the tile over the peers'
// partials (DSMEM) in fixed rank order -- deterministic and parallel.
#include <cooperative_groups.h>

#include "common.cuh"
#include "kernels.h"

namespace hjb {

// WM row-warps x 4 column-warps per TILE x TILE tile (TILE = 32 WM); each
// warp owns 32 rows x TILE/4 columns (NI = TILE/32 8x8 fragments per row
// block), so every SM keeps 16 warps of DMMA chains in flight
template <typename T, int WM, int KC, int STAGES>
struct GramCfg {
  static constexpr int TILE = 32 * WM;
  static constexpr int WC = 4;                 // column-warps
  static constexpr int NI = TILE / (8 * WC);   // 8-column fragments per warp
  static constexpr int NT = 32 * WM * WC;
  static constexpr int PAD = S<T>::cx ? 4 : 4;
  static constexpr int KCP = KC + PAD;                      // elements per staged column
  static constexpr int STAGE_ELEMS = 2 * TILE * KCP;        // X and Y tiles
  static constexpr size_t SMEM = size_t(STAGES) * STAGE_ELEMS * sizeof(T);
};

// (X^H Y) fragment products: real a*b; complex conj(a)*b on 4 DMMAs.
template <typename T> struct GramAcc;
template <> struct GramAcc<double> {
  double v[2];
  __device__ void zero() { v[0] = v[1] = 0.0; }
  __device__ void mma(double a, double b) { dmma(v[0], v[1], a, b); }
  __device__ double get(int q) const { return v[q]; }
};
template <> struct GramAcc<cplx> {
  // four independent DMMA chains (no dependent pair per k step):
  // conj(a) b = (ar br + ai bi) + i (ar bi - ai br)
  double rr[2], ii[2], ri[2], ir[2];
  __device__ void zero() { rr[0] = rr[1] = ii[0] = ii[1] = ri[0] = ri[1] = ir[0] = ir[1] = 0.0; }
  __device__ void mma(cplx a, cplx b) {
    dmma(rr[0], rr[1], a.x, b.x);
    dmma(ii[0], ii[1], a.y, b.y);
    dmma(ri[0], ri[1], a.x, b.y);
    dmma(ir[0], ir[1], a.y, b.x);
  }
  __device__ cplx get(int q) const { return make_double2(rr[q] + ii[q], ri[q] - ir[q]); }
};

template <typename T, int WM, int KC, int STAGES, int VEC, int CL>
__global__ void __launch_bounds__(GramCfg<T, WM, KC, STAGES>::NT)
    gram_kernel(GramArgs a) {
  using Cfg = GramCfg<T, WM, KC, STAGES>;
  constexpr int TILE = Cfg::TILE, NT = Cfg::NT, KCP = Cfg::KCP;
  constexpr int EPP = VEC / int(sizeof(T));       // elements per cp.async piece
  constexpr int PPC = KC / EPP;                   // pieces per staged column
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T *smem = reinterpret_cast<T *>(smem_raw);
  __shared__ int s_last;

  const int tiles = a.tiles;
  const int tile_id = blockIdx.x / CL;
  const int ti = tile_id / tiles, tj = tile_id % tiles;
  const int split = blockIdx.x % CL;  // == rank in the cluster
  const int item_id = blockIdx.z;
  const Item it = a.items[item_id];
  const bool dense = it.nj == 0;
  const int nX = it.ni, nY = dense ? it.ni : it.nj;
  const int oX = it.oi + ti * TILE, oY = (dense ? it.oi : it.oj) + tj * TILE;
  const int cX = min(TILE, nX - ti * TILE), cY = min(TILE, nY - tj * TILE);  // may be <= 0
  const int64_t k0 = int64_t(split) * a.ksplit;
  const int64_t k1 = min(a.m, k0 + a.ksplit);
  const int nchunks = k1 > k0 ? int((k1 - k0 + KC - 1) / KC) : 0;
  const T *G = reinterpret_cast<const T *>(a.G);

  constexpr int NI = Cfg::NI, WC = Cfg::WC;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp / WC, wn = warp % WC;

  auto load_stage = [&](int stage, int chunk) {
    T *Xs = smem + stage * Cfg::STAGE_ELEMS;
    T *Ys = Xs + TILE * KCP;
    const int64_t kb = k0 + int64_t(chunk) * KC;
    for (int pc = tid; pc < 2 * TILE * PPC; pc += NT) {
      const int which = pc / (TILE * PPC);
      const int rem = pc % (TILE * PPC);
      const int col = rem / PPC, within = rem % PPC;
      const int64_t row = kb + within * EPP;
      const int ccount = which ? cY : cX;
      const int coff = which ? oY : oX;
      int64_t valid = (col < ccount) ? min(int64_t(EPP), k1 - row) : 0;
      if (valid < 0) valid = 0;
      const T *src = valid > 0 ? G + int64_t(coff + col) * a.ldg + row : G;
      T *dst = (which ? Ys : Xs) + col * KCP + within * EPP;
      if (VEC == 16)
        cp_async16(dst, src, int(valid * sizeof(T)));
      else
        cp_async8(dst, src, int(valid * sizeof(T)));
    }
  };

  GramAcc<T> acc[4][NI];
#pragma unroll
  for (int mi = 0; mi < 4; ++mi)
#pragma unroll
    for (int ni = 0; ni < NI; ++ni) acc[mi][ni].zero();
  double dx[4] = {0, 0, 0, 0}, dy[NI];
#pragma unroll
  for (int ni = 0; ni < NI; ++ni) dy[ni] = 0.0;
  const bool do_dx = !dense && tj == 0 && wn == 0;
  const bool do_dy = !dense && ti == 0 && wm == 0;

#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < nchunks) load_stage(s, s);
    cp_async_commit();
  }
  for (int c = 0; c < nchunks; ++c) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    {
      const int nxt = c + STAGES - 1;
      if (nxt < nchunks) load_stage(nxt % STAGES, nxt);
      cp_async_commit();
    }
    const T *Xs = smem + (c % STAGES) * Cfg::STAGE_ELEMS;
    const T *Ys = Xs + TILE * KCP;
#pragma unroll
    for (int kk = 0; kk < KC; kk += 4) {
      T fa[4], fb[NI];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
        fa[mi] = Xs[(wm * 32 + mi * 8 + (lane >> 2)) * KCP + kk + (lane & 3)];
#pragma unroll
      for (int ni = 0; ni < NI; ++ni)
        fb[ni] = Ys[(wn * 8 * NI + ni * 8 + (lane >> 2)) * KCP + kk + (lane & 3)];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < NI; ++ni) acc[mi][ni].mma(fa[mi], fb[ni]);
      if (do_dx) {
#pragma unroll
        for (int mi = 0; mi < 4; ++mi) dx[mi] += abs2(fa[mi]);
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
  for (int mi = 0; mi < 4; ++mi) {
    dx[mi] += __shfl_xor_sync(0xffffffffu, dx[mi], 1);
    dx[mi] += __shfl_xor_sync(0xffffffffu, dx[mi], 2);
  }
#pragma unroll
  for (int ni = 0; ni < NI; ++ni) {
    dy[ni] += __shfl_xor_sync(0xffffffffu, dy[ni], 1);
    dy[ni] += __shfl_xor_sync(0xffffffffu, dy[ni], 2);
  }
  const int bmax = a.bmax;
  const int64_t asz = int64_t(bmax) * bmax;
  T *Af = reinterpret_cast<T *>(a.A) + int64_t(item_id) * asz;
  double *Df = a.D + int64_t(item_id) * 2 * bmax;
  if constexpr (CL == 1) {
#pragma unroll
    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
      for (int ni = 0; ni < NI; ++ni)
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const int r = ti * TILE + wm * 32 + mi * 8 + (lane >> 2);
          const int cc = tj * TILE + wn * 8 * NI + ni * 8 + 2 * (lane & 3) + q;
          if (r < bmax && cc < bmax) Af[r + int64_t(cc) * bmax] = acc[mi][ni].get(q);
        }
    if ((lane & 3) == 0) {
#pragma unroll
      for (int mi = 0; mi < 4; ++mi) {
        const int r = ti * TILE + wm * 32 + mi * 8 + (lane >> 2);
        if (do_dx && r < bmax) Df[r] = dx[mi];
      }
#pragma unroll
      for (int ni = 0; ni < NI; ++ni) {
        const int cc = tj * TILE + wn * 8 * NI + ni * 8 + (lane >> 2);
        if (do_dy && cc < bmax) Df[bmax + cc] = dy[ni];
      }
    }
  } else {
    // ---- split-K reduction over the cluster (DSMEM), fixed rank order ----
    namespace cg = cooperative_groups;
    cg::cluster_group cluster = cg::this_cluster();
    __syncthreads();  // staging buffers are free
    T *P = smem;                                               // [TILE][TILE] column-major partial
    double *Pd = reinterpret_cast<double *>(smem + TILE * TILE);  // [2][TILE] norm partials
#pragma unroll
    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
      for (int ni = 0; ni < NI; ++ni)
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const int r = wm * 32 + mi * 8 + (lane >> 2);
          const int cc = wn * 8 * NI + ni * 8 + 2 * (lane & 3) + q;
          P[r + cc * TILE] = acc[mi][ni].get(q);
        }
    if ((lane & 3) == 0) {
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
        if (do_dx) Pd[wm * 32 + mi * 8 + (lane >> 2)] = dx[mi];
#pragma unroll
      for (int ni = 0; ni < NI; ++ni)
        if (do_dy) Pd[TILE + wn * 8 * NI + ni * 8 + (lane >> 2)] = dy[ni];
    }
    cluster.sync();
    constexpr int E = TILE * TILE, SL = (E + CL - 1) / CL;
    for (int e = split * SL + tid; e < min(E, (split + 1) * SL); e += NT) {
      const int r = ti * TILE + (e % TILE), cc = tj * TILE + (e / TILE);
      T v = *cluster.map_shared_rank(P + e, 0);
#pragma unroll
      for (int q = 1; q < CL; ++q) v = add(v, *cluster.map_shared_rank(P + e, q));
      if (r < bmax && cc < bmax) Af[r + int64_t(cc) * bmax] = v;
    }
    if (!dense && split == CL - 1) {
      for (int e = tid; e < 2 * TILE; e += NT) {
        const bool y = e >= TILE;
        const int idx = (y ? tj : ti) * TILE + (e % TILE);
        if ((y ? ti != 0 : tj != 0) || idx >= bmax) continue;
        double v = *cluster.map_shared_rank(Pd + e, 0);
#pragma unroll
        for (int q = 1; q < CL; ++q) v += *cluster.map_shared_rank(Pd + e, q);
        Df[(y ? bmax : 0) + idx] = v;
      }
    }
    cluster.sync();  // peers' partials stay alive until every slice is read
  }
}

template <typename T, int WM, int KC, int STAGES, int VEC, int CL>
static cudaError_t launch_gram_cl(const GramArgs &a, cudaStream_t st) {
  using Cfg = GramCfg<T, WM, KC, STAGES>;
  static_assert(Cfg::TILE * Cfg::TILE * sizeof(T) + 2 * Cfg::TILE * sizeof(double) <= Cfg::SMEM,
                "partial tile fits the staging buffers");
  auto k = gram_kernel<T, WM, KC, STAGES, VEC, CL>;
  static DeviceFlags attr_flags;
  bool *attr = attr_flags.here();
  if (!attr) return cudaErrorInvalidDevice;
  if (!*attr) {
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(Cfg::SMEM));
    if (e != cudaSuccess) return e;
    if (CL > 8) {
      e = cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      if (e != cudaSuccess) return e;
    }
    *attr = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(a.tiles * a.tiles * CL, 1, a.count);
  cfg.blockDim = dim3(Cfg::NT);
  cfg.dynamicSmemBytes = Cfg::SMEM;
  cfg.stream = st;
  cudaLaunchAttribute attrs[1];
  attrs[0].id = cudaLaunchAttributeClusterDimension;
  attrs[0].val.clusterDim.x = CL;
  attrs[0].val.clusterDim.y = 1;
  attrs[0].val.clusterDim.z = 1;
  cfg.attrs = attrs;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k, a);
}

template <typename T, int WM, int KC, int STAGES, int VEC>
static cudaError_t launch_gram_t(const GramArgs &a, cudaStream_t st) {
  switch (a.splits) {
    case 1: return launch_gram_cl<T, WM, KC, STAGES, VEC, 1>(a, st);
    case 2: return launch_gram_cl<T, WM, KC, STAGES, VEC, 2>(a, st);
    case 4: return launch_gram_cl<T, WM, KC, STAGES, VEC, 4>(a, st);
    case 8: return launch_gram_cl<T, WM, KC, STAGES, VEC, 8>(a, st);
    case 16: return launch_gram_cl<T, WM, KC, STAGES, VEC, 16>(a, st);
  }
  return cudaErrorInvalidConfiguration;
}

int gram_tile(int bmax) { return bmax <= 32 ? 32 : 64; }

cudaError_t launch_gram(bool cx, GramArgs a, cudaStream_t st) {
  const int tile = gram_tile(a.bmax);
  a.tiles = (a.bmax + tile - 1) / tile;
  const bool v16 = cx || (a.ldg % 2 == 0);
  if (cx) {
    if (tile == 32) return launch_gram_t<cplx, 1, 16, 2, 16>(a, st);
    return launch_gram_t<cplx, 2, 16, 2, 16>(a, st);
  }
  if (tile == 32)
    return v16 ? launch_gram_t<double, 1, 32, 2, 16>(a, st) : launch_gram_t<double, 1, 32, 2, 8>(a, st);
  return v16 ? launch_gram_t<double, 2, 32, 2, 16>(a, st) : launch_gram_t<double, 2, 32, 2, 8>(a, st);
}

int gram_kc(bool cx) { return cx ? 16 : 32; }

}  // namespace hjb
