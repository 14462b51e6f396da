// Latency / throughput probes for the pivot-kernel design (FP64 on sm_100a).
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

__global__ void dfma_lat(double *out, int iters, double a, double b) {
  double x = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) x = fma(x, a, b);
  long long t1 = clock64();
  if (threadIdx.x == 0) { out[0] = double(t1 - t0) / iters; }
  out[1 + threadIdx.x] = x;
}
__global__ void dfma_tput(double *out, int iters, double a, double b) {
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
    x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = double(t1 - t0) / iters;  // cycles per 8 x blockDim FMAs
  out[1 + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
__global__ void rsqrt_lat(double *out, int iters) {
  double x = 2.0 + threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) x = rsqrt(x) + 1.5;
  long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = double(t1 - t0) / iters;
  out[1 + threadIdx.x] = x;
}
__global__ void sqrt_lat(double *out, int iters) {
  double x = 2.0 + threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) x = sqrt(x) + 1.5;
  long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = double(t1 - t0) / iters;
  out[1 + threadIdx.x] = x;
}
__global__ void div_lat(double *out, int iters) {
  double x = 2.0 + threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) x = 3.0 / x + 1.0;
  long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = double(t1 - t0) / iters;
  out[1 + threadIdx.x] = x;
}
__global__ void shfl_lat(double *out, int iters) {
  double x = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) x += __shfl_xor_sync(0xffffffffu, x, 1);
  long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = double(t1 - t0) / iters;
  out[1 + threadIdx.x] = x;
}
__global__ void sync_lat(double *out, int iters) {
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = double(t1 - t0) / iters;
}
__global__ void cluster_sync_lat(double *out, int iters) {
  auto cl = cg::this_cluster();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) cl.sync();
  long long t1 = clock64();
  if (threadIdx.x == 0 && cl.block_rank() == 0) out[0] = double(t1 - t0) / iters;
}
// DSMEM ping: CTA 0 writes a flag into CTA 1 smem, CTA 1 echoes back (relaxed polling)
__global__ void dsmem_pingpong(double *out, int iters) {
  auto cl = cg::this_cluster();
  __shared__ volatile int flag;
  flag = -1;
  cl.sync();
  int me = cl.block_rank();
  volatile int *peer = cl.map_shared_rank((int *)&flag, 1 - me);
  long long t0 = clock64();
  if (threadIdx.x == 0) {
    for (int i = 0; i < iters; ++i) {
      if (me == 0) {
        *peer = i;
        while (flag != i) {}
      } else {
        while (flag != i) {}
        *peer = i;
      }
    }
  }
  long long t1 = clock64();
  cl.sync();
  if (threadIdx.x == 0 && me == 0) out[0] = double(t1 - t0) / iters / 2;  // one-way
}

template <typename K, typename... A>
float run(K k, int blocks, int threads, int cluster, A... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(blocks);
  cfg.blockDim = dim3(threads);
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = cluster; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  cfg.attrs = at; cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, k, args...);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) printf("err %s\n", cudaGetErrorString(e));
  return 0;
}

int main() {
  double *d; cudaMalloc(&d, 4096 * sizeof(double));
  double h;
  auto get = [&]() { cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost); return h; };
  run(dfma_lat, 1, 32, 1, d, 4096, 1.0000001, 1e-9); printf("DFMA dependent latency: %.1f cycles\n", get());
  for (int th : {128, 256, 512, 1024}) {
    run(dfma_tput, 1, th, 1, d, 4096, 1.0000001, 1e-9);
    double c = get();
    printf("DFMA throughput (1 CTA, %d thr): %.1f FMA/clk/SM\n", th, 8.0 * th / c);
  }
  run(rsqrt_lat, 1, 32, 1, d, 1024); printf("rsqrt(double) chain latency: %.1f cycles (incl. 1 DADD)\n", get());
  run(sqrt_lat, 1, 32, 1, d, 1024); printf("sqrt(double) chain latency: %.1f cycles (incl. 1 DADD)\n", get());
  run(div_lat, 1, 32, 1, d, 1024); printf("div(double) chain latency: %.1f cycles (incl. 1 DADD)\n", get());
  run(shfl_lat, 1, 32, 1, d, 4096); printf("shfl_xor(double)+DADD latency: %.1f cycles\n", get());
  run(sync_lat, 1, 256, 1, d, 4096); printf("__syncthreads (256 thr): %.1f cycles\n", get());
  for (int c : {2, 4, 8}) { run(cluster_sync_lat, c, 256, c, d, 4096); printf("cluster.sync (C=%d, 256 thr): %.1f cycles\n", c, get()); }
  run(dsmem_pingpong, 2, 32, 2, d, 2048); printf("DSMEM one-way flag latency: %.1f cycles\n", get());
  return 0;
}
