#include <cstdio>
#include <cuda_runtime.h>
__global__ void shfl_tput(double *out, int iters) {
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    x0 = __shfl_sync(0xffffffffu, x0, (threadIdx.x + 4) & 31);
    x1 = __shfl_sync(0xffffffffu, x1, (threadIdx.x + 4) & 31);
    x2 = __shfl_sync(0xffffffffu, x2, (threadIdx.x + 4) & 31);
    x3 = __shfl_sync(0xffffffffu, x3, (threadIdx.x + 4) & 31);
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = double(t1 - t0) / iters;
  out[1 + threadIdx.x] = x0 + x1 + x2 + x3;
}
__global__ void lds_tput(double *out, int iters) {
  __shared__ double buf[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) buf[i] = i;
  __syncthreads();
  double a = 0;
  int idx = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    a += buf[(idx + i * 32) & 4095];
    a += buf[(idx + i * 32 + 1024) & 4095];
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = double(t1 - t0) / iters;
  out[1 + threadIdx.x] = a;
}
int main() {
  double *d; cudaMalloc(&d, 8192 * 8); double h;
  for (int th : {256, 512, 1024}) {
    shfl_tput<<<1, th>>>(d, 4096); cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    // each iteration: 4 double shuffles = 8 32-bit SHFL per thread
    printf("SHFL (32-bit) throughput, %d thr: %.2f warp-SHFL/clk/SM\n", th, 8.0 * th / 32 / h);
    lds_tput<<<1, th>>>(d, 4096); cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("LDS.64 throughput, %d thr: %.2f warp-LDS/clk/SM (%.0f B/clk)\n", th, 2.0 * th / 32 / h, 2.0 * th * 8 / h);
  }
  return 0;
}
