// Per-round cost of the pivot kernel's cluster partial exchange in isolation:
// every CTA pushes P2 partials to each peer with st.async + mbarrier
// complete_tx, waits for its own barrier, sums, re-arms (double buffered).
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;
__device__ __forceinline__ uint32_t su32(const void *p) { return uint32_t(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint32_t mapa(uint32_t a, int r) { uint32_t o; asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(o) : "r"(a), "r"(r)); return o; }
__device__ __forceinline__ void arm(uint64_t *b, unsigned tx) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(tx) : "memory"); }
__device__ __forceinline__ void wait(uint64_t *b, unsigned par) {
  asm volatile("{\n .reg .pred p;\nW_%=:\n mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n @!p bra W_%=;\n}" ::"r"(su32(b)), "r"(par) : "memory");
}
__device__ __forceinline__ void sta(uint32_t ra, double v, uint32_t rb) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(ra), "l"(__double_as_longlong(v)), "r"(rb) : "memory");
}
template <int C, int P2, int NT>
__global__ void __launch_bounds__(NT, 1) xchg(double *out, int rounds, int mode) {
  constexpr int TPP = NT / P2;
  __shared__ double part[2][C][P2];
  __shared__ uint64_t mbar[2];
  auto cl = cg::this_cluster();
  const int crank = cl.block_rank(), tid = threadIdx.x, slot = tid / TPP, lane = tid % TPP;
  constexpr unsigned TX = (C - 1) * P2 * 8;
  if (tid == 0) {
    for (int b = 0; b < 2; ++b) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&mbar[b])));
    asm volatile("fence.mbarrier_init.release.cluster;");
    arm(&mbar[0], TX); arm(&mbar[1], TX);
  }
  cl.sync();
  double v = tid * 1e-3;
  long long t0 = clock64();
  for (int g = 0; g < rounds; ++g) {
    const int buf = g & 1;
    double *mine = &part[buf][crank][slot];
    const uint32_t la = su32(mine), lb = su32(&mbar[buf]);
    for (int q = lane; q < C; q += TPP) {
      if (q == crank) *mine = v; else sta(mapa(la, q), v, mapa(lb, q));
    }
    if (mode >= 1) __syncthreads();
    if (tid < P2) {
      wait(&mbar[buf], (g >> 1) & 1);
      double acc = 0;
      for (int r = 0; r < C; ++r) acc += part[buf][r][tid];
      v = acc * 0.5;
    }
    __syncthreads();
    if (tid == NT - 1) arm(&mbar[buf], TX);
    if (mode >= 2) __syncthreads();
  }
  long long t1 = clock64();
  if (tid == 0 && crank == 0) out[blockIdx.x / C] = double(t1 - t0) / rounds;
  cl.sync();
}
template <int C>
void run(double *d, int mode) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(C * 4);
  cfg.blockDim = dim3(256);
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = C; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  cfg.attrs = at; cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, xchg<C, 64, 256>, d, 2000, mode);
  cudaError_t e = cudaDeviceSynchronize();
  double h; cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("C=%d mode=%d: %.0f cycles/round %s\n", C, mode, h, e ? cudaGetErrorString(e) : "");
}
int main() {
  double *d; cudaMalloc(&d, 1024);
  for (int mode = 0; mode < 3; ++mode) { run<2>(d, mode); run<4>(d, mode); run<8>(d, mode); }
  return 0;
}
