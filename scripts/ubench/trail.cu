// isolate the trailing update of qp_chol.cuh: step k=0 at T=15, 6 update warps
#include <cstdio>
#include "qp_chol.cuh"
#ifndef VAR
#define VAR 0
#endif
__global__ void __launch_bounds__(256, 1) kt(long long* out, int T, int k) {
  extern __shared__ double sm[];
  for (int e = threadIdx.x; e < qpchol::tile_doubles(8 * T); e += 256) sm[e] = 1e-3 * (e % 17);
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  long long t0 = clock64();
  if ((wid & 3) != 0) qpchol::trailing_update<6>(sm, T, k, wid - 1 - (wid >> 2), lane);
  long long t1 = clock64();
  __syncthreads();
  long long t2 = clock64();
  if (lane == 0) out[wid] = t1 - t0;
  if (threadIdx.x == 0) out[8] = t2 - t0;
}
int main() {
  long long* d; cudaMalloc(&d, 9 * 8);
  const int T = 15;
  const size_t smem = 8 * qpchol::tile_doubles(8 * T);
  cudaFuncSetAttribute(kt, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  for (int k : {0, 0, 4, 8, 12}) {
    kt<<<1, 256, smem>>>(d, T, k);
    long long h[9]; cudaMemcpy(h, d, 72, cudaMemcpyDeviceToHost);
    int tiles = (T - k - 1) * (T - k) / 2 - 1;
    printf("k=%2d tiles=%3d: per-warp", k, tiles);
    for (int w = 0; w < 8; ++w) printf(" %lld", h[w]);
    printf(" | block %lld cycles\n", h[8]);
  }
}
