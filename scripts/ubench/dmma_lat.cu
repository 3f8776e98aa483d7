#include <cstdio>
__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b, double c0, double c1) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%4,%5};"
               : "=d"(d0), "=d"(d1) : "d"(a), "d"(b), "d"(c0), "d"(c1));
}
__global__ void k(double* out, long long* cyc, int nwarps_active) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double a = 1e-3 * lane, b = 1e-3 * (lane + 1);
  double c0 = 1, c1 = 2, e0 = 3, e1 = 4, f0 = 5, f1 = 6, g0 = 7, g1 = 8;
  __syncthreads();
  long long t0 = clock64();
  if (wid < nwarps_active) {
#pragma unroll 1
    for (int i = 0; i < 256; ++i) dmma884(c0, c1, a, b, c0, c1);
  }
  long long t1 = clock64();
  __syncthreads();
  long long t2 = clock64();
  if (wid < nwarps_active) {
#pragma unroll 1
    for (int i = 0; i < 256; ++i) {
      dmma884(c0, c1, a, b, c0, c1);
      dmma884(e0, e1, a, b, e0, e1);
      dmma884(f0, f1, a, b, f0, f1);
      dmma884(g0, g1, a, b, g0, g1);
    }
  }
  long long t3 = clock64();
  double x = c0, y = 1.0000001;
  __syncthreads();
  long long t4 = clock64();
  if (wid < nwarps_active) {
#pragma unroll 1
    for (int i = 0; i < 256; ++i) {
      x = fma(x, y, 1e-9); e0 = fma(e0, y, 1e-9); f0 = fma(f0, y, 1e-9); g0 = fma(g0, y, 1e-9);
    }
  }
  long long t5 = clock64();
  if (threadIdx.x == 0) { cyc[0] = (t1 - t0) / 256; cyc[1] = (t3 - t2) / 256; cyc[2] = (t5 - t4) / 256; }
  out[threadIdx.x] = c0 + c1 + e0 + e1 + f0 + f1 + g0 + g1 + x;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 8 * 1024); cudaMalloc(&c, 64);
  for (int nw : {1, 4, 8, 16}) {
    k<<<1, 512>>>(o, c, nw); cudaDeviceSynchronize();
    long long h[3]; cudaMemcpy(h, c, 24, cudaMemcpyDeviceToHost);
    printf("warps %2d: dependent DMMA %lld cyc, 4 indep DMMA per iter %lld cyc, 4 indep DFMA per iter %lld cyc\n", nw, h[0], h[1], h[2]);
  }
}
