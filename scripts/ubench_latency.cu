// Micro-benchmark of the latencies that bound the single-CTA QP solver:
// dependent DFMA chain, fp64 rsqrt / sqrt / div, shfl, LDS round trip,
// __syncthreads with 16 warps, named barrier.  nvcc -arch=sm_100a -O3.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_lat(double* out, long long* cyc, double seed) {
  __shared__ double sm[1024];
  const int tid = threadIdx.x;
  sm[tid] = seed + tid;
  __syncthreads();
  double x = seed + tid * 1e-3, y = 1.0000001;
  long long t0, t1;
  // 1. dependent DFMA chain
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1024; ++i) x = fma(x, y, 1e-9);
  t1 = clock64();
  if (tid == 0) cyc[0] = (t1 - t0);
  // 2. rsqrt chain
  double z = x;
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 256; ++i) z = rsqrt(z + 2.0);
  t1 = clock64();
  if (tid == 0) cyc[1] = (t1 - t0);
  // 3. sqrt + div chain
  double w = z;
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 256; ++i) w = 1.0 / sqrt(w + 2.0);
  t1 = clock64();
  if (tid == 0) cyc[2] = (t1 - t0);
  // 4. shfl chain
  double v = w;
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1024; ++i) v = __shfl_sync(0xffffffffu, v, (i + 1) & 31) + 1e-9;
  t1 = clock64();
  if (tid == 0) cyc[3] = (t1 - t0);
  // 5. LDS dependent chain (pointer chasing through an index)
  int idx = tid & 7;
  int* si = (int*)sm;
  __syncthreads();
  if (tid < 256) si[tid] = (tid * 7 + 3) & 255;
  __syncthreads();
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1024; ++i) idx = si[idx];
  t1 = clock64();
  if (tid == 0) cyc[4] = (t1 - t0);
  __syncthreads();
  // 6. __syncthreads round trips with all warps
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1024; ++i) __syncthreads();
  t1 = clock64();
  if (tid == 0) cyc[5] = (t1 - t0);
  // 7. DMUL then dependent DADD
  double a = v;
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1024; ++i) a = a * y + 1e-12;
  t1 = clock64();
  if (tid == 0) cyc[6] = (t1 - t0);
  // 8. independent DFMA throughput per warp (8 chains)
  double c0 = x, c1 = x + 1, c2 = x + 2, c3 = x + 3, c4 = x + 4, c5 = x + 5, c6 = x + 6, c7 = x + 7;
  t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1024; ++i) {
    c0 = fma(c0, y, 1e-9); c1 = fma(c1, y, 1e-9); c2 = fma(c2, y, 1e-9); c3 = fma(c3, y, 1e-9);
    c4 = fma(c4, y, 1e-9); c5 = fma(c5, y, 1e-9); c6 = fma(c6, y, 1e-9); c7 = fma(c7, y, 1e-9);
  }
  t1 = clock64();
  if (tid == 0) cyc[7] = (t1 - t0);
  out[tid] = x + z + w + v + idx + a + c0 + c1 + c2 + c3 + c4 + c5 + c6 + c7;
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 1024 * sizeof(double));
  cudaMallocManaged(&cyc, 16 * sizeof(long long));
  const char* names[] = {"DFMA dep (per op)", "rsqrt(f64) dep", "1/sqrt(f64) dep", "shfl dep",
                         "LDS dep", "__syncthreads", "DMUL+DADD dep (fma-contracted?)",
                         "DFMA 8 chains (per 8 ops)"};
  const int counts[] = {1024, 256, 256, 1024, 1024, 1024, 1024, 1024};
  for (int threads : {32, 512}) {
    k_lat<<<1, threads>>>(out, cyc, 1.5);
    cudaDeviceSynchronize();
    k_lat<<<1, threads>>>(out, cyc, 1.5);
    cudaDeviceSynchronize();
    printf("threads=%d\n", threads);
    for (int i = 0; i < 8; ++i) printf("  %-34s %8.1f cycles\n", names[i], (double)cyc[i] / counts[i]);
  }
  return 0;
}
