// Micro-benchmark of the K-QP Cholesky step pieces on one CTA (n = 140):
// factor_pivot chain, look-ahead body, panel rows, rank-4 update groups.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_2602_17601_b200/csrc chol_parts.cu
#include "../../paper_2602_17601_b200/csrc/k_qp.cu"
#include <cstdio>

__global__ void k_parts(int n, const double* A, long long* cyc, double* sink) {
  extern __shared__ double K[];
  __shared__ double pv[32];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  for (int c = 0; c < n; ++c)
    for (int r = c + tid; r < n; r += blockDim.x) K[colbase(c, n) + r] = A[r * n + c];
  if (tid < 32) pv[tid] = 0.5 + 0.01 * tid;
  __syncthreads();
  double acc = 0.0;
  // 1. factor_pivot chain (thread 0), 35 dependent calls
  if (tid == 0) {
    double E[4][4];
    for (int a = 0; a < 4; ++a)
      for (int b = 0; b < 4; ++b) E[a][b] = (a == b) ? 4.0 + K[a] : 0.1 * K[a + b];
    long long t0 = clock64();
    for (int s = 0; s < 35; ++s) {
      factor_pivot(E, 4, pv);
      E[0][0] = 4.0 + pv[0] * 1e-3;  // dependence on the previous factor
    }
    long long t1 = clock64();
    cyc[0] = (t1 - t0) / 35;
  }
  __syncthreads();
  // 2. look-ahead body (thread 0): loads, E update, factor
  if (tid == 0) {
    long long t0 = clock64();
    for (int s = 0; s < 34; ++s) {
      const int j = 4 * s, j2 = j + 4;
      int cjq[4];
      for (int q = 0; q < 4; ++q) cjq[q] = colbase(j + q, n);
      double La[4][4];
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        const int r = min(j2 + a, n - 1);
#pragma unroll
        for (int q = 0; q < 4; ++q) La[a][q] = K[cjq[q] + r];
      }
      double E[4][4];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          if (b <= a) {
            const int idx = colbase(j2 + b, n) + j2 + a;
            E[a][b] = K[idx] - fma(La[a][3], La[b][3], fma(La[a][2], La[b][2], fma(La[a][1], La[b][1], La[a][0] * La[b][0])));
          } else E[a][b] = 0.0;
        }
      E[0][0] = fabs(E[0][0]) + 10.0 + pv[0] * 1e-9;
      E[1][1] = fabs(E[1][1]) + 10.0; E[2][2] = fabs(E[2][2]) + 10.0; E[3][3] = fabs(E[3][3]) + 10.0;
      factor_pivot(E, 4, pv);
    }
    long long t1 = clock64();
    cyc[1] = (t1 - t0) / 34;
  }
  __syncthreads();
  // 3. panel rows (all threads): 35 steps, barrier each
  {
    long long t0 = clock64();
    for (int s = 0; s < 34; ++s) {
      const int j = 4 * s, j2 = j + 4;
      int cjq[4];
      for (int q = 0; q < 4; ++q) cjq[q] = colbase(j + q, n);
      for (int r = j2 + tid; r < n; r += blockDim.x) {
        double w[4], x[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) w[q] = K[cjq[q] + r];
        lrow4(w, pv, x);
#pragma unroll
        for (int q = 0; q < 4; ++q) acc += x[q];
      }
      __syncthreads();
    }
    long long t1 = clock64();
    if (tid == 0) cyc[2] = (t1 - t0) / 34;
  }
  // 4. barrier only
  {
    long long t0 = clock64();
    for (int s = 0; s < 34; ++s) __syncthreads();
    long long t1 = clock64();
    if (tid == 0) cyc[3] = (t1 - t0) / 34;
  }
  // 5. update groups (warps 1..7), per step, then barrier
  {
    long long t0 = clock64();
    long long tw = 0;
    for (int s = 0; s < 34; ++s) {
      const int j = 4 * s, j2 = j + 4, pe = min(n, j2 + 4);
      int cjq[4];
      for (int q = 0; q < 4; ++q) cjq[q] = colbase(j + q, n);
      if (wid > 0) {
        long long ta = clock64();
        double Lr[5][4];
#pragma unroll
        for (int t = 0; t < 5; ++t) {
          const int r = min(lane + 32 * t, n - 1);
#pragma unroll
          for (int q = 0; q < 4; ++q) Lr[t][q] = K[cjq[q] + r] * 1e-6;
        }
        for (int c0g = j2 + 4 * (wid - 1); c0g < n; c0g += 4 * 7)
          update_group_dispatch<5, 0>(max(c0g, pe) >> 5, K, n, c0g, pe, cjq, Lr, lane);
        tw += clock64() - ta;
      }
      __syncthreads();
    }
    long long t1 = clock64();
    if (tid == 0) cyc[4] = (t1 - t0) / 34;
    if (tid == 32) cyc[5] = tw / 34;
  }
  // 6. one step at j = 0: single warp doing every group, then 7 warps
  for (int nw = 1; nw <= 7; nw += 6) {
    __syncthreads();
    const int j = 0, j2 = 4, pe = 8;
    int cjq[4];
    for (int q = 0; q < 4; ++q) cjq[q] = colbase(j + q, n);
    long long t0 = clock64();
    if (wid >= 1 && wid <= nw) {
      double Lr[5][4];
#pragma unroll
      for (int t = 0; t < 5; ++t) {
        const int r = min(lane + 32 * t, n - 1);
#pragma unroll
        for (int q = 0; q < 4; ++q) Lr[t][q] = K[cjq[q] + r] * 1e-6;
      }
      for (int c0g = j2 + 4 * (wid - 1); c0g < n; c0g += 4 * nw)
        update_group_dispatch<5, 0>(max(c0g, pe) >> 5, K, n, c0g, pe, cjq, Lr, lane);
    }
    __syncthreads();
    long long t1 = clock64();
    if (tid == 0) cyc[nw == 1 ? 6 : 7] = t1 - t0;
  }
  // 7. DMMA tiles at j = 0 with 7 warps, and the average step
  {
    __syncthreads();
    const int j = 0, j2 = 4, pe = 8;
    int cjq[4];
    for (int q = 0; q < 4; ++q) cjq[q] = colbase(j + q, n);
    long long t0 = clock64();
    if (wid >= 1) update_tiles(K, n, 4, j2, pe, cjq, wid - 1, 7, lane);
    __syncthreads();
    long long t1 = clock64();
    if (tid == 0) cyc[8] = t1 - t0;
    t0 = clock64();
    for (int s = 0; s < 34; ++s) {
      const int jj = 4 * s, jj2 = jj + 4, ppe = min(n, jj2 + 4);
      int cq[4];
      for (int q = 0; q < 4; ++q) cq[q] = colbase(jj + q, n);
      if (wid >= 1) update_tiles(K, n, 4, jj2, ppe, cq, wid - 1, 7, lane);
      __syncthreads();
    }
    t1 = clock64();
    if (tid == 0) cyc[9] = (t1 - t0) / 34;
  }
  sink[tid] = acc + pv[3];
}

int main() {
  const int n = 140;
  double* hA = new double[n * n];
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) hA[i * n + j] = (i == j) ? n + 1.0 : 1.0 / (1.0 + i + j);
  double *dA, *sink;
  long long* cyc;
  cudaMalloc(&dA, sizeof(double) * n * n);
  cudaMalloc(&sink, sizeof(double) * 256);
  cudaMalloc(&cyc, sizeof(long long) * 16);
  cudaMemcpy(dA, hA, sizeof(double) * n * n, cudaMemcpyHostToDevice);
  size_t sm = sizeof(double) * n * (n + 1) / 2;
  cudaFuncSetAttribute(k_parts, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  for (int rep = 0; rep < 2; ++rep) k_parts<<<1, 256, sm>>>(n, dA, cyc, sink);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[16];
  cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  printf("err=%s\nfactor_pivot %lld\nlookahead %lld\npanel+bar %lld\nbarrier %lld\nupdate+bar %lld\nupdate(warp1) %lld\nj0 1warp %lld\nj0 7warps %lld\nj0 dmma %lld\ndmma step avg %lld\n",
         cudaGetErrorString(e), h[0], h[1], h[2], h[3], h[4], h[5], h[6], h[7], h[8], h[9]);
  return 0;
}
