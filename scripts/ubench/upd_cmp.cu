// DMMA vs DFMA rank-4 trailing update of the K-QP Cholesky: results and cycles.
#include "../../paper_2602_17601_b200/csrc/k_qp.cu"
#include <cstdio>

__global__ void k_upd(int n, const double* A, int mode, int j, double* out, long long* cyc) {
  extern __shared__ double K[];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  for (int c = 0; c < n; ++c)
    for (int r = c + tid; r < n; r += blockDim.x) K[colbase(c, n) + r] = A[r * n + c];
  __syncthreads();
  const int j2 = j + 4, pe = min(n, j2 + 4);
  int cjq[4];
  for (int q = 0; q < 4; ++q) cjq[q] = colbase(j + q, n);
  long long t0 = clock64();
  for (int rep = 0; rep < 8; ++rep) {
    if (mode == 0) {
      if (wid > 0) {
        double Lr[5][4];
#pragma unroll
        for (int t = 0; t < 5; ++t) {
          const int r = min(lane + 32 * t, n - 1);
#pragma unroll
          for (int q = 0; q < 4; ++q) Lr[t][q] = K[cjq[q] + r];
        }
        for (int c0g = j2 + 4 * (wid - 1); c0g < n; c0g += 4 * 7)
          update_group_dispatch<5, 0>(max(c0g, pe) >> 5, K, n, c0g, pe, cjq, Lr, lane);
      }
    } else {
      if (wid > 0) update_tiles(K, n, 4, j2, pe, cjq, wid - 1, 7, lane);
    }
    __syncthreads();
  }
  long long t1 = clock64();
  if (tid == 0) cyc[0] = (t1 - t0) / 8;
  for (int t = tid; t < n * (n + 1) / 2; t += blockDim.x) out[t] = K[t];
}

int main() {
  const int n = 140, np = n * (n + 1) / 2;
  double* hA = new double[n * n];
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) hA[i * n + j] = (i == j) ? 2.0 : 0.01 * ((i * 7 + j * 3) % 11) / (1.0 + (i > j ? i - j : j - i));
  double *dA, *o0, *o1;
  long long* cyc;
  cudaMalloc(&dA, sizeof(double) * n * n);
  cudaMalloc(&o0, sizeof(double) * np);
  cudaMalloc(&o1, sizeof(double) * np);
  cudaMalloc(&cyc, sizeof(long long) * 4);
  cudaMemcpy(dA, hA, sizeof(double) * n * n, cudaMemcpyHostToDevice);
  size_t sm = sizeof(double) * np;
  cudaFuncSetAttribute(k_upd, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  double* h0 = new double[np];
  double* h1 = new double[np];
  for (int j : {0, 4, 60, 64, 128, 132}) {
    long long c[2];
    for (int mode = 0; mode < 2; ++mode) {
      k_upd<<<1, 256, sm>>>(n, dA, mode, j, mode ? o1 : o0, cyc);
      cudaDeviceSynchronize();
      cudaMemcpy(&c[mode], cyc, sizeof(long long), cudaMemcpyDeviceToHost);
    }
    cudaMemcpy(h0, o0, sizeof(double) * np, cudaMemcpyDeviceToHost);
    cudaMemcpy(h1, o1, sizeof(double) * np, cudaMemcpyDeviceToHost);
    double md = 0;
    for (int t = 0; t < np; ++t) md = fmax(md, fabs(h0[t] - h1[t]));
    printf("j=%3d  dfma %6lld  dmma %6lld cycles/step   max|diff| %.3e  err=%s\n", j, c[0], c[1], md,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
