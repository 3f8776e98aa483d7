// build_k tile pass in isolation: generic vs shared-asserted pointers
#include <cstdio>
#include "qp_chol.cuh"
__device__ __forceinline__ int colbase(int c, int n) { return c * n - ((c * (c + 1)) >> 1); }
template <bool ASSUME, int VAR, int U = 3>
__device__ __noinline__ void tiles(double* K, const double* Hp, const double* Cg, const double* wg, int n, int ldc, int ng, int T, const unsigned short* tij = nullptr) {
  if (ASSUME) { QP_SMEM(K); QP_SMEM(Hp); QP_SMEM(Cg); QP_SMEM(wg); }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int i = lane >> 2, p = lane & 3;
  const int ntiles = T * (T + 1) / 2;
  constexpr int NW = 8;
  for (int t0 = wid; t0 < ntiles; t0 += U * NW) {
    int r[U], ca[U], rb[U];
    double h0[U], h1[U];
    bool live[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int tt = t0 + u * NW;
      live[u] = tt < ntiles;
      int I;
      if (VAR == 3) { const unsigned v = tij[min(tt, ntiles - 1)]; I = v >> 8; } else
      if (VAR == 2) { I = tt >> 3; if (I >= T) I = T - 1; } else {
      I = (int)((sqrtf(8.0f * tt + 1.0f) - 1.0f) * 0.5f);
      while (I * (I + 1) / 2 > tt) --I;
      while ((I + 1) * (I + 2) / 2 <= tt) ++I; }
      const int J = VAR == 3 ? (tij[min(tt, ntiles - 1)] & 255) : tt - I * (I + 1) / 2;
      r[u] = 8 * I + i; ca[u] = 8 * J + 2 * p; rb[u] = 8 * J + i;
      const int cb = ca[u] + 1;
      h0[u] = (live[u] && r[u] < n && ca[u] < n && r[u] > ca[u]) ? 2.0 * Hp[colbase(ca[u], n) + r[u]] : 0.0;
      h1[u] = (live[u] && r[u] < n && cb < n && r[u] > cb) ? 2.0 * Hp[colbase(cb, n) + r[u]] : 0.0;
    }
    for (int g0 = 0; g0 < ng; g0 += 4) {
      const int g = g0 + p;
      const double* cg = Cg + (long long)min(g, ng - 1) * ldc;
      const double wgg = g < ng ? wg[g] : 0.0;
      double av[U], bv[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        av[u] = (g < ng && r[u] < n) ? wgg * cg[r[u]] : 0.0;
        bv[u] = (g < ng && rb[u] < n) ? cg[rb[u]] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) { if (VAR == 1) { h0[u] = fma(av[u], bv[u], h0[u]); h1[u] += av[u]; } else qpchol::dmma884(h0[u], h1[u], av[u], bv[u]); }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (!live[u]) continue;
      const int cb = ca[u] + 1;
      if (r[u] >= n || ca[u] >= n) h0[u] = r[u] == ca[u] ? 1.0 : 0.0;
      if (r[u] >= n || cb >= n) h1[u] = r[u] == cb ? 1.0 : 0.0;
      if (r[u] >= ca[u]) K[qpchol::gel(r[u], ca[u])] = h0[u];
      if (r[u] >= cb) K[qpchol::gel(r[u], cb)] = h1[u];
    }
  }
}
__global__ void __launch_bounds__(256, 1) k(long long* cyc, double* out) {
  extern __shared__ double sm[];
  const int n = 120, ldc = 140, ng = 20, T = 15;
  double* K = sm; double* Hp = K + qpchol::tile_doubles(n); double* Cg = Hp + n * (n + 1) / 2; double* wg = Cg + ng * ldc;
  for (int e = threadIdx.x; e < qpchol::tile_doubles(n) + n * (n + 1) / 2 + ng * ldc + ng; e += 256) sm[e] = 1e-3 * (e % 13);
  __syncthreads();
  for (int rep = 0; rep < 2; ++rep) {
    long long t0 = clock64();
    tiles<false, 0>(K, Hp, Cg, wg, n, ldc, ng, T);
    __syncthreads();
    long long t1 = clock64();
    tiles<true, 0>(K, Hp, Cg, wg, n, ldc, ng, T);
    __syncthreads();
    long long t2 = clock64();
    tiles<true, 1>(K, Hp, Cg, wg, n, ldc, ng, T);
    __syncthreads();
    long long t3 = clock64();
    tiles<true, 2>(K, Hp, Cg, wg, n, ldc, ng, T);
    __syncthreads();
    long long t4 = clock64();
    __shared__ unsigned short tij[528];
    for (int t = threadIdx.x; t < T * (T + 1) / 2; t += 256) { int I = 0; while ((I + 1) * (I + 2) / 2 <= t) ++I; tij[t] = (I << 8) | (t - I * (I + 1) / 2); }
    __syncthreads();
    long long t5 = clock64();
    tiles<true, 3>(K, Hp, Cg, wg, n, ldc, ng, T, tij);
    __syncthreads();
    long long t6 = clock64();
    tiles<true, 3, 5>(K, Hp, Cg, wg, n, ldc, ng, T, tij);
    __syncthreads();
    long long t7 = clock64();
    if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t6 - t5; cyc[5] = t7 - t6; }
  }
  out[threadIdx.x] = K[threadIdx.x];
}
int main() {
  long long* c; double* o; cudaMalloc(&c, 64); cudaMalloc(&o, 256 * 8);
  size_t smem = 8 * (qpchol::tile_doubles(120) + 120 * 121 / 2 + 20 * 140 + 20);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k<<<1, 256, smem>>>(c, o);
  long long h[6]; cudaMemcpy(h, c, 48, cudaMemcpyDeviceToHost);
  printf("tile pass: generic %lld | shared %lld | no-DMMA %lld | no-decode %lld | table %lld | table U=5 %lld cycles\n", h[0], h[1], h[2], h[3], h[4], h[5]);
}
