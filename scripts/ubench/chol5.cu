// Standalone check + cycle count of the tiled Cholesky in csrc/qp_chol.cuh.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_2602_17601_b200/csrc chol5.cu -o chol5
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#include "qp_chol.cuh"

#ifndef NTH
#define NTH 512
#endif
constexpr int NT = NTH;

__global__ void __launch_bounds__(NT, 1) kfac(int n, const double* A, double* L, long long* cyc, int reps, int* okp, long long* prof, const double* bvec, double* xout) {
  extern __shared__ double sm[];
  __shared__ int flag;
  const int T = qpchol::tiles_for(n);
  double* Kt = sm;
  double* dinv = sm + qpchol::tile_doubles(n);
  double* X = dinv + 8 * T;
  double* scratch = X + T * qpchol::kTS;
  double* y = scratch + 64 * (NT / 32);
  double* tmp = y + 8 * T;
  long long best = 1LL << 60;
  bool ok = true;
  for (int rep = 0; rep < reps; ++rep) {
    for (int e = threadIdx.x; e < 64 * T * T; e += NT) {
      const int R = e / (8 * T), C = e % (8 * T);
      if (C > R) continue;
      double v = (R < n && C < n) ? A[(size_t)R * n + C] : (R == C ? 1.0 : 0.0);
      Kt[qpchol::gel(R, C)] = v;
    }
    if (threadIdx.x == 0) flag = 0;
    __syncthreads();
    const long long t0 = clock64();
    ok = qpchol::factor<NT>(Kt, T, dinv, &flag, rep == reps - 1 ? prof : nullptr);
    const long long t1 = clock64();
    if (t1 - t0 < best) best = t1 - t0;
    __syncthreads();
  }
  const long long t2 = clock64();
  qpchol::invert_full<NT>(Kt, T, dinv, X, scratch);
  const long long t3 = clock64();
  for (int r = threadIdx.x; r < 8 * T; r += NT) y[r] = r < n ? bvec[r] : 0.0;
  __syncthreads();
  const long long t4 = clock64();
  qpchol::apply_x<NT>(Kt, T, y, tmp);
  const long long t5 = clock64();
  qpchol::apply_xt<NT>(Kt, T, y, tmp);
  const long long t6 = clock64();
  for (int r = threadIdx.x; r < n; r += NT) xout[r] = y[r];
  if (threadIdx.x == 0) {
    *cyc = best;
    *okp = ok;
    cyc[1] = t3 - t2;
    cyc[2] = t5 - t4;
    cyc[3] = t6 - t5;
  }
  for (int e = threadIdx.x; e < n * n; e += NT) {
    const int R = e / n, C = e % n;
    L[e] = C <= R ? Kt[qpchol::gel(R, C)] : 0.0;
  }
}

__global__ void kf8(const double* A, double* out, long long* cyc) {
  double a[8][8], d[8];
  for (int r = 0; r < 8; ++r)
    for (int c = 0; c <= r; ++c) a[r][c] = A[r * 8 + c];
  long long t0 = clock64();
  for (int it = 0; it < 16; ++it) {
    qpchol::factor8(a, d);
    a[0][0] += d[7];  // keep a dependence between calls
  }
  long long t1 = clock64();
  double s = 0;
  for (int r = 0; r < 8; ++r)
    for (int c = 0; c <= r; ++c) s += a[r][c];
  out[0] = s;
  cyc[0] = (t1 - t0) / 16;
}

int main(int argc, char** argv) {
  {
    double hA[64];
    for (int r = 0; r < 8; ++r)
      for (int c = 0; c < 8; ++c) hA[r * 8 + c] = (r == c) ? 4.0 : 0.1;
    double *dA, *dO;
    long long* dc;
    cudaMalloc(&dA, 512);
    cudaMalloc(&dO, 8);
    cudaMalloc(&dc, 8);
    cudaMemcpy(dA, hA, 512, cudaMemcpyHostToDevice);
    kf8<<<1, 1>>>(dA, dO, dc);
    long long c;
    cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost);
    printf("factor8 alone: %lld cycles per 8x8 factorisation\n", c);
  }
  std::mt19937_64 rng(1);
  std::normal_distribution<double> nd;
  std::uniform_real_distribution<double> ud(-2, 10);
  for (int n : {120, 70, 140, 200}) {
    for (int wide : {0, 1}) {
      std::vector<double> G((size_t)n * n), A((size_t)n * n);
      for (auto& g : G) g = nd(rng);
      for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) {
          double s = 0;
          for (int k = 0; k < n; ++k) s += G[(size_t)i * n + k] * G[(size_t)j * n + k];
          A[(size_t)i * n + j] = s / n;
        }
      for (int i = 0; i < n; ++i) A[(size_t)i * n + i] += wide ? std::pow(10.0, ud(rng)) : 1.0;
      double *dA, *dL;
      long long* dc;
      int* dok;
      cudaMalloc(&dA, 8 * A.size());
      cudaMalloc(&dL, 8 * A.size());
      cudaMalloc(&dc, 32);
      cudaMalloc(&dok, 4);
      std::vector<double> bv(n);
      for (auto& v : bv) v = nd(rng);
      double *db, *dx;
      cudaMalloc(&db, 8 * n);
      cudaMalloc(&dx, 8 * n);
      cudaMemcpy(db, bv.data(), 8 * n, cudaMemcpyHostToDevice);
      long long* dprof;
      cudaMalloc(&dprof, 8 * 8);
      cudaMemset(dprof, 0, 64);
      cudaMemcpy(dA, A.data(), 8 * A.size(), cudaMemcpyHostToDevice);
      const int T = qpchol::tiles_for(n);
      const size_t smem = 8 * (qpchol::tile_doubles(n) + 8 * T + T * qpchol::kTS + 64 * (NT / 32) + 16 * T);
      cudaFuncSetAttribute(kfac, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      kfac<<<1, NT, smem>>>(n, dA, dL, dc, 5, dok, dprof, db, dx);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) {
        printf("n=%d CUDA error %s\n", n, cudaGetErrorString(e));
        return 1;
      }
      std::vector<double> L(A.size());
      long long cyc, cy4[4];
      int ok;
      std::vector<double> xv(n);
      cudaMemcpy(xv.data(), dx, 8 * n, cudaMemcpyDeviceToHost);
      cudaMemcpy(cy4, dc, 32, cudaMemcpyDeviceToHost);
      // relative residual |A x - b| / (|A| |x| + |b|)
      double rmax = 0, xm = 0, bm = 0, am = 0;
      for (int i = 0; i < n; ++i) {
        long double sacc = 0;
        for (int j = 0; j < n; ++j) sacc += (long double)A[(size_t)i * n + j] * xv[j];
        rmax = std::fmax(rmax, std::fabs((double)(sacc - bv[i])));
        xm = std::fmax(xm, std::fabs(xv[i]));
        bm = std::fmax(bm, std::fabs(bv[i]));
        for (int j = 0; j < n; ++j) am = std::fmax(am, std::fabs(A[(size_t)i * n + j]));
      }
      cudaMemcpy(L.data(), dL, 8 * L.size(), cudaMemcpyDeviceToHost);
      cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost);
      cudaMemcpy(&ok, dok, 4, cudaMemcpyDeviceToHost);
      // residual |L L' - A| / |A|
      double emax = 0, amax = 0;
      for (int i = 0; i < n; ++i)
        for (int j = 0; j <= i; ++j) {
          long double s = 0;
          for (int k = 0; k <= j; ++k) s += (long double)L[(size_t)i * n + k] * L[(size_t)j * n + k];
          emax = std::fmax(emax, std::fabs((double)(s - A[(size_t)i * n + j])));
          amax = std::fmax(amax, std::fabs(A[(size_t)i * n + j]));
        }
      printf("n=%3d wide=%d ok=%d factor %lld cycles (%.1f us @1.965GHz)  |LL'-A|/|A| = %.2e\n", n, wide, ok, cyc,
             cyc / 1965.0, emax / amax);
      printf("   invert %lld | fwd %lld | bwd %lld cycles | solve resid %.2e\n", cy4[1], cy4[2], cy4[3], rmax / (am * xm + bm));
      long long pr[8];
      cudaMemcpy(pr, dprof, 64, cudaMemcpyDeviceToHost);
      const int T1 = T - 1;
      printf("   per step: w0 panel %lld | w0 E done %lld | w0 factor done %lld | others panel %lld | bar1 %lld | trailing max %lld/%lld | step %lld\n",
             pr[0] / T1, pr[1] / T1, pr[2] / T1, pr[3] / T1, pr[4] / T1, pr[5] / T1, pr[6] / T1, pr[7] / T1);
      cudaFree(dA);
      cudaFree(dL);
      cudaFree(dc);
      cudaFree(dok);
    }
  }
  return 0;
}
