// Latency calibration for one 256-thread CTA (fp64 IPM phases).
#include <cstdio>
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__global__ void __launch_bounds__(256, 1) k(double* out, long long* cyc) {
  __shared__ double a[512], b[512], c[512], red[8];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  for (int i = tid; i < 512; i += 256) { a[i] = i * 1e-3; b[i] = 1.0 + i; c[i] = 0; }
  __syncthreads();
  long long t0, t1;
  double acc = 0;
  // 1: 100 bare __syncthreads
  t0 = clock64();
  for (int it = 0; it < 100; ++it) __syncthreads();
  t1 = clock64();
  if (tid == 0) cyc[0] = (t1 - t0) / 100;
  // 2: elementwise loop over m=280 (2 loads, 1 store) + barrier
  t0 = clock64();
  for (int it = 0; it < 100; ++it) {
    for (int r = tid; r < 280; r += 256) c[r] = a[r] * b[r] + c[r];
    __syncthreads();
  }
  t1 = clock64();
  if (tid == 0) cyc[1] = (t1 - t0) / 100;
  // 3: block max reduction (shfl + 2 barriers + shfl) as k_qp's block_reduce
  t0 = clock64();
  for (int it = 0; it < 100; ++it) {
    double v = a[(tid + it) & 511];
    v = warp_max(v);
    __syncthreads();
    if (lane == 0) red[wid] = v;
    __syncthreads();
    double r = red[lane & 7];
#pragma unroll
    for (int o = 4; o > 0; o >>= 1) r = fmax(r, __shfl_xor_sync(0xffffffffu, r, o));
    acc += r;
  }
  t1 = clock64();
  if (tid == 0) cyc[2] = (t1 - t0) / 100;
  // 4: dependent smem load chain (pointer chase through doubles)
  t0 = clock64();
  int idx = tid & 7;
  for (int it = 0; it < 100; ++it) idx = ((int)b[idx]) & 511;
  t1 = clock64();
  if (tid == 0) cyc[3] = (t1 - t0) / 100;
  // 5: dependent double shuffle
  double s = a[tid];
  t0 = clock64();
  for (int it = 0; it < 100; ++it) s = __shfl_xor_sync(0xffffffffu, s, 1) + 1.0;
  t1 = clock64();
  if (tid == 0) cyc[4] = (t1 - t0) / 100;
  // 6: dependent DFMA
  double f = a[tid];
  t0 = clock64();
  for (int it = 0; it < 100; ++it) f = fma(f, 1.0000001, 1e-9);
  t1 = clock64();
  if (tid == 0) cyc[5] = (t1 - t0) / 100;
  // 7: warp-0-only elementwise over 280 (9 per lane) + syncwarp
  t0 = clock64();
  if (wid == 0)
    for (int it = 0; it < 100; ++it) {
#pragma unroll 3
      for (int r = lane; r < 280; r += 32) c[r] = a[r] * b[r] + c[r];
      __syncwarp();
    }
  t1 = clock64();
  if (tid == 0) cyc[6] = (t1 - t0) / 100;
  // 8: warp max reduce (5 levels)
  t0 = clock64();
  double wv = a[tid];
  for (int it = 0; it < 100; ++it) wv = warp_max(wv) + 1e-9;
  t1 = clock64();
  if (tid == 0) cyc[7] = (t1 - t0) / 100;
  // 9: rsqrt and division chain
  double q = 2.0 + a[tid];
  t0 = clock64();
  for (int it = 0; it < 100; ++it) q = rsqrt(q) + 1.5;
  t1 = clock64();
  if (tid == 0) cyc[8] = (t1 - t0) / 100;
  t0 = clock64();
  for (int it = 0; it < 100; ++it) q = 1.0 / q + 1.5;
  t1 = clock64();
  if (tid == 0) cyc[9] = (t1 - t0) / 100;
  out[tid] = acc + c[tid] + idx + s + f + wv + q;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 8 * 256); cudaMalloc(&c, 8 * 16);
  for (int rep = 0; rep < 2; ++rep) {
    k<<<1, 256>>>(o, c); cudaDeviceSynchronize();
    long long h[10]; cudaMemcpy(h, c, 80, cudaMemcpyDeviceToHost);
    printf("syncthreads %lld | elementwise m=280 + bar %lld | block_reduce %lld | smem dep load %lld | dshfl %lld | dfma %lld | warp0 elementwise 280 %lld | warp_max %lld | rsqrt %lld | div %lld\n",
           h[0], h[1], h[2], h[3], h[4], h[5], h[6], h[7], h[8], h[9]);
  }
}
