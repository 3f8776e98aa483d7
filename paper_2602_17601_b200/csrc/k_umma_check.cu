// Known-answer check of the tcgen05 3xTF32 Gram path used by K-COND's H
// accumulation (umma.cuh): S = G' Q where G, Q are K x P fp32 (row-major),
// streamed through shared memory in chunks of 48 rows, accumulated in TMEM.
// Exported as gm_gram_check for the GPU tests (tests/test_gpu_umma.py).
#include "common.cuh"
#include "umma.cuh"

namespace {

constexpr int kChunk = 48;                     // K rows per shared-memory chunk
constexpr uint32_t kSbo = (kChunk / 4) * 128;  // 1536 B between 8-row groups
constexpr int kBuf = 128 / 8 * kSbo;           // one 128-row operand buffer, 24 KB

__global__ void __launch_bounds__(256, 1) k_gram_check(int K, int P, const float* G, const float* Q,
                                                        float* S) {
  extern __shared__ __align__(1024) unsigned char sm[];
  unsigned char* a_hi = sm;
  unsigned char* a_lo = sm + kBuf;
  unsigned char* b_hi = sm + 2 * kBuf;
  unsigned char* b_lo = sm + 3 * kBuf;
  uint64_t* mbar = (uint64_t*)(sm + 4 * kBuf);
  uint32_t* tslot = (uint32_t*)(mbar + 1);
  const int tid = threadIdx.x, warp = tid >> 5;
  const int N = ((P + 15) / 16) * 16;
  const uint32_t idesc = umma::idesc_tf32(128, N);
  if (warp == 0) umma::tmem_alloc<128>(tslot);
  if (tid == 32) umma::mbar_init(mbar, 1);
  for (int t = tid; t < 4 * kBuf / 4; t += blockDim.x) ((float*)sm)[t] = 0.f;
  umma::fence_before();
  __syncthreads();
  umma::fence_after();
  const uint32_t tmem = *tslot;
  uint32_t phase = 0;
  const int chunks = (K + kChunk - 1) / kChunk;
  for (int c = 0; c < chunks; ++c) {
    if (c > 0) {  // previous chunk's MMAs must be done before its operands are overwritten
      umma::mbar_wait(mbar, phase);
      phase ^= 1;
      umma::fence_after();
    }
    const int k0 = c * kChunk, kc = min(kChunk, K - k0);
    for (int t = tid; t < kChunk * P; t += blockDim.x) {
      const int k = t / P, p = t - k * P;
      const float g = k < kc ? G[(int64_t)(k0 + k) * P + p] : 0.f;
      const float q = k < kc ? Q[(int64_t)(k0 + k) * P + p] : 0.f;
      umma::put_split(a_hi, a_lo, p, k, kSbo, g);
      umma::put_split(b_hi, b_lo, p, k, kSbo, q);
    }
    umma::fence_async_smem();
    __syncthreads();
    if (tid == 0) {
      umma::fence_after();
      umma::gram_3xtf32(tmem, a_hi, a_lo, kSbo, b_hi, b_lo, kSbo, kChunk / 8, idesc, c > 0);
      umma::commit(mbar);
    }
    __syncwarp();
  }
  umma::mbar_wait(mbar, phase);
  umma::fence_after();
  // warps w and w + 4 share TMEM lanes (w % 4) * 32 .. +31; split the columns
  const int lane_row = (warp & 3) * 32 + (tid & 31);
  const int cbeg = (warp >> 2) * 64;
  for (int c0 = cbeg; c0 < cbeg + 64; c0 += 16) {
    float v[16];
    umma::tmem_ld16(tmem + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)c0, v);
    if (lane_row < P)
#pragma unroll
      for (int j = 0; j < 16; ++j)
        if (c0 + j < P) S[(int64_t)lane_row * P + c0 + j] = v[j];
  }
  umma::fence_before();
  __syncthreads();
  if (warp == 0) umma::tmem_free<128>(tmem);
}

}  // namespace

extern "C" int gm_gram_check(gm_ctx* ctx, int K, int P, const float* G, const float* Q, float* S,
                             void* stream) {
  int rc = gm_need_device(ctx);
  if (rc) return rc;
  if (K < 1 || P < 1 || P > 128) return gm_fail(ctx, GM_ERR_CONFIG, "gram check needs K >= 1, 1 <= P <= 128");
  const size_t sm = 4 * (size_t)kBuf + 64;
  GM_CUDA(ctx, cudaFuncSetAttribute(k_gram_check, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  k_gram_check<<<1, 256, sm, (cudaStream_t)stream>>>(K, P, G, Q, S);
  GM_LAUNCH_CHECK(ctx, "k_gram_check");
  return GM_OK;
}
