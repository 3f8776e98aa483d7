// Halo pack / unpack for the node-partitioned recursion (partition.py).
//
// The reference has no multi-device path; its node-chunk thread pool
// (condensing.py:208-227) is what the row-slab partition generalises.  Per
// horizon stage a rank sends the Gamma rows of its boundary nodes to the
// ranks whose owned nodes read them, and receives its halo rows.  The rows of
// one stage are strided in the work array (node stride (N+1)*nx*ld floats),
// so they are gathered into a contiguous send buffer and scattered back from
// the receive buffer by these kernels (index lists live on the device, built
// once per partition).  8-byte words, one thread per word, coalesced within a
// row; a row of one node-stage block is nx*ld*4 = 3 KB at cfg5.
#include "common.cuh"

namespace {

__global__ void k_gather_rows(const unsigned long long* __restrict__ src,
                              unsigned long long* __restrict__ dst, const int* __restrict__ idx,
                              int n_idx, int64_t row_words, int64_t row_stride_words, int n_outer,
                              int64_t outer_stride_words) {
  const int64_t total = (int64_t)n_outer * n_idx * row_words;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t w = t % row_words;
    const int64_t r = t / row_words;  // (outer, i)
    const int i = (int)(r % n_idx);
    const int o = (int)(r / n_idx);
    dst[t] = src[o * outer_stride_words + (int64_t)idx[i] * row_stride_words + w];
  }
}

__global__ void k_scatter_rows(const unsigned long long* __restrict__ src,
                               unsigned long long* __restrict__ dst, const int* __restrict__ idx,
                               int n_idx, int64_t row_words, int64_t row_stride_words, int n_outer,
                               int64_t outer_stride_words) {
  const int64_t total = (int64_t)n_outer * n_idx * row_words;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t w = t % row_words;
    const int64_t r = t / row_words;
    const int i = (int)(r % n_idx);
    const int o = (int)(r / n_idx);
    dst[o * outer_stride_words + (int64_t)idx[i] * row_stride_words + w] = src[t];
  }
}

int check_rows(gm_ctx* ctx, const void* a, const void* b, int64_t row_bytes, int64_t row_stride,
               int64_t outer_stride) {
  if (((uintptr_t)a & 7) || ((uintptr_t)b & 7) || (row_bytes & 7) || (row_stride & 7) ||
      (outer_stride & 7))
    return gm_fail(ctx, GM_ERR_CONFIG, "halo rows must be 8-byte aligned multiples of 8 bytes");
  return GM_OK;
}

}  // namespace

extern "C" {

int gm_gather_rows(gm_ctx* ctx, const void* src, void* dst, const int32_t* idx, int n_idx,
                   int64_t row_bytes, int64_t row_stride_bytes, int n_outer,
                   int64_t outer_stride_bytes, void* stream) {
  int rc = gm_need_device(ctx);
  if (rc) return rc;
  if (n_idx <= 0 || n_outer <= 0 || row_bytes <= 0) return GM_OK;
  rc = check_rows(ctx, src, dst, row_bytes, row_stride_bytes, outer_stride_bytes);
  if (rc) return rc;
  const int64_t total = (int64_t)n_outer * n_idx * (row_bytes / 8);
  const int blocks = (int)std::min<int64_t>((total + 255) / 256, 8 * ctx->sm_count);
  k_gather_rows<<<blocks, 256, 0, (cudaStream_t)stream>>>(
      (const unsigned long long*)src, (unsigned long long*)dst, idx, n_idx, row_bytes / 8,
      row_stride_bytes / 8, n_outer, outer_stride_bytes / 8);
  GM_LAUNCH_CHECK(ctx, "k_gather_rows");
  return GM_OK;
}

int gm_scatter_rows(gm_ctx* ctx, const void* src, void* dst, const int32_t* idx, int n_idx,
                    int64_t row_bytes, int64_t row_stride_bytes, int n_outer,
                    int64_t outer_stride_bytes, void* stream) {
  int rc = gm_need_device(ctx);
  if (rc) return rc;
  if (n_idx <= 0 || n_outer <= 0 || row_bytes <= 0) return GM_OK;
  rc = check_rows(ctx, src, dst, row_bytes, row_stride_bytes, outer_stride_bytes);
  if (rc) return rc;
  const int64_t total = (int64_t)n_outer * n_idx * (row_bytes / 8);
  const int blocks = (int)std::min<int64_t>((total + 255) / 256, 8 * ctx->sm_count);
  k_scatter_rows<<<blocks, 256, 0, (cudaStream_t)stream>>>(
      (const unsigned long long*)src, (unsigned long long*)dst, idx, n_idx, row_bytes / 8,
      row_stride_bytes / 8, n_outer, outer_stride_bytes / 8);
  GM_LAUNCH_CHECK(ctx, "k_scatter_rows");
  return GM_OK;
}

}  // extern "C"
