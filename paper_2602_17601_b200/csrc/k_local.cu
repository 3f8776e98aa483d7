// Per-node condensing (Eqs. 16-17 of the paper) and its assembly.
//
// Reference: local_hessian_gradient (condensing.py:231-243), condense_local
// (:285-295) and assemble_qp (:334-360).  The fused K-COND / K-HG reduce H
// and g over the nodes inside the kernel; this path keeps each node's
// contribution, which the reference exposes as public API (and pins to the
// fused result, tests/test_condensing.py:264-278).
//
// k_node_hg: one CTA per (instance, node).  The node's Gamma rows (all N+1
// stages, all n0 = N*nu input columns: arbitrary user maps need not be
// causal) are staged from the fp32 work array into shared memory; H^i =
// sum_k G_k' Qs_k G_k with Qs_k = (Q_k + Q_k')/2 (= the reference's
// 0.5 (h + h') of h = sum_k G_k' Q_k G_k) is formed in 4x4 register tiles of
// the upper triangle, fp64 products and accumulation, and mirrored;
// g^i = sum_k G_k' (2 Q_k Gamma_x,k + q_lin,k) one thread per column.
// Bound: fp64 FMA, ~(N+1) nx n0^2 (1 + nx/4) flops per node (3.6 MFLOP at
// cfg3) -- a test-path API, not the per-step hot path.
//
// k_sum_nodes: dst = base + sum_i src_i in ascending i (the reference's loop
// order, condensing.py:344-346), fp64, one thread per output element,
// optionally symmetrised 0.5 (S + S') (condensing.py:355).
#include "common.cuh"

namespace {

constexpr int kLocThreads = 256;

struct NodeHgArgs {
  int M, N, nx, nu, ld, lo, nodes;
  const float* W;        // (B*M, N+1, nx, ld)
  const double* q;       // (B, M, N+1, nx, nx) + b*q_stride
  int64_t q_stride;
  const double* qlin;    // (B, M, N+1, nx) + b*ql_stride
  int64_t ql_stride;
  double* H;             // (B, nodes, n0, n0)
  double* g;             // (B, nodes, n0)
};

__global__ void __launch_bounds__(kLocThreads) k_node_hg(const NodeHgArgs a) {
  extern __shared__ __align__(16) unsigned char smraw[];
  const int N = a.N, nx = a.nx, n0 = N * a.nu, S1 = N + 1;
  const int li = blockIdx.x, b = blockIdx.y;
  const int node = a.lo + li;
  const float* Wn = a.W + ((int64_t)b * a.M + node) * S1 * nx * a.ld;
  const double* Qn = a.q + b * a.q_stride + (int64_t)node * S1 * nx * nx;
  const double* Ln = a.qlin + b * a.ql_stride + (int64_t)node * S1 * nx;
  // shared: G (S1*nx, n0) fp32 | Qs (S1, nx, nx) fp64 | w (S1, nx) fp64
  float* G = reinterpret_cast<float*>(smraw);
  double* Qs = reinterpret_cast<double*>(smraw + ((sizeof(float) * (size_t)S1 * nx * n0 + 15) & ~size_t(15)));
  double* w = Qs + S1 * nx * nx;
  const int tid = threadIdx.x;
  for (int t = tid; t < S1 * nx * n0; t += blockDim.x) {
    const int row = t / n0, c = t - row * n0;
    G[t] = Wn[(int64_t)row * a.ld + c];
  }
  for (int t = tid; t < S1 * nx * nx; t += blockDim.x) {
    const int k = t / (nx * nx), e = t - k * nx * nx, r = e / nx, c = e - r * nx;
    Qs[t] = 0.5 * (Qn[(int64_t)k * nx * nx + r * nx + c] + Qn[(int64_t)k * nx * nx + c * nx + r]);
  }
  for (int t = tid; t < S1 * nx; t += blockDim.x) {
    const int k = t / nx, r = t - k * nx;
    double s = 0.0;
    for (int c = 0; c < nx; ++c)
      s += Qn[(int64_t)k * nx * nx + r * nx + c] * (double)Wn[((int64_t)k * nx + c) * a.ld + n0];
    w[t] = 2.0 * s + Ln[t];
  }
  __syncthreads();
  double* Hn = a.H + ((int64_t)b * a.nodes + li) * n0 * n0;
  double* gn = a.g + ((int64_t)b * a.nodes + li) * n0;
  // g^i (condensing.py:240-241)
  for (int c = tid; c < n0; c += blockDim.x) {
    double s0 = 0.0, s1 = 0.0;
    for (int row = 0; row < S1 * nx; row += 2) {
      s0 = fma((double)G[row * n0 + c], w[row], s0);
      if (row + 1 < S1 * nx) s1 = fma((double)G[(row + 1) * n0 + c], w[row + 1], s1);
    }
    gn[c] = s0 + s1;
  }
  // H^i in 4x4 tiles of the upper triangle (tile row P <= tile col Q)
  const int nt4 = (n0 + 3) / 4;
  const int ntiles = nt4 * (nt4 + 1) / 2;
  for (int t = tid; t < ntiles; t += blockDim.x) {
    int Q = (int)((sqrtf(8.f * t + 1.f) - 1.f) * 0.5f);
    while ((Q + 1) * (Q + 2) / 2 <= t) ++Q;
    while (Q * (Q + 1) / 2 > t) --Q;
    const int P = t - Q * (Q + 1) / 2;
    const int p0 = 4 * P, q0 = 4 * Q;
    double acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
    for (int k = 0; k < S1; ++k) {
      const double* Qk = Qs + k * nx * nx;
      const float* Gk = G + (int64_t)k * nx * n0;
      for (int r = 0; r < nx; ++r) {
        // (Qs G)[r][q0..q0+3]
        double y[4] = {0.0, 0.0, 0.0, 0.0};
        for (int c = 0; c < nx; ++c) {
          const double qrc = Qk[r * nx + c];
#pragma unroll
          for (int j = 0; j < 4; ++j)
            y[j] = fma(qrc, q0 + j < n0 ? (double)Gk[c * n0 + q0 + j] : 0.0, y[j]);
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const double x = p0 + i < n0 ? (double)Gk[r * n0 + p0 + i] : 0.0;
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[i][j] = fma(x, y[j], acc[i][j]);
        }
      }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int p = p0 + i, q = q0 + j;
        if (p < n0 && q < n0 && p <= q) {
          Hn[(int64_t)p * n0 + q] = acc[i][j];
          Hn[(int64_t)q * n0 + p] = acc[i][j];
        }
      }
  }
}

__global__ void k_sum_nodes(int count, int len, int sym_n, const double* __restrict__ src,
                            const double* __restrict__ base, double* __restrict__ dst) {
  const int b = blockIdx.y;
  const double* S = src + (int64_t)b * count * len;
  const double* Bb = base ? base + (int64_t)b * len : nullptr;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < len; e += gridDim.x * blockDim.x) {
    double s = Bb ? Bb[e] : 0.0;
    for (int i = 0; i < count; ++i) s += S[(int64_t)i * len + e];
    if (sym_n > 0) {
      const int p = e / sym_n, q = e - p * sym_n;
      const int et = q * sym_n + p;
      double st = Bb ? Bb[et] : 0.0;
      for (int i = 0; i < count; ++i) st += S[(int64_t)i * len + et];
      s = 0.5 * (s + st);
    }
    dst[(int64_t)b * len + e] = s;
  }
}

}  // namespace

extern "C" {

int gm_node_hessians(gm_ctx* ctx, int B, int N, const float* gamma, int ld, const double* q,
                     int64_t q_stride, const double* q_lin, int64_t qlin_stride, double* H, double* g,
                     void* stream) {
  int rc = gm_need_device(ctx);
  if (rc) return rc;
  if (ctx->M < 1 || ctx->nx < 1 || ctx->n_u < 1) return gm_fail(ctx, GM_ERR_CONFIG, "graph/dimensions not set");
  if (B < 0 || N < 1) return gm_fail(ctx, GM_ERR_CONFIG, "need B >= 0 and horizon >= 1");
  const int nx = ctx->nx, nu = ctx->n_u, n0 = N * nu;
  if (ld < n0 + 1) return gm_fail(ctx, GM_ERR_CONFIG, "gamma leading dimension too small");
  const int64_t lo = ctx->node_lo, nodes = gm_node_hi(ctx) - lo;
  if (B == 0 || nodes == 0) return GM_OK;
  const size_t sm = ((sizeof(float) * (size_t)(N + 1) * nx * n0 + 15) & ~size_t(15)) +
                    sizeof(double) * (size_t)(N + 1) * nx * (nx + 1);
  if (sm > ctx->smem_optin) return gm_fail(ctx, GM_ERR_CONFIG, "node Gamma too large for shared memory");
  GM_CUDA(ctx, cudaFuncSetAttribute(k_node_hg, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  NodeHgArgs a{};
  a.M = (int)ctx->M;
  a.N = N;
  a.nx = nx;
  a.nu = nu;
  a.ld = ld;
  a.lo = (int)lo;
  a.nodes = (int)nodes;
  a.W = gamma;
  a.q = q;
  a.q_stride = q_stride;
  a.qlin = q_lin;
  a.ql_stride = qlin_stride;
  a.H = H;
  a.g = g;
  k_node_hg<<<dim3((unsigned)nodes, (unsigned)B), kLocThreads, sm, (cudaStream_t)stream>>>(a);
  GM_LAUNCH_CHECK(ctx, "k_node_hg");
  return GM_OK;
}

int gm_sum_nodes(gm_ctx* ctx, int B, int count, int len, int sym_n, const double* src,
                 const double* base, double* dst, void* stream) {
  int rc = gm_need_device(ctx);
  if (rc) return rc;
  if (B < 0 || count < 0 || len < 0) return gm_fail(ctx, GM_ERR_CONFIG, "bad sizes");
  if (sym_n > 0 && (int64_t)sym_n * sym_n != len) return gm_fail(ctx, GM_ERR_CONFIG, "sym_n^2 != len");
  if (B == 0 || len == 0) return GM_OK;
  const int blocks = std::max(1, std::min(gm_ceil_div(len, 256), 4 * ctx->sm_count));
  k_sum_nodes<<<dim3((unsigned)blocks, (unsigned)B), 256, 0, (cudaStream_t)stream>>>(count, len, sym_n, src,
                                                                                       base, dst);
  GM_LAUNCH_CHECK(ctx, "k_sum_nodes");
  return GM_OK;
}

}  // extern "C"
