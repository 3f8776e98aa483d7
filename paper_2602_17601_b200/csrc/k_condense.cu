// K-REC / K-HG / K-CON: condensing on the GPU (stages 2 and 3).
//
// K-REC  condense_gammas (condensing.py:182-228).  Work array
//        W (B*M, N+1, nx, ld) fp32: Gamma_u in columns [0, N*nu), Gamma_x in
//        column XC = N*nu.  Stage n -> n+1 is a block-ELL SpMM over the closed
//        neighbourhood read straight from the CSR (slot 0 = a_self, slot s>0 =
//        a_nbr[ptr[i]+s-1] with source src[...]), so the reference's padded
//        a_pad / phantom node are never built.  One CTA per node, one thread
//        per column: neighbour rows are read as contiguous column runs
//        (coalesced), the 6x6 blocks are CTA-broadcast from shared memory.
//        Causality: only the live columns [0, n*nu) and XC are multiplied;
//        block n receives B_n; everything else is written as zero, so W needs
//        no separate memset.
// K-HG   condense_ocp cost part (condensing.py:376-389, :402-403): the
//        tall-skinny contraction H = R + sum_{k,i} G_ki' Q_ki G_ki is a split-K
//        reduction over nodes; each CTA keeps a 128x128 fp32 tile of H in
//        registers (8x8 per thread), stages the node's rows of G and Q G in
//        shared memory, and skips the non-causal part of every row.  Partials
//        are reduced in a fixed order in fp64 (bitwise reproducible), R-bar is
//        added and H is symmetrised as the reference does.
// K-CON  constraint rows (condensing.py:263-282, :312-323) and
//        expand_soft_constraints (condensing.py:419-439).
#include <algorithm>

#include "common.cuh"

namespace {

// ---------------------------------------------------------------------------
// K-REC
// ---------------------------------------------------------------------------
struct RecArgs {
  int M, E, N, nx, nu, ld, n, lo, nodes;
  const int* ptr;
  const int* src;
  const float* a_self;
  const float* a_nbr;
  const float* b;
  const double* c;
  const double* x0;
  float* W;
};

template <int NXC>
__global__ void __launch_bounds__(128) k_gamma_stage(const RecArgs a) {
  extern __shared__ __align__(16) float sblk[];
  const int nx = a.nx, nu = a.nu, ld = a.ld, N = a.N, n = a.n;
  const int64_t bi = blockIdx.x / a.nodes;
  const int i = a.lo + (int)(blockIdx.x % a.nodes);
  const int64_t gi = bi * a.M + i;
  const int XC = N * nu;
  const int64_t stage_stride = (int64_t)nx * ld;
  const int64_t node_stride = (int64_t)(N + 1) * stage_stride;
  if (n < 0) {  // stage 0: Gamma_u = 0, Gamma_x = x0 (condensing.py:205-206)
    float* Wo = a.W + gi * node_stride;
    for (int col = threadIdx.x; col < ld; col += blockDim.x)
      for (int r = 0; r < nx; ++r)
        Wo[(int64_t)r * ld + col] = (col == XC) ? (float)a.x0[gi * nx + r] : 0.f;
    return;
  }
  const int e0 = a.ptr[i], deg = a.ptr[i + 1] - e0;
  const int nn2 = nx * nx;
  float* As = sblk;                      // (1+deg) blocks
  float* Bs = sblk + (1 + deg) * nn2;    // nx*nu
  float* cs = Bs + nx * nu;              // nx (offset, rounded once to fp32)
  int* js = (int*)(cs + nx);             // neighbour ids
  const int64_t pstage = bi * N + n;
  for (int t = threadIdx.x; t < (1 + deg) * nn2; t += blockDim.x) {
    const int s = t / nn2, q = t - s * nn2;
    As[t] = s == 0 ? a.a_self[(pstage * a.M + i) * nn2 + q]
                   : a.a_nbr[(pstage * a.E + e0 + s - 1) * nn2 + q];
  }
  for (int t = threadIdx.x; t < nx * nu; t += blockDim.x) Bs[t] = a.b[(pstage * a.M + i) * nx * nu + t];
  for (int t = threadIdx.x; t < nx; t += blockDim.x) cs[t] = (float)a.c[(pstage * a.M + i) * nx + t];
  for (int t = threadIdx.x; t <= deg; t += blockDim.x) js[t] = t == 0 ? i : a.src[e0 + t - 1];
  __syncthreads();
  const int live = n * nu;
  float* Wo = a.W + gi * node_stride + (int64_t)(n + 1) * stage_stride;
  for (int col = threadIdx.x; col < ld; col += blockDim.x) {
    float acc[NXC];
#pragma unroll
    for (int r = 0; r < NXC; ++r) acc[r] = 0.f;
    if (col < live || col == XC) {
      for (int s = 0; s <= deg; ++s) {
        const float* Wj = a.W + (bi * a.M + js[s]) * node_stride + (int64_t)n * stage_stride + col;
        const float* A = As + s * nn2;
#pragma unroll
        for (int q = 0; q < NXC; ++q) {
          if (q < nx) {
            const float w = Wj[(int64_t)q * ld];
#pragma unroll
            for (int r = 0; r < NXC; ++r)
              if (r < nx) acc[r] = fmaf(A[r * nx + q], w, acc[r]);
          }
        }
      }
      if (col == XC) {
#pragma unroll
        for (int r = 0; r < NXC; ++r)
          if (r < nx) acc[r] += cs[r];
      }
    } else if (col >= live && col < live + nu) {
#pragma unroll
      for (int r = 0; r < NXC; ++r)
        if (r < nx) acc[r] = Bs[r * nu + (col - live)];
    }
#pragma unroll
    for (int r = 0; r < NXC; ++r)
      if (r < nx) Wo[(int64_t)r * ld + col] = acc[r];
  }
}

int rec_stage(gm_ctx* ctx, int B, int N, int n, const float* a_self, const float* a_nbr,
              const float* b, const double* c, const double* x0, float* W, int ld,
              cudaStream_t st) {
  RecArgs a{};
  a.M = (int)ctx->M;
  a.E = (int)ctx->E;
  a.N = N;
  a.nu = ctx->n_u;
  a.nx = ctx->nx;
  a.ld = ld;
  a.n = n;
  a.lo = (int)ctx->node_lo;
  a.nodes = (int)(gm_node_hi(ctx) - ctx->node_lo);
  a.ptr = ctx->d_ptr;
  a.src = ctx->d_src;
  a.a_self = a_self;
  a.a_nbr = a_nbr;
  a.b = b;
  a.c = c;
  a.x0 = x0;
  a.W = W;
  const int64_t blocks = (int64_t)B * a.nodes;
  if (blocks == 0) return GM_OK;
  const size_t sm = sizeof(float) * ((1 + ctx->dmax) * a.nx * a.nx + a.nx * a.nu + a.nx) +
                    sizeof(int) * (ctx->dmax + 1) + 16;
  if (a.nx <= 2)
    k_gamma_stage<2><<<(unsigned)blocks, 128, sm, st>>>(a);
  else if (a.nx <= 4)
    k_gamma_stage<4><<<(unsigned)blocks, 128, sm, st>>>(a);
  else if (a.nx <= 6)
    k_gamma_stage<6><<<(unsigned)blocks, 128, sm, st>>>(a);
  else if (a.nx <= 8)
    k_gamma_stage<8><<<(unsigned)blocks, 128, sm, st>>>(a);
  else
    k_gamma_stage<16><<<(unsigned)blocks, 128, sm, st>>>(a);
  GM_LAUNCH_CHECK(ctx, "k_gamma_stage");
  return GM_OK;
}

int check_dims(gm_ctx* ctx, int B, int N, int ld) {
  int rc = gm_need_device(ctx);
  if (rc) return rc;
  if (ctx->M < 1) return gm_fail(ctx, GM_ERR_CONFIG, "graph not set");
  if (ctx->nx < 1 || ctx->n_u < 1) return gm_fail(ctx, GM_ERR_CONFIG, "dimensions not set");
  if (B < 0 || N < 1) return gm_fail(ctx, GM_ERR_CONFIG, "need B >= 0 and horizon >= 1");
  if (ld < N * ctx->n_u + 1) return gm_fail(ctx, GM_ERR_CONFIG, "gamma leading dimension too small");
  return GM_OK;
}

// ---------------------------------------------------------------------------
// K-HG
// ---------------------------------------------------------------------------
constexpr int kTile = 128;  // output tile of H per CTA (8x8 per thread, 256 threads)

struct CostArgs {
  int M, N, nx, nu, ld, n0, lo, nodes, splits, tilesT, kc;
  const float* W;
  const double* q;
  int64_t q_stride;
  const double* xref;
  int64_t xref_stride;
  float* partH;  // (B, tilesT*tilesT, splits, 128, 128)
  double* partg; // (B, splits, n0)
};

__global__ void __launch_bounds__(256) k_cost_partial(const CostArgs a) {
  extern __shared__ __align__(16) float sm[];
  const int nx = a.nx, nu = a.nu, ld = a.ld, N = a.N, KC = a.kc;
  const int npair = a.tilesT * a.tilesT;
  const int64_t bi = blockIdx.x / ((int64_t)a.splits * npair);
  const int rem = (int)(blockIdx.x % ((int64_t)a.splits * npair));
  const int split = rem / npair, pair = rem % npair;
  const int ti = pair / a.tilesT, tj = pair % a.tilesT;
  const int c1b = ti * kTile, c2b = tj * kTile;
  const int per = (a.nodes + a.splits - 1) / a.splits;
  const int nb = a.lo + split * per, ne = min(a.lo + a.nodes, nb + per);
  const int rows_max = KC * nx;
  float* G1 = sm;                          // rows x 128 (row tile columns)
  float* G2 = G1 + rows_max * kTile;       // rows x 128 (Q G, column tile)
  double* wv = (double*)(G2 + rows_max * kTile);  // rows
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  float acc[8][8];
#pragma unroll
  for (int u = 0; u < 8; ++u)
#pragma unroll
    for (int v = 0; v < 8; ++v) acc[u][v] = 0.f;
  double gacc = 0.0;
  const bool do_g = (tj == 0);  // g rides on the first column-tile CTAs
  const int gcol = c1b + (threadIdx.x & (kTile - 1));
  const int64_t stage_stride = (int64_t)nx * ld;
  const int XC = N * nu;
  for (int i = nb; i < ne; ++i) {
    const int64_t gi = bi * a.M + i;
    const float* Wi = a.W + gi * (int64_t)(N + 1) * stage_stride;
    const double* Qi = a.q + bi * a.q_stride + (int64_t)i * (N + 1) * nx * nx;
    const double* Xi = a.xref + bi * a.xref_stride + (int64_t)i * (N + 1) * nx;
    for (int k0 = 1; k0 <= N; k0 += KC) {
      const int k1 = min(N + 1, k0 + KC);
      const int live_max = (k1 - 1) * nu;
      if (c1b >= live_max || c2b >= live_max) continue;  // tile entirely non-causal
      const int rows = (k1 - k0) * nx;
      __syncthreads();
      // stage rows: G1 = Gamma rows on the row tile, G2 = Q Gamma on the column tile
      for (int t = threadIdx.x; t < rows * kTile; t += blockDim.x) {
        const int r = t / kTile, cc = t % kTile;
        const int k = k0 + r / nx, ar = r % nx;
        const float* Wk = Wi + (int64_t)k * stage_stride;
        const int c1 = c1b + cc, c2 = c2b + cc;
        const int live = k * nu;
        G1[t] = (c1 < live) ? Wk[(int64_t)ar * ld + c1] : 0.f;
        float s = 0.f;
        if (c2 < live) {
          const double* Qk = Qi + (int64_t)k * nx * nx + ar * nx;
          for (int bb = 0; bb < nx; ++bb) s = fmaf((float)Qk[bb], Wk[(int64_t)bb * ld + c2], s);
        }
        G2[t] = s;
      }
      if (do_g) {
        // w = 2 Q Gamma_x + q_lin, q_lin = -2 Q x_ref (condensing.py:153, :388), fp64
        for (int r = threadIdx.x; r < rows; r += blockDim.x) {
          const int k = k0 + r / nx, ar = r % nx;
          const float* Wk = Wi + (int64_t)k * stage_stride;
          const double* Qk = Qi + (int64_t)k * nx * nx + ar * nx;
          const double* xr = Xi + (int64_t)k * nx;
          double qg = 0.0, qx = 0.0;
          for (int bb = 0; bb < nx; ++bb) {
            qg += Qk[bb] * (double)Wk[(int64_t)bb * ld + XC];
            qx += Qk[bb] * xr[bb];
          }
          wv[r] = 2.0 * qg + (-2.0 * qx);
        }
      }
      __syncthreads();
      for (int r = 0; r < rows; ++r) {
        const int live = (k0 + r / nx) * nu;
        if (c1b + ty * 8 >= live || c2b + tx * 8 >= live) continue;
        const float4 g1a = *(const float4*)(G1 + r * kTile + ty * 8);
        const float4 g1b = *(const float4*)(G1 + r * kTile + ty * 8 + 4);
        const float4 g2a = *(const float4*)(G2 + r * kTile + tx * 8);
        const float4 g2b = *(const float4*)(G2 + r * kTile + tx * 8 + 4);
        const float x[8] = {g1a.x, g1a.y, g1a.z, g1a.w, g1b.x, g1b.y, g1b.z, g1b.w};
        const float y[8] = {g2a.x, g2a.y, g2a.z, g2a.w, g2b.x, g2b.y, g2b.z, g2b.w};
#pragma unroll
        for (int u = 0; u < 8; ++u)
#pragma unroll
          for (int v = 0; v < 8; ++v) acc[u][v] = fmaf(x[u], y[v], acc[u][v]);
      }
      if (do_g && threadIdx.x < kTile) {
        for (int r = 0; r < rows; ++r) gacc += (double)G1[r * kTile + threadIdx.x] * wv[r];
      }
    }
  }
  float* P = a.partH + ((bi * npair + pair) * (int64_t)a.splits + split) * kTile * kTile;
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    float4* dst = (float4*)(P + (int64_t)(ty * 8 + u) * kTile + tx * 8);
    dst[0] = make_float4(acc[u][0], acc[u][1], acc[u][2], acc[u][3]);
    dst[1] = make_float4(acc[u][4], acc[u][5], acc[u][6], acc[u][7]);
  }
  if (do_g && threadIdx.x < kTile && gcol < a.n0)
    a.partg[(bi * a.splits + split) * a.n0 + gcol] = gacc;
}

struct ReduceArgs {
  int N, nu, n0, splits, tilesT, partial;
  const float* partH;
  const double* partg;
  const double* r;
  int64_t r_stride;
  const double* uref;
  int64_t uref_stride;
  double* H;
  double* g;
};

// H = 0.5 (S + S') + R-bar in fp64, splits summed in a fixed order.
__global__ void k_cost_reduce(const ReduceArgs a) {
  const int n0 = a.n0, nu = a.nu;
  const int64_t bi = blockIdx.y;
  const int npair = a.tilesT * a.tilesT;
  auto S = [&](int c1, int c2) -> double {
    const int ti = c1 / kTile, tj = c2 / kTile;
    const float* P = a.partH + ((bi * npair + ti * a.tilesT + tj) * (int64_t)a.splits) * kTile * kTile +
                     (int64_t)(c1 % kTile) * kTile + (c2 % kTile);
    double s = 0.0;
    for (int sp = 0; sp < a.splits; ++sp) s += (double)P[(int64_t)sp * kTile * kTile];
    return s;
  };
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < n0 * n0; idx += gridDim.x * blockDim.x) {
    const int c1 = idx / n0, c2 = idx % n0;
    double h = 0.5 * (S(c1, c2) + S(c2, c1));
    if (!a.partial && c1 / nu == c2 / nu) {
      const int k = c1 / nu;
      const double* Rk = a.r + bi * a.r_stride + (int64_t)k * nu * nu;
      // R-bar is symmetrised with the rest (condensing.py:380-381, :403)
      h += 0.5 * (Rk[(c1 % nu) * nu + (c2 % nu)] + Rk[(c2 % nu) * nu + (c1 % nu)]);
    }
    a.H[bi * (int64_t)n0 * n0 + idx] = h;
  }
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < n0; c += gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int sp = 0; sp < a.splits; ++sp) s += a.partg[(bi * a.splits + sp) * n0 + c];
    if (!a.partial) {
      // r_lin = -2 R u_ref (condensing.py:154)
      const int k = c / nu, row = c % nu;
      const double* Rk = a.r + bi * a.r_stride + (int64_t)k * nu * nu + row * nu;
      const double* uk = a.uref + bi * a.uref_stride + (int64_t)k * nu;
      double ru = 0.0;
      for (int j = 0; j < nu; ++j) ru += Rk[j] * uk[j];
      s = -2.0 * ru + s;
    }
    a.g[bi * n0 + c] = s;
  }
}

// ---------------------------------------------------------------------------
// K-CON
// ---------------------------------------------------------------------------
struct ConArgs {
  int M, N, nx, nu, ld, n0, n_in, n_st;
  const float* W;
  const int* in_stage;
  const double* in_c;
  const double* in_d;
  const int* st_node;
  const int* st_stage;
  const double* st_c;
  const double* st_d;
  double* C;
  double* d;
};

__global__ void k_constraint_rows(const ConArgs a) {
  const int m0 = a.n_in + a.n_st;
  const int64_t bi = blockIdx.y;
  const int row = blockIdx.x;
  if (row >= m0) return;
  double* Cr = a.C + (bi * m0 + row) * (int64_t)a.n0;
  const int nu = a.nu, nx = a.nx;
  if (row < a.n_in) {  // input rows (condensing.py:318-322)
    const int k = a.in_stage[row];
    for (int col = threadIdx.x; col < a.n0; col += blockDim.x)
      Cr[col] = (col / nu == k) ? a.in_c[(int64_t)row * nu + (col % nu)] : 0.0;
    if (threadIdx.x == 0) a.d[bi * m0 + row] = a.in_d[row];
  } else {  // state rows mapped through Gamma (condensing.py:268-269)
    const int sr = row - a.n_in;
    const int node = a.st_node[sr], k = a.st_stage[sr];
    const float* Wk = a.W + ((bi * a.M + node) * (int64_t)(a.N + 1) + k) * nx * a.ld;
    const double* cr = a.st_c + (int64_t)sr * nx;
    for (int col = threadIdx.x; col < a.n0; col += blockDim.x) {
      double s = 0.0;
      for (int q = 0; q < nx; ++q) s += cr[q] * (double)Wk[(int64_t)q * a.ld + col];
      Cr[col] = s;
    }
    if (threadIdx.x == 0) {
      double s = 0.0;
      for (int q = 0; q < nx; ++q) s += cr[q] * (double)Wk[(int64_t)q * a.ld + a.N * nu];
      a.d[bi * m0 + row] = a.st_d[sr] - s;
    }
  }
}

struct SoftArgs {
  int n0, m0, ns;
  const double* H0;
  const double* g0;
  const double* C0;
  const double* d0;
  const int* idx;
  const double* rho1;
  const double* rho2;
  double* H;
  double* g;
  double* C;
  double* d;
};

// expand_soft_constraints (condensing.py:429-439) for one instance per blockIdx.y
__global__ void k_expand_soft(const SoftArgs a) {
  const int n0 = a.n0, m0 = a.m0, ns = a.ns, n = n0 + ns, m = m0 + ns;
  const int64_t bi = blockIdx.y;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (int64_t t = t0; t < (int64_t)n * n; t += stride) {
    const int r = (int)(t / n), c = (int)(t % n);
    double v = 0.0;
    if (r < n0 && c < n0) v = a.H0[bi * n0 * n0 + (int64_t)r * n0 + c];
    else if (r >= n0 && r == c) v = a.rho2[r - n0];
    a.H[bi * (int64_t)n * n + t] = v;
  }
  for (int64_t t = t0; t < n; t += stride)
    a.g[bi * n + t] = t < n0 ? a.g0[bi * n0 + t] : a.rho1[t - n0];
  for (int64_t t = t0; t < (int64_t)m * n; t += stride) {
    const int r = (int)(t / n), c = (int)(t % n);
    double v = 0.0;
    if (r < m0) {
      if (c < n0) v = a.C0[(bi * m0 + r) * (int64_t)n0 + c];
      else if (a.idx[c - n0] == r) v = -1.0;  // C[idx, n + arange(ns)] = -1
    } else if (c - n0 == r - m0) {
      v = -1.0;  // -s <= 0
    }
    a.C[bi * (int64_t)m * n + t] = v;
  }
  for (int64_t t = t0; t < m; t += stride) a.d[bi * m + t] = t < m0 ? a.d0[bi * m0 + t] : 0.0;
}

}  // namespace

extern "C" {

int gm_condense_gammas_stage(gm_ctx* ctx, int B, int N, int n, const float* a_self,
                             const float* a_nbr, const float* b, const double* c,
                             const double* x0, float* gamma, int ld, void* stream) {
  int rc = check_dims(ctx, B, N, ld);
  if (rc) return rc;
  if (n < -1 || n >= N) return gm_fail(ctx, GM_ERR_CONFIG, "stage out of range");
  return rec_stage(ctx, B, N, n, a_self, a_nbr, b, c, x0, gamma, ld, (cudaStream_t)stream);
}

int gm_condense_gammas(gm_ctx* ctx, int B, int N, const float* a_self, const float* a_nbr,
                       const float* b, const double* c, const double* x0, float* gamma, int ld,
                       void* stream) {
  int rc = check_dims(ctx, B, N, ld);
  if (rc) return rc;
  for (int n = -1; n < N; ++n) {
    rc = rec_stage(ctx, B, N, n, a_self, a_nbr, b, c, x0, gamma, ld, (cudaStream_t)stream);
    if (rc) return rc;
  }
  return GM_OK;
}

int gm_condense_cost(gm_ctx* ctx, int B, int N, const float* gamma, int ld, const double* q,
                     int64_t q_stride, const double* x_ref, int64_t xref_stride, const double* r,
                     int64_t r_stride, const double* u_ref, int64_t uref_stride, double* H,
                     double* g, int partial, void* stream) {
  int rc = check_dims(ctx, B, N, ld);
  if (rc) return rc;
  if (B == 0) return GM_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const int nx = ctx->nx, nu = ctx->n_u;
  const int n0 = N * nu;
  const int tilesT = (n0 + kTile - 1) / kTile;
  const int npair = tilesT * tilesT;
  const int nodes = (int)(gm_node_hi(ctx) - ctx->node_lo);
  // split-K over nodes: about two CTAs per SM in total
  int splits = std::max(1, std::min(nodes, (2 * ctx->sm_count + B * npair - 1) / (B * npair)));
  // stage chunk so the staged rows fit the shared-memory budget
  int kc = N;
  auto smem_for = [&](int k) {
    return sizeof(float) * 2 * (size_t)k * nx * kTile + sizeof(double) * (size_t)k * nx + 16;
  };
  while (kc > 1 && smem_for(kc) > 120 * 1024) kc = (kc + 1) / 2;
  const size_t sm = smem_for(kc);
  const size_t partH_bytes = sizeof(float) * (size_t)B * npair * splits * kTile * kTile;
  const size_t partg_bytes = sizeof(double) * (size_t)B * splits * n0;
  char* scr = (char*)gm_scratch(ctx, partH_bytes + partg_bytes + 256);
  if (!scr) return gm_fail(ctx, GM_ERR_CUDA, "scratch allocation failed");
  CostArgs a{};
  a.M = (int)ctx->M;
  a.N = N;
  a.nx = nx;
  a.nu = nu;
  a.ld = ld;
  a.n0 = n0;
  a.lo = (int)ctx->node_lo;
  a.nodes = nodes;
  a.splits = splits;
  a.tilesT = tilesT;
  a.kc = kc;
  a.W = gamma;
  a.q = q;
  a.q_stride = q_stride;
  a.xref = x_ref;
  a.xref_stride = xref_stride;
  a.partH = (float*)scr;
  a.partg = (double*)(scr + ((partH_bytes + 255) & ~size_t(255)));
  GM_CUDA(ctx, cudaFuncSetAttribute(k_cost_partial, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  const int64_t blocks = (int64_t)B * splits * npair;
  k_cost_partial<<<(unsigned)blocks, 256, sm, st>>>(a);
  GM_LAUNCH_CHECK(ctx, "k_cost_partial");
  ReduceArgs ra{};
  ra.N = N;
  ra.nu = nu;
  ra.n0 = n0;
  ra.splits = splits;
  ra.tilesT = tilesT;
  ra.partial = partial;
  ra.partH = a.partH;
  ra.partg = a.partg;
  ra.r = r;
  ra.r_stride = r_stride;
  ra.uref = u_ref;
  ra.uref_stride = uref_stride;
  ra.H = H;
  ra.g = g;
  dim3 grid((unsigned)std::min(64, (n0 * n0 + 255) / 256), (unsigned)B);
  k_cost_reduce<<<grid, 256, 0, st>>>(ra);
  GM_LAUNCH_CHECK(ctx, "k_cost_reduce");
  return GM_OK;
}

int gm_constraint_rows(gm_ctx* ctx, int B, int N, const float* gamma, int ld, int n_in,
                       const int32_t* in_stage, const double* in_c, const double* in_d, int n_st,
                       const int32_t* st_node, const int32_t* st_stage, const double* st_c,
                       const double* st_d, double* C, double* d, void* stream) {
  int rc = check_dims(ctx, B, N, ld);
  if (rc) return rc;
  const int m0 = n_in + n_st;
  if (m0 == 0 || B == 0) return GM_OK;
  ConArgs a{};
  a.M = (int)ctx->M;
  a.N = N;
  a.nx = ctx->nx;
  a.nu = ctx->n_u;
  a.ld = ld;
  a.n0 = N * ctx->n_u;
  a.n_in = n_in;
  a.n_st = n_st;
  a.W = gamma;
  a.in_stage = in_stage;
  a.in_c = in_c;
  a.in_d = in_d;
  a.st_node = st_node;
  a.st_stage = st_stage;
  a.st_c = st_c;
  a.st_d = st_d;
  a.C = C;
  a.d = d;
  dim3 grid((unsigned)m0, (unsigned)B);
  k_constraint_rows<<<grid, 128, 0, (cudaStream_t)stream>>>(a);
  GM_LAUNCH_CHECK(ctx, "k_constraint_rows");
  return GM_OK;
}

int gm_expand_soft(gm_ctx* ctx, int B, int n0, int m0, const double* H0, const double* g0,
                   const double* C0, const double* d0, int ns, const int32_t* soft_idx,
                   const double* rho1, const double* rho2, double* H, double* g, double* C,
                   double* d, void* stream) {
  int rc = gm_need_device(ctx);
  if (rc) return rc;
  if (B == 0) return GM_OK;
  SoftArgs a{};
  a.n0 = n0;
  a.m0 = m0;
  a.ns = ns;
  a.H0 = H0;
  a.g0 = g0;
  a.C0 = C0;
  a.d0 = d0;
  a.idx = soft_idx;
  a.rho1 = rho1;
  a.rho2 = rho2;
  a.H = H;
  a.g = g;
  a.C = C;
  a.d = d;
  const int64_t n = n0 + ns, m = m0 + ns;
  const int64_t work = std::max<int64_t>(n * n, m * n);
  dim3 grid((unsigned)std::max<int64_t>(1, std::min<int64_t>(64, (work + 255) / 256)), (unsigned)B);
  k_expand_soft<<<grid, 256, 0, (cudaStream_t)stream>>>(a);
  GM_LAUNCH_CHECK(ctx, "k_expand_soft");
  return GM_OK;
}

}  // extern "C"
