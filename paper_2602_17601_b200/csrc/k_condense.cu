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
//        reduction over nodes with one persistent CTA per SM; each CTA streams
//        its nodes' Gamma / Q / x_ref rows through a bulk-copy (TMA) ring in
//        shared memory and keeps a 128x128 fp32 tile of H in registers (8x8
//        per thread, upper blocks only), skipping the non-causal part of every
//        row.  Partials are reduced in a fixed order in fp64 (bitwise
//        reproducible), R-bar is added and H is mirrored.
// K-CON  constraint rows (condensing.py:263-282, :312-323) and
//        expand_soft_constraints (condensing.py:419-439).
#include <algorithm>

#include "common.cuh"

namespace {

// ---------------------------------------------------------------------------
// K-REC
// ---------------------------------------------------------------------------
struct RecArgs {
  int M, E, N, nx, nu, ld, n, lo, nodes, B;
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

// K-REC, warp form (nx = 6, 16-byte aligned rows): one warp per (instance,
// node), lane l owns the column chunks 4l + 128 j of all six rows, so every
// neighbour row is one coalesced 512-byte float4 sweep and each lane keeps
// 6 x 4 accumulators; the node's 6x6 blocks are staged once per warp in
// shared memory (no CTA barrier) and read as broadcast vectors.  Chunks with
// no causal column skip the neighbour loads.  Per-column FMA order is that of
// k_gamma_stage (neighbour slot, then state index), so Gamma is bitwise
// identical to it and to the fused K-COND.
constexpr int kRecWarps = 8;
__global__ void __launch_bounds__(32 * kRecWarps) k_gamma_stage_w6(const RecArgs a, int dmax) {
  constexpr int NX = 6;
  extern __shared__ __align__(16) float rsm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t wg = (int64_t)blockIdx.x * kRecWarps + warp;
  const int nu = a.nu, ld = a.ld, N = a.N, n = a.n;
  const int64_t bi = wg / a.nodes;
  if (bi >= a.B) return;
  const int i = a.lo + (int)(wg - bi * a.nodes);
  const int64_t gi = bi * a.M + i;
  const int XC = N * nu;
  const int64_t stage_stride = (int64_t)NX * ld;
  const int64_t node_stride = (int64_t)(N + 1) * stage_stride;
  if (n < 0) {  // stage 0: Gamma_u = 0, Gamma_x = x0 (condensing.py:205-206)
    float* Wo = a.W + gi * node_stride;
    for (int c0 = lane * 4; c0 < ld; c0 += 128)
#pragma unroll
      for (int r = 0; r < NX; ++r) {
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        const float x = (float)a.x0[gi * NX + r];
        if (c0 == XC) v.x = x;
        if (c0 + 1 == XC) v.y = x;
        if (c0 + 2 == XC) v.z = x;
        if (c0 + 3 == XC) v.w = x;
        *reinterpret_cast<float4*>(Wo + (int64_t)r * ld + c0) = v;
      }
    return;
  }
  const int e0 = a.ptr[i], deg = a.ptr[i + 1] - e0;
  float* As = rsm + warp * ((dmax + 2) * NX * NX);  // (1+deg) A blocks, then B (nx x nu)
  float* Bs = As + (dmax + 1) * NX * NX;
  const int64_t pstage = bi * N + n;
  for (int t = lane; t < (1 + deg) * NX * NX; t += 32) {
    const int s = t / (NX * NX), q = t - s * NX * NX;
    As[t] = s == 0 ? a.a_self[(pstage * a.M + i) * NX * NX + q] : a.a_nbr[(pstage * a.E + e0 + s - 1) * NX * NX + q];
  }
  for (int t = lane; t < NX * nu; t += 32) Bs[t] = a.b[(pstage * a.M + i) * NX * nu + t];
  __syncwarp();
  const int live = n * nu;
  float* Wo = a.W + gi * node_stride + (int64_t)(n + 1) * stage_stride;
  for (int c0 = lane * 4; c0 < ld; c0 += 128) {
    float acc[NX][4];
#pragma unroll
    for (int r = 0; r < NX; ++r)
#pragma unroll
      for (int e = 0; e < 4; ++e) acc[r][e] = 0.f;
    if (c0 < live || (XC >= c0 && XC < c0 + 4)) {
      for (int s = 0; s <= deg; ++s) {
        const int j = s == 0 ? i : __ldg(a.src + e0 + s - 1);
        const float* Wj = a.W + (bi * a.M + j) * node_stride + (int64_t)n * stage_stride + c0;
        float4 w[NX];
#pragma unroll
        for (int q = 0; q < NX; ++q) w[q] = __ldcg(reinterpret_cast<const float4*>(Wj + (int64_t)q * ld));
        const float* A = As + s * NX * NX;
#pragma unroll
        for (int q = 0; q < NX; ++q)
#pragma unroll
          for (int r = 0; r < NX; ++r) {
            const float ar = A[r * NX + q];
            acc[r][0] = fmaf(ar, w[q].x, acc[r][0]);
            acc[r][1] = fmaf(ar, w[q].y, acc[r][1]);
            acc[r][2] = fmaf(ar, w[q].z, acc[r][2]);
            acc[r][3] = fmaf(ar, w[q].w, acc[r][3]);
          }
      }
    }
#pragma unroll
    for (int r = 0; r < NX; ++r) {
      float o[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int col = c0 + e;
        if (col < live) {
          o[e] = acc[r][e];
        } else if (col == XC) {
          o[e] = acc[r][e] + (float)a.c[pstage * a.M * NX + (int64_t)i * NX + r];
        } else if (col < live + nu) {
          o[e] = Bs[r * nu + (col - live)];
        } else {
          o[e] = 0.f;
        }
      }
      *reinterpret_cast<float4*>(Wo + (int64_t)r * ld + c0) = make_float4(o[0], o[1], o[2], o[3]);
    }
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
  a.B = B;
  const int64_t blocks = (int64_t)B * a.nodes;
  if (blocks == 0) return GM_OK;
  if (a.nx == 6 && ld % 4 == 0 && ((uintptr_t)W & 15) == 0 && ctx->cond_mode != 1) {
    const int dmax = (int)ctx->dmax;
    const size_t smw = sizeof(float) * (size_t)kRecWarps * (dmax + 2) * 36;
    k_gamma_stage_w6<<<(unsigned)((blocks + kRecWarps - 1) / kRecWarps), 32 * kRecWarps, smw, st>>>(a, dmax);
    GM_LAUNCH_CHECK(ctx, "k_gamma_stage_w6");
    return GM_OK;
  }
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
constexpr int kTile = 128;   // output tile of H per CTA (8x8 per thread, 256 threads)
constexpr int kRing = 3;     // bulk-copy ring depth (stage chunks in flight per CTA)

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  } while (!done);
}
// 1-D bulk copy global -> shared (TMA engine), completion counted on `bar`
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

struct CostArgs {
  int M, N, nx, nu, ld, n0, lo, nodes, splits, tilesT, npairU, kc, bulk;
  const float* W;
  const double* q;
  int64_t q_stride;
  const double* xref;
  int64_t xref_stride;
  float* partH;  // (B, npairU, splits, 128, 128); upper 8x8 blocks only on diagonal pairs
  double* partg; // (B, splits, n0)
};

// Split-K over nodes, one persistent CTA per (instance, upper tile pair, node
// range).  The rows of Gamma / Q / x_ref a CTA needs are contiguous per
// (node, stage chunk), so each chunk is ONE bulk copy per array into a
// kRing-deep shared-memory ring (mbarrier complete_tx), issued kRing chunks
// ahead of the consumer: the CTA streams its ~64 KB per node at copy-engine
// rate instead of one dependent global load chain per element.
//   per chunk:  QG = Qs G (column tile; Qs = (Q+Q')/2 so S = G' Qs G is already
//               the symmetrised sum 0.5(S+S') of condensing.py:403),
//               w  = 2 Q Gamma_x - 2 Q x_ref (fp64, condensing.py:153, :388)
//               acc += G(:, row tile)' QG         (8x8 fp32 per thread)
//               g   += G(:, row tile)' w          (fp64, diagonal pairs)
// Rows of stage k only reach columns < k*nu: chunks whose live columns end
// before the column tile are never copied, and per row a thread skips when its
// column block is non-causal.  On diagonal tile pairs only the 136 upper 8x8
// blocks are computed, packed onto the first 136 threads.
__global__ void __launch_bounds__(256, 1) k_cost_partial(const CostArgs a) {
  extern __shared__ __align__(128) unsigned char smraw[];
  const int nx = a.nx, nu = a.nu, ld = a.ld, N = a.N, KC = a.kc;
  const int rows_max = KC * nx;
  const int64_t slotW = (int64_t)rows_max * ld;            // floats
  const int64_t slotQ = (int64_t)rows_max * nx;            // doubles
  uint64_t* full = (uint64_t*)smraw;                       // kRing mbarriers
  float* Wr = (float*)(smraw + 128);                       // kRing * slotW (+ kTile pad)
  float* QG = Wr + kRing * slotW + kTile;                  // rows_max x 128
  double* Qr = (double*)(QG + (int64_t)rows_max * kTile);  // kRing * slotQ
  double* Xr = Qr + kRing * slotQ;                         // kRing * rows_max
  double* wv = Xr + kRing * rows_max;                      // rows_max

  const int64_t bi = blockIdx.x / ((int64_t)a.splits * a.npairU);
  const int rem = (int)(blockIdx.x % ((int64_t)a.splits * a.npairU));
  const int split = rem / a.npairU, pair = rem % a.npairU;
  int ti = 0, tj = pair;
  while (tj >= a.tilesT - ti) { tj -= a.tilesT - ti; ++ti; }
  tj += ti;
  const int c1b = ti * kTile, c2b = tj * kTile;
  const bool diag = ti == tj;
  const int per = (a.nodes + a.splits - 1) / a.splits;
  const int nb = a.lo + split * per, ne = min(a.lo + a.nodes, nb + per);
  const int cpn = (N + KC - 1) / KC;
  int g0 = 0;  // first stage chunk whose live columns reach the column tile
  while (g0 < cpn && min(N, (g0 + 1) * KC) * nu <= c2b) ++g0;
  const int act = cpn - g0;
  const int nchunks = ne > nb ? (ne - nb) * act : 0;

  // thread -> 8x8 block of the tile
  int ty = threadIdx.x >> 4, tx = threadIdx.x & 15;
  bool active = true;
  if (diag) {
    int t = threadIdx.x;
    active = t < 136;
    ty = 0;
    while (ty < 16 && t >= 16 - ty) { t -= 16 - ty; ++ty; }
    tx = ty + t;
    if (!active) { ty = 15; tx = 15; }
  }
  const bool do_g = diag;
  const int64_t stage_stride = (int64_t)nx * ld;
  const int XC = N * nu;

  auto chunk_src = [&](int c, int& node, int& k0, int& k1) {
    node = nb + c / act;
    const int grp = g0 + c % act;
    k0 = 1 + grp * KC;
    k1 = min(N + 1, k0 + KC);
  };
  auto issue = [&](int c) {  // one thread
    int node, k0, k1;
    chunk_src(c, node, k0, k1);
    const int slot = c % kRing;
    const int nk = k1 - k0;
    const int64_t gi = bi * a.M + node;
    const uint32_t bw = (uint32_t)(nk * stage_stride * sizeof(float));
    const uint32_t bq = (uint32_t)(nk * nx * nx * sizeof(double));
    const uint32_t bx = (uint32_t)(nk * nx * sizeof(double));
    mbar_expect_tx(&full[slot], bw + bq + bx);
    bulk_g2s(Wr + slot * slotW, a.W + (gi * (N + 1) + k0) * stage_stride, bw, &full[slot]);
    bulk_g2s(Qr + slot * slotQ, a.q + bi * a.q_stride + ((int64_t)node * (N + 1) + k0) * nx * nx, bq,
             &full[slot]);
    bulk_g2s(Xr + slot * rows_max, a.xref + bi * a.xref_stride + ((int64_t)node * (N + 1) + k0) * nx, bx,
             &full[slot]);
  };
  auto load_sync = [&](int c) {  // all threads, when bulk copies are not usable
    int node, k0, k1;
    chunk_src(c, node, k0, k1);
    const int slot = c % kRing;
    const int nk = k1 - k0;
    const int64_t gi = bi * a.M + node;
    const float* sw = a.W + (gi * (N + 1) + k0) * stage_stride;
    const double* sq = a.q + bi * a.q_stride + ((int64_t)node * (N + 1) + k0) * nx * nx;
    const double* sx = a.xref + bi * a.xref_stride + ((int64_t)node * (N + 1) + k0) * nx;
    for (int64_t t = threadIdx.x; t < nk * stage_stride; t += blockDim.x) Wr[slot * slotW + t] = sw[t];
    for (int t = threadIdx.x; t < nk * nx * nx; t += blockDim.x) Qr[slot * slotQ + t] = sq[t];
    for (int t = threadIdx.x; t < nk * nx; t += blockDim.x) Xr[slot * rows_max + t] = sx[t];
  };

  if (threadIdx.x == 0) {
    for (int s = 0; s < kRing; ++s) mbar_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int t = threadIdx.x; t < kTile; t += blockDim.x) Wr[kRing * slotW + t] = 0.f;
  __syncthreads();
  if (a.bulk && threadIdx.x == 0)
    for (int c = 0; c < min(kRing, nchunks); ++c) issue(c);

  float acc[8][8];
#pragma unroll
  for (int u = 0; u < 8; ++u)
#pragma unroll
    for (int v = 0; v < 8; ++v) acc[u][v] = 0.f;
  double gacc = 0.0;

  for (int c = 0; c < nchunks; ++c) {
    int node, k0, k1;
    chunk_src(c, node, k0, k1);
    const int slot = c % kRing;
    const int rows = (k1 - k0) * nx;
    if (a.bulk) mbar_wait(&full[slot], (uint32_t)((c / kRing) & 1));
    else load_sync(c);
    if (!a.bulk) __syncthreads();
    const float* Ws = Wr + slot * slotW;
    const double* Qs = Qr + slot * slotQ;
    // QG on the column tile
    for (int t = threadIdx.x; t < rows * kTile; t += blockDim.x) {
      const int r = t >> 7, cc = t & (kTile - 1);
      const int kk = r / nx, ar = r - kk * nx;
      const double* Qk = Qs + (int64_t)kk * nx * nx;
      const float* Wk = Ws + (int64_t)kk * stage_stride + c2b + cc;
      float s = 0.f;
      for (int b2 = 0; b2 < nx; ++b2)
        s = fmaf((float)(0.5 * (Qk[ar * nx + b2] + Qk[b2 * nx + ar])), Wk[(int64_t)b2 * ld], s);
      QG[t] = s;
    }
    if (do_g) {
      for (int r = threadIdx.x; r < rows; r += blockDim.x) {
        const int kk = r / nx, ar = r - kk * nx;
        const double* Qk = Qs + (int64_t)kk * nx * nx + ar * nx;
        const float* Wk = Ws + (int64_t)kk * stage_stride + XC;
        const double* xr = Xr + slot * rows_max + kk * nx;
        double qg = 0.0, qx = 0.0;
        for (int b2 = 0; b2 < nx; ++b2) {
          qg += Qk[b2] * (double)Wk[(int64_t)b2 * ld];
          qx += Qk[b2] * xr[b2];
        }
        wv[r] = 2.0 * qg + (-2.0 * qx);
      }
    }
    __syncthreads();
    if (active) {
      const int cb2 = c2b + tx * 8;
      for (int r = 0; r < rows; ++r) {
        const int live = (k0 + r / nx) * nu;
        if (cb2 >= live) continue;
        const float* Gr = Ws + (int64_t)(r / nx) * stage_stride + (int64_t)(r % nx) * ld + c1b + ty * 8;
        const float4 g1a = *(const float4*)(Gr);
        const float4 g1b = *(const float4*)(Gr + 4);
        const float4 g2a = *(const float4*)(QG + r * kTile + tx * 8);
        const float4 g2b = *(const float4*)(QG + r * kTile + tx * 8 + 4);
        const float x[8] = {g1a.x, g1a.y, g1a.z, g1a.w, g1b.x, g1b.y, g1b.z, g1b.w};
        const float y[8] = {g2a.x, g2a.y, g2a.z, g2a.w, g2b.x, g2b.y, g2b.z, g2b.w};
#pragma unroll
        for (int u = 0; u < 8; ++u)
#pragma unroll
          for (int v = 0; v < 8; ++v) acc[u][v] = fmaf(x[u], y[v], acc[u][v]);
      }
    }
    if (do_g && threadIdx.x < kTile) {
      for (int r = 0; r < rows; ++r)
        gacc += (double)Ws[(int64_t)(r / nx) * stage_stride + (int64_t)(r % nx) * ld + c1b + threadIdx.x] *
                wv[r];
    }
    __syncthreads();  // slot and QG free
    if (a.bulk && threadIdx.x == 0 && c + kRing < nchunks) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(c + kRing);
    }
  }
  float* P = a.partH + ((bi * a.npairU + pair) * (int64_t)a.splits + split) * kTile * kTile;
  if (active) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      float4* dst = (float4*)(P + (int64_t)(ty * 8 + u) * kTile + tx * 8);
      dst[0] = make_float4(acc[u][0], acc[u][1], acc[u][2], acc[u][3]);
      dst[1] = make_float4(acc[u][4], acc[u][5], acc[u][6], acc[u][7]);
    }
  }
  const int gcol = c1b + threadIdx.x;
  if (do_g && threadIdx.x < kTile && gcol < a.n0)
    a.partg[(bi * a.splits + split) * a.n0 + gcol] = gacc;
}

struct ReduceArgs {
  int N, nu, n0, splits, tilesT, groups, partial;
  const float* partH;
  const double* partg;
  double* tmpH;  // (B, groups, n0, n0)
  double* tmpg;  // (B, groups, n0)
  const double* r;
  int64_t r_stride;
  const double* uref;
  int64_t uref_stride;
  double* H;
  double* g;
};

__device__ __forceinline__ int upper_pair(int ti, int tj, int T) { return ti * T - ti * (ti - 1) / 2 + (tj - ti); }

// pass 1: sum the splits of one group for every upper element (c1 <= c2), in
// a fixed order (bitwise reproducible); coalesced over c2.
__global__ void k_cost_reduce1(const ReduceArgs a) {
  const int n0 = a.n0;
  const int64_t bi = blockIdx.z;
  const int grp = blockIdx.y;
  const int per = (a.splits + a.groups - 1) / a.groups;
  const int s0 = grp * per, s1 = min(a.splits, s0 + per);
  const int npairU = a.tilesT * (a.tilesT + 1) / 2;
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx < n0 * n0) {
    const int c1 = idx / n0, c2 = idx - c1 * n0;
    if (c1 <= c2) {
      const int pr = upper_pair(c1 / kTile, c2 / kTile, a.tilesT);
      const float* P = a.partH + ((bi * npairU + pr) * (int64_t)a.splits) * kTile * kTile +
                       (int64_t)(c1 % kTile) * kTile + (c2 % kTile);
      double s = 0.0;
#pragma unroll 4
      for (int sp = s0; sp < s1; ++sp) s += (double)P[(int64_t)sp * kTile * kTile];
      a.tmpH[(bi * a.groups + grp) * (int64_t)n0 * n0 + idx] = s;
    }
  }
  if (idx < n0) {
    double s = 0.0;
    for (int sp = s0; sp < s1; ++sp) s += a.partg[(bi * a.splits + sp) * n0 + idx];
    a.tmpg[(bi * a.groups + grp) * n0 + idx] = s;
  }
}

// pass 2: H = S + R-bar (mirrored), g = sum + r_lin.
__global__ void k_cost_reduce2(const ReduceArgs a) {
  const int n0 = a.n0, nu = a.nu;
  const int64_t bi = blockIdx.y;
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx < n0 * n0) {
    const int c1 = idx / n0, c2 = idx - c1 * n0;
    if (c1 <= c2) {
      double h = 0.0;
      for (int grp = 0; grp < a.groups; ++grp) h += a.tmpH[(bi * a.groups + grp) * (int64_t)n0 * n0 + idx];
      if (!a.partial && c1 / nu == c2 / nu) {
        const int k = c1 / nu;
        const double* Rk = a.r + bi * a.r_stride + (int64_t)k * nu * nu;
        // R-bar is symmetrised with the rest (condensing.py:380-381, :403)
        h += 0.5 * (Rk[(c1 % nu) * nu + (c2 % nu)] + Rk[(c2 % nu) * nu + (c1 % nu)]);
      }
      a.H[bi * (int64_t)n0 * n0 + (int64_t)c1 * n0 + c2] = h;
      a.H[bi * (int64_t)n0 * n0 + (int64_t)c2 * n0 + c1] = h;
    }
  }
  if (idx < n0) {
    double s = 0.0;
    for (int grp = 0; grp < a.groups; ++grp) s += a.tmpg[(bi * a.groups + grp) * n0 + idx];
    if (!a.partial) {
      // r_lin = -2 R u_ref (condensing.py:154)
      const int k = idx / nu, row = idx % nu;
      const double* Rk = a.r + bi * a.r_stride + (int64_t)k * nu * nu + row * nu;
      const double* uk = a.uref + bi * a.uref_stride + (int64_t)k * nu;
      double ru = 0.0;
      for (int j = 0; j < nu; ++j) ru += Rk[j] * uk[j];
      s = -2.0 * ru + s;
    }
    a.g[bi * n0 + idx] = s;
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
  // K-HG through the fused condensing kernel without its recursion: the
  // SIMT one (fp32 FMA, round-to-nearest) by default, the tcgen05 3xTF32 one
  // when forced (gm_set_condense_mode(3)); the per-tile kernel below for
  // shapes without an instantiation
  {
    rc = gm_fused_cost(ctx, ctx->cond_mode == 3, B, N, gamma, ld, q, q_stride, x_ref, xref_stride,
                       r, r_stride, u_ref, uref_stride, H, g, partial, stream);
    if (rc != 1) return rc;
  }
  cudaStream_t st = (cudaStream_t)stream;
  const int nx = ctx->nx, nu = ctx->n_u;
  const int n0 = N * nu;
  const int tilesT = (n0 + kTile - 1) / kTile;
  const int npairU = tilesT * (tilesT + 1) / 2;
  const int nodes = (int)(gm_node_hi(ctx) - ctx->node_lo);
  // split-K over nodes: one persistent CTA per SM in total
  const int splits = std::max(1, std::min(nodes, (ctx->sm_count + B * npairU - 1) / (B * npairU)));
  // stage chunk: the largest balanced chunk whose ring fits shared memory
  auto smem_for = [&](int k) {
    const size_t rows = (size_t)k * nx;
    return 128 + sizeof(float) * (kRing * rows * ld + kTile + rows * kTile) +
           sizeof(double) * (kRing * rows * nx + kRing * rows + rows);
  };
  const size_t budget = std::min<size_t>(ctx->smem_optin, 200 * 1024);
  int kmax = N;
  while (kmax > 1 && smem_for(kmax) > budget) --kmax;
  if (smem_for(kmax) > budget) return gm_fail(ctx, GM_ERR_CONFIG, "gamma rows too wide for K-HG tiles");
  const int kc = gm_ceil_div(N, gm_ceil_div(N, kmax));
  const size_t sm = smem_for(kc);
  // bulk copies need 16-byte aligned sources and sizes
  auto al = [](const void* p) { return ((uintptr_t)p & 15) == 0; };
  const int bulk = al(gamma) && al(q) && al(x_ref) && (ld % 4 == 0) && (nx % 2 == 0) &&
                   (q_stride % 2 == 0) && (xref_stride % 2 == 0);
  const int groups = std::min(splits, 16);
  const size_t partH_bytes = sizeof(float) * (size_t)B * npairU * splits * kTile * kTile;
  const size_t partg_bytes = sizeof(double) * (size_t)B * splits * n0;
  const size_t tmpH_bytes = sizeof(double) * (size_t)B * groups * n0 * n0;
  const size_t tmpg_bytes = sizeof(double) * (size_t)B * groups * n0;
  auto up = [](size_t x) { return (x + 255) & ~size_t(255); };
  char* scr = (char*)gm_scratch(ctx, up(partH_bytes) + up(partg_bytes) + up(tmpH_bytes) + tmpg_bytes + 256);
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
  a.npairU = npairU;
  a.kc = kc;
  a.bulk = bulk;
  a.W = gamma;
  a.q = q;
  a.q_stride = q_stride;
  a.xref = x_ref;
  a.xref_stride = xref_stride;
  a.partH = (float*)scr;
  a.partg = (double*)(scr + up(partH_bytes));
  GM_CUDA(ctx, cudaFuncSetAttribute(k_cost_partial, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  const int64_t blocks = (int64_t)B * splits * npairU;
  k_cost_partial<<<(unsigned)blocks, 256, sm, st>>>(a);
  GM_LAUNCH_CHECK(ctx, "k_cost_partial");
  ReduceArgs ra{};
  ra.N = N;
  ra.nu = nu;
  ra.n0 = n0;
  ra.splits = splits;
  ra.tilesT = tilesT;
  ra.groups = groups;
  ra.partial = partial;
  ra.partH = a.partH;
  ra.partg = a.partg;
  ra.tmpH = (double*)(scr + up(partH_bytes) + up(partg_bytes));
  ra.tmpg = (double*)(scr + up(partH_bytes) + up(partg_bytes) + up(tmpH_bytes));
  ra.r = r;
  ra.r_stride = r_stride;
  ra.uref = u_ref;
  ra.uref_stride = uref_stride;
  ra.H = H;
  ra.g = g;
  const unsigned eb = (unsigned)gm_ceil_div((int64_t)n0 * n0, 256);
  k_cost_reduce1<<<dim3(eb, (unsigned)groups, (unsigned)B), 256, 0, st>>>(ra);
  GM_LAUNCH_CHECK(ctx, "k_cost_reduce1");
  k_cost_reduce2<<<dim3(eb, (unsigned)B), 256, 0, st>>>(ra);
  GM_LAUNCH_CHECK(ctx, "k_cost_reduce2");
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
