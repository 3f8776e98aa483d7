// K-LIN v2: layer-wise GNN linearisation (stage 1) as a chain of large GEMMs.
//
// Reference: _linearize_batch (gnn.py:237-298), _forward_parts
// (gnn.py:129-150), mlp_jacobian (mlp.py:132-145), step_array
// (gnn.py:153-159).  Same formulas as the fused per-tile kernel
// (k_linearize.cu), but every MLP layer of every node / edge of every
// linearisation point is ONE register-tiled GEMM launch over all rows:
//
//   rows      layer GEMM (K x N)                       precision  epilogue
//   edges     psi forward  6->32->32->16               fp64       +bias, ReLU mask
//   nodes     phi forward 28->64->64->3                fp64       +bias, ReLU mask
//   nodes*3   phi Jacobian from the output side 64->64->28   fp32  mask of the row's node
//   edges*3   psi VJP seeded with J_m[dst]   16->32->32->6   fp32  mask of the row's edge
//
// Per-CTA fused tiles hold only ~16 nodes (shared memory), which left every
// layer latency- and load-bound; here each launch is a plain GEMM with the
// weights and a transposed input tile in shared memory and an RT x CT register
// tile per thread, and the intermediates stream through L2/HBM (~170 MB at
// cfg3, L2-resident; ~34 GB at the 1e5-node mesh, ~5 ms of HBM time against
// ~39 ms for the fused kernel).  Masks are stored as bytes, activations in
// fp64 / fp32 exactly as the fused kernel keeps them on chip, so results are
// identical to it up to summation order within a dot product.
#include <algorithm>

#include "common.cuh"

namespace {

constexpr int kLT = 256;

enum { kFwdHidden = 0, kFwdLast = 1, kBwd = 2 };

// out[r][c] = epi(sum_k in[r][k] W[k][c]), W (K, N) row-major.  Block: BR rows
// x all N columns; thread (rg, cg) owns rows rg*RT.., columns cg*CT..
template <typename T, int RT, int CT, int MODE>
__global__ void __launch_bounds__(kLT) k_layer(const T* __restrict__ in, int ldi, int R, int K,
                                               const T* __restrict__ W, int N, const T* __restrict__ bias,
                                               T* __restrict__ out, int ldo, uint8_t* __restrict__ mask,
                                               int ldm, int rows_per) {
  extern __shared__ __align__(16) unsigned char sm[];
  const int tid = threadIdx.x;
  const int CG = N / CT, RGB = kLT / CG, BR = RGB * RT, ldx = BR + 1;
  T* Ws = (T*)sm;      // K x N
  T* Xs = Ws + K * N;  // K x ldx: transposed input tile
  const int rb = blockIdx.x * BR;
  for (int t = tid; t < K * N; t += kLT) Ws[t] = W[t];
#pragma unroll 8
  for (int t = tid; t < BR * K; t += kLT) {
    const int r = t / K, k = t - r * K;
    const int gr = rb + r;
    Xs[k * ldx + r] = gr < R ? in[(int64_t)gr * ldi + k] : T(0);
  }
  __syncthreads();
  const int cg = tid % CG, rg = tid / CG;
  const int c0 = cg * CT, rl = min(rg, RGB - 1) * RT;  // idle threads (rg >= RGB) shadow the last group
  T acc[RT][CT];
#pragma unroll
  for (int t = 0; t < RT; ++t)
#pragma unroll
    for (int u = 0; u < CT; ++u) acc[t][u] = T(0);
#pragma unroll 4
  for (int k = 0; k < K; ++k) {
    T w[CT], x[RT];
#pragma unroll
    for (int u = 0; u < CT; ++u) w[u] = Ws[k * N + c0 + u];
#pragma unroll
    for (int t = 0; t < RT; ++t) x[t] = Xs[k * ldx + rl + t];
#pragma unroll
    for (int t = 0; t < RT; ++t)
#pragma unroll
      for (int u = 0; u < CT; ++u) acc[t][u] = fma(x[t], w[u], acc[t][u]);
  }
  // epilogue into a row-major output tile in shared memory (the input tile is
  // dead), then coalesced row-contiguous stores of values and mask bytes
  __syncthreads();
  const int ldt = N + 1;
  T* Os = Xs;                                            // BR x ldt
  uint8_t* Ms = (uint8_t*)(Xs + (size_t)BR * ldt);        // BR x N (hidden layers)
  if (rg < RGB) {
#pragma unroll
    for (int t = 0; t < RT; ++t) {
      const int rloc = rl + t;
      const int r = rb + rloc;
      const int mrow = MODE == kBwd ? r / rows_per : r;
#pragma unroll
      for (int u = 0; u < CT; ++u) {
        const int c = c0 + u;
        T v = acc[t][u];
        if constexpr (MODE == kFwdHidden) {
          v += bias[c];
          const bool m = v > T(0);  // strict: derivative 0 at the kink (mlp.py:143)
          Ms[rloc * N + c] = m;
          v = m ? v : T(0);
        } else if constexpr (MODE == kFwdLast) {
          v += bias[c];
        } else {
          if (mask && r < R && !mask[(int64_t)mrow * ldm + c]) v = T(0);
        }
        Os[rloc * ldt + c] = v;
      }
    }
  }
  __syncthreads();
  const int rows = min(BR, R - rb);
  for (int t = tid; t < rows * N; t += kLT) {
    const int rloc = t / N, c = t - rloc * N;
    out[(int64_t)(rb + rloc) * ldo + c] = Os[rloc * ldt + c];
    if constexpr (MODE == kFwdHidden) mask[(int64_t)(rb + rloc) * ldm + c] = Ms[rloc * N + c];
  }
}

template <typename T, int RT, int MODE>
int launch_layer(gm_ctx* ctx, const T* in, int ldi, int64_t R, int K, const T* W, int N, const T* bias,
                 T* out, int ldo, uint8_t* mask, int ldm, int rows_per, cudaStream_t st) {
  if (R <= 0) return GM_OK;
  if (R >= (int64_t(1) << 31)) return gm_fail(ctx, GM_ERR_CONFIG, "too many rows for one layer launch");
  auto go = [&](auto kern, int CT) -> int {
    const int CG = N / CT, BR = (kLT / CG) * RT;
    const size_t tile_in = sizeof(T) * (size_t)K * (BR + 1);
    const size_t tile_out = sizeof(T) * (size_t)BR * (N + 1) + (size_t)BR * N;
    const size_t smem = sizeof(T) * (size_t)K * N + ((std::max(tile_in, tile_out) + 15) & ~size_t(15));
    if (smem > ctx->smem_optin) return gm_fail(ctx, GM_ERR_CONFIG, "layer too wide for the layer GEMM");
    GM_CUDA(ctx, cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const int64_t blocks = (R + BR - 1) / BR;
    kern<<<(unsigned)blocks, kLT, smem, st>>>(in, ldi, (int)R, K, W, N, bias, out, ldo, mask, ldm, rows_per);
    GM_LAUNCH_CHECK(ctx, "k_layer");
    return GM_OK;
  };
  if (N % 4 == 0) return go(k_layer<T, RT, 4, MODE>, 4);
  if (N % 2 == 0) return go(k_layer<T, RT, 2, MODE>, 2);
  return go(k_layer<T, RT, 1, MODE>, 1);
}

struct LinDims {
  int M, nx, nu, n_p, n_m, nin, lo, nN, e0, nE;
  int P, Rn, Re;  // every element count below stays < 2^31 (host check)
};

// edge features e = (x_dst - x_src) / s_x over all (point, owned edge)
__global__ void k_lin_edges(const LinDims d, const int* __restrict__ dst, const int* __restrict__ src,
                            const double* __restrict__ X, const double* __restrict__ norm, double* ef) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= d.Re * d.nx) return;
  const int re = t / d.nx;
  const int k = (int)(t - re * d.nx);
  const int p = re / d.nE;
  const int e = d.e0 + (int)(re - p * d.nE);
  const double* Xp = X + p * (int64_t)d.M * d.nx;
  ef[t] = (Xp[(int64_t)dst[e] * d.nx + k] - Xp[(int64_t)src[e] * d.nx + k]) / norm[d.nx + k];
}

// z = [(x - mu)/s, sum of in-edge messages (edge order), (u - mu_u)/s_u]
__global__ void k_lin_z(const LinDims d, const int* __restrict__ ptr, const double* __restrict__ X,
                        const double* __restrict__ U, const double* __restrict__ norm,
                        const double* __restrict__ msg, int ldmsg, double* z) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= d.Rn * d.nin) return;
  const int rn = t / d.nin;
  const int k = (int)(t - rn * d.nin);
  const int p = rn / d.nN;
  const int i = d.lo + (int)(rn - p * d.nN);
  const int nx = d.nx;
  double v;
  if (k < nx) {
    v = (X[(p * d.M + i) * nx + k] - norm[k]) / norm[nx + k];
  } else if (k < nx + d.n_m) {
    const int m = k - nx;
    v = 0.0;
    for (int e = ptr[i]; e < ptr[i + 1]; ++e) v += msg[(p * d.nE + (e - d.e0)) * ldmsg + m];
  } else {
    const int j = k - nx - d.n_m;
    v = (U[p * d.nu + j] - norm[2 * nx + j]) / norm[2 * nx + d.nu + j];
  }
  z[t] = v;
}

// f = step_array: v' = v + dv, p' = p + dt v' (gnn.py:157-158)
__global__ void k_lin_f(const LinDims d, double dt, const double* __restrict__ X,
                        const double* __restrict__ dv, int ldv, double* f, double* f_next) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= d.Rn * d.nx) return;
  const int rn = t / d.nx;
  const int k = (int)(t - rn * d.nx);
  const int p = rn / d.nN;
  const int i = d.lo + (int)(rn - p * d.nN);
  const double* xi = X + (p * d.M + i) * d.nx;
  const int n_p = d.n_p;
  double val;
  if (k >= n_p) {
    val = xi[k] + dv[rn * ldv + (k - n_p)];
  } else {
    const double v1 = xi[n_p + k] + dv[rn * ldv + k];
    val = xi[k] + dt * v1;
  }
  f[t] = val;
  if (f_next) f_next[(p * d.M + i) * d.nx + k] = val;
}

// phi Jacobian seed: row (node, ro) = W_L[ro] masked by the node's last hidden layer
__global__ void k_lin_seed_phi(const LinDims d, const float* __restrict__ wL, int wl,
                               const uint8_t* __restrict__ mphi, int hphi, int mo, float* q, int ldq) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= d.Rn * d.n_p * wl) return;
  const int r = t / wl;
  const int j = (int)(t - r * wl);
  const int rn = r / d.n_p;
  const int ro = (int)(r - rn * d.n_p);
  q[r * ldq + j] = mphi[rn * hphi + mo + j] ? wL[ro * wl + j] : 0.f;
}

// psi VJP seed: row (edge, ro) = J_m of the edge's destination node
__global__ void k_lin_seed_psi(const LinDims d, const int* __restrict__ dst, const float* __restrict__ jphi,
                               float* q, int ldq) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= d.Re * d.n_p * d.n_m) return;
  const int r = t / d.n_m;
  const int m = (int)(t - r * d.n_m);
  const int re = r / d.n_p;
  const int ro = (int)(r - re * d.n_p);
  const int p = re / d.nE;
  const int e = d.e0 + (int)(re - p * d.nE);
  const int rn = p * d.nN + (dst[e] - d.lo);
  q[r * ldq + m] = jphi[(rn * d.n_p + ro) * d.nin + d.nx + m];
}

// a_nbr blocks of every (point, owned edge) (gnn.py:266, :282-285)
__global__ void k_lin_nbr(const LinDims d, float dtf, const double* __restrict__ norm,
                          const float* __restrict__ Pe, int E, float* a_nbr) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  const int nx = d.nx, n_p = d.n_p;
  if (t >= d.Re * n_p * nx) return;
  const int re = t / (n_p * nx);
  const int rem = (int)(t - re * n_p * nx), r = rem / nx, cc = rem - r * nx;
  const int p = re / d.nE;
  const int e = d.e0 + (int)(re - p * d.nE);
  const float inv_sx = (float)(1.0 / norm[nx + cc]);
  const float jv = -Pe[(re * n_p + r) * nx + cc] * inv_sx;
  float* blk = a_nbr + (p * E + e) * (int64_t)nx * nx;
  blk[r * nx + cc] = dtf * jv;
  blk[(n_p + r) * nx + cc] = jv;
}

// a_self and b blocks of every (point, owned node) (gnn.py:262-288)
__global__ void k_lin_self(const LinDims d, float dtf, const int* __restrict__ ptr,
                           const double* __restrict__ norm, const float* __restrict__ jphi,
                           const float* __restrict__ Pe, float* a_self, float* b) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  const int nx = d.nx, nu = d.nu, n_p = d.n_p, w = nx + nu;
  if (t >= d.Rn * n_p * w) return;
  const int rn = t / (n_p * w);
  const int rem = (int)(t - rn * n_p * w), r = rem / w, cc = rem - r * w;
  const int p = rn / d.nN;
  const int i = d.lo + (int)(rn - p * d.nN);
  const float* jr = jphi + (rn * n_p + r) * d.nin;
  if (cc < nx) {
    float s = 0.f;
    for (int e = ptr[i]; e < ptr[i + 1]; ++e) s += Pe[((p * d.nE + (e - d.e0)) * n_p + r) * nx + cc];
    const float inv_sx = (float)(1.0 / norm[nx + cc]);
    const float dvdx = (jr[cc] + s) * inv_sx + (cc == n_p + r ? 1.f : 0.f);
    float* blk = a_self + (p * d.M + i) * (int64_t)nx * nx;
    blk[r * nx + cc] = (r == cc ? 1.f : 0.f) + dtf * dvdx;
    blk[(n_p + r) * nx + cc] = dvdx;
  } else {
    const int cu = cc - nx;
    const float inv_su = (float)(1.0 / norm[2 * nx + nu + cu]);
    const float jv = jr[nx + d.n_m + cu] * inv_su;
    float* blk = b + (p * d.M + i) * (int64_t)nx * nu;
    blk[r * nu + cu] = dtf * jv;
    blk[(n_p + r) * nu + cu] = jv;
  }
}

// affine offset in fp64 from the stored fp32 blocks (gnn.py:291-297)
__global__ void k_lin_c(const LinDims d, int E, const int* __restrict__ ptr, const int* __restrict__ src,
                        const double* __restrict__ X, const double* __restrict__ U, const double* __restrict__ f,
                        const float* __restrict__ a_self, const float* __restrict__ a_nbr,
                        const float* __restrict__ b, double* c) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  const int nx = d.nx, nu = d.nu;
  if (t >= d.Rn * nx) return;
  const int rn = t / nx;
  const int r = (int)(t - rn * nx);
  const int p = rn / d.nN;
  const int i = d.lo + (int)(rn - p * d.nN);
  const double* Xp = X + p * (int64_t)d.M * nx;
  const double* xi = Xp + (int64_t)i * nx;
  const float* As = a_self + ((p * d.M + i) * nx + r) * nx;
  double s = f[t];
  for (int k = 0; k < nx; ++k) s -= (double)As[k] * xi[k];
  const float* Bs = b + ((p * d.M + i) * nx + r) * nu;
  for (int k = 0; k < nu; ++k) s -= (double)Bs[k] * U[p * nu + k];
  for (int e = ptr[i]; e < ptr[i + 1]; ++e) {
    const float* An = a_nbr + ((p * E + e) * nx + r) * nx;
    const double* xj = Xp + (int64_t)src[e] * nx;
    for (int k = 0; k < nx; ++k) s -= (double)An[k] * xj[k];
  }
  c[(p * d.M + i) * nx + r] = s;
}

inline unsigned grid_for(int64_t n) { return (unsigned)((n + 255) / 256); }
inline int pld(int w) { return w | 1; }
inline size_t al(size_t x) { return (x + 255) & ~size_t(255); }

}  // namespace

namespace {

int layers_chunk(gm_ctx* ctx, int64_t P, const double* X, const double* U, float* a_self, float* a_nbr,
                 float* b, double* c, double* f_next, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t lo = ctx->node_lo, hi = gm_node_hi(ctx);
  LinDims d{};
  d.M = (int)ctx->M;
  d.nx = ctx->m_nx;
  d.nu = ctx->m_nu;
  d.n_p = ctx->n_p;
  d.n_m = ctx->n_m;
  d.nin = ctx->phi.dims[0];
  d.lo = (int)lo;
  d.nN = (int)(hi - lo);
  d.e0 = (int)ctx->h_ptr[lo];
  d.nE = (int)(ctx->h_ptr[hi] - ctx->h_ptr[lo]);
  d.P = (int)P;  // chunked by the caller: every element count fits in int
  d.Rn = (int)(P * (hi - lo));
  d.Re = (int)(P * (ctx->h_ptr[hi] - ctx->h_ptr[lo]));
  const MlpView psi = ctx->psi.view(), phi = ctx->phi.view();
  const int wpsi = ctx->psi.max_width(), wphi = ctx->phi.max_width();
  const int hpsi = ctx->psi.hidden_sum(), hphi = ctx->phi.hidden_sum();
  const int n_p = d.n_p, nx = d.nx;
  // scratch carve-up
  const size_t n64 = (size_t)std::max(d.Re * pld(wpsi), d.Rn * pld(wphi));
  const size_t n32 = (size_t)std::max(d.Rn * n_p * pld(wphi), d.Re * n_p * pld(wpsi));
  size_t o = 0;
  const size_t o_ef = o;  o = al(o + sizeof(double) * d.Re * nx);
  const size_t o_ha = o;  o = al(o + sizeof(double) * n64);
  const size_t o_hb = o;  o = al(o + sizeof(double) * n64);
  const size_t o_z = o;   o = al(o + sizeof(double) * d.Rn * d.nin);
  const size_t o_f = o;   o = al(o + sizeof(double) * d.Rn * nx);
  const size_t o_mp = o;  o = al(o + (size_t)d.Re * hpsi);
  const size_t o_mf = o;  o = al(o + (size_t)d.Rn * hphi);
  const size_t o_qa = o;  o = al(o + sizeof(float) * n32);
  const size_t o_qb = o;  o = al(o + sizeof(float) * n32);
  const size_t o_j = o;   o = al(o + sizeof(float) * d.Rn * n_p * d.nin);
  const size_t o_pe = o;  o = al(o + sizeof(float) * d.Re * n_p * nx);
  unsigned char* base = (unsigned char*)gm_scratch(ctx, o);
  if (!base) return gm_fail(ctx, GM_ERR_CUDA, "linearisation workspace allocation failed");
  double* ef = (double*)(base + o_ef);
  double* ha = (double*)(base + o_ha);
  double* hb = (double*)(base + o_hb);
  double* z = (double*)(base + o_z);
  double* fb = (double*)(base + o_f);
  uint8_t* mpsi = base + o_mp;
  uint8_t* mphi = base + o_mf;
  float* qa = (float*)(base + o_qa);
  float* qb = (float*)(base + o_qb);
  float* jphi = (float*)(base + o_j);
  float* Pe = (float*)(base + o_pe);
  auto mask_off = [](const MlpView& m, int l) {
    int s = 0;
    for (int q = 0; q < l; ++q) s += m.dims[q + 1];
    return s;
  };
  int rc;
  // psi forward over every (point, owned edge)
  const double* msg = nullptr;
  int ldmsg = 0;
  if (d.Re > 0) {
    k_lin_edges<<<grid_for(d.Re * nx), 256, 0, st>>>(d, ctx->d_dst, ctx->d_src, X, ctx->d_norm, ef);
    GM_LAUNCH_CHECK(ctx, "k_lin_edges");
    const double* cur = ef;
    int ldc = nx;
    for (int l = 0; l < psi.L; ++l) {
      double* outp = (l & 1) ? hb : ha;
      const int N = psi.dims[l + 1];
      const bool relu = l < psi.L - 1;
      rc = relu ? launch_layer<double, 4, kFwdHidden>(ctx, cur, ldc, d.Re, psi.dims[l], psi.wt64[l], N,
                                                     psi.b64[l], outp, pld(N), mpsi + mask_off(psi, l), hpsi,
                                                     1, st)
                : launch_layer<double, 4, kFwdLast>(ctx, cur, ldc, d.Re, psi.dims[l], psi.wt64[l], N,
                                                   psi.b64[l], outp, pld(N), nullptr, 0, 1, st);
      if (rc) return rc;
      cur = outp;
      ldc = pld(N);
    }
    msg = cur;
    ldmsg = ldc;
  }
  k_lin_z<<<grid_for(d.Rn * d.nin), 256, 0, st>>>(d, ctx->d_ptr, X, U, ctx->d_norm, msg, ldmsg, z);
  GM_LAUNCH_CHECK(ctx, "k_lin_z");
  // phi forward over every (point, owned node); the output buffer must not
  // alias msg (ha/hb hold it), so phi starts in the buffer psi did not end in
  double* pbuf[2] = {(msg == ha) ? hb : ha, (msg == ha) ? ha : hb};
  const double* cur = z;
  int ldc = d.nin;
  for (int l = 0; l < phi.L; ++l) {
    double* outp = pbuf[l & 1];
    const int N = phi.dims[l + 1];
    const bool relu = l < phi.L - 1;
    rc = relu ? launch_layer<double, 4, kFwdHidden>(ctx, cur, ldc, d.Rn, phi.dims[l], phi.wt64[l], N, phi.b64[l],
                                                   outp, pld(N), mphi + mask_off(phi, l), hphi, 1, st)
              : launch_layer<double, 4, kFwdLast>(ctx, cur, ldc, d.Rn, phi.dims[l], phi.wt64[l], N, phi.b64[l],
                                                 outp, pld(N), nullptr, 0, 1, st);
    if (rc) return rc;
    cur = outp;
    ldc = pld(N);
  }
  k_lin_f<<<grid_for(d.Rn * nx), 256, 0, st>>>(d, ctx->dt, X, cur, ldc, fb, f_next);
  GM_LAUNCH_CHECK(ctx, "k_lin_f");
  // phi Jacobian, n_p rows per node, accumulated from the output side
  const int64_t Rj = d.Rn * n_p;
  if (phi.L == 1) {
    return gm_fail(ctx, GM_ERR_CONFIG, "single-layer phi is handled by the fused kernel");
  }
  {
    const int L = phi.L, wl = phi.dims[L - 1];
    k_lin_seed_phi<<<grid_for(Rj * wl), 256, 0, st>>>(d, phi.w32[L - 1], wl, mphi, hphi, mask_off(phi, L - 2), qa,
                                                      pld(wl));
    GM_LAUNCH_CHECK(ctx, "k_lin_seed_phi");
    const float* qc = qa;
    int ldq = pld(wl);
    for (int l = L - 2; l >= 0; --l) {
      const int KK = phi.dims[l];
      float* outp = (l == 0) ? jphi : ((qc == qa) ? qb : qa);
      uint8_t* mk = (l >= 1) ? mphi + mask_off(phi, l - 1) : nullptr;
      rc = launch_layer<float, 8, kBwd>(ctx, qc, ldq, Rj, phi.dims[l + 1], phi.w32[l], KK, nullptr, outp,
                                        l == 0 ? KK : pld(KK), mk, hphi, n_p, st);
      if (rc) return rc;
      qc = outp;
      ldq = pld(KK);
    }
  }
  // psi VJP seeded with J_m[dst], n_p rows per edge
  const int64_t Rv = d.Re * n_p;
  if (d.Re > 0) {
    k_lin_seed_psi<<<grid_for(Rv * d.n_m), 256, 0, st>>>(d, ctx->d_dst, jphi, qa, pld(d.n_m));
    GM_LAUNCH_CHECK(ctx, "k_lin_seed_psi");
    const float* qc = qa;
    int ldq = pld(d.n_m);
    for (int l = psi.L - 1; l >= 0; --l) {
      const int KK = psi.dims[l];
      float* outp = (l == 0) ? Pe : ((qc == qa) ? qb : qa);
      uint8_t* mk = (l >= 1) ? mpsi + mask_off(psi, l - 1) : nullptr;
      rc = launch_layer<float, 8, kBwd>(ctx, qc, ldq, Rv, psi.dims[l + 1], psi.w32[l], KK, nullptr, outp,
                                        l == 0 ? KK : pld(KK), mk, hpsi, n_p, st);
      if (rc) return rc;
      qc = outp;
      ldq = pld(KK);
    }
    k_lin_nbr<<<grid_for(Rv * nx), 256, 0, st>>>(d, (float)ctx->dt, ctx->d_norm, Pe, (int)ctx->E, a_nbr);
    GM_LAUNCH_CHECK(ctx, "k_lin_nbr");
  }
  k_lin_self<<<grid_for(Rj * (nx + d.nu)), 256, 0, st>>>(d, (float)ctx->dt, ctx->d_ptr, ctx->d_norm, jphi, Pe,
                                                        a_self, b);
  GM_LAUNCH_CHECK(ctx, "k_lin_self");
  k_lin_c<<<grid_for(d.Rn * nx), 256, 0, st>>>(d, (int)ctx->E, ctx->d_ptr, ctx->d_src, X, U, fb, a_self, a_nbr,
                                               b, c);
  GM_LAUNCH_CHECK(ctx, "k_lin_c");
  return GM_OK;
}

// largest per-point element count of any intermediate buffer
int64_t per_point_elements(const gm_ctx* ctx) {
  const int64_t nN = gm_node_hi(ctx) - ctx->node_lo;
  const int64_t nE = ctx->h_ptr[gm_node_hi(ctx)] - ctx->h_ptr[ctx->node_lo];
  const int64_t wpsi = pld(ctx->psi.max_width()), wphi = pld(ctx->phi.max_width()), n_p = ctx->n_p;
  const int64_t nin = ctx->phi.dims[0];
  int64_t m = std::max({nE * n_p * wpsi, nN * n_p * wphi, nN * n_p * nin, nE * wpsi, nN * wphi,
                        (int64_t)nE * ctx->psi.hidden_sum(), (int64_t)nN * ctx->phi.hidden_sum()});
  return std::max<int64_t>(m, 1);
}

}  // namespace

// Layer-wise linearisation over P points (owned node range); same contract
// as gm_linearize.  Points are processed in chunks so every buffer index fits
// in 32 bits and the workspace stays below ~2^30 elements per buffer.
int launch_linearize_layers(gm_ctx* ctx, int64_t P, const double* X, const double* U, float* a_self,
                            float* a_nbr, float* b, double* c, double* f_next, void* stream) {
  const int64_t M = ctx->M, E = ctx->E;
  const int nx = ctx->m_nx, nu = ctx->m_nu;
  const int64_t chunk = std::max<int64_t>(1, (int64_t(1) << 30) / per_point_elements(ctx));
  for (int64_t p0 = 0; p0 < P; p0 += chunk) {
    const int64_t np = std::min(chunk, P - p0);
    const int rc = layers_chunk(ctx, np, X + p0 * M * nx, U + p0 * nu, a_self + p0 * M * nx * nx,
                                a_nbr ? a_nbr + p0 * E * nx * nx : nullptr, b + p0 * M * nx * nu, c + p0 * M * nx,
                                f_next ? f_next + p0 * M * nx : nullptr, stream);
    if (rc) return rc;
  }
  return GM_OK;
}
