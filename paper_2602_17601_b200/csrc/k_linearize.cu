// K-LIN: fused GNN forward + exact per-node linearisation (stage 1).
//
// Reference: _linearize_batch (gnn.py:237-298), _forward_parts
// (gnn.py:129-150), mlp_jacobian (mlp.py:132-145), step_array
// (gnn.py:153-159).
//
// One CTA owns a tile of TN consecutive nodes at one linearisation point p
// (p = instance*K + stage).  Because edges are stored node-major, the tile's
// in-edges are one contiguous range [ptr[i0], ptr[i1]) and every edge belongs
// to exactly one tile -- the whole stage is computed with no inter-CTA
// traffic and no intermediate arrays in HBM:
//
//   1. edge features e = (x_dst - x_src)/s_x, psi forward (fp64)      gnn.py:137-140
//   2. messages summed per node in edge order (fp64)                  gnn.py:141-143
//   3. phi forward on z = [(x-mu)/s, agg, (u-mu_u)/s_u] (fp64)         gnn.py:146-149
//   4. f = step_array(x, u) (fp64)                                      gnn.py:153-159
//   5. J_phi (n_p x nin) from the output side, ReLU masks of step 3    mlp.py:138-145
//   6. psi VJP: seed J_m[dst] (n_p x n_m) pushed back through psi with the
//      edge's own masks -> P_e = J_m J_psi (n_p x nx)                  gnn.py:259-266
//      (n_p rows instead of the reference's n_m-row J_psi: ~n_m/n_p less work)
//   7. assembly of a_self, a_nbr, b and the fp64 offset c              gnn.py:272-297
//
// Precision: the forward passes run in fp64 so every ReLU mask decision
// matches the fp64 reference (an fp32 pre-activation near 0 would flip a mask
// and change a Jacobian block by O(1)); the Jacobian chains run in fp32.  c is
// evaluated in fp64 from the *stored* fp32 blocks, so the affine model is exact
// at the linearisation point to fp64 round-off.
#include <algorithm>

#include "common.cuh"

int launch_linearize_layers(gm_ctx* ctx, int64_t P, const double* X, const double* U, float* a_self,
                            float* a_nbr, float* b, double* c, double* f_next, void* stream);

namespace {

constexpr int kLinThreads = 256;

struct LinPlan {
  int TN, EM, nin, wpsi, wphi, hpsi, hphi;
  size_t o_ef, o_z, o_p64a, o_p64b, o_f, o_mpsi, o_mphi, o_p32a, o_p32b, o_jphi, o_P, o_bself,
      o_bnbr, o_bb, o_bc, total;
};

__host__ __device__ inline size_t al16(size_t x) { return (x + 15) & ~size_t(15); }
// odd leading dimension for activation rows: rows read by different row
// groups of a warp then fall into different banks
__host__ __device__ inline int pld(int w) { return w | 1; }

__host__ __device__ inline LinPlan make_plan(int TN, int EM, int nx, int nu, int n_p, int nin,
                                             int wpsi, int wphi, int hpsi, int hphi) {
  LinPlan p{};
  p.TN = TN;
  p.EM = EM;
  p.nin = nin;
  p.wpsi = wpsi;
  p.wphi = wphi;
  p.hpsi = hpsi;
  p.hphi = hphi;
  size_t o = 0;
  const size_t f64ping = (size_t)max(EM * pld(wpsi), TN * pld(wphi));
  const size_t f32ping = (size_t)max(TN * n_p * pld(wphi), EM * n_p * pld(wpsi));
  p.o_ef = o;    o = al16(o + sizeof(double) * EM * nx);
  p.o_z = o;     o = al16(o + sizeof(double) * TN * nin);
  p.o_p64a = o;  o = al16(o + sizeof(double) * f64ping);
  p.o_p64b = o;  o = al16(o + sizeof(double) * f64ping);
  p.o_f = o;     o = al16(o + sizeof(double) * TN * nx);
  p.o_mpsi = o;  o = al16(o + (size_t)EM * hpsi);
  p.o_mphi = o;  o = al16(o + (size_t)TN * hphi);
  p.o_p32a = o;  o = al16(o + sizeof(float) * f32ping);
  p.o_p32b = o;  o = al16(o + sizeof(float) * f32ping);
  p.o_jphi = o;  o = al16(o + sizeof(float) * TN * n_p * nin);
  p.o_P = o;     o = al16(o + sizeof(float) * EM * n_p * nx);
  p.o_bself = o; o = al16(o + sizeof(float) * TN * nx * nx);
  p.o_bnbr = o;  o = al16(o + sizeof(float) * EM * nx * nx);
  p.o_bb = o;    o = al16(o + sizeof(float) * TN * nx * nu);
  p.o_bc = o;    o = al16(o + sizeof(double) * TN * nx);
  p.total = o;
  return p;
}

struct LinArgs {
  int M, E, nx, nu, n_p, n_m;
  double dt;
  const int* ptr;
  const int* src;
  const int* dst;
  const double* norm;
  MlpView psi, phi;
  const double* X;
  const double* U;
  float* a_self;
  float* a_nbr;
  float* b;
  double* c;
  double* f_next;
  int lo, hi, tiles, jac;
  LinPlan plan;
};

// Register-tiled micro-GEMM shared by every layer:
//   out[r][c] = epi(r, c, sum_k in[r][k] W[k][c]),  W row-major (K, N).
// Each thread owns RT x CT outputs: per k it loads RT inputs (warp
// broadcasts: neighbouring threads share rows) and CT weights (contiguous,
// vector loads through L1), i.e. RT*CT FMAs per RT + CT loads.  N % CT == 0.
template <typename T, int RT, int CT, typename Epi>
__device__ __forceinline__ void tile_gemm(const T* in, int ldi, int R, int K, const T* __restrict__ W, int N,
                                          Epi epi) {
  const int CG = N / CT, RG = (R + RT - 1) / RT;
  for (int idx = threadIdx.x; idx < RG * CG; idx += blockDim.x) {
    const int c0 = (idx % CG) * CT;
    const int r0 = (idx / CG) * RT;
    const T* x[RT];
#pragma unroll
    for (int t = 0; t < RT; ++t) x[t] = in + (size_t)min(r0 + t, R - 1) * ldi;
    T acc[RT][CT];
#pragma unroll
    for (int t = 0; t < RT; ++t)
#pragma unroll
      for (int u = 0; u < CT; ++u) acc[t][u] = T(0);
    const T* wp = W + c0;
#pragma unroll 4
    for (int k = 0; k < K; ++k) {
      T w[CT];
#pragma unroll
      for (int u = 0; u < CT; ++u) w[u] = __ldg(wp + u);
      wp += N;
#pragma unroll
      for (int t = 0; t < RT; ++t) {
        const T xv = x[t][k];
#pragma unroll
        for (int u = 0; u < CT; ++u) acc[t][u] = fma(xv, w[u], acc[t][u]);
      }
    }
#pragma unroll
    for (int t = 0; t < RT; ++t)
      if (r0 + t < R)
#pragma unroll
        for (int u = 0; u < CT; ++u) epi(r0 + t, c0 + u, acc[t][u]);
  }
}

// Largest micro-tile that still gives every thread of the CTA an output
// block (the per-CTA row counts are small: 32 nodes, ~64 edges, x n_p).
template <typename T, typename Epi>
__device__ __forceinline__ void gemm_dispatch(const T* in, int ldi, int R, int K, const T* __restrict__ W, int N,
                                              Epi epi) {
  const int nt = blockDim.x;
  auto items = [&](int rt, int ct) { return ((R + rt - 1) / rt) * (N / ct); };
  constexpr bool wide = sizeof(T) == 4;  // fp64 tiles capped at 2 x 4 (register budget)
  if (wide && N % 8 == 0 && items(4, 8) >= nt)
    tile_gemm<T, 4, 8>(in, ldi, R, K, W, N, epi);
  else if (wide && N % 4 == 0 && items(4, 4) >= nt)
    tile_gemm<T, 4, 4>(in, ldi, R, K, W, N, epi);
  else if (N % 4 == 0 && items(2, 4) >= nt)
    tile_gemm<T, 2, 4>(in, ldi, R, K, W, N, epi);
  else if (N % 2 == 0 && items(2, 2) >= nt)
    tile_gemm<T, 2, 2>(in, ldi, R, K, W, N, epi);
  else if (N % 2 == 0)
    tile_gemm<T, 1, 2>(in, ldi, R, K, W, N, epi);
  else
    tile_gemm<T, 1, 1>(in, ldi, R, K, W, N, epi);
}

// out[r][j] = act(sum_k in[r][k] W[j][k] + bias[j]); Wt is (K, Nout), fp64.
__device__ void fwd_layer(const double* in, int ldi, int R, int K, const double* __restrict__ Wt,
                          const double* __restrict__ bias, int Nout, double* out, int ldo,
                          uint8_t* mask, int ldm, bool relu) {
  gemm_dispatch<double>(in, ldi, R, K, Wt, Nout, [&](int r, int j, double s) {
    s += __ldg(bias + j);
    if (relu) {
      const bool m = s > 0.0;  // strict: derivative 0 at the kink (mlp.py:143)
      mask[(size_t)r * ldm + j] = m;
      out[(size_t)r * ldo + j] = m ? s : 0.0;
    } else {
      out[(size_t)r * ldo + j] = s;
    }
  });
}

// out[r][kk] = (sum_j in[r][j] W[j][kk]) * mask[r / rows_per][kk]; W is (J, KK)
// row-major (reference layout), fp32.
__device__ void bwd_layer(const float* in, int ldi, int R, int J, const float* __restrict__ W,
                          int KK, float* out, int ldo, const uint8_t* mask, int ldm, int rows_per) {
  gemm_dispatch<float>(in, ldi, R, J, W, KK, [&](int r, int kk, float v) {
    if (mask && !mask[(size_t)(r / rows_per) * ldm + kk]) v = 0.f;
    out[(size_t)r * ldo + kk] = v;
  });
}

__device__ inline int mask_off(const MlpView& m, int l) {  // column offset of hidden layer l
  int o = 0;
  for (int q = 0; q < l; ++q) o += m.dims[q + 1];
  return o;
}

__global__ void __launch_bounds__(kLinThreads, 3) k_linearize(const LinArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const LinPlan& pl = a.plan;
  const int nx = a.nx, nu = a.nu, n_p = a.n_p, n_m = a.n_m, nin = pl.nin;
  const int64_t p = blockIdx.x / a.tiles;
  const int tile = blockIdx.x % a.tiles;
  const int i0 = a.lo + tile * pl.TN;
  const int i1 = min(i0 + pl.TN, a.hi);
  const int nN = i1 - i0;
  const int e0 = a.ptr[i0], e1 = a.ptr[i1];
  const int nE = e1 - e0;
  const double* Xp = a.X + p * (int64_t)a.M * nx;
  const double* Up = a.U + p * nu;
  const double* smean = a.norm;
  const double* sscale = a.norm + nx;
  const double* umean = a.norm + 2 * nx;
  const double* uscale = a.norm + 2 * nx + nu;

  double* ef = (double*)(smem + pl.o_ef);
  double* z = (double*)(smem + pl.o_z);
  double* pa = (double*)(smem + pl.o_p64a);
  double* pb = (double*)(smem + pl.o_p64b);
  double* fb = (double*)(smem + pl.o_f);
  uint8_t* mpsi = smem + pl.o_mpsi;
  uint8_t* mphi = smem + pl.o_mphi;
  const int tid = threadIdx.x, nt = blockDim.x;

  // 1. edge features and the state / input parts of z (gnn.py:137-146)
  for (int t = tid; t < nE * nx; t += nt) {
    const int el = t / nx, k = t - el * nx;
    const int e = e0 + el;
    const int i = a.dst[e], j = a.src[e];
    ef[t] = (Xp[(int64_t)i * nx + k] - Xp[(int64_t)j * nx + k]) / sscale[k];
  }
  for (int t = tid; t < nN * nin; t += nt) {
    const int li = t / nin, k = t - li * nin;
    if (k < nx)
      z[t] = (Xp[(int64_t)(i0 + li) * nx + k] - smean[k]) / sscale[k];
    else if (k >= nx + n_m)
      z[t] = (Up[k - nx - n_m] - umean[k - nx - n_m]) / uscale[k - nx - n_m];
  }
  __syncthreads();

  // 2. psi forward over the tile's edges, keep hidden ReLU masks
  const double* msg = nullptr;
  int ldmsg = 0;
  if (nE > 0) {
    const double* cur = ef;
    int ldc = nx;
    for (int l = 0; l < a.psi.L; ++l) {
      double* out = (l & 1) ? pb : pa;
      const bool relu = l < a.psi.L - 1;
      fwd_layer(cur, ldc, nE, a.psi.dims[l], a.psi.wt64[l], a.psi.b64[l], a.psi.dims[l + 1], out,
                pld(a.psi.dims[l + 1]), relu ? mpsi + mask_off(a.psi, l) : nullptr, pl.hpsi, relu);
      __syncthreads();
      cur = out;
      ldc = pld(a.psi.dims[l + 1]);
    }
    msg = cur;
    ldmsg = ldc;
  }
  // messages summed per node in canonical edge order (gnn.py:141-143)
  for (int t = tid; t < nN * n_m; t += nt) {
    const int li = t / n_m, m = t - li * n_m;
    double s = 0.0;
    for (int e = a.ptr[i0 + li]; e < a.ptr[i0 + li + 1]; ++e) s += msg[(size_t)(e - e0) * ldmsg + m];
    z[li * nin + nx + m] = s;
  }
  __syncthreads();

  // 3. phi forward (gnn.py:149)
  const double* dv;
  {
    const double* cur = z;
    int ldc = nin;
    for (int l = 0; l < a.phi.L; ++l) {
      double* out = (l & 1) ? pb : pa;
      const bool relu = l < a.phi.L - 1;
      fwd_layer(cur, ldc, nN, a.phi.dims[l], a.phi.wt64[l], a.phi.b64[l], a.phi.dims[l + 1], out,
                pld(a.phi.dims[l + 1]), relu ? mphi + mask_off(a.phi, l) : nullptr, pl.hphi, relu);
      __syncthreads();
      cur = out;
      ldc = pld(a.phi.dims[l + 1]);
    }
    dv = cur;  // (nN, n_p), leading dimension ldv
  }
  const int ldv = pld(n_p);
  {
  }

  // 4. f = step_array: v' = v + dv, p' = p + dt v' (gnn.py:157-158)
  for (int t = tid; t < nN * nx; t += nt) {
    const int li = t / nx, k = t - li * nx;
    const double* xi = Xp + (int64_t)(i0 + li) * nx;
    double val;
    if (k >= n_p) {
      val = xi[k] + dv[li * ldv + (k - n_p)];
    } else {
      const double v1 = xi[n_p + k] + dv[li * ldv + k];
      val = xi[k] + a.dt * v1;
    }
    fb[t] = val;
    if (a.f_next) a.f_next[(p * a.M + i0 + li) * nx + k] = val;
  }
  if (!a.jac) return;
  __syncthreads();

  float* qa = (float*)(smem + pl.o_p32a);
  float* qb = (float*)(smem + pl.o_p32b);
  float* jphi = (float*)(smem + pl.o_jphi);
  float* Pe = (float*)(smem + pl.o_P);

  // 5. J_phi = W_L D_{L-1} W_{L-1} ... D_0 W_0 accumulated from the output side
  {
    const int L = a.phi.L;
    const int R = nN * n_p;
    if (L == 1) {
      for (int t = tid; t < R * nin; t += nt) {
        const int r = t / nin, k = t - r * nin;
        jphi[t] = a.phi.w32[0][(r % n_p) * nin + k];
      }
    } else {
      const int wl = a.phi.dims[L - 1];
      const int mo = mask_off(a.phi, L - 2);
      for (int t = tid; t < R * wl; t += nt) {
        const int r = t / wl, j = t - r * wl;
        const int li = r / n_p, ro = r - li * n_p;
        qa[r * pld(wl) + j] = mphi[li * pl.hphi + mo + j] ? a.phi.w32[L - 1][ro * wl + j] : 0.f;
      }
      __syncthreads();
      const float* cur = qa;
      int ldc = pld(wl);
      for (int l = L - 2; l >= 0; --l) {
        const int KK = a.phi.dims[l];
        float* out = (l == 0) ? jphi : ((cur == qa) ? qb : qa);
        const uint8_t* mk = (l >= 1) ? mphi + mask_off(a.phi, l - 1) : nullptr;
        bwd_layer(cur, ldc, R, a.phi.dims[l + 1], a.phi.w32[l], KK, out, l == 0 ? KK : pld(KK), mk, pl.hphi,
                  n_p);
        __syncthreads();
        cur = out;
        ldc = pld(KK);
      }
    }
  }
  __syncthreads();

  // 6. psi VJP with seed J_m[dst] (gnn.py:259-266 reformulated)
  if (nE > 0) {
    const int L = a.psi.L;
    const int R = nE * n_p;
    for (int t = tid; t < R * n_m; t += nt) {
      const int r = t / n_m, m = t - r * n_m;
      const int el = r / n_p, ro = r - el * n_p;
      const int li = a.dst[e0 + el] - i0;
      qa[r * pld(n_m) + m] = jphi[(li * n_p + ro) * nin + nx + m];
    }
    __syncthreads();
    const float* cur = qa;
    int ldc = pld(n_m);
    for (int l = L - 1; l >= 0; --l) {
      const int KK = a.psi.dims[l];
      float* out = (l == 0) ? Pe : ((cur == qa) ? qb : qa);
      const uint8_t* mk = (l >= 1) ? mpsi + mask_off(a.psi, l - 1) : nullptr;
      bwd_layer(cur, ldc, R, a.psi.dims[l + 1], a.psi.w32[l], KK, out, l == 0 ? KK : pld(KK), mk, pl.hpsi,
                n_p);
      __syncthreads();
      cur = out;
      ldc = pld(KK);
    }
  }

  // 7. assembly (gnn.py:272-288)
  float* bs = (float*)(smem + pl.o_bself);
  float* bn = (float*)(smem + pl.o_bnbr);
  float* bbk = (float*)(smem + pl.o_bb);
  double* bc = (double*)(smem + pl.o_bc);
  const float dtf = (float)a.dt;
  for (int t = tid; t < nN * n_p * nx; t += nt) {
    const int li = t / (n_p * nx);
    const int r = (t / nx) % n_p, cc = t % nx;
    float s = 0.f;
    for (int e = a.ptr[i0 + li]; e < a.ptr[i0 + li + 1]; ++e)
      s += Pe[((e - e0) * n_p + r) * nx + cc];
    const float inv_sx = (float)(1.0 / sscale[cc]);
    const float dvdx = (jphi[(li * n_p + r) * nin + cc] + s) * inv_sx + (cc == n_p + r ? 1.f : 0.f);
    float* blk = bs + li * nx * nx;
    blk[r * nx + cc] = (r == cc ? 1.f : 0.f) + dtf * dvdx;
    blk[(n_p + r) * nx + cc] = dvdx;
  }
  for (int t = tid; t < nE * n_p * nx; t += nt) {
    const int el = t / (n_p * nx);
    const int r = (t / nx) % n_p, cc = t % nx;
    const float inv_sx = (float)(1.0 / sscale[cc]);
    const float jv = -Pe[(el * n_p + r) * nx + cc] * inv_sx;
    float* blk = bn + el * nx * nx;
    blk[r * nx + cc] = dtf * jv;
    blk[(n_p + r) * nx + cc] = jv;
  }
  for (int t = tid; t < nN * n_p * nu; t += nt) {
    const int li = t / (n_p * nu);
    const int r = (t / nu) % n_p, cu = t % nu;
    const float inv_su = (float)(1.0 / uscale[cu]);
    const float jv = jphi[(li * n_p + r) * nin + nx + n_m + cu] * inv_su;
    float* blk = bbk + li * nx * nu;
    blk[r * nu + cu] = dtf * jv;
    blk[(n_p + r) * nu + cu] = jv;
  }
  __syncthreads();
  // affine offset in fp64 from the stored fp32 blocks (gnn.py:291-297)
  for (int t = tid; t < nN * nx; t += nt) {
    const int li = t / nx, r = t - li * nx;
    const int i = i0 + li;
    const double* xi = Xp + (int64_t)i * nx;
    const float* As = bs + li * nx * nx + r * nx;
    double s = fb[t];
    for (int k = 0; k < nx; ++k) s -= (double)As[k] * xi[k];
    const float* Bs = bbk + li * nx * nu + r * nu;
    for (int k = 0; k < nu; ++k) s -= (double)Bs[k] * Up[k];
    for (int e = a.ptr[i]; e < a.ptr[i + 1]; ++e) {
      const float* An = bn + (e - e0) * nx * nx + r * nx;
      const double* xj = Xp + (int64_t)a.src[e] * nx;
      for (int k = 0; k < nx; ++k) s -= (double)An[k] * xj[k];
    }
    bc[t] = s;
  }
  __syncthreads();
  // coalesced write-out of the tile's contiguous block ranges
  {
    const int64_t nn2 = (int64_t)nx * nx;
    float* g_self = a.a_self + (p * a.M + i0) * nn2;
    for (int t = tid; t < nN * nn2; t += nt) g_self[t] = bs[t];
    float* g_nbr = a.a_nbr + (p * a.E + e0) * nn2;
    for (int t = tid; t < nE * nn2; t += nt) g_nbr[t] = bn[t];
    float* g_b = a.b + (p * a.M + i0) * (int64_t)nx * nu;
    for (int t = tid; t < nN * nx * nu; t += nt) g_b[t] = bbk[t];
    double* g_c = a.c + (p * a.M + i0) * (int64_t)nx;
    for (int t = tid; t < nN * nx; t += nt) g_c[t] = bc[t];
  }
}

int launch_linearize(gm_ctx* ctx, int64_t P, const double* X, const double* U, float* a_self,
                     float* a_nbr, float* b, double* c, double* f_next, int jac, void* stream) {
  int rc = gm_need_device(ctx);
  if (rc) return rc;
  if (!ctx->has_model) return gm_fail(ctx, GM_ERR_CONFIG, "model not set");
  if (ctx->M < 1) return gm_fail(ctx, GM_ERR_CONFIG, "graph not set");
  if (P < 0) return gm_fail(ctx, GM_ERR_CONFIG, "negative point count");
  const int64_t lo = ctx->node_lo, hi = gm_node_hi(ctx);
  if (P == 0 || hi <= lo) return GM_OK;
  // Jacobians beyond a few thousand node points: the layer-wise path
  // (k_linearize_layers.cu; with the fused per-row MLP chains of the
  // reference architecture it beats the per-tile kernel from ~8 K node points:
  // M = 600 0.12 vs 0.16 ms, M = 1000 0.21 vs 0.25 ms, M = 1e4 1.0 vs 2.1 ms at
  // N = 20; the per-layer GEMM form only from ~200 K); the fused per-tile
  // kernel below serves small problems, step_array (no Jacobian) and a
  // single-layer phi
  const int64_t kLayerMinRows = gm_lin_chains(ctx) ? 8000 : 200000;
  const bool big = P * (hi - lo) >= kLayerMinRows;
  if (jac && ctx->phi.L >= 2 && ctx->psi.L >= 1 && (ctx->lin_mode >= 2 || (ctx->lin_mode == 0 && big)))
    return launch_linearize_layers(ctx, P, X, U, a_self, a_nbr, b, c, f_next, stream);
  const int nx = ctx->m_nx, nu = ctx->m_nu, n_p = ctx->n_p;
  const int nin = ctx->phi.dims[0];
  const int wpsi = ctx->psi.max_width(), wphi = ctx->phi.max_width();
  const int hpsi = ctx->psi.hidden_sum(), hphi = ctx->phi.hidden_sum();
  const int dmax = (int)ctx->dmax;
  // largest node tile whose working set keeps >= 2 CTAs per SM resident
  const size_t budget = std::min<size_t>(ctx->smem_optin, 110 * 1024);
  LinPlan plan{};
  int TN = 32;
  for (; TN >= 1; TN >>= 1) {
    plan = make_plan(TN, TN * dmax, nx, nu, n_p, nin, wpsi, wphi, hpsi, hphi);
    if (plan.total <= budget) break;
  }
  if (TN < 1) {
    plan = make_plan(1, dmax, nx, nu, n_p, nin, wpsi, wphi, hpsi, hphi);
    if (plan.total > ctx->smem_optin)
      return gm_fail(ctx, GM_ERR_CONFIG, "model too wide for the on-chip linearisation tile");
    TN = 1;
  }
  LinArgs a{};
  a.M = (int)ctx->M;
  a.E = (int)ctx->E;
  a.nx = nx;
  a.nu = nu;
  a.n_p = n_p;
  a.n_m = ctx->n_m;
  a.dt = ctx->dt;
  a.ptr = ctx->d_ptr;
  a.src = ctx->d_src;
  a.dst = ctx->d_dst;
  a.norm = ctx->d_norm;
  a.psi = ctx->psi.view();
  a.phi = ctx->phi.view();
  a.X = X;
  a.U = U;
  a.a_self = a_self;
  a.a_nbr = a_nbr;
  a.b = b;
  a.c = c;
  a.f_next = f_next;
  a.lo = (int)lo;
  a.hi = (int)hi;
  a.tiles = gm_ceil_div(hi - lo, TN);
  a.jac = jac;
  a.plan = plan;
  const int64_t blocks = P * a.tiles;
  if (blocks >= (int64_t(1) << 31)) return gm_fail(ctx, GM_ERR_CONFIG, "too many linearisation tiles");
  GM_CUDA(ctx, cudaFuncSetAttribute(k_linearize, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)plan.total));
  k_linearize<<<(unsigned)blocks, kLinThreads, plan.total, (cudaStream_t)stream>>>(a);
  GM_LAUNCH_CHECK(ctx, "k_linearize");
  return GM_OK;
}

}  // namespace

extern "C" {

int gm_linearize(gm_ctx* ctx, int64_t P, const double* X, const double* U, float* a_self,
                 float* a_nbr, float* b, double* c, double* f_next, void* stream) {
  if (!a_self || !b || !c || (ctx && ctx->E > 0 && !a_nbr))
    return gm_fail(ctx, GM_ERR_CONFIG, "null output buffer");
  return launch_linearize(ctx, P, X, U, a_self, a_nbr, b, c, f_next, 1, stream);
}

int gm_set_linearize_mode(gm_ctx* ctx, int mode) {
  if (!ctx) return GM_ERR_CONFIG;
  if (mode < 0 || mode > 4) return gm_fail(ctx, GM_ERR_CONFIG, "linearize mode must be 0 .. 4");
  ctx->lin_mode = mode;
  return GM_OK;
}

int gm_step(gm_ctx* ctx, int64_t P, const double* X, const double* U, double* f, void* stream) {
  if (!f) return gm_fail(ctx, GM_ERR_CONFIG, "null output buffer");
  return launch_linearize(ctx, P, X, U, nullptr, nullptr, nullptr, nullptr, f, 0, stream);
}

}  // extern "C"
