// Batched training gradients of the dynamics model: loss_gradients
// (training.py:99-150), fp64 like the reference.
//
// The loss is the O-weighted one-step prediction error of a batch of B
// records plus an l2 penalty; the gradient is reverse mode through the
// message-passing step (gnn.py:129-159).  On the device:
//
//   k_tr_edges   e = (x_dst - x_src) / s_x                      (B*E rows)
//   k_mlp_fwd    psi forward, layer inputs kept                 (B*E rows)
//   k_tr_z       z = [(x - mu)/s, sum_in-edges msg, (u - mu_u)/s_u] (B*M rows)
//   k_mlp_fwd    phi forward
//   k_tr_out     pred, residual, per-row loss, dL/d(dv)  (p' = p + dt v'
//                folds the position error into the velocity channel)
//   k_mlp_bwd    phi backward: per-layer deltas, dL/dz
//   k_tr_gmsg    dL/dmsg_e = dL/dagg[dst(e)]
//   k_mlp_bwd    psi backward: per-layer deltas
//   k_wgrad      dW_l = sum_rows delta_l' a_l, db_l = sum_rows delta_l
//                (split over row chunks, partials summed in a fixed order:
//                bitwise reproducible), + 2 lambda p
//   k_tr_loss    sum of the per-row losses (fixed order) + lambda |p|^2
//
// The MLP passes process a tile of 32 rows per CTA with the tile's
// activations in shared memory; weights are read from the context's fp64
// transposed copies (L1/L2 resident).  Offline path: the
// per-step controller never calls it.
#include "common.cuh"

namespace {

constexpr int kRows = 32;   // rows per CTA tile
constexpr int kThr = 256;

struct MlpDev {
  int L;
  int dims[GM_MAX_LAYERS + 1];
  const double* wt[GM_MAX_LAYERS];  // (in, out) transposed
  const double* b[GM_MAX_LAYERS];
  int in_off[GM_MAX_LAYERS];   // column offset of layer l's input in the acts buffer
  int d_off[GM_MAX_LAYERS];    // column offset of layer l's output delta in the delta buffer
  int acts_w, delta_w, maxw;
};

MlpDev mlp_dev(const MlpHost& m) {
  MlpDev d{};
  d.L = m.L;
  int ao = 0, dd = 0, mw = 0;
  for (int l = 0; l <= m.L; ++l) {
    d.dims[l] = m.dims[l];
    mw = std::max(mw, m.dims[l]);
  }
  for (int l = 0; l < m.L; ++l) {
    d.wt[l] = m.d_wt64 + m.w_off[l];
    d.b[l] = m.d_b64 + m.b_off[l];
    d.in_off[l] = ao;
    ao += m.dims[l];
    d.d_off[l] = dd;
    dd += m.dims[l + 1];
  }
  d.acts_w = ao;
  d.delta_w = dd;
  d.maxw = mw;
  return d;
}

// forward over R rows: X (R, D0) -> out (R, DL); acts (R, acts_w) keeps every
// layer's input (post-ReLU activations), so masks are acts > 0
__global__ void __launch_bounds__(kThr) k_mlp_fwd(const MlpDev m, int64_t R, const double* __restrict__ X,
                                                  double* __restrict__ acts, double* __restrict__ out) {
  extern __shared__ double sm[];
  double* a = sm;                       // kRows x maxw
  double* z = sm + kRows * m.maxw;      // kRows x maxw
  const int64_t r0 = (int64_t)blockIdx.x * kRows;
  const int nr = (int)(R - r0 < kRows ? R - r0 : (int64_t)kRows);
  const int D0 = m.dims[0];
  for (int t = threadIdx.x; t < nr * D0; t += blockDim.x) {
    const int r = t / D0, c = t - r * D0;
    a[r * m.maxw + c] = X[(r0 + r) * D0 + c];
  }
  __syncthreads();
  for (int l = 0; l < m.L; ++l) {
    const int in = m.dims[l], ou = m.dims[l + 1];
    const bool last = l == m.L - 1;
    for (int t = threadIdx.x; t < nr * in; t += blockDim.x) {  // keep layer input
      const int r = t / in, c = t - r * in;
      acts[(r0 + r) * m.acts_w + m.in_off[l] + c] = a[r * m.maxw + c];
    }
    const double* wt = m.wt[l];
    for (int t = threadIdx.x; t < nr * ou; t += blockDim.x) {
      const int r = t / ou, o = t - r * ou;
      const double* ar = a + r * m.maxw;
      double s0 = m.b[l][o], s1 = 0.0;
      int i = 0;
      for (; i + 1 < in; i += 2) {
        s0 = fma(wt[(int64_t)i * ou + o], ar[i], s0);
        s1 = fma(wt[(int64_t)(i + 1) * ou + o], ar[i + 1], s1);
      }
      if (i < in) s0 = fma(wt[(int64_t)i * ou + o], ar[i], s0);
      const double v = s0 + s1;
      z[r * m.maxw + o] = last ? v : fmax(v, 0.0);
    }
    __syncthreads();
    double* tmp = a;
    a = z;
    z = tmp;
  }
  const int DL = m.dims[m.L];
  for (int t = threadIdx.x; t < nr * DL; t += blockDim.x) {
    const int r = t / DL, c = t - r * DL;
    out[(r0 + r) * DL + c] = a[r * m.maxw + c];
  }
}

// backward over R rows: g (R, DL) = dL/dout -> delta (R, delta_w) per layer
// (dL/d pre-activation), gin (R, D0) = dL/dinput (may be NULL)
__global__ void __launch_bounds__(kThr) k_mlp_bwd(const MlpDev m, int64_t R, const double* __restrict__ acts,
                                                  const double* __restrict__ g, double* __restrict__ delta,
                                                  double* __restrict__ gin) {
  extern __shared__ double sm[];
  double* d = sm;
  double* e = sm + kRows * m.maxw;
  const int64_t r0 = (int64_t)blockIdx.x * kRows;
  const int nr = (int)(R - r0 < kRows ? R - r0 : (int64_t)kRows);
  const int DL = m.dims[m.L];
  for (int t = threadIdx.x; t < nr * DL; t += blockDim.x) {
    const int r = t / DL, c = t - r * DL;
    d[r * m.maxw + c] = g[(r0 + r) * DL + c];
  }
  __syncthreads();
  for (int l = m.L - 1; l >= 0; --l) {
    const int in = m.dims[l], ou = m.dims[l + 1];
    for (int t = threadIdx.x; t < nr * ou; t += blockDim.x) {
      const int r = t / ou, o = t - r * ou;
      delta[(r0 + r) * m.delta_w + m.d_off[l] + o] = d[r * m.maxw + o];
    }
    if (l == 0 && !gin) break;
    const double* wt = m.wt[l];
    for (int t = threadIdx.x; t < nr * in; t += blockDim.x) {
      const int r = t / in, i = t - r * in;
      const double* dr = d + r * m.maxw;
      const double* wi = wt + (int64_t)i * ou;
      double s0 = 0.0, s1 = 0.0;
      int o = 0;
      for (; o + 1 < ou; o += 2) {
        s0 = fma(wi[o], dr[o], s0);
        s1 = fma(wi[o + 1], dr[o + 1], s1);
      }
      if (o < ou) s0 = fma(wi[o], dr[o], s0);
      double v = s0 + s1;
      // ReLU mask of layer l's input (mlp.py:121-122, strict > 0)
      if (l > 0 && !(acts[(r0 + r) * m.acts_w + m.in_off[l] + i] > 0.0)) v = 0.0;
      e[r * m.maxw + i] = v;
    }
    __syncthreads();
    double* tmp = d;
    d = e;
    e = tmp;
  }
  if (gin) {
    const int D0 = m.dims[0];
    for (int t = threadIdx.x; t < nr * D0; t += blockDim.x) {
      const int r = t / D0, c = t - r * D0;
      gin[(r0 + r) * D0 + c] = d[r * m.maxw + c];
    }
  }
}

// weight / bias gradients of every layer: partial sums over row chunk y
__global__ void k_wgrad(const MlpDev m, int64_t R, int64_t chunk, const double* __restrict__ acts,
                        const double* __restrict__ delta, int nparam, double* __restrict__ part) {
  const int64_t ra = (int64_t)blockIdx.y * chunk, rb = (R < ra + chunk ? R : ra + chunk);
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < nparam; p += gridDim.x * blockDim.x) {
    // parameter p -> (layer, weight (o, i) or bias o), order: all weights of
    // every layer, then all biases (training.py:_params per MLP)
    int rest = p, l = 0, isb = 0, o = 0, i = -1;
    for (l = 0; l < m.L; ++l) {
      const int nw = m.dims[l] * m.dims[l + 1];
      if (rest < nw) break;
      rest -= nw;
    }
    if (l == m.L) {
      isb = 1;
      for (l = 0; l < m.L; ++l) {
        if (rest < m.dims[l + 1]) break;
        rest -= m.dims[l + 1];
      }
      o = rest;
    } else {
      o = rest / m.dims[l];
      i = rest - o * m.dims[l];
    }
    const double* dcol = delta + m.d_off[l] + o;
    const double* acol = acts + m.in_off[l] + (isb ? 0 : i);
    double s0 = 0.0, s1 = 0.0;
    int64_t r = ra;
    for (; r + 1 < rb; r += 2) {
      s0 = fma(dcol[r * m.delta_w], isb ? 1.0 : acol[r * m.acts_w], s0);
      s1 = fma(dcol[(r + 1) * m.delta_w], isb ? 1.0 : acol[(r + 1) * m.acts_w], s1);
    }
    if (r < rb) s0 = fma(dcol[r * m.delta_w], isb ? 1.0 : acol[r * m.acts_w], s0);
    part[(int64_t)blockIdx.y * nparam + p] = s0 + s1;
  }
}

// grads = sum over chunks (ascending) + 2 lambda p; params in the same order
__global__ void k_wgrad_sum(const MlpDev m, int nchunks, int nparam, const double* __restrict__ part,
                            double lam, double* __restrict__ grads) {
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < nparam; p += gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int c = 0; c < nchunks; ++c) s += part[(int64_t)c * nparam + p];
    if (lam > 0.0) {
      int rest = p, l = 0;
      double v;
      for (l = 0; l < m.L; ++l) {
        const int nw = m.dims[l] * m.dims[l + 1];
        if (rest < nw) break;
        rest -= nw;
      }
      if (l < m.L) {
        const int o = rest / m.dims[l], i = rest - o * m.dims[l];
        v = m.wt[l][(int64_t)i * m.dims[l + 1] + o];
      } else {
        for (l = 0; l < m.L; ++l) {
          if (rest < m.dims[l + 1]) break;
          rest -= m.dims[l + 1];
        }
        v = m.b[l][rest];
      }
      s += 2.0 * lam * v;
    }
    grads[p] = s;
  }
}

struct TrArgs {
  int B, M, E, nx, nu, np, nm;
  double dt;
  const int* ptr;
  const int* src;
  const int* dst;
  const double* norm;  // mean_x, s_x, mean_u, s_u
  const double* X;     // (B, M, nx)
  const double* U;     // (B, nu)
  const double* Xn;    // (B, M, nx)
  const double* Wt;    // (M, nx) state weights
};

__global__ void k_tr_edges(const TrArgs a, double* __restrict__ ef) {
  const int64_t tot = (int64_t)a.B * a.E * a.nx;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < tot; t += (int64_t)gridDim.x * blockDim.x) {
    const int k = (int)(t % a.nx);
    const int64_t be = t / a.nx;
    const int e = (int)(be % a.E);
    const int64_t b = be / a.E;
    const double* Xb = a.X + b * a.M * a.nx;
    ef[t] = (Xb[(int64_t)a.dst[e] * a.nx + k] - Xb[(int64_t)a.src[e] * a.nx + k]) / a.norm[a.nx + k];
  }
}

// z = [(x - mu)/s, agg, (u - mu_u)/s_u]; agg sums the in-edge messages of
// node i in edge order (the reference's padded gather-sum, gnn.py:140-143)
__global__ void k_tr_z(const TrArgs a, const double* __restrict__ msg, double* __restrict__ z) {
  const int zw = a.nx + a.nm + a.nu;
  const int64_t tot = (int64_t)a.B * a.M * zw;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < tot; t += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(t % zw);
    const int64_t bi = t / zw;
    const int i = (int)(bi % a.M);
    const int64_t b = bi / a.M;
    double v;
    if (c < a.nx) {
      v = (a.X[bi * a.nx + c] - a.norm[c]) / a.norm[a.nx + c];
    } else if (c < a.nx + a.nm) {
      v = 0.0;
      for (int e = a.ptr[i]; e < a.ptr[i + 1]; ++e) v += msg[(b * a.E + e) * a.nm + (c - a.nx)];
    } else {
      const int k = c - a.nx - a.nm;
      v = (a.U[b * a.nu + k] - a.norm[2 * a.nx + k]) / a.norm[2 * a.nx + a.nu + k];
    }
    z[t] = v;
  }
}

// prediction, residual, per-row weighted loss, g_dv (training.py:126-135)
__global__ void k_tr_out(const TrArgs a, const double* __restrict__ dv, double* __restrict__ rowloss,
                         double* __restrict__ gdv) {
  const int64_t rows = (int64_t)a.B * a.M;
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < rows; r += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(r % a.M);
    const double* x = a.X + r * a.nx;
    const double* xn = a.Xn + r * a.nx;
    const double* w = a.Wt + (int64_t)i * a.nx;
    double lsum = 0.0;
    for (int k = 0; k < a.np; ++k) {
      const double vnew = x[a.np + k] + dv[r * a.np + k];
      const double pnew = x[k] + a.dt * vnew;
      const double rp = pnew - xn[k], rv = vnew - xn[a.np + k];
      lsum += w[k] * rp * rp;
      lsum += w[a.np + k] * rv * rv;
      const double gp = 2.0 * w[k] * rp / a.B, gv = 2.0 * w[a.np + k] * rv / a.B;
      gdv[r * a.np + k] = gv + a.dt * gp;
    }
    rowloss[r] = lsum;
  }
}

__global__ void k_tr_gmsg(const TrArgs a, const double* __restrict__ gz, double* __restrict__ gmsg) {
  const int zw = a.nx + a.nm + a.nu;
  const int64_t tot = (int64_t)a.B * a.E * a.nm;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < tot; t += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(t % a.nm);
    const int64_t be = t / a.nm;
    const int e = (int)(be % a.E);
    const int64_t b = be / a.E;
    gmsg[t] = gz[(b * a.M + a.dst[e]) * zw + a.nx + c];
  }
}

// loss = sum rows (ascending) / B + lambda (|psi|^2 + |phi|^2); one block
__global__ void k_tr_loss(int64_t rows, int B, const double* __restrict__ rowloss, double lam,
                          const MlpDev psi, const MlpDev phi, double* __restrict__ out) {
  __shared__ double red[kThr];
  double s = 0.0;
  // fixed per-thread strided partials, then a fixed tree: reproducible
  for (int64_t r = threadIdx.x; r < rows; r += blockDim.x) s += rowloss[r];
  double pn = 0.0;
  if (lam > 0.0) {
    for (int which = 0; which < 2; ++which) {
      const MlpDev& m = which == 0 ? psi : phi;
      for (int l = 0; l < m.L; ++l) {
        const int nw = m.dims[l] * m.dims[l + 1];
        for (int p = threadIdx.x; p < nw; p += blockDim.x) pn += m.wt[l][p] * m.wt[l][p];
        for (int p = threadIdx.x; p < m.dims[l + 1]; p += blockDim.x) pn += m.b[l][p] * m.b[l][p];
      }
    }
  }
  red[threadIdx.x] = s;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  const double tot = red[0];
  __syncthreads();
  red[threadIdx.x] = pn;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[0] = tot / B + lam * red[0];
}

inline int grid_for(int64_t n, int sm) { return (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 8 * sm)); }

int mlp_params(const MlpHost& m) {
  int n = 0;
  for (int l = 0; l < m.L; ++l) n += m.dims[l] * m.dims[l + 1] + m.dims[l + 1];
  return n;
}

int wgrad(gm_ctx* ctx, const MlpDev& m, int nparam, int64_t R, const double* acts, const double* delta,
          double* part, double lam, double* grads, cudaStream_t st) {
  const int64_t chunk = 4096;
  const int nchunks = (int)std::max<int64_t>(1, (R + chunk - 1) / chunk);
  const unsigned gx = (unsigned)std::max(1, std::min((nparam + 255) / 256, 64));
  if (R > 0) {
    k_wgrad<<<dim3(gx, (unsigned)nchunks), 256, 0, st>>>(m, R, chunk, acts, delta, nparam, part);
    GM_LAUNCH_CHECK(ctx, "k_wgrad");
  }
  k_wgrad_sum<<<gx, 256, 0, st>>>(m, R > 0 ? nchunks : 0, nparam, part, lam, grads);
  GM_LAUNCH_CHECK(ctx, "k_wgrad_sum");
  return GM_OK;
}

}  // namespace

extern "C" {

int gm_param_count(const gm_ctx* ctx) {
  if (!ctx || !ctx->has_model) return -1;
  return mlp_params(ctx->psi) + mlp_params(ctx->phi);
}

int gm_loss_gradients(gm_ctx* ctx, int B, const double* X, const double* U, const double* Xn,
                      const double* weights, double l2_lambda, double* loss, double* grads,
                      void* stream) {
  int rc = gm_need_device(ctx);
  if (rc) return rc;
  if (!ctx->has_model || ctx->M < 1) return gm_fail(ctx, GM_ERR_CONFIG, "model / graph not set");
  if (B < 1) return gm_fail(ctx, GM_ERR_CONFIG, "empty batch");
  if (l2_lambda < 0) return gm_fail(ctx, GM_ERR_CONFIG, "l2_lambda must be nonnegative");
  cudaStream_t st = (cudaStream_t)stream;
  const MlpDev psi = mlp_dev(ctx->psi), phi = mlp_dev(ctx->phi);
  const int nx = ctx->m_nx, nu = ctx->m_nu, nm = ctx->n_m, np_ = ctx->n_p;
  const int64_t M = ctx->M, E = ctx->E;
  const int64_t Re = (int64_t)B * E, Rn = (int64_t)B * M;
  const int npsi = mlp_params(ctx->psi), nphi = mlp_params(ctx->phi);
  const int64_t nchunk = std::max<int64_t>(1, (std::max(Re, Rn) + 4095) / 4096);
  // workspace (fp64): ef, psi acts, msg, psi delta, gmsg | z, phi acts, dv,
  // phi delta, gz, gdv, rowloss | chunk partials
  const int64_t zw = nx + nm + nu;
  const int64_t sizes[] = {Re * nx, Re * psi.acts_w, Re * nm, Re * psi.delta_w, Re * nm,
                           Rn * zw, Rn * phi.acts_w, Rn * np_, Rn * phi.delta_w, Rn * zw, Rn * np_, Rn,
                           nchunk * std::max(npsi, nphi)};
  int64_t total = 0, off[13];
  for (int k = 0; k < 13; ++k) {
    off[k] = total;
    total += (sizes[k] + 31) & ~int64_t(31);
  }
  double* w = (double*)gm_scratch(ctx, sizeof(double) * (size_t)total);
  if (!w) return gm_fail(ctx, GM_ERR_CUDA, "training workspace allocation failed");
  double *ef = w + off[0], *pa = w + off[1], *msg = w + off[2], *pd = w + off[3], *gmsg = w + off[4];
  double *z = w + off[5], *fa = w + off[6], *dv = w + off[7], *fd = w + off[8], *gz = w + off[9];
  double *gdv = w + off[10], *rl = w + off[11], *part = w + off[12];
  TrArgs a{};
  a.B = B;
  a.M = (int)M;
  a.E = (int)E;
  a.nx = nx;
  a.nu = nu;
  a.np = np_;
  a.nm = nm;
  a.dt = ctx->dt;
  a.ptr = ctx->d_ptr;
  a.src = ctx->d_src;
  a.dst = ctx->d_dst;
  a.norm = ctx->d_norm;
  a.X = X;
  a.U = U;
  a.Xn = Xn;
  a.Wt = weights;
  const size_t smp = sizeof(double) * 2 * kRows * psi.maxw, smf = sizeof(double) * 2 * kRows * phi.maxw;
  if (smp > ctx->smem_optin || smf > ctx->smem_optin) return gm_fail(ctx, GM_ERR_CONFIG, "MLP too wide");
  GM_CUDA(ctx, cudaFuncSetAttribute(k_mlp_fwd, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)std::max(smp, smf)));
  GM_CUDA(ctx, cudaFuncSetAttribute(k_mlp_bwd, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)std::max(smp, smf)));
  if (E > 0) {
    k_tr_edges<<<grid_for(Re * nx, ctx->sm_count), 256, 0, st>>>(a, ef);
    GM_LAUNCH_CHECK(ctx, "k_tr_edges");
    k_mlp_fwd<<<(unsigned)((Re + kRows - 1) / kRows), kThr, smp, st>>>(psi, Re, ef, pa, msg);
    GM_LAUNCH_CHECK(ctx, "k_mlp_fwd(psi)");
  }
  k_tr_z<<<grid_for(Rn * zw, ctx->sm_count), 256, 0, st>>>(a, msg, z);
  GM_LAUNCH_CHECK(ctx, "k_tr_z");
  k_mlp_fwd<<<(unsigned)((Rn + kRows - 1) / kRows), kThr, smf, st>>>(phi, Rn, z, fa, dv);
  GM_LAUNCH_CHECK(ctx, "k_mlp_fwd(phi)");
  k_tr_out<<<grid_for(Rn, ctx->sm_count), 256, 0, st>>>(a, dv, rl, gdv);
  GM_LAUNCH_CHECK(ctx, "k_tr_out");
  k_mlp_bwd<<<(unsigned)((Rn + kRows - 1) / kRows), kThr, smf, st>>>(phi, Rn, fa, gdv, fd, E > 0 ? gz : nullptr);
  GM_LAUNCH_CHECK(ctx, "k_mlp_bwd(phi)");
  // gradient layout (training.py:_params): psi W, psi b, phi W, phi b
  if (E > 0) {
    k_tr_gmsg<<<grid_for(Re * nm, ctx->sm_count), 256, 0, st>>>(a, gz, gmsg);
    GM_LAUNCH_CHECK(ctx, "k_tr_gmsg");
    k_mlp_bwd<<<(unsigned)((Re + kRows - 1) / kRows), kThr, smp, st>>>(psi, Re, pa, gmsg, pd, nullptr);
    GM_LAUNCH_CHECK(ctx, "k_mlp_bwd(psi)");
  }
  rc = wgrad(ctx, psi, npsi, Re, pa, pd, part, l2_lambda, grads, st);
  if (rc) return rc;
  rc = wgrad(ctx, phi, nphi, Rn, fa, fd, part, l2_lambda, grads + npsi, st);
  if (rc) return rc;
  k_tr_loss<<<1, kThr, 0, st>>>(Rn, B, rl, l2_lambda, psi, phi, loss);
  GM_LAUNCH_CHECK(ctx, "k_tr_loss");
  return GM_OK;
}

}  // extern "C"
