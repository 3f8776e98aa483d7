// K-QP: batched dense interior-point QP solver in fp64, one CTA per problem.
//
// Reference: solve_qp (qpsolver.py:112-235), _residuals (:90-97),
// _split_single_nonzero_rows (:100-109), _max_step (:238-243).  Same
// algorithm step by step -- Mehrotra predictor-corrector on
//   2Hu + g + C'lam = 0,  Cu + s = d,  lam_i s_i = mu
// with the reference's scale references, stopping and infeasibility tests,
// best-iterate bookkeeping, escalating Cholesky regularisation and status
// semantics -- so statuses and iteration counts match the reference.
//
// B200 mapping: the whole IPM loop runs on the device inside one CTA per QP
// (no host round trips); the Schur matrix K lives in shared memory
// (column-major lower triangle, odd leading dimension => conflict-free row and
// column walks), single-nonzero constraint rows are never touched densely
// (diagonal Schur contribution + a per-column row list), general rows are
// staged once into shared memory.  Batches of independent QPs (cfg4) fill the
// GPU with one CTA each.
#include <algorithm>
#include <cfloat>

#include "common.cuh"

namespace {

constexpr int kQpThreads = 512;
constexpr int kQpWarps = kQpThreads / 32;

struct QpArgs {
  int n, m, ldk, k_smem;
  size_t smem_bytes;
  const double* H;
  const double* g;
  const double* C;
  const double* d;
  const double* warm;
  double tol, reg, tau;
  int max_it;
  double* u_out;
  double* lam_out;
  int* status;
  int* iters;
  double* resid;
  double* gws;       // per-instance global workspace (K and/or Cg when they do not fit)
  int64_t gws_stride;
};

struct QpLayout {
  size_t o_vec, o_ints, o_cg, o_k, total;
  int nvec_n, nvec_m;
};

__host__ __device__ inline size_t qal(size_t x) { return (x + 15) & ~size_t(15); }

// n-vectors: g, u, hu, rdual, rhs, du, ubest, dinv, ctl          (9)
// m-vectors: d, s, lam, cu, rpri, t, dl, ds, dla, dsa, w, lbest,  (13)
//            rval
__host__ __device__ inline QpLayout qp_layout(int n, int m, int ldk, int ng, bool k_smem,
                                              bool cg_smem) {
  QpLayout L{};
  L.nvec_n = 9;
  L.nvec_m = 13;
  size_t o = 0;
  L.o_vec = o;
  o = qal(o + sizeof(double) * ((size_t)L.nvec_n * n + (size_t)L.nvec_m * m + 64));
  L.o_ints = o;  // rcol(m) gpos(m) grow(m) colptr(n+1) colrows(m)
  o = qal(o + sizeof(int) * ((size_t)4 * m + n + 1 + 8));
  L.o_k = o;
  if (k_smem) o = qal(o + sizeof(double) * (size_t)ldk * n);
  L.o_cg = o;
  if (cg_smem) o = qal(o + sizeof(double) * (size_t)ng * n);
  L.total = o;
  return L;
}

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ double warp_min(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// block-wide reductions; every thread gets the result.  op: 0 max, 1 min, 2 sum
template <int OP>
__device__ double block_reduce(double v, double* red) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  v = OP == 0 ? warp_max(v) : (OP == 1 ? warp_min(v) : warp_sum(v));
  __syncthreads();  // protect red[] from the previous use
  if (lane == 0) red[wid] = v;
  __syncthreads();
  double r = red[0];
  for (int w = 1; w < kQpWarps; ++w) r = OP == 0 ? fmax(r, red[w]) : (OP == 1 ? fmin(r, red[w]) : r + red[w]);
  return r;
}

// Right-looking Cholesky of the lower triangle of K (column-major, leading
// dimension ldk) in place; returns false on a non-positive / NaN pivot
// (LAPACK potrf's failure condition).  On success column j holds L[:, j] and
// dinv[j] = 1 / L[j][j].
__device__ bool chol_factor(double* K, int n, int ldk, double* dinv, double* red) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int j = 0; j < n; ++j) {
    const double piv = K[(size_t)j * ldk + j];
    if (!(piv > 0.0)) {
      __syncthreads();
      return false;
    }
    const double ipiv = 1.0 / piv;
    const double* colj = K + (size_t)j * ldk;
    for (int c = j + 1 + wid; c < n; c += kQpWarps) {
      const double f = colj[c] * ipiv;
      double* colc = K + (size_t)c * ldk;
      for (int r = c + lane; r < n; r += 32) colc[r] = fma(-colj[r], f, colc[r]);
    }
    __syncthreads();
  }
  // scale columns: L[r][j] = Kt[r][j] / sqrt(piv_j)
  for (int j = wid; j < n; j += kQpWarps) {
    double* colj = K + (size_t)j * ldk;
    const double piv = colj[j];
    const double ljj = sqrt(piv);
    const double inv = 1.0 / ljj;
    for (int r = j + 1 + lane; r < n; r += 32) colj[r] *= inv;
    __syncwarp();
    if (lane == 0) {
      colj[j] = ljj;
      dinv[j] = inv;
    }
  }
  __syncthreads();
  return true;
}

// x = K^{-1} b with K = L L' (L from chol_factor); b, x shared vectors (may alias).
// Column-oriented substitution by warp 0; the other warps wait at the barrier.
__device__ void chol_solve(const double* K, int n, int ldk, const double* dinv, const double* b,
                           double* x) {
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    for (int r = lane; r < n; r += 32) x[r] = b[r];
    __syncwarp();
    for (int j = 0; j < n; ++j) {  // L y = b
      const double yj = x[j] * dinv[j];
      const double* colj = K + (size_t)j * ldk;
      for (int r = j + 1 + lane; r < n; r += 32) x[r] = fma(-colj[r], yj, x[r]);
      __syncwarp();
      if (lane == 0) x[j] = yj;
      __syncwarp();
    }
    for (int j = n - 1; j >= 0; --j) {  // L' x = y
      const double xj = x[j] * dinv[j];
      for (int r = lane; r < j; r += 32) x[r] = fma(-K[(size_t)r * ldk + j], xj, x[r]);
      __syncwarp();
      if (lane == 0) x[j] = xj;
      __syncwarp();
    }
  }
  __syncthreads();
}

__global__ void __launch_bounds__(kQpThreads) k_solve_qp(const QpArgs A) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ double red[kQpWarps];
  __shared__ int sh_int[4];
  const int n = A.n, m = A.m, ldk = A.ldk;
  const int64_t bi = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nt = blockDim.x;
  const double* H = A.H + bi * (int64_t)n * n;
  const double* gg = A.g + bi * (int64_t)n;
  const double* C = A.C + bi * (int64_t)m * n;
  const double* dd = A.d + bi * (int64_t)m;
  double* gws = A.gws ? A.gws + bi * A.gws_stride : nullptr;

  // ---- classify rows once (qpsolver.py:100-109): single-nonzero vs general
  // first pass into registers of the layout-independent arrays
  const QpLayout L0 = qp_layout(n, m, ldk, 0, false, false);
  double* vec = (double*)(smem + L0.o_vec);
  double* v_g = vec;
  double* v_u = v_g + n;
  double* v_hu = v_u + n;
  double* v_rd = v_hu + n;
  double* v_rhs = v_rd + n;
  double* v_du = v_rhs + n;
  double* v_ub = v_du + n;
  double* v_dinv = v_ub + n;
  double* v_ctl = v_dinv + n;
  double* v_d = v_ctl + n;
  double* v_s = v_d + m;
  double* v_lam = v_s + m;
  double* v_cu = v_lam + m;
  double* v_rp = v_cu + m;
  double* v_t = v_rp + m;
  double* v_dl = v_t + m;
  double* v_ds = v_dl + m;
  double* v_dla = v_ds + m;
  double* v_dsa = v_dla + m;
  double* v_w = v_dsa + m;
  double* v_lb = v_w + m;
  double* v_rval = v_lb + m;
  int* rcol = (int*)(smem + L0.o_ints);  // col of a single row, -1 for general rows
  int* gpos = rcol + m;                  // general index of row r
  int* grow = gpos + m;                  // row of general index g
  int* colptr = grow + m;                // CSC of single rows, ascending row order
  int* colrows = colptr + n + 1;

  for (int r = wid; r < m; r += kQpWarps) {
    const double* Cr = C + (int64_t)r * n;
    int cnt = 0, first = n;
    double fval = 0.0;
    for (int c0 = 0; c0 < n; c0 += 32) {
      const int c = c0 + lane;
      const double v = c < n ? Cr[c] : 0.0;
      const unsigned bal = __ballot_sync(0xffffffffu, v != 0.0);
      cnt += __popc(bal);
      if (bal && first == n) {
        const int src = __ffs(bal) - 1;
        first = c0 + src;
        fval = __shfl_sync(0xffffffffu, v, src);
      }
    }
    if (lane == 0) {
      rcol[r] = cnt == 1 ? first : -1;
      v_rval[r] = cnt == 1 ? fval : 0.0;
    }
  }
  __syncthreads();
  if (tid == 0) {
    int ng = 0;
    for (int r = 0; r < m; ++r) {
      if (rcol[r] < 0) {
        gpos[r] = ng;
        grow[ng++] = r;
      } else {
        gpos[r] = -1;
      }
    }
    for (int c = 0; c <= n; ++c) colptr[c] = 0;
    for (int r = 0; r < m; ++r)
      if (rcol[r] >= 0) colptr[rcol[r] + 1]++;
    for (int c = 0; c < n; ++c) colptr[c + 1] += colptr[c];
    for (int r = 0; r < m; ++r)  // counting sort: ascending row order per column
      if (rcol[r] >= 0) colrows[colptr[rcol[r]]++] = r;
    for (int c = n; c > 0; --c) colptr[c] = colptr[c - 1];
    colptr[0] = 0;
    sh_int[0] = ng;
  }
  __syncthreads();
  const int ng = sh_int[0];
  // general rows on-chip when they fit next to K, else in the global workspace
  const bool cg_smem = qp_layout(n, m, ldk, ng, A.k_smem != 0, true).total <= A.smem_bytes;
  const QpLayout LY = qp_layout(n, m, ldk, ng, A.k_smem != 0, cg_smem);
  double* K = A.k_smem ? (double*)(smem + LY.o_k) : gws;
  double* Cg = cg_smem ? (double*)(smem + LY.o_cg) : (gws + (A.k_smem ? 0 : (int64_t)ldk * n));
  for (int t = tid; t < ng * n; t += nt) {
    const int gi = t / n, c = t - gi * n;
    Cg[t] = C[(int64_t)grow[gi] * n + c];
  }
  for (int t = tid; t < n; t += nt) v_g[t] = gg[t];
  for (int t = tid; t < m; t += nt) v_d[t] = dd[t];
  __syncthreads();

  // scale references (qpsolver.py:124-127)
  double hmax = 0.0, gmax = 0.0;
  for (int t = tid; t < n * n; t += nt) hmax = fmax(hmax, fabs(H[t]));
  for (int t = tid; t < n; t += nt) gmax = fmax(gmax, fabs(v_g[t]));
  hmax = block_reduce<0>(hmax, red);
  gmax = block_reduce<0>(gmax, red);
  const double norm_g = n ? gmax : 0.0;
  const double scale_k = fmin(1.0, fmax(n ? hmax : 0.0, norm_g));
  const double scale_g = scale_k + norm_g;
  const double comp_ref = scale_k;
  const double tol = A.tol, reg = A.reg, tau = A.tau;

  // (C' t) into out[n], t over all m rows
  auto ct_apply = [&](const double* tv, double* out) {
    for (int c = tid; c < n; c += nt) {
      double s = 0.0;
      for (int q = colptr[c]; q < colptr[c + 1]; ++q) {
        const int r = colrows[q];
        s = fma(v_rval[r], tv[r], s);
      }
      for (int gi = 0; gi < ng; ++gi) s = fma(Cg[(int64_t)gi * n + c], tv[grow[gi]], s);
      out[c] = s;
    }
  };
  // (C x) into out[m]
  auto c_apply = [&](const double* xv, double* out) {
    for (int r = tid; r < m; r += nt) {
      if (rcol[r] >= 0) out[r] = v_rval[r] * xv[rcol[r]];
    }
    for (int gi = wid; gi < ng; gi += kQpWarps) {
      const double* row = Cg + (int64_t)gi * n;
      double s = 0.0;
      for (int c = lane; c < n; c += 32) s = fma(row[c], xv[c], s);
      s = warp_sum(s);
      if (lane == 0) out[grow[gi]] = s;
    }
  };
  // K = 2H + (reg or 0) I + boost I + diag(single) + Cg' W Cg, lower triangle,
  // column-major.  Optionally hu = H u in the same pass over H.
  auto build_k = [&](double diag_reg, double boost, bool with_terms, bool want_hu) {
    for (int r = wid; r < n; r += kQpWarps) {
      const double* Hr = H + (int64_t)r * n;
      double* Kc = K + (int64_t)r * ldk;  // column r of K holds rows c >= r (symmetry)
      double s = 0.0;
      for (int c = lane; c < n; c += 32) {
        const double h = Hr[c];
        if (want_hu) s = fma(h, v_u[c], s);
        if (c >= r) Kc[c] = 2.0 * h + (c == r ? diag_reg : 0.0);
      }
      if (want_hu) {
        s = warp_sum(s);
        if (lane == 0) v_hu[r] = s;
      }
    }
    __syncthreads();
    if (with_terms) {
      for (int c = tid; c < n; c += nt) {  // np.bincount(s_cols, weights=w*val*val)
        double s = 0.0;
        for (int q = colptr[c]; q < colptr[c + 1]; ++q) {
          const int r = colrows[q];
          s += v_w[r] * v_rval[r] * v_rval[r];
        }
        K[(int64_t)c * ldk + c] += s;
      }
      if (ng > 0) {
        for (int c = wid; c < n; c += kQpWarps) {
          double* Kc = K + (int64_t)c * ldk;
          for (int r = c + lane; r < n; r += 32) {
            double s = 0.0;
            for (int gi = 0; gi < ng; ++gi) {
              const double* row = Cg + (int64_t)gi * n;
              s = fma(row[r] * v_w[grow[gi]], row[c], s);
            }
            Kc[r] += s;
          }
        }
      }
    }
    if (boost != 0.0)
      for (int c = tid; c < n; c += nt) K[(int64_t)c * ldk + c] += boost;
    __syncthreads();
  };

  double* uo = A.u_out + bi * (int64_t)n;
  double* lo = A.lam_out + bi * (int64_t)m;

  // ---- unconstrained problems (qpsolver.py:131-144)
  if (m == 0) {
    const double boosts[4] = {0.0, reg, reg * 1e3, reg * 1e6};
    bool ok = false;
    for (int t = 0; t < 4 && !ok; ++t) {
      build_k(0.0, boosts[t], false, false);
      ok = chol_factor(K, n, ldk, v_dinv, red);
    }
    if (!ok) {
      for (int t = tid; t < n; t += nt) uo[t] = 0.0;
      if (tid == 0) {
        A.status[bi] = GM_QP_NUMERICAL_FAILURE;
        A.iters[bi] = 0;
        A.resid[bi * 3 + 0] = A.resid[bi * 3 + 1] = A.resid[bi * 3 + 2] = INFINITY;
      }
      return;
    }
    for (int t = tid; t < n; t += nt) v_rhs[t] = -v_g[t];
    __syncthreads();
    chol_solve(K, n, ldk, v_dinv, v_rhs, v_u);
    // stationarity max|2Hu + g|
    double rs = 0.0;
    for (int r = wid; r < n; r += kQpWarps) {
      double s = 0.0;
      for (int c = lane; c < n; c += 32) s = fma(2.0 * H[(int64_t)r * n + c], v_u[c], s);
      s = warp_sum(s);
      rs = fmax(rs, fabs(s + v_g[r]));
    }
    rs = block_reduce<0>(rs, red);
    for (int t = tid; t < n; t += nt) uo[t] = v_u[t];
    if (tid == 0) {
      A.status[bi] = GM_QP_OPTIMAL;
      A.iters[bi] = 0;
      A.resid[bi * 3 + 0] = rs;
      A.resid[bi * 3 + 1] = 0.0;
      A.resid[bi * 3 + 2] = 0.0;
    }
    return;
  }

  // ---- start point (qpsolver.py:146-150)
  for (int t = tid; t < n; t += nt) v_u[t] = A.warm ? A.warm[bi * (int64_t)n + t] : 0.0;
  __syncthreads();
  c_apply(v_u, v_cu);
  __syncthreads();
  for (int r = tid; r < m; r += nt) {
    v_s[r] = fmax(v_d[r] - v_cu[r], 1.0) * 1.1;
    v_lam[r] = 1.0;
  }
  __syncthreads();

  double best_metric = INFINITY, b_rs = 0, b_rp = 0, b_rc = 0;
  int status = -1, iters = 0;
  double f_rs = 0, f_rp = 0, f_rc = 0;
  bool use_best = false;

  // residuals at (u, lam) with best-iterate tracking (qpsolver.py:158-165);
  // leaves r_dual in v_rd and C u in v_cu
  auto residuals = [&](bool want_k, double& rs, double& rp, double& rc) {
    for (int r = tid; r < m; r += nt) v_w[r] = v_lam[r] / v_s[r];
    __syncthreads();
    build_k(reg, 0.0, want_k, true);  // hu = H u (and K for this iteration)
    ct_apply(v_lam, v_ctl);
    c_apply(v_u, v_cu);
    __syncthreads();
    double a_rs = 0.0, a_rp = 0.0, a_rc = 0.0;
    for (int c = tid; c < n; c += nt) {
      const double rd = (2.0 * v_hu[c] + v_g[c]) + v_ctl[c];
      v_rd[c] = rd;
      a_rs = fmax(a_rs, fabs(rd));
    }
    for (int r = tid; r < m; r += nt) {
      const double viol = v_cu[r] - v_d[r];
      a_rp = fmax(a_rp, viol);
      a_rc = fmax(a_rc, fabs(v_lam[r] * viol));
    }
    rs = block_reduce<0>(a_rs, red);
    rp = fmax(0.0, block_reduce<0>(a_rp, red));  // max(0, max viol)
    rc = block_reduce<0>(a_rc, red);
    const double metric = fmax(fmax(rs / scale_g, rp), rc / fmax(comp_ref, 1e-300));
    if (metric < best_metric) {
      best_metric = metric;
      b_rs = rs;
      b_rp = rp;
      b_rc = rc;
      for (int t = tid; t < n; t += nt) v_ub[t] = v_u[t];
      for (int t = tid; t < m; t += nt) v_lb[t] = v_lam[t];
    }
    __syncthreads();
  };

  // step length to the boundary (qpsolver.py:238-243)
  auto max_step = [&](const double* x, const double* dx) {
    double a = 1.0;
    for (int r = tid; r < m; r += nt)
      if (dx[r] < 0.0) a = fmin(a, -x[r] / dx[r]);
    return block_reduce<1>(a, red);
  };

  // KKT direction for complementarity target rc_vec (in v_t on entry is
  // overwritten): du -> v_du, dlam -> v_dl, ds -> v_ds (qpsolver.py:204-209)
  auto kkt_step = [&](const double* rcv) {
    for (int r = tid; r < m; r += nt) v_t[r] = (rcv[r] + v_lam[r] * v_rp[r]) / v_s[r];
    __syncthreads();
    ct_apply(v_t, v_ctl);
    __syncthreads();
    for (int c = tid; c < n; c += nt) v_rhs[c] = -v_rd[c] - v_ctl[c];
    __syncthreads();
    chol_solve(K, n, ldk, v_dinv, v_rhs, v_du);
    c_apply(v_du, v_t);  // C du
    __syncthreads();
    for (int r = tid; r < m; r += nt) {
      const double ds = -v_rp[r] - v_t[r];
      v_ds[r] = ds;
      v_dl[r] = (rcv[r] - v_lam[r] * ds) / v_s[r];
    }
    __syncthreads();
  };

  for (int it = 0; it < A.max_it; ++it) {
    double rs, rp, rc;
    residuals(true, rs, rp, rc);
    if (rs <= tol * scale_g && rp <= tol && rc <= tol * comp_ref) {
      status = GM_QP_OPTIMAL;
      iters = it;
      f_rs = rs;
      f_rp = rp;
      f_rc = rc;
      break;
    }
    double lmax = 0.0;
    for (int r = tid; r < m; r += nt) lmax = fmax(lmax, v_lam[r]);
    lmax = block_reduce<0>(lmax, red);
    if (lmax > 1e12 && rp > 1e-6) {
      status = GM_QP_PRIMAL_INFEASIBLE;
      iters = it;
      use_best = true;
      break;
    }
    // Cholesky with escalating regularisation (qpsolver.py:186-198)
    bool ok = chol_factor(K, n, ldk, v_dinv, red);
    double boost = 0.0;
    for (int att = 1; att < 4 && !ok; ++att) {
      boost = boost == 0.0 ? fmax(reg * 1e3, 1e-12) : boost * 1e3;
      build_k(reg, boost, true, false);
      ok = chol_factor(K, n, ldk, v_dinv, red);
    }
    if (!ok) {
      status = GM_QP_NUMERICAL_FAILURE;
      iters = it;
      use_best = true;
      break;
    }
    // r_pri = C u + s - d, mu = lam.s / m
    double mu_loc = 0.0;
    for (int r = tid; r < m; r += nt) {
      v_rp[r] = v_cu[r] + v_s[r] - v_d[r];
      mu_loc += v_lam[r] * v_s[r];
    }
    const double mu = block_reduce<2>(mu_loc, red) / m;
    // affine direction
    for (int r = tid; r < m; r += nt) v_dsa[r] = -v_lam[r] * v_s[r];  // rc target, temp
    __syncthreads();
    kkt_step(v_dsa);
    const double ap = max_step(v_s, v_ds);
    const double ad = max_step(v_lam, v_dl);
    double maff = 0.0;
    for (int r = tid; r < m; r += nt) maff += (v_lam[r] + ad * v_dl[r]) * (v_s[r] + ap * v_ds[r]);
    const double mu_aff = block_reduce<2>(maff, red) / m;
    const double sigma = mu > 0.0 ? (mu_aff / mu) * (mu_aff / mu) * (mu_aff / mu) : 0.0;
    // corrector with centring: rc = -lam s - dlam_a ds_a + sigma mu
    for (int r = tid; r < m; r += nt) {
      const double dla = v_dl[r], dsa = v_ds[r];
      v_dla[r] = -v_lam[r] * v_s[r] - dla * dsa + sigma * mu;
    }
    __syncthreads();
    kkt_step(v_dla);
    const double alpha = fmin(tau * max_step(v_s, v_ds), tau * max_step(v_lam, v_dl));
    bool finite = true;
    for (int c = tid; c < n; c += nt) {
      v_u[c] = v_u[c] + alpha * v_du[c];
      if (!isfinite(v_u[c])) finite = false;
    }
    for (int r = tid; r < m; r += nt) {
      v_s[r] = v_s[r] + alpha * v_ds[r];
      v_lam[r] = v_lam[r] + alpha * v_dl[r];
      if (!isfinite(v_s[r]) || !isfinite(v_lam[r])) finite = false;
    }
    const int all_finite = __syncthreads_and(finite ? 1 : 0);
    if (!all_finite) {
      status = GM_QP_NUMERICAL_FAILURE;
      iters = it + 1;
      use_best = true;
      break;
    }
  }
  if (status < 0) {  // iteration cap (qpsolver.py:231-235)
    double rs, rp, rc;
    residuals(false, rs, rp, rc);
    iters = A.max_it;
    if (rs <= tol * scale_g && rp <= tol && rc <= tol * comp_ref) {
      status = GM_QP_OPTIMAL;
      f_rs = rs;
      f_rp = rp;
      f_rc = rc;
    } else {
      status = GM_QP_MAX_ITERATIONS;
      use_best = true;
    }
  }
  const double* us = use_best ? v_ub : v_u;
  const double* ls = use_best ? v_lb : v_lam;
  for (int t = tid; t < n; t += nt) uo[t] = us[t];
  for (int t = tid; t < m; t += nt) lo[t] = ls[t];
  if (tid == 0) {
    A.status[bi] = status;
    A.iters[bi] = iters;
    A.resid[bi * 3 + 0] = use_best ? b_rs : f_rs;
    A.resid[bi * 3 + 1] = use_best ? b_rp : f_rp;
    A.resid[bi * 3 + 2] = use_best ? b_rc : f_rc;
  }
}

}  // namespace

extern "C" int gm_solve_qp(gm_ctx* ctx, int B, int n, int m, const double* H, const double* g,
                           const double* C, const double* d, const double* warm,
                           const gm_qp_settings* settings, double* u, double* lam, int32_t* status,
                           int32_t* iterations, double* resid, void* stream) {
  int rc = gm_need_device(ctx);
  if (rc) return rc;
  if (B < 0 || n < 1 || m < 0) return gm_fail(ctx, GM_ERR_CONFIG, "bad QP dimensions");
  if (B == 0) return GM_OK;
  gm_qp_settings s{1e-8, 50, 1e-9, 0.995};
  if (settings) s = *settings;
  if (!(s.tolerance > 0)) return gm_fail(ctx, GM_ERR_CONFIG, "tolerance must be positive");
  const int ldk = n | 1;  // odd leading dimension: conflict-free column and row walks
  // placement: vectors always on-chip; K on-chip when it fits; the general
  // constraint rows (count known only on the device) go on-chip if room is left.
  const size_t cap = ctx->smem_optin - 1024;
  bool k_smem = qp_layout(n, m, ldk, 0, true, false).total <= cap;
  if (qp_layout(n, m, ldk, 0, false, false).total > cap)
    return gm_fail(ctx, GM_ERR_CONFIG, "QP too large for the on-chip vectors");
  const size_t want = qp_layout(n, m, ldk, m, k_smem, true).total;
  const size_t smem_bytes = std::min(cap, want);
  const int64_t gws_stride = (k_smem ? 0 : (int64_t)ldk * n) + (int64_t)m * n;
  double* gws = (double*)gm_scratch(ctx, sizeof(double) * (size_t)gws_stride * B);
  if (!gws) return gm_fail(ctx, GM_ERR_CUDA, "QP workspace allocation failed");
  QpArgs a{};
  a.n = n;
  a.m = m;
  a.ldk = ldk;
  a.k_smem = k_smem;
  a.smem_bytes = smem_bytes;
  a.H = H;
  a.g = g;
  a.C = C;
  a.d = d;
  a.warm = warm;
  a.tol = s.tolerance;
  a.reg = s.regularization;
  a.tau = s.fraction_to_boundary;
  a.max_it = s.max_iterations;
  a.u_out = u;
  a.lam_out = lam;
  a.status = status;
  a.iters = iterations;
  a.resid = resid;
  a.gws = gws;
  a.gws_stride = gws_stride;
  GM_CUDA(ctx, cudaFuncSetAttribute(k_solve_qp, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_bytes));
  k_solve_qp<<<B, kQpThreads, smem_bytes, (cudaStream_t)stream>>>(a);
  GM_LAUNCH_CHECK(ctx, "k_solve_qp");
  return GM_OK;
}
