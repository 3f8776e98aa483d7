// K-QP: batched dense interior-point QP solver in fp64, one CTA per problem.
//
// Reference: solve_qp (qpsolver.py:112-235), _residuals (:90-97),
// _split_single_nonzero_rows (:100-109), _max_step (:238-243).  Same
// algorithm step by step -- Mehrotra predictor-corrector on
//   2Hu + g + C'lam = 0,  Cu + s = d,  lam_i s_i = mu
// with the reference's scale references, stopping / infeasibility tests,
// best-iterate bookkeeping, escalating Cholesky regularisation and status
// semantics, so statuses and iteration counts match the reference.
//
// Latency model (measured on B200, scripts/ubench_latency.cu): a dependent
// fp64 FMA costs 23 cycles, rsqrt(f64) 84, 1/sqrt(f64) 185, a double shuffle
// 54.  An IPM iteration is a chain of ~n dependent pivots, so the design
// shortens that chain and keeps every other loop free of long dependences:
//  * one CTA per QP, the whole IPM loop on the device (no host round trips);
//    batches of independent QPs fill the GPU (cfg4);
//  * the Schur matrix K is a packed lower triangle in shared memory;
//  * factorisation = block elimination with 2x2 pivots: one reciprocal per
//    two columns on the critical path, and the next pivot block is updated
//    and inverted one step ahead by warp 0 while warps 1..15 apply the
//    rank-2 update to the trailing matrix (one CTA barrier per 2 columns);
//    a final parallel pass turns the result into the Cholesky factor L;
//  * the 32x32 diagonal blocks of L are inverted in parallel, so the
//    triangular solves are 5 short block mat-vecs, not n scalar steps;
//  * every dot product uses 4 independent accumulators; loads of H (L2
//    resident when it does not fit on chip) are issued in batches;
//  * single-nonzero constraint rows (box bounds, slack signs) only touch the
//    diagonal; general rows are staged once into shared memory.
#include <algorithm>
#include <cfloat>

#include "common.cuh"
#include "qp_chol.cuh"

namespace {

#ifndef QP_THREADS
#define QP_THREADS 256
#endif
constexpr int kQpThreads = QP_THREADS;
constexpr int kQpWarps = kQpThreads / 32;
constexpr int kTB = 32;  // triangular-solve block

__host__ __device__ inline size_t qal(size_t x) { return (x + 15) & ~size_t(15); }
__host__ __device__ inline int64_t packed_size(int n) { return (int64_t)n * (n + 1) / 2; }

struct QpLayout {
  size_t o_vec, o_ints, o_k, o_x, o_h, o_cg, o_gv, total;
};

// n-vectors: g u hu rd rhs du ub ctl ytmp kee hde ea          (12)
// m-vectors: d s lam cu rp t dl ds tmp w lb rval              (12)
// ng-vectors (after the row classification): wg ga cf         (3)
// nf: dimension of the factorised system, <= n.  K: lower 8x8 tiles of the
// padded Schur matrix (qp_chol.cuh), overwritten by its Cholesky factor L;
// X region: the inverted diagonal tiles of L, per-warp scratch tiles (the
// coupling tiles of the 16x16 block inverses of solve_mw16), 1/diag(L), the
// padded solve vector and its staging copy.
__host__ __device__ inline size_t xregion_doubles(int nf) {
  const size_t T = qpchol::tiles_for(nf);
  return T * qpchol::kTS + 64 * kQpWarps + 24 * T;
}
// gv_smem = false: the three ng-vectors live in the global workspace (many
// general rows), so they take no shared memory
__host__ __device__ inline QpLayout qp_layout(int n, int m, int ng, bool h_smem, bool cg_smem, int nf = -1,
                                              bool gv_smem = true) {
  QpLayout L{};
  if (nf < 0) nf = n;
  size_t o = 0;
  L.o_vec = o;
  o = qal(o + sizeof(double) * (12 * (size_t)n + 12 * (size_t)m + 64));
  L.o_ints = o;  // rcol(m) grow(m) colptr(n+1) colrows(m) cstart(n+1) kidx(n) eidx(n) egi(n) ge(m) elig(n)
  o = qal(o + sizeof(int) * (4 * (size_t)m + 6 * (size_t)n + 2 + 8));
  L.o_gv = o;
  if (gv_smem) o = qal(o + sizeof(double) * 3 * (size_t)ng);
  L.o_k = o;
  o = qal(o + sizeof(double) * (size_t)qpchol::tile_doubles(nf));
  L.o_x = o;
  o = qal(o + sizeof(double) * xregion_doubles(nf));
  L.o_cg = o;
  if (cg_smem) o = qal(o + sizeof(double) * (size_t)ng * n);
  L.o_h = o;
  if (h_smem) o = qal(o + sizeof(double) * packed_size(nf));
  L.total = o;
  return L;
}

struct QpArgs {
  int n, m;
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
  double* gws;  // per-instance global workspace: packed H / general rows when off-chip
  int64_t gws_stride;
};

// optional per-phase cycle accounting (block 0, thread 0), read back with
// gm_qp_phase_cycles(); enabled by gm_qp_profile(1)
__device__ unsigned long long g_qp_prof[16];
__device__ int g_qp_prof_on;
// 1: the K-QP profile's slots 13-15 account the Cholesky pivot chain instead
// of the Schur-build phases (diagnostics)
__device__ int g_qp_chol_split;

struct Qs {  // per-CTA views
  // n: variables; nf: variables kept in the factorised (reduced) system.
  // Variables with a diagonal-only Hessian row that meet at most one general
  // constraint row (the soft-constraint slacks of expand_soft_constraints,
  // condensing.py:419-439) are eliminated exactly by a Schur complement:
  // kidx[0..nf) / eidx[0..ne) list kept / eliminated variables, egi[e] is the
  // general row of eliminated e (or -1) with coefficient ea[e], ge[gi] the
  // eliminated variable of general row gi (or -1) with coefficient ga[gi].
  int n, m, ng, nblk, nf, ne, T;
  int *kidx, *eidx, *egi, *ge, *elig;
  double *kee, *hde, *ea, *wg, *ga, *cf;
  double *K, *X, *Hp, *Cg, *scr, *yv;
  double *g, *u, *hu, *rd, *rhs, *du, *ub, *ctl, *ytmp, *dinv;
  double *d, *s, *lam, *cu, *rp, *t, *dl, *ds, *tmp, *w, *lb, *rval;
  int *rcol, *grow, *colptr, *colrows, *cstart;
  const unsigned short* tij;  // lower tile (I, J) of linear index t, row major
  double* red;
  double* pv;  // 2 x 16 pivot-block factors (double buffered)
  double* ys;  // 32-entry staging vector of the triangular solves
  int* flag;
  bool prof;
  long long last;
};

// the accounting is compiled in with -DGM_QP_PROF only (make EXTRA=-DGM_QP_PROF):
// its branches cost instruction-cache footprint in the IPM loop
#ifdef GM_QP_PROF
constexpr bool kQpProf = true;
#else
constexpr bool kQpProf = false;
#endif
__device__ __forceinline__ void qmark(Qs& S, int phase) {
  if (kQpProf && S.prof && threadIdx.x == 0) {
    const long long t = clock64();
    atomicAdd(&g_qp_prof[phase], (unsigned long long)(t - S.last));
    S.last = t;
  }
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// block-wide reductions (every thread gets the result); op 0 max, 1 min, 2 sum.
// Warp partials go through shared memory and every thread folds them in a
// fixed order (bitwise reproducible); block_reduce_n reduces K values with
// one pair of barriers.
template <int OP>
__device__ __forceinline__ double rop(double a, double b) {
  return OP == 0 ? fmax(a, b) : (OP == 1 ? fmin(a, b) : a + b);
}
template <int OP>
__device__ double block_reduce(double v, double* red) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = rop<OP>(v, __shfl_xor_sync(0xffffffffu, v, o));
  __syncthreads();
  if (lane == 0) red[wid] = v;
  __syncthreads();
  double w[kQpWarps];
#pragma unroll
  for (int i = 0; i < kQpWarps; i += 2) {
    const double2 t = *reinterpret_cast<const double2*>(red + i);
    w[i] = t.x;
    w[i + 1] = t.y;
  }
#pragma unroll
  for (int o = kQpWarps / 2; o > 0; o >>= 1)
#pragma unroll
    for (int i = 0; i < o; ++i) w[i] = rop<OP>(w[i], w[i + o]);
  return w[0];
}
template <int OP, int K>
__device__ void block_reduce_n(double (&v)[K], double* red, double* sum = nullptr) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double sv = sum ? *sum : 0.0;  // optional extra value, summed
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
#pragma unroll
    for (int q = 0; q < K; ++q) v[q] = rop<OP>(v[q], __shfl_xor_sync(0xffffffffu, v[q], o));
    if (sum) sv += __shfl_xor_sync(0xffffffffu, sv, o);
  }
  __syncthreads();
  if (lane == 0) {
#pragma unroll
    for (int q = 0; q < K; ++q) red[q * kQpWarps + wid] = v[q];
    if (sum) red[K * kQpWarps + wid] = sv;
  }
  __syncthreads();
  if (sum) {
    double w[kQpWarps];
#pragma unroll
    for (int i = 0; i < kQpWarps; i += 2) {
      const double2 t = *reinterpret_cast<const double2*>(red + K * kQpWarps + i);
      w[i] = t.x;
      w[i + 1] = t.y;
    }
#pragma unroll
    for (int o = kQpWarps / 2; o > 0; o >>= 1)
#pragma unroll
      for (int i = 0; i < o; ++i) w[i] = w[i] + w[i + o];
    *sum = w[0];
  }
#pragma unroll
  for (int q = 0; q < K; ++q) {
    double w[kQpWarps];
#pragma unroll
    for (int i = 0; i < kQpWarps; i += 2) {
      const double2 t = *reinterpret_cast<const double2*>(red + q * kQpWarps + i);
      w[i] = t.x;
      w[i + 1] = t.y;
    }
#pragma unroll
    for (int o = kQpWarps / 2; o > 0; o >>= 1)
#pragma unroll
      for (int i = 0; i < o; ++i) w[i] = rop<OP>(w[i], w[i + o]);
    v[q] = w[0];
  }
}

// ---------------------------------------------------------------------------
// factorisation and solves (qp_chol.cuh): tiled Cholesky of the reduced Schur
// matrix, blocked substitution solves (solve_mw16; X = L^{-1} variants behind
// QP_SOLVE_XXT)
// ---------------------------------------------------------------------------
// Packed lower triangle of H, column-major: element (r, c), r >= c, at
// colbase(c, n) + r.
__device__ __forceinline__ int colbase(int c, int n) { return c * n - ((c * (c + 1)) >> 1); }

// Cholesky factor of the padded Schur matrix (qp_chol.cuh)
__device__ __forceinline__ bool chol_factor(Qs& S) {
  if (S.T == 0) return true;  // every variable eliminated
  if (threadIdx.x == 0) *S.flag = 0;
  __syncthreads();
#ifdef QP_CHOL_SYNC
  const bool ok = qpchol::factor<kQpThreads>(S.K, S.T, S.dinv, S.flag);
#else
  const bool ok = qpchol::factor_la<kQpThreads>(S.K, S.T, S.dinv, S.flag,
                                                (kQpProf && S.prof && g_qp_chol_split) ? g_qp_prof + 13 : nullptr);
#endif
  __syncthreads();
  return ok;
}

// Solve strategies per IPM iteration (cycles per iteration at cfg3,
// scripts/qp_phases.py): (default) the diagonal-tile inverses plus the
// 16x16 block-inverse coupling tiles (3.6 K) and an all-warp blocked
// substitution with a one-block look-ahead (solve_mw16; the two solves
// 30.6 K incl. the reduced-system prep) -- 119.8 K per iteration;
// (QP_SOLVE_MW8) the same with 8-row blocks, 123.4 K; (QP_SOLVE_XXT, round
// 1) X = L^{-1} formed in place (23 K) and every solve two parallel mat-vecs,
// 133 K; (QP_SOLVE_SUBST) single-warp substitution (~24 K per solve).
#if !defined(QP_SOLVE_SUBST) && defined(QP_SOLVE_XXT)
__device__ __forceinline__ void invert_diag_blocks(Qs& S) {
  if (S.T == 0) return;
  qpchol::invert_full<kQpThreads>(S.K, S.T, S.dinv, S.X, S.scr);
}
#else
// inverses of the diagonal tiles of L (into the X region); L stays in K;
// with T <= 16 also the coupling tiles of the 16x16 block inverses (into
// the scratch area) for solve_mw16
__device__ __forceinline__ void invert_diag_blocks(Qs& S) {
  if (S.T == 0) return;
  qpchol::diag_inverses<kQpThreads>(S.K, S.T, S.dinv, S.X);
  __syncthreads();
#if !defined(QP_SOLVE_SUBST) && !defined(QP_SOLVE_MW8)
  if (S.T <= 16 && 64 * kQpWarps >= 512) qpchol::diag16<kQpThreads>(S.K, S.T, S.X, S.scr);
#endif
}
#endif

// x = K^{-1} b = X' (X b) through the padded solve vector S.yv (padding stays
// zero); b and x are shared nf-vectors (x may alias b).  Call with all threads.
__device__ void chol_solve(Qs& S, const double* b, double* x) {
#if defined(QP_SOLVE_SUBST)
  if (S.T > 0) qpchol::solve_llt<kQpThreads>(S.K, S.X, S.T, S.nf, b, x, S.yv);
#elif defined(QP_SOLVE_XXT)
  if (S.T > 0) qpchol::solve_xxt<kQpThreads>(S.K, S.T, S.nf, b, x, S.yv + 8 * S.T);
#else
  if (S.T > 0) {
#ifndef QP_SOLVE_MW8
    if (S.T <= 16 && 64 * kQpWarps >= 512)
      qpchol::solve_mw16<kQpThreads>(S.K, S.X, S.scr, S.T, S.nf, b, x, S.yv);
    else
#endif
      qpchol::solve_mw<kQpThreads>(S.K, S.X, S.T, S.nf, b, x, S.yv);
  }
#endif
}

// ---------------------------------------------------------------------------
// QP building blocks
// ---------------------------------------------------------------------------

// explicit shared-window loads: the on-chip / workspace choice of H and the
// general rows is made at run time, so their pointers are generic and the
// compiler emits LD.E (generic, 64-bit address math) even with
// __builtin_assume(__isShared(...)); these helpers force LDS
__device__ __forceinline__ uint32_t sh_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
// (not volatile: a pure load of data no thread writes during the caller, so
// the compiler may hoist and batch these loads ahead of the DMMAs)
__device__ __forceinline__ double lds64(uint32_t a) {
  double v;
  asm("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
  return v;
}
// element i of a double array: shared window when SH (base = sh_addr), else generic
template <bool SH>
__device__ __forceinline__ double ldv(const double* p, uint32_t base, int i) {
  return SH ? lds64(base + 8u * (uint32_t)i) : p[i];
}

// out = C' tv.  General rows are stored column-permuted: Cg[gi][k] is the
// coefficient of kept variable kidx[k]; a row's eliminated variable (if any)
// is (ge[gi], ga[gi]).
// RHS: write -rd - (C' tv) instead (the KKT right-hand side, fused)
template <bool RHS = false>
__device__ void ct_apply(const Qs& S, const double* tv, double* out) {
#pragma unroll 1
  for (int k = threadIdx.x; k < S.nf; k += blockDim.x) {
    const int c = S.kidx[k];
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
#pragma unroll 1
    for (int q = S.colptr[c]; q < S.colptr[c + 1]; ++q) {
      const int r = S.colrows[q];
      s0 = fma(S.rval[r], tv[r], s0);
    }
    const double* cg = S.Cg + k;
    int gi = 0;
#pragma unroll 1
    for (; gi + 3 < S.ng; gi += 4) {
      s0 = fma(cg[(int64_t)gi * S.n], tv[S.grow[gi]], s0);
      s1 = fma(cg[(int64_t)(gi + 1) * S.n], tv[S.grow[gi + 1]], s1);
      s2 = fma(cg[(int64_t)(gi + 2) * S.n], tv[S.grow[gi + 2]], s2);
      s3 = fma(cg[(int64_t)(gi + 3) * S.n], tv[S.grow[gi + 3]], s3);
    }
#pragma unroll 1
    for (; gi < S.ng; ++gi) s0 = fma(cg[(int64_t)gi * S.n], tv[S.grow[gi]], s0);
    const double v = (s0 + s1) + (s2 + s3);
    out[c] = RHS ? -S.rd[c] - v : v;
  }
  // eliminated variables on the threads the kept loop leaves idle
  int e = (int)threadIdx.x - S.nf % (int)blockDim.x;
  if (e < 0) e += blockDim.x;
  for (; e < S.ne; e += blockDim.x) {
    const int c = S.eidx[e];
    double s0 = 0.0;
#pragma unroll 1
    for (int q = S.colptr[c]; q < S.colptr[c + 1]; ++q) {
      const int r = S.colrows[q];
      s0 = fma(S.rval[r], tv[r], s0);
    }
    if (S.egi[e] >= 0) s0 = fma(S.ea[e], tv[S.grow[S.egi[e]]], s0);
    out[c] = RHS ? -S.rd[c] - s0 : s0;
  }
}

// out[r] = (C xv)[r].  General rows: one 8-lane group per row (all rows at
// once for ng <= NT/8; a 3-level shuffle instead of a warp-wide 5-level one),
// two FMA chains per lane.
__device__ void c_apply(const Qs& S, const double* xv, double* out) {
  constexpr int G = 8;
  const int lg = threadIdx.x & (G - 1), grp = threadIdx.x / G;
#pragma unroll 1
  for (int r = threadIdx.x; r < S.m; r += blockDim.x)
    if (S.rcol[r] >= 0) out[r] = S.rval[r] * xv[S.rcol[r]];
  for (int g0 = 0; g0 < S.ng; g0 += kQpThreads / G) {
    const int gi = g0 + grp;
    double s = 0.0, s1 = 0.0;
    if (gi < S.ng) {
      const double* row = S.Cg + (int64_t)gi * S.n;
      int k = lg;
#pragma unroll 1
      for (; k + G < S.nf; k += 2 * G) {
        s = fma(row[k], xv[S.kidx[k]], s);
        s1 = fma(row[k + G], xv[S.kidx[k + G]], s1);
      }
      if (k < S.nf) s = fma(row[k], xv[S.kidx[k]], s);
      s += s1;
    }
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (gi < S.ng && lg == 0) {
      if (S.ge[gi] >= 0) s = fma(S.ga[gi], xv[S.eidx[S.ge[gi]]], s);
      out[S.grow[gi]] = s;
    }
  }
}

// hu = H u over the kept variables (packed lower H, column major) plus the
// diagonal of the eliminated ones.  One pass over the columns serves both
// triangles: warp w takes columns c = w, w + NW, ...; lane-rows r >= c
// (contiguous, conflict free) accumulate H[r][c] u_c into per-lane row
// partials (lower part) and H[r][c] u_r into the column's sum (upper part,
// r > c), 4 columns in flight so their warp reductions overlap.  Row
// partials of the warps meet in the (free at this point) K tile region and
// are added in a fixed order.  Call with all threads; out is complete after
// the call's final barrier.
__device__ void h_apply_rows(const Qs& S, const double* uv, double* out);
// (out of line: the H-in-global-memory case, kept out of the hot code)
__device__ __noinline__ void h_apply_cols(const double* Hp, const int* kidx, const int* eidx, const double* hde,
                                          double* K, int n, int ne, const double* uv, double* out) {
  constexpr int TM = 8;  // n <= 256
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double* part = K;                        // NW x n row partials
  double* colsum = K + kQpWarps * n;       // n upper-part sums
  double uk[TM], acc[TM];
#pragma unroll
  for (int t = 0; t < TM; ++t) {
    const int r = lane + 32 * t;
    uk[t] = r < n ? uv[kidx[r]] : 0.0;
    acc[t] = 0.0;
  }
  for (int c0 = wid; c0 < n; c0 += 4 * kQpWarps) {
    double cs[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int c = c0 + q * kQpWarps;
      cs[q] = 0.0;
      if (c < n) {
        const double uc = uv[kidx[c]];
        const double* col = Hp + colbase(c, n);
#pragma unroll
        for (int t = 0; t < TM; ++t) {
          const int r = lane + 32 * t;
          if (r >= c && r < n) {
            const double h = col[r];
            acc[t] = fma(h, uc, acc[t]);
            if (r > c) cs[q] = fma(h, uk[t], cs[q]);
          }
        }
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
#pragma unroll
      for (int q = 0; q < 4; ++q) cs[q] += __shfl_xor_sync(0xffffffffu, cs[q], o);
    if (lane == 0) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int c = c0 + q * kQpWarps;
        if (c < n) colsum[c] = cs[q];
      }
    }
  }
#pragma unroll
  for (int t = 0; t < TM; ++t) {
    const int r = lane + 32 * t;
    if (r < n) part[wid * n + r] = acc[t];
  }
  __syncthreads();
#pragma unroll 1
  for (int r = threadIdx.x; r < n; r += blockDim.x) {
    double v = colsum[r];
#pragma unroll
    for (int w = 0; w < kQpWarps; ++w) v += part[w * n + r];
    out[kidx[r]] = v;
  }
#pragma unroll 1
  for (int e = threadIdx.x; e < ne; e += blockDim.x) out[eidx[e]] = hde[e] * uv[eidx[e]];
  __syncthreads();
}
__device__ void h_apply(const Qs& S, const double* uv, double* out) {
  if (__isShared(S.Hp) && S.nf <= (int)blockDim.x && uv != out)
    h_apply_rows(S, uv, out);
  else
    h_apply_cols(S.Hp, S.kidx, S.eidx, S.hde, S.K, S.nf, S.ne, uv, out);
}

// out = H u with packed H on chip: one thread per kept row r, the row read
// as column r's lower part below the diagonal (H[c][r], consecutive rows ->
// consecutive words) and column r itself above it, four independent
// accumulators; no shuffles or cross-warp partials (the warp-per-column form
// above is for H left in global memory, where it batches the L2 round trips).
__device__ void h_apply_rows(const Qs& S, const double* uv, double* out) {
  const int n = S.nf;
  const double* Hp = S.Hp;
  const uint32_t hb = sh_addr(Hp);  // the caller checked __isShared(S.Hp)
  double* uk = out;
  // two threads per row when n <= blockDim/2 (halves of the column range,
  // combined in a fixed order)
  const bool split = 2 * n <= (int)blockDim.x;
  const int half = split ? (int)threadIdx.x / (blockDim.x / 2) : 0;
  const int r = split ? (int)threadIdx.x % (blockDim.x / 2) : (int)threadIdx.x;
  const int cmid = split ? n / 2 : n;
  const int c_lo = half ? cmid : 0, c_hi = half ? n : cmid;
  double uv_r = 0.0;
  if (half == 0 && r < n) uv_r = uv[S.kidx[r]];
  __syncthreads();
  if (half == 0 && r < n) uk[r] = uv_r;
  __syncthreads();
  double acc = 0.0;
  if (r < n) {
    auto hl = [&](int i) { return lds64(hb + 8u * (uint32_t)i); };
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    int c = c_lo;
    const int cl = min(r, c_hi);
#pragma unroll 1
    for (; c + 3 < cl; c += 4) {
      a0 = fma(hl(colbase(c, n) + r), uk[c], a0);
      a1 = fma(hl(colbase(c + 1, n) + r), uk[c + 1], a1);
      a2 = fma(hl(colbase(c + 2, n) + r), uk[c + 2], a2);
      a3 = fma(hl(colbase(c + 3, n) + r), uk[c + 3], a3);
    }
#pragma unroll 1
    for (; c < cl; ++c) a0 = fma(hl(colbase(c, n) + r), uk[c], a0);
    const int colr = colbase(r, n);
    c = max(c, r);
#pragma unroll 1
    for (; c + 3 < c_hi; c += 4) {
      a0 = fma(hl(colr + c), uk[c], a0);
      a1 = fma(hl(colr + c + 1), uk[c + 1], a1);
      a2 = fma(hl(colr + c + 2), uk[c + 2], a2);
      a3 = fma(hl(colr + c + 3), uk[c + 3], a3);
    }
#pragma unroll 1
    for (; c < c_hi; ++c) a0 = fma(hl(colr + c), uk[c], a0);
    acc = (a0 + a1) + (a2 + a3);
  }
  double* part = S.K;  // free at this point (rebuilt by build_k)
  if (split && half == 1 && r < n) part[r] = acc;
  __syncthreads();
  if (split && half == 0 && r < n) acc += part[r];
  if (half == 0 && r < n) out[S.kidx[r]] = acc;
#pragma unroll 1
  for (int e = threadIdx.x; e < S.ne; e += blockDim.x) out[S.eidx[e]] = S.hde[e] * uv[S.eidx[e]];
  __syncthreads();
}

// K = 2H + diag_add I + diag(sum_single w val^2) + Cg' W Cg  (qpsolver.py:178-184)
// on the reduced system: with an eliminated variable e in general row g,
//   K_ee = 2 H_ee + diag_add + sum_single w val^2 + w_g a^2,
//   K_red = K_kk - K_ke K_ee^{-1} K_ek  =  ... + w'_g Cg_g' Cg_g,
//   w'_g = w_g - (w_g a)^2 / K_ee            (a rank-one change per such row).
// build_k returns false when an eliminated pivot K_ee is not positive
// (potrf's failure rule applied to the eliminated block).
// Lower 8x8 tiles of 2H + Cg' diag(wg) Cg on the fp64 tensor cores: the C
// fragment (row i, cols 2p, 2p+1) starts from 2H, ng/4 DMMAs add the general
// rows (A[i][g] = wg_g Cg[g][row], B[g][j] = Cg[g][col]); padding rows / cols
// (>= n) become the identity.  One warp per tile, U tiles in flight.  The
// operand loads are branch-free with 32-bit offsets: padding rows / cols read
// a clamped (finite) index, which only touches C entries of that padding row /
// col, overwritten afterwards; SH: H, Cg and wg are in shared memory.
template <bool SH>
__device__ __noinline__ void build_tiles(const double* Cg, const double* Hp, const double* wg, double* K,
                                         const unsigned short* tij, int T, int n, int ng, int ldc) {
  const uint32_t cgb = SH ? sh_addr(Cg) : 0u, hpb = SH ? sh_addr(Hp) : 0u, wgb = SH ? sh_addr(wg) : 0u;
  QP_SMEM(K);
  QP_SMEM(tij);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int i = lane >> 2, p = lane & 3;
  const int ntiles = T * (T + 1) / 2;
  constexpr int U = 2;  // tiles in flight per warp (A/B on one box: 2 < 3 < 4 < 5)
  for (int t0 = wid; t0 < ntiles; t0 += U * kQpWarps) {
    int r[U], ca[U], ra[U], rbc[U];
    double h0[U], h1[U];
    bool live[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int tt = t0 + u * kQpWarps;
      live[u] = tt < ntiles;
      const int ij = tij[min(tt, ntiles - 1)];  // (I << 8) | J, built once
      const int I = ij >> 8, J = ij & 255;
      r[u] = 8 * I + i;
      ca[u] = 8 * J + 2 * p;
      const int rb = 8 * J + i;  // B operand column
      ra[u] = min(r[u], n - 1);
      rbc[u] = min(rb, n - 1);
      const int cb = ca[u] + 1;
      // strictly lower entries start from 2H; the diagonal is completed below
      h0[u] = (live[u] && r[u] < n && ca[u] < n && r[u] > ca[u]) ? 2.0 * ldv<SH>(Hp, hpb, colbase(ca[u], n) + r[u])
                                                                  : 0.0;
      h1[u] = (live[u] && r[u] < n && cb < n && r[u] > cb) ? 2.0 * ldv<SH>(Hp, hpb, colbase(cb, n) + r[u]) : 0.0;
    }
    // software-pipelined over the general-row steps: the operands of step
    // g0 + 4 are loaded before the DMMAs of step g0 are issued
    double xa[U], xb[U], wnext;
    auto load = [&](int g0) {
      const int g = g0 + p;
      const bool gv = g < ng;
      const int rowo = (gv ? g : ng - 1) * ldc;
      wnext = gv ? ldv<SH>(wg, wgb, g) : 0.0;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        xa[u] = ldv<SH>(Cg, cgb, rowo + ra[u]);
        xb[u] = ldv<SH>(Cg, cgb, rowo + rbc[u]);
      }
    };
    if (ng > 0) load(0);
    for (int g0 = 0; g0 < ng; g0 += 4) {
      const double wgg = wnext;
      double av[U], bv[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        av[u] = wgg * xa[u];
        bv[u] = xb[u];
      }
      if (g0 + 4 < ng) load(g0 + 4);
#pragma unroll
      for (int u = 0; u < U; ++u) qpchol::dmma884(h0[u], h1[u], av[u], bv[u]);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (!live[u]) continue;
      const int cb = ca[u] + 1;
      if (r[u] >= n || ca[u] >= n) h0[u] = r[u] == ca[u] ? 1.0 : 0.0;
      if (r[u] >= n || cb >= n) h1[u] = r[u] == cb ? 1.0 : 0.0;
      if (r[u] >= ca[u]) K[qpchol::gel(r[u], ca[u])] = h0[u];
      if (r[u] >= cb) K[qpchol::gel(r[u], cb)] = h1[u];
    }
  }
}

__device__ bool build_k(const Qs& S, double diag_add, bool terms) {
  const int n = S.nf, ng = terms ? S.ng : 0;
  bool ok = true;
#pragma unroll 1
  for (int e = threadIdx.x; e < S.ne; e += blockDim.x) {
    const int c = S.eidx[e];
    double dsum = 0.0;
    if (terms)
  #pragma unroll 1
    for (int q = S.colptr[c]; q < S.colptr[c + 1]; ++q) {
        const int r = S.colrows[q];
        dsum += S.w[r] * S.rval[r] * S.rval[r];
      }
    double kee = (2.0 * S.hde[e] + diag_add) + dsum;
    if (terms && S.egi[e] >= 0) kee += S.w[S.grow[S.egi[e]]] * S.ea[e] * S.ea[e];
    if (!(kee > 0.0)) ok = false;
    S.kee[e] = kee;
  }
  __syncthreads();
#pragma unroll 1
  for (int gi = threadIdx.x; gi < ng; gi += blockDim.x) {
    const double wgi = S.w[S.grow[gi]];
    double wr = wgi;
    if (S.ge[gi] >= 0) {
      const double t = wgi * S.ga[gi];
      wr = wgi - t * t / S.kee[S.ge[gi]];
    }
    S.wg[gi] = wr;
  }
  __syncthreads();
  if (!g_qp_chol_split) qmark(const_cast<Qs&>(S), 13);
  // lower 8x8 tiles of 2H + Cg' diag(wg) Cg on the fp64 tensor cores
  // (build_tiles); on-chip H and Cg take the shared-address instantiation
  if (__isShared(S.Cg) && __isShared(S.Hp) && __isShared(S.wg))
    build_tiles<true>(S.Cg, S.Hp, S.wg, S.K, S.tij, S.T, n, ng, S.n);
  else
    build_tiles<false>(S.Cg, S.Hp, S.wg, S.K, S.tij, S.T, n, ng, S.n);
  __syncthreads();
  if (!g_qp_chol_split) qmark(const_cast<Qs&>(S), 14);
  // diagonal (holds only the general-row term so far): (2H + reg) +
  // bincount(single rows) first, then the general-row term, as the
  // reference orders it
#pragma unroll 1
  for (int k = threadIdx.x; k < n; k += blockDim.x) {
    const int c = S.kidx[k];
    double dsum = 0.0;
    if (terms)
  #pragma unroll 1
    for (int q = S.colptr[c]; q < S.colptr[c + 1]; ++q) {
        const int r = S.colrows[q];
        dsum += S.w[r] * S.rval[r] * S.rval[r];
      }
    const int dc = qpchol::gel(k, k);
    S.K[dc] = ((2.0 * S.Hp[colbase(k, n) + k] + diag_add) + dsum) + S.K[dc];
  }

  const bool all_ok = __syncthreads_and(ok ? 1 : 0) != 0;
  if (!g_qp_chol_split) qmark(const_cast<Qs&>(S), 15);
  return all_ok;
}

// step lengths of (s, ds) and (lam, dl) with one block reduction
__device__ __forceinline__ void max_step2(const Qs& S, double& ap, double& ad) {
  double a[2] = {1.0, 1.0};
#pragma unroll 1
  for (int r = threadIdx.x; r < S.m; r += blockDim.x) {
    if (S.ds[r] < 0.0) a[0] = fmin(a[0], -S.s[r] / S.ds[r]);
    if (S.dl[r] < 0.0) a[1] = fmin(a[1], -S.lam[r] / S.dl[r]);
  }
  block_reduce_n<1, 2>(a, S.red);
  ap = a[0];
  ad = a[1];
}

// largest step in [0, 1] with x + a dx > 0 (qpsolver.py:238-243)
__device__ double max_step(const Qs& S, const double* x, const double* dx) {
  double a = 1.0;
#pragma unroll 1
  for (int r = threadIdx.x; r < S.m; r += blockDim.x)
    if (dx[r] < 0.0) a = fmin(a, -x[r] / dx[r]);
  return block_reduce<1>(a, S.red);
}

// x = K^{-1} b for the full Schur matrix through the reduced system:
//   b_red = b_k - K_ke K_ee^{-1} b_e,  K_red x_k = b_red,
//   x_e = (b_e - K_ek x_k) / K_ee,   K_ke = w_g a Cg_g (kept part).
// Uses ytmp (reduced rhs / solution) and cf (per-row coefficients).
__device__ void reduced_solve(Qs& S, const double* b, double* x) {
  double* yr = S.ytmp;
  double* coef = S.cf;
  if (S.ne == 0) {
#pragma unroll 1
    for (int k = threadIdx.x; k < S.nf; k += blockDim.x) yr[k] = b[S.kidx[k]];
    __syncthreads();
    chol_solve(S, yr, yr);
#pragma unroll 1
    for (int k = threadIdx.x; k < S.nf; k += blockDim.x) x[S.kidx[k]] = yr[k];
    __syncthreads();
    return;
  }
#pragma unroll 1
  for (int gi = threadIdx.x; gi < S.ng; gi += blockDim.x) {
    const int e = S.ge[gi];
    coef[gi] = e >= 0 ? S.w[S.grow[gi]] * S.ga[gi] * b[S.eidx[e]] / S.kee[e] : 0.0;
  }
  __syncthreads();
#pragma unroll 1
  for (int k = threadIdx.x; k < S.nf; k += blockDim.x) {
    double s = b[S.kidx[k]];
    for (int gi = 0; gi < S.ng; ++gi) s = fma(-coef[gi], S.Cg[(int64_t)gi * S.n + k], s);
    yr[k] = s;
  }
  __syncthreads();
  chol_solve(S, yr, yr);
#pragma unroll 1
  for (int k = threadIdx.x; k < S.nf; k += blockDim.x) x[S.kidx[k]] = yr[k];
  // eliminated: one 8-lane group per eliminated variable, all groups at once
  constexpr int G = 8;
  const int lg = threadIdx.x & (G - 1);
  for (int e0 = 0; e0 < S.ne; e0 += kQpThreads / G) {
    const int e = e0 + (int)threadIdx.x / G;
    const bool live = e < S.ne;
    const int gi = live ? S.egi[e] : -1;
    double s = 0.0;
    if (gi >= 0) {
      const double* row = S.Cg + (int64_t)gi * S.n;
      double s1 = 0.0;
      int k = lg;
#pragma unroll 1
      for (; k + G < S.nf; k += 2 * G) {
        s = fma(row[k], yr[k], s);
        s1 = fma(row[k + G], yr[k + G], s1);
      }
      if (k < S.nf) s = fma(row[k], yr[k], s);
      s += s1;
    }
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (live && lg == 0) {
      if (gi >= 0) s *= S.w[S.grow[gi]] * S.ea[e];
      x[S.eidx[e]] = (b[S.eidx[e]] - s) / S.kee[e];
    }
  }
  __syncthreads();
}

// du, dlam, ds for complementarity target rcv (qpsolver.py:204-209)
__device__ void kkt_step(Qs& S, const double* rcv) {
#pragma unroll 1
  for (int r = threadIdx.x; r < S.m; r += blockDim.x)
    S.t[r] = (rcv[r] + S.lam[r] * S.rp[r]) / S.s[r];
  __syncthreads();
  ct_apply<true>(S, S.t, S.rhs);  // rhs = -rd - C' t
  __syncthreads();
  qmark(S, 10);
  reduced_solve(S, S.rhs, S.du);
  qmark(S, 11);
  c_apply(S, S.du, S.t);  // C du
  __syncthreads();
#pragma unroll 1
  for (int r = threadIdx.x; r < S.m; r += blockDim.x) {
    const double ds = -S.rp[r] - S.t[r];
    S.ds[r] = ds;
    S.dl[r] = (rcv[r] - S.lam[r] * ds) / S.s[r];
  }
  __syncthreads();
}

struct Resid {
  double rs, rp, rc, lmax, musum;
};

// residuals at (u, lam) (qpsolver.py:90-97); leaves r_dual in rd, C u in cu
__device__ Resid residuals(Qs& S) {
  qmark(S, 1);
  h_apply(S, S.u, S.hu);
  qmark(S, 12);
  ct_apply(S, S.lam, S.ctl);
  c_apply(S, S.u, S.cu);
  __syncthreads();
  double a_rs = 0.0, a_rp = -INFINITY, a_rc = 0.0, a_lm = 0.0, a_mu = 0.0;
#pragma unroll 1
  for (int c = threadIdx.x; c < S.n; c += blockDim.x) {
    const double rd = (2.0 * S.hu[c] + S.g[c]) + S.ctl[c];
    S.rd[c] = rd;
    a_rs = fmax(a_rs, fabs(rd));
  }
#pragma unroll 1
  for (int r = threadIdx.x; r < S.m; r += blockDim.x) {
    const double viol = S.cu[r] - S.d[r];
    a_rp = fmax(a_rp, viol);
    a_rc = fmax(a_rc, fabs(S.lam[r] * viol));
    a_lm = fmax(a_lm, S.lam[r]);  // max lam for the infeasibility test
    S.rp[r] = S.cu[r] + S.s[r] - S.d[r];  // r_pri and mu of this iterate
    a_mu += S.lam[r] * S.s[r];
  }
  Resid R;
  double r3[4] = {a_rs, a_rp, a_rc, a_lm};
  block_reduce_n<0, 4>(r3, S.red, &a_mu);
  R.rs = r3[0];
  R.rp = fmax(0.0, r3[1]);
  R.rc = r3[2];
  R.lmax = r3[3];
  R.musum = a_mu;
  return R;
}

__global__ void __launch_bounds__(kQpThreads, 1) k_solve_qp(const QpArgs A) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ __align__(16) double red[5 * kQpWarps];
  __shared__ double pvbuf[32];
  __shared__ double ysbuf[kTB];
  __shared__ int sh_int[4];
  const int n = A.n, m = A.m;
  const int64_t bi = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nt = blockDim.x;
  const double* H = A.H + bi * (int64_t)n * n;
  const double* C = A.C + bi * (int64_t)m * n;
  double* gws = A.gws + bi * A.gws_stride;

  Qs S;
  S.n = n;
  S.m = m;
  S.nblk = (n + kTB - 1) / kTB;
  S.red = red;
  S.pv = pvbuf;
  S.ys = ysbuf;
  S.flag = &sh_int[1];
  S.prof = kQpProf && g_qp_prof_on && blockIdx.x == 0;
  S.last = clock64();
  {
    const QpLayout L0 = qp_layout(n, m, 0, false, false);
    double* v = (double*)(smem + L0.o_vec);
    S.g = v; v += n;
    S.u = v; v += n;
    S.hu = v; v += n;
    S.rd = v; v += n;
    S.rhs = v; v += n;
    S.du = v; v += n;
    S.ub = v; v += n;
    S.ctl = v; v += n;
    S.ytmp = v; v += n;
    S.kee = v; v += n;
    S.hde = v; v += n;
    S.ea = v; v += n;
    S.d = v; v += m;
    S.s = v; v += m;
    S.lam = v; v += m;
    S.cu = v; v += m;
    S.rp = v; v += m;
    S.t = v; v += m;
    S.dl = v; v += m;
    S.ds = v; v += m;
    S.tmp = v; v += m;
    S.w = v; v += m;
    S.lb = v; v += m;
    S.rval = v;
    int* ip = (int*)(smem + L0.o_ints);
    S.rcol = ip;
    S.grow = ip + m;
    S.colptr = ip + 2 * m;
    S.colrows = ip + 2 * m + n + 1;
    S.cstart = ip + 3 * m + n + 1;
    S.kidx = ip + 3 * m + 2 * n + 2;
    S.eidx = S.kidx + n;
    S.egi = S.eidx + n;
    S.ge = S.egi + n;
    S.elig = S.ge + m;
    S.K = (double*)(smem + L0.o_k);
    S.X = (double*)(smem + L0.o_x);
  }

  // ---- classify rows (qpsolver.py:100-109): single-nonzero vs general.
  // Setup runs once per solve; every pass below is a flat, independent-load
  // sweep or a warp-wide ballot/match compaction (no single-thread loops over
  // m or n: they cost ~100 us of L2/shared latency per solve).
  // Pass 1 over C: per-row nonzero count (rcol) and first nonzero column
  // (grow), by shared atomics.
#pragma unroll 1
  for (int r = tid; r < m; r += nt) {
    S.rcol[r] = 0;
    S.grow[r] = n;
  }
  for (int c = tid; c <= n; c += nt) {
    S.colptr[c] = 0;
    S.cstart[c] = c * n - (c * (c - 1)) / 2;
  }
#pragma unroll 1
  for (int c = tid; c < n; c += nt) S.elig[c] = m > 0 ? 1 : 0;
  __syncthreads();
  {
    const int64_t mn = (int64_t)m * n;
    for (int64_t t0 = tid; t0 < mn; t0 += 8 * (int64_t)nt) {
      double v[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int64_t t = t0 + (int64_t)j * nt;
        v[j] = t < mn ? __ldg(C + t) : 0.0;
      }
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (v[j] != 0.0) {
          const int64_t t = t0 + (int64_t)j * nt;
          const int r = (int)(t / n), c = (int)(t - (int64_t)r * n);
          atomicAdd(&S.rcol[r], 1);
          atomicMin(&S.grow[r], c);
        }
    }
  }
  // Pass over H: the scale reference max|H| (qpsolver.py:124) and the
  // eliminable-variable test below (no off-diagonal Hessian entry in the row)
  double hmax_loc = 0.0;
  {
    const int64_t nn2 = (int64_t)n * n;
    for (int64_t t0 = tid; t0 < nn2; t0 += 8 * (int64_t)nt) {
      double v[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int64_t t = t0 + (int64_t)j * nt;
        v[j] = t < nn2 ? __ldg(H + t) : 0.0;
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        hmax_loc = fmax(hmax_loc, fabs(v[j]));
        if (v[j] != 0.0) {
          const int64_t t = t0 + (int64_t)j * nt;
          const int r = (int)(t / n), c = (int)(t - (int64_t)r * n);
          if (r != c) S.elig[r] = 0;
        }
      }
    }
  }
  __syncthreads();
#pragma unroll 1
  for (int r = tid; r < m; r += nt) {
    const int cnt = S.rcol[r], first = S.grow[r];
    S.rcol[r] = cnt == 1 ? first : -1;
    S.rval[r] = cnt == 1 ? C[(int64_t)r * n + first] : 0.0;
    if (cnt == 1) atomicAdd(&S.colptr[first + 1], 1);
  }
  __syncthreads();
  if (wid == 0) {
    const unsigned lt = (1u << lane) - 1u;
    // general rows, ascending
    int ng = 0;
    for (int r0 = 0; r0 < m; r0 += 32) {
      const int r = r0 + lane;
      const bool gen = r < m && S.rcol[r] < 0;
      const unsigned bg = __ballot_sync(0xffffffffu, gen);
      if (gen) S.grow[ng + __popc(bg & lt)] = r;
      ng += __popc(bg);
    }
    // column starts: exclusive prefix of the per-column counts in colptr[c + 1]
    int run = 0;
    for (int c0 = 0; c0 <= n; c0 += 32) {
      const int c = c0 + lane;
      int v = c <= n ? S.colptr[c] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += y;
      }
      if (c <= n) S.colptr[c] = run + v;
      run += __shfl_sync(0xffffffffu, v, 31);
    }
    __syncwarp();
    // stable counting sort (ascending rows per column); running offsets in kidx
    for (int c = lane; c < n; c += 32) S.kidx[c] = S.colptr[c];
    __syncwarp();
    for (int r0 = 0; r0 < m; r0 += 32) {
      const int r = r0 + lane;
      const int c = r < m ? S.rcol[r] : -1;
      const unsigned peers = __match_any_sync(0xffffffffu, c);
      if (c >= 0) S.colrows[S.kidx[c] + __popc(peers & lt)] = r;
      __syncwarp();
      if (c >= 0 && (peers & lt) == 0) S.kidx[c] += __popc(peers);
      __syncwarp();
    }
    if (lane == 0) sh_int[0] = ng;
  }
  __syncthreads();
  S.ng = sh_int[0];
  // the ng-vectors (and with them everything placed after them) go on-chip
  // only when the base layout with them still fits; else to the workspace
  const bool gv_smem = qp_layout(n, m, S.ng, false, false).total <= A.smem_bytes;
  {
    double* gv = gv_smem ? (double*)(smem + qp_layout(n, m, S.ng, false, false).o_gv)
                         : gws + packed_size(n) + (int64_t)m * n;
    S.wg = gv;
    S.ga = gv + S.ng;
    S.cf = gv + 2 * S.ng;
  }
  // ---- eliminable variables: diagonal-only Hessian row (elig, from the H
  // pass), at most one general row, and alone in that row (otherwise K_ee
  // would not be diagonal)
#pragma unroll 1
  for (int c = tid; c < n; c += nt) {
    if (!S.elig[c]) { S.egi[c] = -1; continue; }
    int cnt = 0, gs = -1;
    for (int gi = 0; gi < S.ng; ++gi)
      if (C[(int64_t)S.grow[gi] * n + c] != 0.0) { ++cnt; gs = gi; }
    S.egi[c] = gs;  // temporarily indexed by column
    if (cnt > 1) S.elig[c] = 0;
  }
#pragma unroll 1
  for (int gi = tid; gi < S.ng; gi += nt) S.ge[gi] = 0;
  __syncthreads();
#pragma unroll 1
  for (int c = tid; c < n; c += nt)  // rows meeting several candidates keep them all
    if (S.elig[c] && S.egi[c] >= 0) atomicAdd(&S.ge[S.egi[c]], 1);
  __syncthreads();
#pragma unroll 1
  for (int c = tid; c < n; c += nt)
    if (S.elig[c] && S.egi[c] >= 0 && S.ge[S.egi[c]] > 1) S.elig[c] = 0;
  __syncthreads();
  if (wid == 0) {
    const unsigned lt = (1u << lane) - 1u;
    for (int gi = lane; gi < S.ng; gi += 32) S.ge[gi] = -1;
    __syncwarp();
    int nf = 0, ne = 0;
    for (int c0 = 0; c0 < n; c0 += 32) {
      const int c = c0 + lane;
      const bool el = c < n && S.elig[c] != 0;
      const int gs = el ? S.egi[c] : -1;
      const unsigned be = __ballot_sync(0xffffffffu, el);
      const unsigned bk = __ballot_sync(0xffffffffu, c < n && !el);
      if (el) {
        const int e = ne + __popc(be & lt);
        S.eidx[e] = c;
        S.hde[e] = H[(int64_t)c * n + c];
        if (gs >= 0) {
          const double a = C[(int64_t)S.grow[gs] * n + c];
          S.ge[gs] = e;
          S.ga[gs] = a;
          S.ea[e] = a;
        } else {
          S.ea[e] = 0.0;
        }
        S.elig[e] = gs;  // egi by eliminated index, staged (e <= c: slots already read)
      } else if (c < n) {
        S.kidx[nf + __popc(bk & lt)] = c;
      }
      ne += __popc(be);
      nf += __popc(bk);
      __syncwarp();
    }
    for (int e = lane; e < ne; e += 32) S.egi[e] = S.elig[e];
    if (lane == 0) {
      sh_int[2] = nf;
      sh_int[3] = ne;
    }
  }
  __syncthreads();
  S.nf = sh_int[2];
  S.ne = sh_int[3];
  S.nblk = (S.nf + kTB - 1) / kTB;
  {
    const bool cg_smem = qp_layout(n, m, S.ng, false, true, S.nf, gv_smem).total <= A.smem_bytes;
    const bool h_smem = qp_layout(n, m, S.ng, true, cg_smem, S.nf, gv_smem).total <= A.smem_bytes;
    const QpLayout LY = qp_layout(n, m, S.ng, h_smem, cg_smem, S.nf, gv_smem);
    S.K = (double*)(smem + LY.o_k);
    S.X = (double*)(smem + LY.o_x);
    S.T = qpchol::tiles_for(S.nf);
    S.scr = S.X + S.T * qpchol::kTS;
    S.dinv = S.scr + 64 * kQpWarps;
    S.yv = S.dinv + 8 * S.T;
    S.Cg = cg_smem ? (double*)(smem + LY.o_cg) : gws + packed_size(n);
    S.Hp = h_smem ? (double*)(smem + LY.o_h) : gws;
  }
  for (int t = tid; t < 16 * S.T; t += nt) S.yv[t] = 0.0;
  {
    __shared__ unsigned short tij[32 * 33 / 2];
    for (int t = tid; t < S.T * (S.T + 1) / 2; t += nt) {
      int I = 0;
      while ((I + 1) * (I + 2) / 2 <= t) ++I;
      tij[t] = (unsigned short)((I << 8) | (t - I * (I + 1) / 2));
    }
    S.tij = tij;
  }
  // general rows, column-permuted to the kept variables
  for (int t = tid; t < S.ng * S.nf; t += nt) {
    const int gi = t / S.nf, k = t - gi * S.nf;
    S.Cg[(int64_t)gi * n + k] = C[(int64_t)S.grow[gi] * n + S.kidx[k]];
  }
  // pack H's lower triangle over the kept variables
  for (int kr = wid; kr < S.nf; kr += kQpWarps) {
    const double* Hr = H + (int64_t)S.kidx[kr] * n;
    for (int kc = lane; kc <= kr; kc += 32) S.Hp[colbase(kc, S.nf) + kr] = Hr[S.kidx[kc]];
  }
#pragma unroll 1
  for (int t = tid; t < n; t += nt) S.g[t] = A.g[bi * (int64_t)n + t];
#pragma unroll 1
  for (int t = tid; t < m; t += nt) S.d[t] = A.d[bi * (int64_t)m + t];
  __syncthreads();

  // scale references (qpsolver.py:124-127)
  double hmax = hmax_loc, gmax = 0.0;
#pragma unroll 1
  for (int t = tid; t < n; t += nt) gmax = fmax(gmax, fabs(S.g[t]));
  hmax = block_reduce<0>(hmax, red);
  gmax = block_reduce<0>(gmax, red);
  const double norm_g = gmax;
  const double scale_k = fmin(1.0, fmax(hmax, norm_g));
  const double scale_g = scale_k + norm_g;
  const double comp_ref = scale_k;
  const double tol = A.tol, reg = A.reg, tau = A.tau;
  double* uo = A.u_out + bi * (int64_t)n;
  double* lo = A.lam_out + bi * (int64_t)m;

  // ---- unconstrained problems (qpsolver.py:131-144)
  if (m == 0) {
    bool ok = false;
    for (int t = 0; t < 4 && !ok; ++t) {
      const double boost = t == 0 ? 0.0 : (t == 1 ? reg : (t == 2 ? reg * 1e3 : reg * 1e6));
      build_k(S, boost, false);
      ok = chol_factor(S);
    }
    if (!ok) {
#pragma unroll 1
      for (int t = tid; t < n; t += nt) uo[t] = 0.0;
      if (tid == 0) {
        A.status[bi] = GM_QP_NUMERICAL_FAILURE;
        A.iters[bi] = 0;
        A.resid[bi * 3 + 0] = A.resid[bi * 3 + 1] = A.resid[bi * 3 + 2] = INFINITY;
      }
      return;
    }
    invert_diag_blocks(S);
#pragma unroll 1
    for (int t = tid; t < n; t += nt) S.rhs[t] = -S.g[t];
    __syncthreads();
    chol_solve(S, S.rhs, S.u);
    h_apply(S, S.u, S.hu);
    __syncthreads();
    double rs = 0.0;
#pragma unroll 1
    for (int c = tid; c < n; c += nt) rs = fmax(rs, fabs(2.0 * S.hu[c] + S.g[c]));
    rs = block_reduce<0>(rs, red);
#pragma unroll 1
    for (int t = tid; t < n; t += nt) uo[t] = S.u[t];
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
#pragma unroll 1
  for (int t = tid; t < n; t += nt) S.u[t] = A.warm ? A.warm[bi * (int64_t)n + t] : 0.0;
  __syncthreads();
  c_apply(S, S.u, S.cu);
  __syncthreads();
#pragma unroll 1
  for (int r = tid; r < m; r += nt) {
    S.s[r] = fmax(S.d[r] - S.cu[r], 1.0) * 1.1;
    S.lam[r] = 1.0;
  }
  __syncthreads();

  double best_metric = INFINITY, b_rs = 0, b_rp = 0, b_rc = 0;
  double f_rs = 0, f_rp = 0, f_rc = 0;
  int status = -1, iters = 0;
  bool use_best = false;

  qmark(S, 0);
  for (int it = 0; it < A.max_it; ++it) {
    const Resid R = residuals(S);
    qmark(S, 1);
    const double metric = fmax(fmax(R.rs / scale_g, R.rp), R.rc / fmax(comp_ref, 1e-300));
    if (metric < best_metric) {  // record_best (qpsolver.py:158-165)
      best_metric = metric;
      b_rs = R.rs;
      b_rp = R.rp;
      b_rc = R.rc;
#pragma unroll 1
      for (int t = tid; t < n; t += nt) S.ub[t] = S.u[t];
#pragma unroll 1
      for (int t = tid; t < m; t += nt) S.lb[t] = S.lam[t];
    }
    if (R.rs <= tol * scale_g && R.rp <= tol && R.rc <= tol * comp_ref) {
      status = GM_QP_OPTIMAL;
      iters = it;
      f_rs = R.rs;
      f_rp = R.rp;
      f_rc = R.rc;
      break;
    }
    if (R.lmax > 1e12 && R.rp > 1e-6) {
      status = GM_QP_PRIMAL_INFEASIBLE;
      iters = it;
      use_best = true;
      break;
    }
    qmark(S, 2);
    // Schur matrix and Cholesky with escalating regularisation (qpsolver.py:178-198)
#pragma unroll 1
    for (int r = tid; r < m; r += nt) S.w[r] = S.lam[r] / S.s[r];
    __syncthreads();
    // build + factor with escalating regularisation: one copy in the code
    bool ok = false;
    double boost = 0.0;
#pragma unroll 1
    for (int att = 0; att < 4; ++att) {
      if (att > 0) boost = boost == 0.0 ? fmax(reg * 1e3, 1e-12) : boost * 1e3;
      ok = build_k(S, reg + boost, true);
      if (att == 0) qmark(S, 3);
      ok = ok && chol_factor(S);
      if (att == 0) qmark(S, 4);
      if (ok) break;
    }
    if (!ok) {
      status = GM_QP_NUMERICAL_FAILURE;
      iters = it;
      use_best = true;
      break;
    }
    invert_diag_blocks(S);
    __syncthreads();
    qmark(S, 5);
    // r_pri = C u + s - d and mu = lam.s / m came with the residuals
    const double mu = R.musum / m;
    // affine direction (rc = -lam s), then the corrector with centring (rc =
    // -lam s - dlam_a ds_a + sigma mu): one copy of the KKT step in the code,
    // run twice (the instruction working set of an iteration)
#pragma unroll 1
    for (int r = tid; r < m; r += nt) S.tmp[r] = -S.lam[r] * S.s[r];
    __syncthreads();
    qmark(S, 6);
#pragma unroll 1
    for (int pass = 0; pass < 2; ++pass) {
      kkt_step(S, S.tmp);
      qmark(S, 7);
      if (pass == 1) break;
      double ap, ad;
      max_step2(S, ap, ad);
      double maff = 0.0;
#pragma unroll 1
      for (int r = tid; r < m; r += nt) maff += (S.lam[r] + ad * S.dl[r]) * (S.s[r] + ap * S.ds[r]);
      const double mu_aff = block_reduce<2>(maff, red) / m;
      const double sigma = mu > 0.0 ? (mu_aff / mu) * (mu_aff / mu) * (mu_aff / mu) : 0.0;
#pragma unroll 1
      for (int r = tid; r < m; r += nt) S.tmp[r] = -S.lam[r] * S.s[r] - S.dl[r] * S.ds[r] + sigma * mu;
      __syncthreads();
      qmark(S, 8);
    }
    double ap_f, ad_f;
    max_step2(S, ap_f, ad_f);
    const double alpha = fmin(tau * ap_f, tau * ad_f);
    bool finite = true;
#pragma unroll 1
    for (int c = tid; c < n; c += nt) {
      S.u[c] = S.u[c] + alpha * S.du[c];
      if (!isfinite(S.u[c])) finite = false;
    }
#pragma unroll 1
    for (int r = tid; r < m; r += nt) {
      S.s[r] = S.s[r] + alpha * S.ds[r];
      S.lam[r] = S.lam[r] + alpha * S.dl[r];
      if (!isfinite(S.s[r]) || !isfinite(S.lam[r])) finite = false;
    }
    const int all_finite = __syncthreads_and(finite ? 1 : 0);
    qmark(S, 9);
    if (!all_finite) {
      status = GM_QP_NUMERICAL_FAILURE;
      iters = it + 1;
      use_best = true;
      break;
    }
  }
  if (status < 0) {  // iteration cap (qpsolver.py:231-235)
    const Resid R = residuals(S);
    const double metric = fmax(fmax(R.rs / scale_g, R.rp), R.rc / fmax(comp_ref, 1e-300));
    if (metric < best_metric) {
      best_metric = metric;
      b_rs = R.rs;
      b_rp = R.rp;
      b_rc = R.rc;
#pragma unroll 1
      for (int t = tid; t < n; t += nt) S.ub[t] = S.u[t];
#pragma unroll 1
      for (int t = tid; t < m; t += nt) S.lb[t] = S.lam[t];
    }
    iters = A.max_it;
    if (R.rs <= tol * scale_g && R.rp <= tol && R.rc <= tol * comp_ref) {
      status = GM_QP_OPTIMAL;
      f_rs = R.rs;
      f_rp = R.rp;
      f_rc = R.rc;
    } else {
      status = GM_QP_MAX_ITERATIONS;
      use_best = true;
    }
  }
  __syncthreads();
  const double* us = use_best ? S.ub : S.u;
  const double* ls = use_best ? S.lb : S.lam;
#pragma unroll 1
  for (int t = tid; t < n; t += nt) uo[t] = us[t];
#pragma unroll 1
  for (int t = tid; t < m; t += nt) lo[t] = ls[t];
  if (tid == 0) {
    A.status[bi] = status;
    A.iters[bi] = iters;
    A.resid[bi * 3 + 0] = use_best ? b_rs : f_rs;
    A.resid[bi * 3 + 1] = use_best ? b_rp : f_rp;
    A.resid[bi * 3 + 2] = use_best ? b_rc : f_rc;
  }
}

// Diagnostic kernel: factor a dense SPD A (n x n) with the solver's own
// chol_factor / invert_diag_blocks / chol_solve and return L and A^{-1} b.
__global__ void __launch_bounds__(kQpThreads, 1) k_chol_check(int n, const double* A, const double* b,
                                                               double* L, double* x, int* ok) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ int sh_int[4];
  Qs S;
  S.n = n;
  S.nf = n;
  S.ne = 0;
  S.m = 0;
  S.ng = 0;
  S.T = qpchol::tiles_for(n);
  S.flag = &sh_int[1];
  S.prof = false;
  const QpLayout L0 = qp_layout(n, 0, 0, false, false);
  double* v = (double*)(smem + L0.o_vec);
  S.rhs = v;
  S.du = v + n;
  S.K = (double*)(smem + L0.o_k);
  S.X = (double*)(smem + L0.o_x);
  S.scr = S.X + S.T * qpchol::kTS;
  S.dinv = S.scr + 64 * kQpWarps;
  S.yv = S.dinv + 8 * S.T;
  for (int t = threadIdx.x; t < 16 * S.T; t += blockDim.x) S.yv[t] = 0.0;
  for (int e = threadIdx.x; e < 64 * S.T * S.T; e += blockDim.x) {
    const int r = e / (8 * S.T), c = e - r * (8 * S.T);
    if (c > r) continue;
    S.K[qpchol::gel(r, c)] = (r < n && c < n) ? A[(int64_t)r * n + c] : (r == c ? 1.0 : 0.0);
  }
#pragma unroll 1
  for (int r = threadIdx.x; r < n; r += blockDim.x) S.rhs[r] = b[r];
  __syncthreads();
  const bool good = chol_factor(S);
  if (threadIdx.x == 0) *ok = good ? 1 : 0;
  if (!good) return;
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
    const int r = e / n, c = e - r * n;
    L[e] = r >= c ? S.K[qpchol::gel(r, c)] : 0.0;
  }
  __syncthreads();
  invert_diag_blocks(S);
  __syncthreads();
  chol_solve(S, S.rhs, S.du);
#pragma unroll 1
  for (int r = threadIdx.x; r < n; r += blockDim.x) x[r] = S.du[r];
}

}  // namespace

extern "C" int gm_chol_check(gm_ctx* ctx, int n, const double* A, const double* b, double* L,
                             double* x, int32_t* ok, void* stream) {
  int rc = gm_need_device(ctx);
  if (rc) return rc;
  if (n < 1 || n > 256) return gm_fail(ctx, GM_ERR_CONFIG, "n must be in [1, 256]");
  const size_t sm = qp_layout(n, 0, 0, false, false).total;
  if (sm > ctx->smem_optin) return gm_fail(ctx, GM_ERR_CONFIG, "matrix too large for the on-chip factorisation");
  GM_CUDA(ctx, cudaFuncSetAttribute(k_chol_check, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  k_chol_check<<<1, kQpThreads, sm, (cudaStream_t)stream>>>(n, A, b, L, x, ok);
  GM_LAUNCH_CHECK(ctx, "k_chol_check");
  return GM_OK;
}

extern "C" int gm_qp_profile(int on) {
  if (on && !kQpProf) return GM_ERR_CONFIG;  // built without -DGM_QP_PROF
  const int split = on == 2 ? 1 : 0;
  on = on != 0 ? 1 : 0;
  cudaMemcpyToSymbol(g_qp_prof_on, &on, sizeof(int));
  cudaMemcpyToSymbol(g_qp_chol_split, &split, sizeof(int));
  unsigned long long z[16] = {0};
  cudaMemcpyToSymbol(g_qp_prof, z, sizeof(z));
  return GM_OK;
}

extern "C" int gm_qp_phase_cycles(unsigned long long* out) {
  return cudaMemcpyFromSymbol(out, g_qp_prof, sizeof(unsigned long long) * 16) == cudaSuccess
             ? GM_OK
             : GM_ERR_CUDA;
}

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
  // vectors, the packed Schur matrix and the inverted diagonal blocks always
  // live on-chip; general rows, then packed H, go on-chip when room is left
  const size_t cap = ctx->smem_optin - 2048;  // static shared arrays of the kernel
  const QpLayout base = qp_layout(n, m, 0, false, false);
  if (base.total > cap) return gm_fail(ctx, GM_ERR_CONFIG, "QP too large for the on-chip solver");
  const size_t smem_bytes = std::min(cap, qp_layout(n, m, m, true, true).total);
  const int64_t gws_stride = packed_size(n) + (int64_t)m * n + 3 * (int64_t)m;
  double* gws = (double*)gm_scratch(ctx, sizeof(double) * (size_t)gws_stride * B);
  if (!gws) return gm_fail(ctx, GM_ERR_CUDA, "QP workspace allocation failed");
  QpArgs a{};
  a.n = n;
  a.m = m;
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
  if (n > 256) return gm_fail(ctx, GM_ERR_CONFIG, "QP with n > 256 variables is not supported by this build");
  GM_CUDA(ctx, cudaFuncSetAttribute(k_solve_qp, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_bytes));
  k_solve_qp<<<B, kQpThreads, smem_bytes, (cudaStream_t)stream>>>(a);
  GM_LAUNCH_CHECK(ctx, "k_solve_qp");
  return GM_OK;
}
