// Tiled fp64 Cholesky factorisation and triangular solves for K-QP (one CTA
// per QP, whole matrix on chip).
//
// Storage.  The n x n SPD matrix is padded to 8T x 8T (T = ceil(n/8)) with an
// identity block and held as its lower 8x8 tiles (I >= J) in shared memory,
// row-major tile order ti(I, J) = I(I+1)/2 + J, tile stride kTS doubles.
// Inside a tile, element (r, c) sits at c*8 + (r ^ ((c & 2) << 1)): column
// major with a 4-row swizzle on columns 2,3,6,7 so the DMMA fragment loads of
// the trailing update hit distinct banks; kTS = 72 (a multiple of 8 but not
// of 16) keeps row-per-thread accesses of consecutive tiles conflict free.
//
// Factorisation (right-looking, 8-column steps, look-ahead depth 1).  The
// critical path of a small Cholesky is the chain of pivots: rsqrt of the
// updated diagonal -> scale -> update of the next diagonal.  Measured B200
// latencies (scripts/ubench_latency.cu): dependent DFMA 23 cycles, rsqrt(f64)
// 84, double shuffle 54, so one pivot costs ~130 cycles when a single thread
// holds the whole 8x8 pivot tile in registers and nothing else is on the path.
// Step k:
//   warp 0  : panel rows of tile (k+1, k) [x = w L_kk^{-T}], publishes them
//             (named barrier arrive), updates tile (k+1, k+1) with them and
//             lane 0 factors it (8 pivots in registers);
//   warps 1+: panel rows of tiles (I, k), I >= k+2, wait for warp 0's rows,
//             then the rank-8 trailing update C_IJ -= P_I P_J' of every tile
//             k+1 <= J <= I < T except (k+1, k+1), on the fp64 tensor cores
//             (mma.sync m8n8k4 f64, 2 per tile), 4 tiles in flight per warp;
//   one CTA barrier per step.
// The trailing work of a step (<= ~1000 cycles at T = 15) hides under warp
// 0's chain (~1500 cycles), so a factorisation costs ~T chains.
#pragma once

#include <cuda_runtime.h>

namespace qpchol {

constexpr int kTS = 72;  // tile stride (doubles)

// Pointers into shared memory that travel through structs / non-inlined
// calls lose their address space and compile to generic LD/ST; asserting it
// restores LDS/STS.
#define QP_SMEM(p) __builtin_assume(__isShared(p))

__device__ __forceinline__ int ti(int I, int J) { return ((I * (I + 1)) >> 1) + J; }
__device__ __forceinline__ int eo(int r, int c) { return c * 8 + (r ^ ((c & 2) << 1)); }
// element (R, C) with R >= C of the padded matrix
__device__ __forceinline__ int gel(int R, int C) { return ti(R >> 3, C >> 3) * kTS + eo(R & 7, C & 7); }
__host__ __device__ inline int tiles_for(int n) { return (n + 7) >> 3; }
__host__ __device__ inline int tile_doubles(int n) {
  const int T = tiles_for(n);
  return T * (T + 1) / 2 * kTS;
}

__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}
__device__ __forceinline__ void bar_arrive(int id, int nthreads) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
__device__ __forceinline__ void bar_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// Factor the 8x8 lower tile held in a[r][c] (r >= c) in place: a[r][c] <- L,
// d[j] <- 1/L[j][j].  False on a non-positive / NaN pivot (potrf's rule).
__device__ __forceinline__ bool factor8(double (&a)[8][8], double (&d)[8]) {
  bool ok = true;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const double p = a[j][j];
    if (!(p > 0.0)) ok = false;
    const double r = rsqrt(p);
    d[j] = r;
    a[j][j] = p * r;
#pragma unroll
    for (int i = j + 1; i < 8; ++i) a[i][j] *= r;
#pragma unroll
    for (int i = j + 1; i < 8; ++i)
#pragma unroll
      for (int c = j + 1; c <= i; ++c) a[i][c] = fma(-a[i][j], a[c][j], a[i][c]);
  }
  return ok;
}

// x = w L^{-T} for one row w of a panel tile, L = tile Lt (factored), d = 1/diag
__device__ __forceinline__ void panel_row(const double* Lt, const double* d, double (&w)[8]) {
  double l[8][8];
#pragma unroll
  for (int q = 1; q < 8; ++q)
#pragma unroll
    for (int p = 0; p < q; ++p) l[q][p] = Lt[eo(q, p)];
#pragma unroll
  for (int p = 0; p < 8; ++p) {
    w[p] *= d[p];
#pragma unroll
    for (int q = p + 1; q < 8; ++q) w[q] = fma(-l[q][p], w[p], w[q]);
  }
}

__device__ __forceinline__ void load_row(const double* t, int r, double (&w)[8]) {
#pragma unroll
  for (int q = 0; q < 8; ++q) w[q] = t[eo(r, q)];
}
__device__ __forceinline__ void store_row(double* t, int r, const double (&w)[8]) {
#pragma unroll
  for (int q = 0; q < 8; ++q) t[eo(r, q)] = w[q];
}

// Lower pair (a, b), a >= b, of the 36 entries of an 8x8 lower triangle.
__device__ __forceinline__ void pair36(int l, int& a, int& b) {
  // rows: 0:1 entry, 1:2, ... 7:8 -> cumulative 1,3,6,10,15,21,28,36
  a = (l >= 1) + (l >= 3) + (l >= 6) + (l >= 10) + (l >= 15) + (l >= 21) + (l >= 28);
  b = l - ((a * (a + 1)) >> 1);
}

// Rank-8 trailing update of step k: C_IJ -= P_I P_J' for every tile
// k+1 <= J <= I < T except (k+1, k+1), P_I = tile (I, k).  Tiles are
// enumerated column by column and dealt round-robin to the NU update warps
// (uw = this warp's rank), 4 tiles in flight per warp.  The transposed tile
// C' = P_J P_I' is accumulated: its DMMA C fragment (row i, cols 2p, 2p+1) is
// C[2p..2p+1][i], two adjacent entries of column i, so C moves with
// conflict-free 128-bit accesses; the P fragments are conflict free through
// the swizzle.
template <int NU, int NB = 6>
__device__ __forceinline__ void trailing_update(double* Kt, int T, int k, int uw, int lane) {
  QP_SMEM(Kt);
  const int i = lane >> 2, p = lane & 3;
  int I = k + 2, J = k + 1;  // first tile after (k+1, k+1)
  auto adv = [&](int s) {
    I += s;
    while (J < T && I >= T) {
      I -= T - (J + 1);
      ++J;
    }
  };
  adv(uw);
  while (J < T) {
    int off[NB], cnt = 0;
    double a0[NB], a1[NB], b0[NB], b1[NB];
    double2 cv[NB];
#pragma unroll
    for (int u = 0; u < NB; ++u) {
      if (J < T) {
        const double* PI = Kt + ti(I, k) * kTS;
        const double* PJ = Kt + ti(J, k) * kTS;
        off[u] = ti(I, J) * kTS + eo(2 * p, i);
        a0[u] = -PJ[eo(i, p)];
        a1[u] = -PJ[eo(i, p + 4)];
        b0[u] = PI[eo(i, p)];
        b1[u] = PI[eo(i, p + 4)];
        cv[u] = *reinterpret_cast<const double2*>(Kt + off[u]);
        ++cnt;
        adv(NU);
      }
    }
#pragma unroll
    for (int u = 0; u < NB; ++u)
      if (u < cnt) dmma884(cv[u].x, cv[u].y, a0[u], b0[u]);
#pragma unroll
    for (int u = 0; u < NB; ++u)
      if (u < cnt) dmma884(cv[u].x, cv[u].y, a1[u], b1[u]);
#pragma unroll
    for (int u = 0; u < NB; ++u)
      if (u < cnt) *reinterpret_cast<double2*>(Kt + off[u]) = cv[u];
  }
}

// Factor the padded SPD matrix in Kt (T x T lower tiles) in place.  dinv
// (8T) receives 1/L[j][j].  flag: shared int, zero on entry.  All NT threads
// call; returns false (uniformly) on a failed pivot.
template <int NT>
__device__ __noinline__ bool factor(double* Kt, int T, double* dinv, int* flag, long long* prof = nullptr) {
  QP_SMEM(Kt);
  QP_SMEM(dinv);
  QP_SMEM(flag);
  constexpr int NW = NT / 32;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  long long pr[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  if (tid == 0) {
    double a[8][8], d[8];
    double* t = Kt;
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int c = 0; c <= r; ++c) a[r][c] = t[eo(r, c)];
    if (!factor8(a, d)) *flag = 1;
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      dinv[r] = d[r];
#pragma unroll
      for (int c = 0; c <= r; ++c) t[eo(r, c)] = a[r][c];
    }
  }
  __syncthreads();
  for (int k = 0; k < T; ++k) {
    if (*flag) return false;
    if (k + 1 >= T) break;
    const double* Lkk = Kt + ti(k, k) * kTS;
    const double* dk = dinv + 8 * k;
    const long long t0 = prof ? clock64() : 0;
    if (wid == 0) {
      double* P = Kt + ti(k + 1, k) * kTS;
      if (lane < 8) {
        double w[8];
        load_row(P, lane, w);
        panel_row(Lkk, dk, w);
        store_row(P, lane, w);
      }
      __syncwarp();
      __threadfence_block();
      if (prof && lane == 0) pr[0] += clock64() - t0;
      bar_arrive(1, NT);
      // E = A_{k+1,k+1} - P P'  (36 lower entries over 32 lanes)
      double* Dt = Kt + ti(k + 1, k + 1) * kTS;
      {
        // lanes 0..31 own entry lane, lanes 0..3 also entry 32 + lane; both
        // dot products run with independent accumulators
        int ra, ca, rb, cb;
        pair36(lane, ra, ca);
        pair36(32 + (lane & 3), rb, cb);
        double x0 = Dt[eo(ra, ca)], x1 = 0.0, y0 = Dt[eo(rb, cb)], y1 = 0.0;
#pragma unroll
        for (int q = 0; q < 8; q += 2) {
          x0 = fma(-P[eo(ra, q)], P[eo(ca, q)], x0);
          x1 = fma(-P[eo(ra, q + 1)], P[eo(ca, q + 1)], x1);
          y0 = fma(-P[eo(rb, q)], P[eo(cb, q)], y0);
          y1 = fma(-P[eo(rb, q + 1)], P[eo(cb, q + 1)], y1);
        }
        Dt[eo(ra, ca)] = x0 + x1;
        if (lane < 4) Dt[eo(rb, cb)] = y0 + y1;
      }
      __syncwarp();
      if (prof && lane == 0) pr[1] += clock64() - t0;
      if (lane == 0) {
        double a[8][8], d[8];
#pragma unroll
        for (int r = 0; r < 8; ++r)
#pragma unroll
          for (int c = 0; c <= r; ++c) a[r][c] = Dt[eo(r, c)];
        if (!factor8(a, d)) *flag = 1;
#pragma unroll
        for (int r = 0; r < 8; ++r) {
          dinv[8 * (k + 1) + r] = d[r];
#pragma unroll
          for (int c = 0; c <= r; ++c) Dt[eo(r, c)] = a[r][c];
        }
        if (prof) pr[2] += clock64() - t0;
      }
    } else {
      // panel rows of tiles I >= k+2
      const int rows = 8 * (T - k - 2);
      for (int t = tid - 32; t < rows; t += NT - 32) {
        double* P = Kt + ti(k + 2 + (t >> 3), k) * kTS;
        double w[8];
        load_row(P, t & 7, w);
        panel_row(Lkk, dk, w);
        store_row(P, t & 7, w);
      }
      if (prof && tid == 32) pr[3] += clock64() - t0;
      bar_sync(1, NT);
      if (prof && tid == 32) pr[4] += clock64() - t0;
      // Warps sharing warp 0's sub-partition (wid % 4 == 0) stay off the
      // FP64 pipe: a DMMA holds it ~16 cycles and would stall the pivot
      // chain's dependent DFMAs.
#ifndef CHOL_SKIP_TRAIL
      if ((wid & 3) != 0) trailing_update<NW - NW / 4>(Kt, T, k, wid - 1 - (wid >> 2), lane);
#endif
      if (prof && lane == 0) pr[5] += clock64() - t0;
    }
    __syncthreads();
    if (prof && tid == 0) pr[7] += clock64() - t0;
  }
  if (prof) {
    if (tid == 0)
      for (int q : {0, 1, 2, 7}) prof[q] = pr[q];
    if (tid == 32)
      for (int q : {3, 4}) prof[q] = pr[q];
    if (lane == 0 && wid > 0) atomicMax((unsigned long long*)&prof[5 + (wid & 1)], (unsigned long long)pr[5]);
  }
  return !*flag;
}

// ---------------------------------------------------------------------------
// Triangular solves through inverted 32 x 32 diagonal superblocks
// ---------------------------------------------------------------------------
// Superblock s covers tiles 4s..4s+3 (rows 32s..32s+31).  X holds, per
// superblock, the 10 lower tiles of X_s = L_ss^{-1} (local tile index
// ti(a, b), a >= b, same in-tile layout; the strict upper part of its
// diagonal tiles is zero).  With X a solve is NSB = ceil(T/4) short steps:
//   forward  y_s = X_s (b_s - sum_{c<s} L_sc y_c),
//   backward x_s = X_s' (y_s - sum_{c>s} L_cs' x_c),
// each a 32-term dot per row by one warp plus a parallel update of the
// remaining rows.
__host__ __device__ inline int superblocks_for(int n) { return (tiles_for(n) + 3) >> 2; }
__host__ __device__ inline int xinv_doubles(int n) { return superblocks_for(n) * 10 * kTS; }

// X_s tiles.  Phase 1: inverse of every diagonal 8x8 tile, one thread per
// (tile, column), forward substitution with progressive accumulation.
// Phase 2: off-diagonal tiles by levels d = a - b = 1, 2, 3:
//   X(a, b) = -Linv_a * sum_{m=b}^{a-1} L(a, m) X(m, b),
// one warp per tile on the fp64 tensor cores (the partial sum is staged in a
// per-warp scratch tile to become a B operand).  scratch: NW * 64 doubles.
template <int NT>
__device__ __noinline__ void invert_superblocks(const double* Kt, int T, const double* dinv, double* X, double* scratch) {
  QP_SMEM(Kt);
  QP_SMEM(dinv);
  QP_SMEM(X);
  QP_SMEM(scratch);
  constexpr int NW = NT / 32;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  for (int t = tid; t < 8 * T; t += NT) {
    const int k = t >> 3, c = t & 7;
    const double* L = Kt + ti(k, k) * kTS;
    double* Xt = X + ((k >> 2) * 10 + ti(k & 3, k & 3)) * kTS;
    double x[8], acc[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      x[r] = 0.0;
      acc[r] = 0.0;
    }
#pragma unroll
    for (int p = 0; p < 8; ++p) {
      if (p == c) x[p] = dinv[8 * k + p];
      if (p > c) x[p] = -dinv[8 * k + p] * acc[p];
      if (p >= c) {
#pragma unroll
        for (int r = p + 1; r < 8; ++r) acc[r] = fma(L[eo(r, p)], x[p], acc[r]);
      }
    }
#pragma unroll
    for (int r = 0; r < 8; ++r) Xt[eo(r, c)] = x[r];
  }
  __syncthreads();
  const int NSB = (T + 3) >> 2;
  const int i = lane >> 2, p = lane & 3;
  double* W = scratch + wid * 64;
  for (int d = 1; d < 4; ++d) {
    // tasks: (superblock s, local column b) with b + d < min(4, T - 4s)
    const int per = 4 - d;
    for (int task = wid; task < NSB * per; task += NW) {
      const int s = task / per, b = task - s * per, a = b + d;
      if (4 * s + a >= T) continue;
      double* Xs = X + s * 10 * kTS;
      double w0 = 0.0, w1 = 0.0;
      for (int m = b; m < a; ++m) {
        const double* L = Kt + ti(4 * s + a, 4 * s + m) * kTS;  // A = L(a, m)
        const double* Xm = Xs + ti(m, b) * kTS;                  // B = X(m, b)
#pragma unroll
        for (int h = 0; h < 8; h += 4) dmma884(w0, w1, L[eo(i, p + h)], Xm[eo(p + h, i)]);
      }
      // W (C fragment: row i, cols 2p, 2p+1) -> scratch -> B fragments
      W[eo(i, 2 * p)] = w0;
      W[eo(i, 2 * p + 1)] = w1;
      __syncwarp();
      const double* La = Xs + ti(a, a) * kTS;  // Linv_a
      double x0 = 0.0, x1 = 0.0;
#pragma unroll
      for (int h = 0; h < 8; h += 4) dmma884(x0, x1, -La[eo(i, p + h)], W[eo(p + h, i)]);
      double* Xab = Xs + ti(a, b) * kTS;
      Xab[eo(i, 2 * p)] = x0;
      Xab[eo(i, 2 * p + 1)] = x1;
      __syncwarp();
    }
    __syncthreads();
  }
}

// In-place forward solve L y = y (y: shared, 8T entries, padding zero).
// stage: 32 doubles.  All NT threads call.
template <int NT>
__device__ __noinline__ void solve_fwd(const double* Kt, int T, const double* X, double* y, double* stage) {
  QP_SMEM(Kt);
  QP_SMEM(X);
  QP_SMEM(y);
  const int tid = threadIdx.x, lane = tid & 31;
  const int NSB = (T + 3) >> 2, N8 = 8 * T;
  for (int s = 0; s < NSB; ++s) {
    const int r0 = 32 * s, nb = min(32, N8 - r0);
    if (tid < 32) {
      const double* Xs = X + s * 10 * kTS;
      double v = 0.0;
      if (lane < nb) {
        const int a = lane >> 3, r = lane & 7;
        double c0 = 0.0, c1 = 0.0, c2 = 0.0, c3 = 0.0;
        for (int m = 0; m <= a; ++m) {
          const double* Xt = Xs + ti(a, m) * kTS;
          const double* yy = y + r0 + 8 * m;
          c0 = fma(Xt[eo(r, 0)], yy[0], c0);
          c1 = fma(Xt[eo(r, 1)], yy[1], c1);
          c2 = fma(Xt[eo(r, 2)], yy[2], c2);
          c3 = fma(Xt[eo(r, 3)], yy[3], c3);
          c0 = fma(Xt[eo(r, 4)], yy[4], c0);
          c1 = fma(Xt[eo(r, 5)], yy[5], c1);
          c2 = fma(Xt[eo(r, 6)], yy[6], c2);
          c3 = fma(Xt[eo(r, 7)], yy[7], c3);
        }
        v = (c0 + c1) + (c2 + c3);
      }
      __syncwarp();
      if (lane < nb) y[r0 + lane] = v;
    }
    __syncthreads();
    if (s + 1 == NSB) break;
    // rows below: y_r -= L[r][r0 .. r0+31] y[r0 ..], two threads per row
    const int rows = N8 - (r0 + 32);
    for (int t0 = 0; t0 < 2 * rows; t0 += NT) {  // warp-uniform trip count (shuffle below)
      const int t = t0 + tid;
      const bool live = t < 2 * rows;
      const int r = r0 + 32 + (live ? t >> 1 : 0), half = t & 1;
      const int R = r >> 3, rr = r & 7;
      double c0 = 0.0, c1 = 0.0, c2 = 0.0, c3 = 0.0;
#pragma unroll
      for (int mm = 0; mm < 2 && live; ++mm) {
        const int m = 4 * s + 2 * half + mm;
        const double* Lt = Kt + ti(R, m) * kTS;
        const double* yy = y + 8 * m;
        c0 = fma(Lt[eo(rr, 0)], yy[0], c0);
        c1 = fma(Lt[eo(rr, 1)], yy[1], c1);
        c2 = fma(Lt[eo(rr, 2)], yy[2], c2);
        c3 = fma(Lt[eo(rr, 3)], yy[3], c3);
        c0 = fma(Lt[eo(rr, 4)], yy[4], c0);
        c1 = fma(Lt[eo(rr, 5)], yy[5], c1);
        c2 = fma(Lt[eo(rr, 6)], yy[6], c2);
        c3 = fma(Lt[eo(rr, 7)], yy[7], c3);
      }
      double v = (c0 + c1) + (c2 + c3);
      v += __shfl_xor_sync(0xffffffffu, v, 1);
      if (live && !half) y[r] -= v;
    }
    __syncthreads();
  }
  (void)stage;
}

// In-place backward solve L' x = x.
template <int NT>
__device__ __noinline__ void solve_bwd(const double* Kt, int T, const double* X, double* x) {
  QP_SMEM(Kt);
  QP_SMEM(X);
  QP_SMEM(x);
  const int tid = threadIdx.x, lane = tid & 31;
  const int NSB = (T + 3) >> 2, N8 = 8 * T;
  for (int s = NSB - 1; s >= 0; --s) {
    const int r0 = 32 * s, nb = min(32, N8 - r0), na = (nb + 7) >> 3;
    if (tid < 32) {
      const double* Xs = X + s * 10 * kTS;
      double v = 0.0;
      if (lane < nb) {
        const int b = lane >> 3, c = lane & 7;
        double c0 = 0.0, c1 = 0.0, c2 = 0.0, c3 = 0.0;
        for (int m = b; m < na; ++m) {  // column c of X tiles (m, b)
          const double* Xt = Xs + ti(m, b) * kTS;
          const double* xx = x + r0 + 8 * m;
          c0 = fma(Xt[eo(0, c)], xx[0], c0);
          c1 = fma(Xt[eo(1, c)], xx[1], c1);
          c2 = fma(Xt[eo(2, c)], xx[2], c2);
          c3 = fma(Xt[eo(3, c)], xx[3], c3);
          c0 = fma(Xt[eo(4, c)], xx[4], c0);
          c1 = fma(Xt[eo(5, c)], xx[5], c1);
          c2 = fma(Xt[eo(6, c)], xx[6], c2);
          c3 = fma(Xt[eo(7, c)], xx[7], c3);
        }
        v = (c0 + c1) + (c2 + c3);
      }
      __syncwarp();
      if (lane < nb) x[r0 + lane] = v;
    }
    __syncthreads();
    if (s == 0) break;
    // rows above: x_c -= sum_{r in superblock s} L[r][c] x_r, two threads per row
    const int rows = r0;
    for (int t0 = 0; t0 < 2 * rows; t0 += NT) {
      const int t = t0 + tid;
      const bool live = t < 2 * rows;
      const int c = live ? t >> 1 : 0, half = t & 1;
      const int C = c >> 3, cc = c & 7;
      double c0 = 0.0, c1 = 0.0, c2 = 0.0, c3 = 0.0;
#pragma unroll
      for (int mm = 0; mm < 2; ++mm) {
        const int m = 4 * s + 2 * half + mm;
        if (live && m < T) {
          const double* Lt = Kt + ti(m, C) * kTS;
          const double* xx = x + 8 * m;
          c0 = fma(Lt[eo(0, cc)], xx[0], c0);
          c1 = fma(Lt[eo(1, cc)], xx[1], c1);
          c2 = fma(Lt[eo(2, cc)], xx[2], c2);
          c3 = fma(Lt[eo(3, cc)], xx[3], c3);
          c0 = fma(Lt[eo(4, cc)], xx[4], c0);
          c1 = fma(Lt[eo(5, cc)], xx[5], c1);
          c2 = fma(Lt[eo(6, cc)], xx[6], c2);
          c3 = fma(Lt[eo(7, cc)], xx[7], c3);
        }
      }
      double v = (c0 + c1) + (c2 + c3);
      v += __shfl_xor_sync(0xffffffffu, v, 1);
      if (live && !half) x[c] -= v;
    }
    __syncthreads();
  }
}

}  // namespace qpchol
