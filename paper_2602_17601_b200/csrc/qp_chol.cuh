// Tiled fp64 Cholesky factorisation and triangular solves for K-QP (one CTA
// per QP, whole matrix on chip).
//
// Storage.  The n x n SPD matrix is padded to 8T x 8T (T = ceil(n/8)) with an
// identity block and held as its lower 8x8 tiles (I >= J) in shared memory,
// row-major tile order ti(I, J) = I(I+1)/2 + J, tile stride kTS doubles.
// Inside a tile, element (r, c) sits at eo(r, c): column major with an XOR
// row swizzle per column pair, so DMMA fragments, rows and columns are all
// conflict free; kTS = 72 (a multiple of 8 but not of 16) keeps
// row-per-thread accesses of consecutive tiles conflict free.
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
#ifdef QP_NO_ASSUME
#define QP_SMEM(p) ((void)0)
#else
#define QP_SMEM(p) __builtin_assume(__isShared(p))
#endif

__device__ __forceinline__ int ti(int I, int J) { return ((I * (I + 1)) >> 1) + J; }
// in-tile offset of (r, c): column major, rows XOR-permuted by s(c) =
// {0,0,4,4,2,2,6,6}[c] so that a column (fixed c), a row (fixed r), the DMMA
// A/B fragments (rows 0..3 x cols 0..3 per half warp) and the transposed C
// fragment pairs all hit distinct banks
#ifdef QP_EO_OLD
__device__ __forceinline__ int eo(int r, int c) { return c * 8 + (r ^ ((c & 2) << 1)); }
#else
__device__ __forceinline__ int eo(int r, int c) { return c * 8 + (r ^ (((c & 2) << 1) | ((c & 4) >> 1))); }
#endif
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
  constexpr int NU = NW - NW / 4;  // update warps (off warp 0's sub-partition)
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
      if ((wid & 3) != 0) trailing_update<NU>(Kt, T, k, wid - 1 - (wid >> 2), lane);
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

// One tile of a rank-8 trailing update: C_IJ -= P_I P_J' (P_X = tile (X, k)),
// transposed-C DMMA form of trailing_update.  One warp.
__device__ __forceinline__ void update_tile(double* Kt, int k, int I, int J, int lane) {
  QP_SMEM(Kt);
  const int i = lane >> 2, p = lane & 3;
  const double* PI = Kt + ti(I, k) * kTS;
  const double* PJ = Kt + ti(J, k) * kTS;
  const int off = ti(I, J) * kTS + eo(2 * p, i);
  double2 cv = *reinterpret_cast<const double2*>(Kt + off);
  dmma884(cv.x, cv.y, -PJ[eo(i, p)], PI[eo(i, p)]);
  dmma884(cv.x, cv.y, -PJ[eo(i, p + 4)], PI[eo(i, p + 4)]);
  *reinterpret_cast<double2*>(Kt + off) = cv;
}

// trailing_update without the look-ahead tiles (k+1, k+1), (k+2, k+1) and
// (k+2, k+2): columns J = k+1 and k+2 start at row k+3
template <int NU, int NB = 6>
__device__ __forceinline__ void trailing_update_la(double* Kt, int T, int k, int uw, int lane) {
  QP_SMEM(Kt);
  const int i = lane >> 2, p = lane & 3;
  auto col_start = [&](int J) { return J <= k + 2 ? k + 3 : J; };
  int J = k + 1, I = col_start(k + 1);
  auto adv = [&](int s) {
    I += s;
    while (J < T && I >= T) {
      const int o = I - T;
      ++J;
      I = col_start(J) + o;
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

// Factorisation with a software-pipelined look-ahead (replaces the
// CTA-wide barrier that ended every step of `factor`).  Warp 0 owns the
// pivot chain: at step k it forms panel (k+1, k), E = A(k+1,k+1) - P P' and
// factors it (lane 0).  It needs only tiles (k+1, k) and (k+1, k+1) from the
// previous trailing update, so update warp 0 refreshes those two first and
// signals warp 0 on named barrier 2; the rest of the trailing update overlaps
// warp 0's next pivot step.  Named barriers:
//   1  (NT):  warp 0 arrives after panel (k+1, k); the others sync after
//             their panel rows -> every column-k panel is final
//   2  (64):  update warp 0 arrives after tiles (k+2, k+1), (k+2, k+2);
//             warp 0 syncs before step k+1
//   3/4 (NT, by step parity): warp 0 arrives after factoring tile (k+1, k+1);
//             the others sync at the start of step k+1 (all of them have
//             finished trailing(k) by then, and L_{k+1,k+1} is published).
//             Parity alternation keeps warp 0, which may run one step ahead,
//             from arriving twice on an open barrier phase.
// No early exit inside the loop (the phases must stay balanced): a failed
// pivot raises *flag and the factorisation runs to the end.
template <int NT>
__device__ __noinline__ bool factor_la(double* Kt, int T, double* dinv, int* flag,
                                       unsigned long long* prof = nullptr) {
  QP_SMEM(Kt);
  QP_SMEM(dinv);
  QP_SMEM(flag);
  constexpr int NW = NT / 32;
  constexpr int NU = NW - NW / 4;  // update warps (off warp 0's sub-partition)
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  if (tid == 0) {
    double a[8][8], d[8];
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int c = 0; c <= r; ++c) a[r][c] = Kt[eo(r, c)];
    if (!factor8(a, d)) *flag = 1;
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      dinv[r] = d[r];
#pragma unroll
      for (int c = 0; c <= r; ++c) Kt[eo(r, c)] = a[r][c];
    }
  }
  __syncthreads();
  if (wid == 0) {
    // optional pivot-chain accounting (prof[0..2]: look-ahead wait, panel + E,
    // 8x8 factor + publish), lane 0 of block 0
    const bool pf = prof && lane == 0;
    long long c0 = 0, c1 = 0, c2 = 0;
    for (int k = 0; k + 1 < T; ++k) {
      if (pf) c0 = clock64();
      if (k >= 1) bar_sync(2, 64);  // tiles (k+1, k), (k+1, k+1) refreshed
      if (pf) c1 = clock64();
      const double* Lkk = Kt + ti(k, k) * kTS;
      const double* dk = dinv + 8 * k;
      double* P = Kt + ti(k + 1, k) * kTS;
      if (lane < 8) {
        double w[8];
        load_row(P, lane, w);
        panel_row(Lkk, dk, w);
        store_row(P, lane, w);
      }
      __syncwarp();
      __threadfence_block();
      bar_arrive(1, NT);
      double* Dt = Kt + ti(k + 1, k + 1) * kTS;
      {
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
      if (pf) c2 = clock64();
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
      }
      __syncwarp();
      __threadfence_block();
      bar_arrive(3 + (k & 1), NT);
      if (pf) {
        const long long c3 = clock64();
        atomicAdd(prof + 0, (unsigned long long)(c1 - c0));
        atomicAdd(prof + 1, (unsigned long long)(c2 - c1));
        atomicAdd(prof + 2, (unsigned long long)(c3 - c2));
      }
    }
  } else {
    const int uw = ((wid & 3) != 0) ? wid - 1 - (wid >> 2) : -1;  // trailing-update rank
    for (int k = 0; k + 1 < T; ++k) {
      if (k >= 1) bar_sync(3 + ((k - 1) & 1), NT);  // L_kk published, trailing(k-1) done
      const double* Lkk = Kt + ti(k, k) * kTS;
      const double* dk = dinv + 8 * k;
      const int rows = 8 * (T - k - 2);
      for (int t = tid - 32; t < rows; t += NT - 32) {
        double* P = Kt + ti(k + 2 + (t >> 3), k) * kTS;
        double w[8];
        load_row(P, t & 7, w);
        panel_row(Lkk, dk, w);
        store_row(P, t & 7, w);
      }
      bar_sync(1, NT);
      if (uw == 0 && k + 2 < T) {  // the look-ahead tiles of warp 0's next step
        update_tile(Kt, k, k + 2, k + 1, lane);
        update_tile(Kt, k, k + 2, k + 2, lane);
        __syncwarp();
        __threadfence_block();
        bar_arrive(2, 64);
      }
      if (uw >= 0) trailing_update_la<NU>(Kt, T, k, uw, lane);
    }
    if (T >= 2) bar_sync(3 + ((T - 2) & 1), NT);  // consume warp 0's last arrival
  }
  __syncthreads();
  return !*flag;
}

// ---------------------------------------------------------------------------
// Full inverse X = L^{-1} in place, and triangular solves as mat-vecs
// ---------------------------------------------------------------------------
// Row wavefront: after row I is processed, tile (I, I) holds Linv_I and tiles
// (I, J < I) hold X_IJ = -Linv_I * sum_{K=J}^{I-1} L_IK X_KJ.  Row I only reads
// row I of L (still intact) and the finished X rows above, so it can be
// computed in place: all of the row's tiles are formed in registers (one warp
// per tile, the K-sum split over two DMMA accumulator chains), then written
// after a barrier.  The diagonal inverses are formed first for all rows (one
// thread per (tile, column), forward substitution) in the scratch area D
// (T tiles) and copied in with their row.  W: per-warp 64-double staging.
// With X, each triangular solve is one parallel mat-vec instead of a chain.
template <int NT>
__device__ __noinline__ void invert_full(double* Kt, int T, const double* dinv, double* D, double* W) {
  QP_SMEM(Kt);
  QP_SMEM(dinv);
  QP_SMEM(D);
  QP_SMEM(W);
  constexpr int NW = NT / 32;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  for (int t = tid; t < 8 * T; t += NT) {
    const int k = t >> 3, c = t & 7;
    const double* L = Kt + ti(k, k) * kTS;
    double* Xt = D + k * kTS;
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
  const int i = lane >> 2, p = lane & 3;
  double* Ws = W + wid * 64;
  // row 0: only its diagonal
  for (int e = tid; e < 64; e += NT) Kt[ti(0, 0) * kTS + e] = D[e];
  for (int I = 1; I < T; ++I) {
    constexpr int MAXR = 4;  // tiles per warp per row (T <= 32)
    double x0[MAXR], x1[MAXR];
    const double* Li = D + I * kTS;  // Linv_I
#pragma unroll
    for (int u = 0; u < MAXR; ++u) {
      const int J = wid + u * NW;
      x0[u] = 0.0;
      x1[u] = 0.0;
      if (J < I) {
        double a0 = 0.0, a1 = 0.0, b0 = 0.0, b1 = 0.0;
        for (int K = J; K < I; K += 2) {
          const double* L0 = Kt + ti(I, K) * kTS;
          const double* X0 = Kt + ti(K, J) * kTS;
#pragma unroll
          for (int h = 0; h < 8; h += 4) dmma884(a0, a1, L0[eo(i, p + h)], X0[eo(p + h, i)]);
          if (K + 1 < I) {
            const double* L1 = Kt + ti(I, K + 1) * kTS;
            const double* X1 = Kt + ti(K + 1, J) * kTS;
#pragma unroll
            for (int h = 0; h < 8; h += 4) dmma884(b0, b1, L1[eo(i, p + h)], X1[eo(p + h, i)]);
          }
        }
        Ws[eo(i, 2 * p)] = a0 + b0;
        Ws[eo(i, 2 * p + 1)] = a1 + b1;
        __syncwarp();
#pragma unroll
        for (int h = 0; h < 8; h += 4) dmma884(x0[u], x1[u], -Li[eo(i, p + h)], Ws[eo(p + h, i)]);
        __syncwarp();
      }
    }
    __syncthreads();  // row I of L fully read
#pragma unroll
    for (int u = 0; u < MAXR; ++u) {
      const int J = wid + u * NW;
      if (J < I) {
        double* Xt = Kt + ti(I, J) * kTS;
        Xt[eo(i, 2 * p)] = x0[u];
        Xt[eo(i, 2 * p + 1)] = x1[u];
      }
    }
    for (int e = tid; e < 64; e += NT) Kt[ti(I, I) * kTS + e] = Li[e];
    __syncthreads();
  }
}

// y <- X y (X = L^{-1} in Kt, lower).  One warp per tile row-block I
// (blocks dealt in mirrored pairs w, 2NW-1-w, ... so every warp sums about
// the same number of tiles); lane (rr, cq) owns row rr and columns 2cq, 2cq+1
// of each tile, two independent FMA chains, then a 4-lane shuffle reduce.
// The two column loads alternate order by cq parity so a warp's first loads
// fall on 16 different bank pairs (2 wavefronts, the minimum).
// y: shared, 8T entries; tmp: 8T doubles.  All NT threads call.
template <int NT>
__device__ __noinline__ void apply_x(const double* Kt, int T, double* y, double* tmp) {
  QP_SMEM(Kt);
  QP_SMEM(y);
  QP_SMEM(tmp);
  constexpr int NW = NT / 32;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int rr = lane >> 2, cq = lane & 3;
  const int ca = 2 * cq + (cq & 1), cb = 2 * cq + 1 - (cq & 1);
  for (int base = 0; base < T; base += 2 * NW) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int I = h == 0 ? base + wid : base + 2 * NW - 1 - wid;
      if (I >= T) continue;
      double s0 = 0.0, s1 = 0.0;
      const double* Xt = Kt + ti(I, 0) * kTS;
      for (int J = 0; J <= I; ++J, Xt += kTS) {
        s0 = fma(Xt[eo(rr, ca)], y[8 * J + ca], s0);
        s1 = fma(Xt[eo(rr, cb)], y[8 * J + cb], s1);
      }
      double v = s0 + s1;
      v += __shfl_xor_sync(0xffffffffu, v, 1);
      v += __shfl_xor_sync(0xffffffffu, v, 2);
      if (cq == 0) tmp[8 * I + rr] = v;
    }
  }
  __syncthreads();
  for (int r = threadIdx.x; r < 8 * T; r += NT) y[r] = tmp[r];
  __syncthreads();
}

// y <- X' y: one warp per tile column-block C (mirrored pairs as above);
// lane (cc, rq) owns column cc and rows 2rq, 2rq+1 of each tile (I, C), I >= C.
template <int NT>
__device__ __noinline__ void apply_xt(const double* Kt, int T, double* y, double* tmp) {
  QP_SMEM(Kt);
  QP_SMEM(y);
  QP_SMEM(tmp);
  constexpr int NW = NT / 32;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int cc = lane >> 2, rq = lane & 3;
  for (int base = 0; base < T; base += 2 * NW) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int C = h == 0 ? base + wid : base + 2 * NW - 1 - wid;
      if (C >= T) continue;
      double s0 = 0.0, s1 = 0.0;
      for (int I = C; I < T; ++I) {
        const double* Xt = Kt + ti(I, C) * kTS;
        s0 = fma(Xt[eo(2 * rq, cc)], y[8 * I + 2 * rq], s0);
        s1 = fma(Xt[eo(2 * rq + 1, cc)], y[8 * I + 2 * rq + 1], s1);
      }
      double v = s0 + s1;
      v += __shfl_xor_sync(0xffffffffu, v, 1);
      v += __shfl_xor_sync(0xffffffffu, v, 2);
      if (rq == 0) tmp[8 * C + cc] = v;
    }
  }
  __syncthreads();
  for (int r = threadIdx.x; r < 8 * T; r += NT) y[r] = tmp[r];
  __syncthreads();
}

// x = X' (X b) = K^{-1} b in one call: two barrier-separated mat-vec phases,
// no staging copies.  Phase 1 (tmp = X b) and phase 2 (x = X' tmp) use the
// warp-per-tile-block scheme of apply_x / apply_xt with the tile loop
// unrolled by two (four independent FMA chains).  b: nf entries (padding rows
// read as zero); x may alias b; tmp: 8T doubles.  All NT threads call.
template <int NT>
__device__ __noinline__ void solve_xxt(const double* Kt, int T, int nf, const double* b, double* x,
                                       double* tmp) {
  QP_SMEM(Kt);
  QP_SMEM(tmp);
  constexpr int NW = NT / 32;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  {
    const int rr = lane >> 2, cq = lane & 3;
    const int ca = 2 * cq + (cq & 1), cb = 2 * cq + 1 - (cq & 1);
    for (int base = 0; base < T; base += 2 * NW) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int I = h == 0 ? base + wid : base + 2 * NW - 1 - wid;
        if (I >= T) continue;
        double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
        const double* Xt = Kt + ti(I, 0) * kTS;
        int J = 0;
        for (; J + 1 <= I; J += 2, Xt += 2 * kTS) {
          const int ja = 8 * J + ca, jb = 8 * J + cb;
          s0 = fma(Xt[eo(rr, ca)], ja < nf ? b[ja] : 0.0, s0);
          s1 = fma(Xt[eo(rr, cb)], jb < nf ? b[jb] : 0.0, s1);
          s2 = fma(Xt[kTS + eo(rr, ca)], ja + 8 < nf ? b[ja + 8] : 0.0, s2);
          s3 = fma(Xt[kTS + eo(rr, cb)], jb + 8 < nf ? b[jb + 8] : 0.0, s3);
        }
        if (J == I) {
          const int ja = 8 * J + ca, jb = 8 * J + cb;
          s0 = fma(Xt[eo(rr, ca)], ja < nf ? b[ja] : 0.0, s0);
          s1 = fma(Xt[eo(rr, cb)], jb < nf ? b[jb] : 0.0, s1);
        }
        double v = (s0 + s1) + (s2 + s3);
        v += __shfl_xor_sync(0xffffffffu, v, 1);
        v += __shfl_xor_sync(0xffffffffu, v, 2);
        if (cq == 0) tmp[8 * I + rr] = v;
      }
    }
  }
  __syncthreads();
  {
    const int cc = lane >> 2, rq = lane & 3;
    for (int base = 0; base < T; base += 2 * NW) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int C = h == 0 ? base + wid : base + 2 * NW - 1 - wid;
        if (C >= T) continue;
        double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
        int I = C;
        for (; I + 1 < T; I += 2) {
          const double* X0 = Kt + ti(I, C) * kTS;
          const double* X1 = Kt + ti(I + 1, C) * kTS;
          s0 = fma(X0[eo(2 * rq, cc)], tmp[8 * I + 2 * rq], s0);
          s1 = fma(X0[eo(2 * rq + 1, cc)], tmp[8 * I + 2 * rq + 1], s1);
          s2 = fma(X1[eo(2 * rq, cc)], tmp[8 * I + 8 + 2 * rq], s2);
          s3 = fma(X1[eo(2 * rq + 1, cc)], tmp[8 * I + 9 + 2 * rq], s3);
        }
        if (I < T) {
          const double* X0 = Kt + ti(I, C) * kTS;
          s0 = fma(X0[eo(2 * rq, cc)], tmp[8 * I + 2 * rq], s0);
          s1 = fma(X0[eo(2 * rq + 1, cc)], tmp[8 * I + 2 * rq + 1], s1);
        }
        double v = (s0 + s1) + (s2 + s3);
        v += __shfl_xor_sync(0xffffffffu, v, 1);
        v += __shfl_xor_sync(0xffffffffu, v, 2);
        if (rq == 0 && 8 * C + cc < nf) x[8 * C + cc] = v;
      }
    }
  }
  __syncthreads();
}

// Inverses of the diagonal tiles only, D_k = L_kk^{-1} (lower), one thread
// per (tile, column): the first phase of invert_full.
template <int NT>
__device__ __noinline__ void diag_inverses(const double* Kt, int T, const double* dinv, double* D) {
  QP_SMEM(Kt);
  QP_SMEM(dinv);
  QP_SMEM(D);
  for (int t = threadIdx.x; t < 8 * T; t += NT) {
    const int k = t >> 3, c = t & 7;
    const double* L = Kt + ti(k, k) * kTS;
    double* Xt = D + k * kTS;
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
}

// x = K^{-1} b = L^{-T} L^{-1} b by blocked substitution in ONE warp (the
// caller's other warps wait at the closing barrier): right-looking, so the
// chain per 8-row block is one 8x8 mat-vec with the diagonal-tile inverse D
// (lane (r, cq): two FMAs + a 4-lane shuffle reduce) followed by the update
// of the remaining rows by that block (independent 8-FMA rows, two chains
// each).  No inverse of L is formed.  b: nf entries (padding reads as zero);
// x may alias b; s: 8T doubles of shared scratch.  All NT threads call.
template <int NT>
__device__ __noinline__ void solve_llt(const double* Kt, const double* D, int T, int nf, const double* b,
                                       double* x, double* s) {
  QP_SMEM(Kt);
  QP_SMEM(D);
  QP_SMEM(s);
  const int lane = threadIdx.x & 31;
  if (threadIdx.x < 32) {
    const int rr = lane >> 2, cq = lane & 3;
    for (int t = lane; t < 8 * T; t += 32) s[t] = t < nf ? b[t] : 0.0;
    __syncwarp();
    // forward: L y = b (y overwrites s block by block)
    for (int J = 0; J < T; ++J) {
      const double* Dj = D + J * kTS;
      double v = fma(Dj[eo(rr, 2 * cq)], s[8 * J + 2 * cq], Dj[eo(rr, 2 * cq + 1)] * s[8 * J + 2 * cq + 1]);
      v += __shfl_xor_sync(0xffffffffu, v, 1);
      v += __shfl_xor_sync(0xffffffffu, v, 2);
      __syncwarp();
      if (cq == 0) s[8 * J + rr] = v;
      __syncwarp();
      for (int row = 8 * (J + 1) + lane; row < 8 * T; row += 32) {
        const double* Lt = Kt + ti(row >> 3, J) * kTS;
        const int r = row & 7;
        double a0 = 0.0, a1 = 0.0;
#pragma unroll
        for (int c = 0; c < 8; c += 2) {
          a0 = fma(Lt[eo(r, c)], s[8 * J + c], a0);
          a1 = fma(Lt[eo(r, c + 1)], s[8 * J + c + 1], a1);
        }
        s[row] -= a0 + a1;
      }
      __syncwarp();
    }
    // backward: L^T x = y (x overwrites s block by block, from the last)
    for (int J = T - 1; J >= 0; --J) {
      const double* Dj = D + J * kTS;
      // x_J[c] = sum_{r >= c} D_J[r][c] t_J[r]; lane (cc = rr, rq = cq)
      double v = fma(Dj[eo(2 * cq, rr)], s[8 * J + 2 * cq], Dj[eo(2 * cq + 1, rr)] * s[8 * J + 2 * cq + 1]);
      v += __shfl_xor_sync(0xffffffffu, v, 1);
      v += __shfl_xor_sync(0xffffffffu, v, 2);
      __syncwarp();
      if (cq == 0) s[8 * J + rr] = v;
      __syncwarp();
      // t_K[c] -= sum_r L_JK[r][c] x_J[r] for every column of the blocks K < J
      for (int col = lane; col < 8 * J; col += 32) {
        const double* Lt = Kt + ti(J, col >> 3) * kTS;
        const int c = col & 7;
        double a0 = 0.0, a1 = 0.0;
#pragma unroll
        for (int r = 0; r < 8; r += 2) {
          a0 = fma(Lt[eo(r, c)], s[8 * J + r], a0);
          a1 = fma(Lt[eo(r + 1, c)], s[8 * J + r + 1], a1);
        }
        s[col] -= a0 + a1;
      }
      __syncwarp();
    }
    for (int t = lane; t < nf; t += 32) x[t] = s[t];
  }
  __syncthreads();
}

// x = K^{-1} b = L^{-T} L^{-1} b by blocked substitution over all warps with
// a look-ahead of one block (the pattern of factor_la): warp 0 runs the chain
// -- apply the previous block's solution to the next block, then the 8x8
// mat-vec with the diagonal-tile inverse D_J -- while warps 1.. update every
// later block with the solution just published.  Named barriers, by step
// parity: Y (warp 0 arrives after publishing block J, the others sync) and
// U (the others arrive after their update with block J, warp 0 syncs two
// steps later, before it needs those contributions).  No L^{-1} is formed:
// only D (diag_inverses).  b: nf entries (padding reads as zero); x may
// alias b; s: 8T doubles of shared scratch.  All NT threads call.
template <int NT>
__device__ __noinline__ void solve_mw(const double* Kt, const double* D, int T, int nf, const double* b, double* x,
                                      double* s) {
  QP_SMEM(Kt);
  QP_SMEM(D);
  QP_SMEM(s);
  constexpr int BY = 8, BU = 10;  // Y: 8, 9; U: 10, 11 (factor_la uses 1-4)
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int rr = lane >> 2, cq = lane & 3;
  for (int t = tid; t < 8 * T; t += NT) s[t] = t < nf ? b[t] : 0.0;
  __syncthreads();
  // warp-0 helpers: 8-vector out[rr] = sum_c M[rr][c] v[c] (lanes (rr, cq)
  // take columns 2cq, 2cq+1; 4-lane reduce), M read through eo (row, col)
  auto mv8 = [&](const double* M, const double* v) {
    double t0 = fma(M[eo(rr, 2 * cq)], v[2 * cq], M[eo(rr, 2 * cq + 1)] * v[2 * cq + 1]);
    t0 += __shfl_xor_sync(0xffffffffu, t0, 1);
    t0 += __shfl_xor_sync(0xffffffffu, t0, 2);
    return t0;
  };
  // transposed: out[rr] = sum_r M[r][rr] v[r]
  auto mv8t = [&](const double* M, const double* v) {
    double t0 = fma(M[eo(2 * cq, rr)], v[2 * cq], M[eo(2 * cq + 1, rr)] * v[2 * cq + 1]);
    t0 += __shfl_xor_sync(0xffffffffu, t0, 1);
    t0 += __shfl_xor_sync(0xffffffffu, t0, 2);
    return t0;
  };
  // ---- forward: y = L^{-1} b (y overwrites s) ----
  if (wid == 0) {
    for (int J = 0; J < T; ++J) {
      if (J >= 2) bar_sync(BU + (J & 1), NT);  // others applied y_0..y_{J-2} to block J
      double* sJ = s + 8 * J;
      if (J >= 1) {  // look-ahead: y_{J-1} into block J
        const double v = mv8(Kt + ti(J, J - 1) * kTS, s + 8 * (J - 1));
        __syncwarp();
        if (cq == 0) sJ[rr] -= v;
        __syncwarp();
      }
      const double y = mv8(D + J * kTS, sJ);
      __syncwarp();
      if (cq == 0) sJ[rr] = y;
      __syncwarp();
      __threadfence_block();
      bar_arrive(BY + (J & 1), NT);
    }
    for (int J = max(T, 2); J < T + 2; ++J) bar_sync(BU + (J & 1), NT);  // the last two U phases
  } else {
    const int ut = tid - 32;
    for (int J = 0; J < T; ++J) {
      bar_sync(BY + (J & 1), NT);  // y_J published
      const double* yJ = s + 8 * J;
      for (int row = 8 * (J + 2) + ut; row < 8 * T; row += NT - 32) {
        const double* Lt = Kt + ti(row >> 3, J) * kTS;
        const int r = row & 7;
        double a0 = 0.0, a1 = 0.0;
#pragma unroll
        for (int c = 0; c < 8; c += 2) {
          a0 = fma(Lt[eo(r, c)], yJ[c], a0);
          a1 = fma(Lt[eo(r, c + 1)], yJ[c + 1], a1);
        }
        s[row] -= a0 + a1;
      }
      __threadfence_block();
      bar_arrive(BU + (J & 1), NT);
    }
  }
  __syncthreads();
  // ---- backward: x = L^{-T} y (x overwrites s), J = T-1 .. 0 ----
  // step index q = T-1-J drives the barrier parity
  if (wid == 0) {
    for (int q = 0; q < T; ++q) {
      const int J = T - 1 - q;
      if (q >= 2) bar_sync(BU + (q & 1), NT);
      double* tJ = s + 8 * J;
      if (q >= 1) {  // look-ahead: x_{J+1} into block J: t_J -= L_{J+1,J}^T x_{J+1}
        const double v = mv8t(Kt + ti(J + 1, J) * kTS, s + 8 * (J + 1));
        __syncwarp();
        if (cq == 0) tJ[rr] -= v;
        __syncwarp();
      }
      const double xv = mv8t(D + J * kTS, tJ);
      __syncwarp();
      if (cq == 0) tJ[rr] = xv;
      __syncwarp();
      __threadfence_block();
      bar_arrive(BY + (q & 1), NT);
    }
    for (int q = max(T, 2); q < T + 2; ++q) bar_sync(BU + (q & 1), NT);
  } else {
    const int ut = tid - 32;
    for (int q = 0; q < T; ++q) {
      const int J = T - 1 - q;
      bar_sync(BY + (q & 1), NT);  // x_J published
      const double* xJ = s + 8 * J;
      // t_K[c] -= sum_r L_JK[r][c] x_J[r] for the blocks K <= J-2
      for (int col = ut; col < 8 * (J - 1); col += NT - 32) {
        const double* Lt = Kt + ti(J, col >> 3) * kTS;
        const int c = col & 7;
        double a0 = 0.0, a1 = 0.0;
#pragma unroll
        for (int r = 0; r < 8; r += 2) {
          a0 = fma(Lt[eo(r, c)], xJ[r], a0);
          a1 = fma(Lt[eo(r + 1, c)], xJ[r + 1], a1);
        }
        s[col] -= a0 + a1;
      }
      __threadfence_block();
      bar_arrive(BU + (q & 1), NT);
    }
  }
  __syncthreads();
  for (int t = tid; t < nf; t += NT) x[t] = s[t];
  __syncthreads();
}

// Off-diagonal parts of the 16x16 diagonal-block inverses: for 16-block j
// (tiles 2j, 2j+1), [[A, 0], [B, C]]^{-1} = [[A^-1, 0], [-C^-1 B A^-1, C^-1]];
// X21_j = -D_{2j+1} L_{2j+1,2j} D_{2j} into X21 (64 doubles per block, eo
// layout).  D from diag_inverses.  All NT threads call.
template <int NT>
__device__ __noinline__ void diag16(const double* Kt, int T, const double* D, double* X21) {
  QP_SMEM(Kt);
  QP_SMEM(D);
  QP_SMEM(X21);
  const int nb = T / 2;  // full 16-blocks
  constexpr int PER = 4;  // items per thread (nb * 64 <= 4 * NT for T <= 16 and NT >= 256)
  double m[PER];
  // M = B A^-1 (into registers), then X21 = -C^-1 M after a barrier
#pragma unroll
  for (int u = 0; u < PER; ++u) {
    const int t = threadIdx.x + u * NT;
    m[u] = 0.0;
    if (t < nb * 64) {
      const int j = t >> 6, r = (t >> 3) & 7, c = t & 7;
      const double* B = Kt + ti(2 * j + 1, 2 * j) * kTS;
      const double* A = D + 2 * j * kTS;
      double a = 0.0;
#pragma unroll
      for (int k = 0; k < 8; ++k) a = fma(B[eo(r, k)], A[eo(k, c)], a);
      m[u] = a;
    }
  }
#pragma unroll
  for (int u = 0; u < PER; ++u) {
    const int t = threadIdx.x + u * NT;
    if (t < nb * 64) {
      const int j = t >> 6, r = (t >> 3) & 7, c = t & 7;
      X21[j * 64 + eo(r, c)] = m[u];
    }
  }
  __syncthreads();
#pragma unroll
  for (int u = 0; u < PER; ++u) {
    const int t = threadIdx.x + u * NT;
    m[u] = 0.0;
    if (t < nb * 64) {
      const int j = t >> 6, r = (t >> 3) & 7, c = t & 7;
      const double* C = D + (2 * j + 1) * kTS;
      const double* Mj = X21 + j * 64;
      double a = 0.0;
#pragma unroll
      for (int k = 0; k < 8; ++k) a = fma(C[eo(r, k)], Mj[eo(k, c)], a);
      m[u] = -a;
    }
  }
  __syncthreads();
#pragma unroll
  for (int u = 0; u < PER; ++u) {
    const int t = threadIdx.x + u * NT;
    if (t < nb * 64) {
      const int j = t >> 6, r = (t >> 3) & 7, c = t & 7;
      X21[j * 64 + eo(r, c)] = m[u];
    }
  }
  __syncthreads();
}

// solve_mw with 16-row blocks (tiles 2j, 2j+1): the chain step is one 16x16
// look-ahead product and one 16x16 mat-vec with the block inverse
// [[D_2j, 0], [X21_j, D_2j+1]]; lane r < 16 owns row r of the block (both
// 8-column halves in the lane: 4 FMA chains, no shuffle on the chain; the
// (row, half) lane-pair form was 1.7 % slower at cfg3) -- half the chain
// steps of solve_mw and no 4-lane reduce.  T <= 16 (X21 in 512 doubles); odd T: the last block is
// 8 rows.  Same arguments as solve_mw plus X21 (diag16).
template <int NT>
__device__ __noinline__ void solve_mw16(const double* Kt, const double* D, const double* X21, int T, int nf,
                                        const double* b, double* x, double* s) {
  QP_SMEM(Kt);
  QP_SMEM(D);
  QP_SMEM(X21);
  QP_SMEM(s);
  constexpr int BY = 8, BU = 10;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int r = lane >> 1, h = lane & 1, rr = r & 7, rh = r >> 3;
  const int T16 = (T + 1) / 2, n8 = 8 * T;
  for (int t = tid; t < n8; t += NT) s[t] = t < nf ? b[t] : 0.0;
  __syncthreads();
  // dot of 8 with two chains
  auto dot8 = [](const double* M, int row, bool trans, const double* v) {
    double a0 = 0.0, a1 = 0.0;
#pragma unroll
    for (int k = 0; k < 8; k += 2) {
      a0 = fma(trans ? M[eo(k, row)] : M[eo(row, k)], v[k], a0);
      a1 = fma(trans ? M[eo(k + 1, row)] : M[eo(row, k + 1)], v[k + 1], a1);
    }
    return a0 + a1;
  };
  // ---- forward ----
  if (wid == 0) {
    // lane q < 16 owns row q of the 16-row block; both halves of every dot
    // in the lane (4 FMA chains), so the chain has no pair shuffles
    const int q16 = lane & 15, qh = q16 >> 3, qr = q16 & 7;
    const bool act = lane < 16;
    for (int j = 0; j < T16; ++j) {
      if (j >= 2) bar_sync(BU + (j & 1), NT);
      const int tr = 2 * j + qh;  // tile row of this lane's row
      const bool live = act && tr < T;
      const int trs = live ? tr : 2 * j;
      if (j >= 1) {  // look-ahead: y of block j-1 (two full tiles) into block j
        const double* y = s + 16 * (j - 1);
        const double v = dot8(Kt + ti(trs, 2 * j - 2) * kTS, qr, false, y) +
                         dot8(Kt + ti(trs, 2 * j - 1) * kTS, qr, false, y + 8);
        __syncwarp();
        if (live) s[16 * j + q16] -= v;
        __syncwarp();
      }
      // rows 0-7: D_2j y_a; rows 8-15: X21 y_a + D_2j+1 y_c (uniform selects)
      const bool two = 2 * j + 1 < T;
      const double* M1 = (qh == 0 || !two) ? D + 2 * j * kTS : X21 + j * 64;
      const double* M2 = two ? D + (2 * j + 1) * kTS : D + 2 * j * kTS;
      const double w2 = (qh == 1 && two) ? 1.0 : 0.0;
      const double* ya = s + 16 * j;
      const double v = dot8(M1, qr, false, ya) + w2 * dot8(M2, qr, false, two ? ya + 8 : ya);
      __syncwarp();
      if (live) s[16 * j + q16] = v;
      __syncwarp();
      __threadfence_block();
      bar_arrive(BY + (j & 1), NT);
    }
    for (int j = max(T16, 2); j < T16 + 2; ++j) bar_sync(BU + (j & 1), NT);
  } else {
    const int ut = tid - 32;
    for (int j = 0; j < T16; ++j) {
      bar_sync(BY + (j & 1), NT);
      const double* y = s + 16 * j;
      const bool two = 2 * j + 1 < T;
      for (int row = 16 * (j + 2) + ut; row < n8; row += NT - 32) {
        const int rt = row >> 3, ri = row & 7;
        double a = dot8(Kt + ti(rt, 2 * j) * kTS, ri, false, y);
        if (two) a += dot8(Kt + ti(rt, 2 * j + 1) * kTS, ri, false, y + 8);
        s[row] -= a;
      }
      __threadfence_block();
      bar_arrive(BU + (j & 1), NT);
    }
  }
  __syncthreads();
  // ---- backward (step q = T16-1-j) ----
  if (wid == 0) {
    const int q16 = lane & 15, qh = q16 >> 3, qr = q16 & 7;
    const bool act = lane < 16;
    for (int q = 0; q < T16; ++q) {
      const int j = T16 - 1 - q;
      if (q >= 2) bar_sync(BU + (q & 1), NT);
      const int tc = 2 * j + qh;  // this lane's row of block j as a column of L
      const bool live = act && tc < T;
      const int tcs = live ? tc : 2 * j;
      if (q >= 1) {  // look-ahead: x of block j+1 into block j
        const bool two1 = 2 * j + 3 < T;
        const double* x1 = s + 16 * (j + 1);
        const double v = dot8(Kt + ti(2 * j + 2, tcs) * kTS, qr, true, x1) +
                         (two1 ? 1.0 : 0.0) * dot8(Kt + ti(two1 ? 2 * j + 3 : 2 * j + 2, tcs) * kTS, qr, true,
                                                   two1 ? x1 + 8 : x1);
        __syncwarp();
        if (live) s[16 * j + q16] -= v;
        __syncwarp();
      }
      // rows 0-7: D_2j' t_a + X21' t_c; rows 8-15: D_2j+1' t_c (uniform selects)
      const bool two = 2 * j + 1 < T;
      const double* ta = s + 16 * j;
      const double* tcv = two ? ta + 8 : ta;
      const double* M1 = (qh == 0 || !two) ? D + 2 * j * kTS : D + (2 * j + 1) * kTS;
      const double w2 = (qh == 0 && two) ? 1.0 : 0.0;
      // (no X21 for a lone last tile: a finite stand-in under the zero weight)
      const double v = dot8(M1, qr, true, qh == 0 ? ta : tcv) +
                       w2 * dot8(two ? X21 + j * 64 : D + 2 * j * kTS, qr, true, tcv);
      __syncwarp();
      if (live) s[16 * j + q16] = v;
      __syncwarp();
      __threadfence_block();
      bar_arrive(BY + (q & 1), NT);
    }
    for (int q = max(T16, 2); q < T16 + 2; ++q) bar_sync(BU + (q & 1), NT);
  } else {
    const int ut = tid - 32;
    for (int q = 0; q < T16; ++q) {
      const int j = T16 - 1 - q;
      bar_sync(BY + (q & 1), NT);
      const double* xj = s + 16 * j;
      const bool two = 2 * j + 1 < T;
      for (int col = ut; col < 16 * (j - 1) && col < n8; col += NT - 32) {
        const int ct = col >> 3, ci = col & 7;
        double a = dot8(Kt + ti(2 * j, ct) * kTS, ci, true, xj);
        if (two) a += dot8(Kt + ti(2 * j + 1, ct) * kTS, ci, true, xj + 8);
        s[col] -= a;
      }
      __threadfence_block();
      bar_arrive(BU + (q & 1), NT);
    }
  }
  __syncthreads();
  for (int t = tid; t < nf; t += NT) x[t] = s[t];
  __syncthreads();
}

}  // namespace qpchol
