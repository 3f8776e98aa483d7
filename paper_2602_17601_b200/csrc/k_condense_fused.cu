// K-COND: fused Gamma recursion + cost reduction (stages 2 and 3a in one
// persistent kernel).
//
// Reference: condense_gammas (condensing.py:182-228) followed by the cost part
// of condense_ocp (condensing.py:376-389, :402-403).
//
// The two-kernel path (k_condense.cu) launches K-REC once per stage (N + 1
// launches, each a few microseconds of work behind a full-device dependency)
// and then re-reads all of Gamma (64 MB at M=1000, N=20) for K-HG.  Here:
//
//   * CTA s owns the node range [s*per, (s+1)*per) of one instance for the
//     whole horizon.  Stage n+1 of a node needs stage n of its neighbours, so
//     instead of a grid-wide barrier per stage a CTA waits only on the CTAs
//     that own its nodes' neighbours (dependency lists built on the host from
//     the CSR), through per-CTA stage counters in global memory
//     (st.release / ld.acquire at gpu scope).  On a chain or mesh a CTA has
//     two neighbours, so stages pipeline across the device like a wavefront.
//     All CTAs are co-resident (grid <= SMs x occupancy; the host checks), so
//     the waits cannot deadlock.  The last CTA to finish resets the counters.
//   * the stage-(n+1) rows a CTA computes stay in shared memory and are
//     folded into H right away: thread t owns the nu x nu block pair (p, q),
//     p <= q, of H, ordered by q, so at stage k exactly the first k(k+1)/2
//     threads are live (Gamma rows of stage k only reach input blocks < k):
//       acc(p,q) += G(:, p-block)' Qs G(:, q-block),   Qs = (Q + Q')/2
//     which is the symmetrised sum 0.5 (S + S') of condensing.py:403.
//     g += G' (2 Q Gamma_x - 2 Q x_ref) in fp64 per column (condensing.py:388).
//   * per-CTA fp32 partials are reduced in a fixed order in fp64 (bitwise
//     reproducible) by two small kernels that add R-bar and mirror H.
//
// Numerics equal the two-kernel path: the same fp32 Gamma recursion (c rounded
// once to fp32, as K-REC), fp32 partial sums, fp64 reduction.
#include <algorithm>
#include <cstdlib>
#include <cstdio>
#include <cmath>

#include <cuda.h>
#include <cudaTypedefs.h>

#include "common.cuh"
#include "umma.cuh"

namespace {

constexpr int kFusedSmemBudget = 160 * 1024;
constexpr int kTcThreads = 512;  // k_condense_tc block size (16 warps: latency hiding for the neighbour loads)

struct FusedArgs {
  int M, E, N, ld, per, splits, sc, npairs, dslot;
  int reg_prefetch;  // k_condense_tc: register prefetch of the next item's neighbour rows
  int rec;           // k_condense_tc: 1 = run the recursion (K-COND), 0 = read Gamma (K-HG on tcgen05)
  int lo, hi;        // node range of the launch (k_condense_tc)
  const int* ptr;
  const int* src;
  const int* dep_ptr;
  const int* dep;
  const float* a_self;
  const float* a_nbr;
  const float* b;
  const double* c;
  const double* x0;
  float* W;
  const double* q;
  int64_t q_stride;
  const double* xref;
  int64_t xref_stride;
  float* partH;   // (B, splits, npairs * nu * nu)
  double* partg;  // (B, splits, n0)
  int* flags;     // (B * splits) stage counters, then one completion counter
  // k_condense_tma: unique closed-neighbourhood nodes per SC-node chunk
  const int* cu_ptr;
  const int* cu_nodes;
  const unsigned char* cu_slot;
  int umax;
  int qg_r8;  // k_condense_tmap: eighths of the Qs*G columns done by the recursion group
  int al16;   // every block base 16-byte aligned: 16-byte cp.async for the item blocks
  int hacc_gl;  // k_condense_tmap: H accumulator in the global partial (shared memory too small)
};

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)),
               "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)),
               "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)),
               "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

// Per-item staging buffer (one (stage, node sub-chunk) work item), double
// buffered: item j+1 is fetched with cp.async while item j computes.
template <int NX, int NU>
struct Stage {
  float* as;    // SC x NX*NX      a_self[n]
  float* an;    // SC*dmax x NX*NX a_nbr[n] of the chunk's edge range
  float* bb;    // SC x NX*NU      b[n]
  double* cc;   // SC x NX         c[n]
  double* qd;   // SC x NX*NX      Q[k]
  double* xd;   // SC x NX         x_ref[k]
  int* src;     // SC*dmax         in-neighbour ids of the chunk's edges
};

template <int NX, int NU>
__device__ __forceinline__ Stage<NX, NU> stage_at(unsigned char* base, int SC, int emax) {
  Stage<NX, NU> s;
  double* d = (double*)base;
  s.cc = d;
  s.qd = s.cc + SC * NX;
  s.xd = s.qd + SC * NX * NX;
  float* f = (float*)(s.xd + SC * NX);
  s.as = f;
  s.an = s.as + SC * NX * NX;
  s.bb = s.an + (int64_t)emax * NX * NX;
  s.src = (int*)(s.bb + SC * NX * NU);
  return s;
}

template <int NX, int NU>
__host__ __device__ inline size_t stage_bytes(int SC, int emax) {
  size_t b = sizeof(double) * ((size_t)SC * NX * 2 + (size_t)SC * NX * NX) +
             sizeof(float) * ((size_t)SC * NX * NX + (size_t)emax * NX * NX + (size_t)SC * NX * NU) +
             sizeof(int) * (size_t)emax;
  return (b + 15) & ~size_t(15);
}

template <int NX, int NU>
__global__ void __launch_bounds__(256, 1) k_condense_fused(const FusedArgs a) {
  extern __shared__ __align__(16) unsigned char smraw[];
  const int N = a.N, ld = a.ld, SC = a.sc, M = a.M;
  const int n0 = N * NU, XC = N * NU;
  const int tid = threadIdx.x, nt = blockDim.x;
  const int64_t bi = blockIdx.x / a.splits;
  const int split = (int)(blockIdx.x % a.splits);
  const bool rec = a.rec != 0;  // 0: read Gamma of [lo, hi) instead of producing it (K-HG)
  const int nb = a.lo + split * a.per, ne = min(a.hi, nb + a.per);
  const int nn = ne - nb;
  const int nsub = (nn + SC - 1) / SC;
  const int emax = SC * (a.dslot - 1) > 0 ? SC * (a.dslot - 1) : 1;
  int* flags = rec ? a.flags + bi * a.splits : nullptr;
  const int64_t stage_stride = (int64_t)NX * ld;
  const int64_t node_stride = (int64_t)(N + 1) * stage_stride;
  float* Wb = a.W + bi * (int64_t)M * node_stride;

  // shared memory carve-up
  const size_t sbytes = stage_bytes<NX, NU>(SC, emax);
  float* Gc = (float*)(smraw + 2 * sbytes);        // SC x NX x ld  current-stage rows
  float* QGc = Gc + (int64_t)SC * NX * ld;         // SC x NX x ld  Qs G (live columns)
  float* Qs = QGc + (int64_t)SC * NX * ld;         // SC x NX*NX    (Q + Q')/2
  double* wv = (double*)(((uintptr_t)(Qs + SC * NX * NX) + 15) & ~(uintptr_t)15);  // SC x NX
  double* gs = wv + SC * NX;                       // n0 (g accumulator)
  int* nptr = (int*)(gs + n0);                     // nn + 1 CSR offsets of the owned nodes

  for (int t = tid; t <= nn; t += nt) nptr[t] = a.ptr[nb + t];
  // block pair owned by this thread (ordered by q, then p)
  int bq = (int)((sqrtf(8.f * tid + 1.f) - 1.f) * 0.5f);
  while ((bq + 1) * (bq + 2) / 2 <= tid) ++bq;
  while (bq * (bq + 1) / 2 > tid) --bq;
  const int bp = tid - bq * (bq + 1) / 2;
  const bool owner = tid < a.npairs;
  float acc[NU][NU];
#pragma unroll
  for (int u = 0; u < NU; ++u)
#pragma unroll
    for (int v = 0; v < NU; ++v) acc[u][v] = 0.f;
  for (int t = tid; t < n0; t += nt) gs[t] = 0.0;
  __syncthreads();

  // work item j = (stage n = j / nsub, sub-chunk j % nsub); cp.async prefetch
  auto prefetch = [&](int j) {
    const int n = j / nsub, s0 = nb + (j % nsub) * SC;
    const int sc = min(SC, ne - s0), k = n + 1;
    const Stage<NX, NU> S = stage_at<NX, NU>(smraw + (j & 1) * sbytes, SC, emax);
    const int64_t pstage = bi * N + n;
    const int eb = nptr[s0 - nb], ee = nptr[s0 - nb + sc];
    const int nE = ee - eb;
    if (rec) {
      const float* gas = a.a_self + (pstage * M + s0) * NX * NX;
      for (int t = tid; t < sc * NX * NX; t += nt) cp_async4(S.as + t, gas + t);
      if (nE > 0) {
        const float* gan = a.a_nbr + (pstage * a.E + eb) * NX * NX;
        for (int t = tid; t < nE * NX * NX; t += nt) cp_async4(S.an + t, gan + t);
        for (int t = tid; t < nE; t += nt) cp_async4(S.src + t, a.src + eb + t);
      }
      const float* gb = a.b + (pstage * M + s0) * NX * NU;
      for (int t = tid; t < sc * NX * NU; t += nt) cp_async4(S.bb + t, gb + t);
      const double* gc = a.c + (pstage * M + s0) * NX;
      for (int t = tid; t < sc * NX; t += nt) cp_async8(S.cc + t, gc + t);
    }
    for (int t = tid; t < sc * NX * NX; t += nt) {
      const int li = t / (NX * NX), e = t - li * NX * NX;
      cp_async8(S.qd + t, a.q + bi * a.q_stride + ((int64_t)(s0 + li) * (N + 1) + k) * NX * NX + e);
    }
    for (int t = tid; t < sc * NX; t += nt) {
      const int li = t / NX, e = t - li * NX;
      cp_async8(S.xd + t, a.xref + bi * a.xref_stride + ((int64_t)(s0 + li) * (N + 1) + k) * NX + e);
    }
    cp_async_commit();
  };
  const int items = N * nsub;
  if (items > 0) prefetch(0);

  // stage 0: Gamma_u = 0, Gamma_x = x0 (condensing.py:205-206)
  if (rec)
    for (int t = tid; t < nn * NX * ld; t += nt) {
      const int li = t / (NX * ld), rem = t - li * NX * ld, r = rem / ld, col = rem - r * ld;
      Wb[(int64_t)(nb + li) * node_stride + rem] =
          (col == XC) ? (float)a.x0[(bi * M + nb + li) * NX + r] : 0.f;
    }
  const int d0 = rec ? a.dep_ptr[split] : 0, d1 = rec ? a.dep_ptr[split + 1] : 0;
  __syncthreads();
  if (rec && tid == 0) {
    __threadfence();
    st_release(&flags[split], 1);
  }

  for (int j = 0; j < items; ++j) {
    const int n = j / nsub, sub = j % nsub;
    const int s0 = nb + sub * SC, sc = min(SC, ne - s0);
    const int k = n + 1;       // stage being produced
    const int live = n * NU;   // live Gamma_u columns of stage n
    const Stage<NX, NU> S = stage_at<NX, NU>(smraw + (j & 1) * sbytes, SC, emax);
    if (sub == 0) {
      // wait until every CTA owning a neighbour has published stage n
      for (int d = d0 + tid; d < d1; d += nt) {
        const int* f = &flags[a.dep[d]];
        while (ld_acquire(f) < k) __nanosleep(32);
      }
    }
    cp_async_wait_all();
    __syncthreads();
    if (j + 1 < items) prefetch(j + 1);  // into the other buffer (free since item j-1 ended)
    for (int t = tid; t < sc * NX * NX; t += nt) {
      const int li = t / (NX * NX), e = t - li * NX * NX, r = e / NX, cc = e - r * NX;
      const double* Qk = S.qd + li * NX * NX;
      Qs[t] = (float)(0.5 * (Qk[r * NX + cc] + Qk[cc * NX + r]));
    }
    const int ebase = nptr[s0 - nb];
    if (!rec) {
      // K-HG: the stage-k rows (causal columns + Gamma_x) come from Gamma
      const int lk1 = k * NU;
      for (int t = tid; t < sc * NX * ld; t += nt) {
        const int li = t / (NX * ld), rem = t - li * NX * ld, col = rem % ld;
        if (col < lk1 || col == XC)
          Gc[t] = __ldcg(Wb + (int64_t)(s0 + li) * node_stride + (int64_t)k * stage_stride + rem);
      }
    }
    // Gamma rows of stage k (condensing.py:213-224), same per-column
    // recursion and FMA order as K-REC: live columns and Gamma_x via the
    // closed neighbourhood, block n <- B_n, zero elsewhere
    for (int t = tid; rec && t < sc * ld; t += nt) {
      const int li = t / ld, col = t - li * ld;
      const int i = s0 + li;
      float r6[NX];
#pragma unroll
      for (int r = 0; r < NX; ++r) r6[r] = 0.f;
      if (col < live || col == XC) {
        const int el0 = nptr[i - nb] - ebase, deg = nptr[i - nb + 1] - nptr[i - nb];
        const float* Wn = Wb + (int64_t)n * stage_stride + col;
        for (int s = 0; s <= deg; s += 4) {
          float w[4][NX];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int ss = s + u;
            if (ss <= deg) {
              const int jn = ss == 0 ? i : S.src[el0 + ss - 1];
              const float* Wj = Wn + (int64_t)jn * node_stride;
#pragma unroll
              for (int qq = 0; qq < NX; ++qq) w[u][qq] = __ldcg(Wj + (int64_t)qq * ld);
            }
          }
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int ss = s + u;
            if (ss <= deg) {
              const float* As = ss == 0 ? S.as + li * NX * NX : S.an + (el0 + ss - 1) * NX * NX;
#pragma unroll
              for (int r = 0; r < NX; ++r)
#pragma unroll
                for (int qq = 0; qq < NX; ++qq) r6[r] = fmaf(As[r * NX + qq], w[u][qq], r6[r]);
            }
          }
        }
        if (col == XC) {
#pragma unroll
          for (int r = 0; r < NX; ++r) r6[r] += (float)S.cc[li * NX + r];
        }
      } else if (col >= live && col < live + NU) {
#pragma unroll
        for (int r = 0; r < NX; ++r) r6[r] = S.bb[(li * NX + r) * NU + (col - live)];
      }
      float* Wo = Wb + (int64_t)i * node_stride + (int64_t)k * stage_stride + col;
      float* Gs = Gc + (int64_t)li * NX * ld + col;
#pragma unroll
      for (int r = 0; r < NX; ++r) {
        Wo[(int64_t)r * ld] = r6[r];
        Gs[(int64_t)r * ld] = r6[r];
      }
    }
    __syncthreads();
    if (rec && sub == nsub - 1 && tid == 0) {  // all of this CTA's stage-k rows are out
      __threadfence();
      st_release(&flags[split], k + 1);
    }
    // Qs G on the live columns of stage k, and w = 2 Q Gamma_x - 2 Q x_ref
    const int lk = k * NU;
    for (int t = tid; t < sc * lk; t += nt) {
      const int li = t / lk, col = t - li * lk;
      const float* Gs = Gc + (int64_t)li * NX * ld + col;
      float gcol[NX];
#pragma unroll
      for (int qq = 0; qq < NX; ++qq) gcol[qq] = Gs[(int64_t)qq * ld];
      const float* Qn = Qs + li * NX * NX;
      float* Os = QGc + (int64_t)li * NX * ld + col;
#pragma unroll
      for (int r = 0; r < NX; ++r) {
        float s = 0.f;
#pragma unroll
        for (int qq = 0; qq < NX; ++qq) s = fmaf(Qn[r * NX + qq], gcol[qq], s);
        Os[(int64_t)r * ld] = s;
      }
    }
    for (int t = tid; t < sc * NX; t += nt) {
      const int li = t / NX, r = t - li * NX;
      const double* Qk = S.qd + li * NX * NX + r * NX;
      const double* xr = S.xd + li * NX;
      const float* gx = Gc + (int64_t)li * NX * ld + XC;
      double qg = 0.0, qx = 0.0;
#pragma unroll
      for (int qq = 0; qq < NX; ++qq) {
        qg += Qk[qq] * (double)gx[(int64_t)qq * ld];
        qx += Qk[qq] * xr[qq];
      }
      wv[t] = 2.0 * qg + (-2.0 * qx);
    }
    __syncthreads();
    // H block pairs live at stage k: q < k  <=>  tid < k(k+1)/2
    if (owner && bq < k) {
      for (int li = 0; li < sc; ++li) {
#pragma unroll
        for (int r = 0; r < NX; ++r) {
          const float* gp = Gc + ((int64_t)li * NX + r) * ld + bp * NU;
          const float* gq = QGc + ((int64_t)li * NX + r) * ld + bq * NU;
          float x[NU], y[NU];
#pragma unroll
          for (int u = 0; u < NU; ++u) {
            x[u] = gp[u];
            y[u] = gq[u];
          }
#pragma unroll
          for (int u = 0; u < NU; ++u)
#pragma unroll
            for (int v = 0; v < NU; ++v) acc[u][v] = fmaf(x[u], y[v], acc[u][v]);
        }
      }
    }
    for (int cidx = tid; cidx < lk; cidx += nt) {
      double s = gs[cidx];
      for (int li = 0; li < sc; ++li)
#pragma unroll
        for (int r = 0; r < NX; ++r)
          s += (double)Gc[((int64_t)li * NX + r) * ld + cidx] * wv[li * NX + r];
      gs[cidx] = s;
    }
    __syncthreads();
  }

  // partials
  const int PU = a.npairs * NU * NU;
  float* P = a.partH + (bi * a.splits + split) * (int64_t)PU;
  if (owner) {
#pragma unroll
    for (int u = 0; u < NU; ++u)
#pragma unroll
      for (int v = 0; v < NU; ++v) P[tid * NU * NU + u * NU + v] = acc[u][v];
  }
  for (int t = tid; t < n0; t += nt) a.partg[(bi * a.splits + split) * n0 + t] = gs[t];
  // the last CTA out resets the stage counters for the next launch
  __syncthreads();
  if (rec && tid == 0) {
    __threadfence();
    int* done = a.flags + (int64_t)gridDim.x;
    if (atomicAdd(done, 1) == (int)gridDim.x - 1) {
      for (int s = 0; s < (int)gridDim.x; ++s) a.flags[s] = 0;
      *done = 0;
      __threadfence();
    }
  }
}

// ---------------------------------------------------------------------------
// K-COND with TMA-staged Gamma tiles (nx = nu = 6, the reference
// architecture; the default fused path).  Same work items, stage flags,
// FMA order and fp32 round-to-nearest H accumulation as k_condense_fused,
// but the neighbour Gamma rows of an item no longer come from per-thread
// global loads (the measured bottleneck: long-scoreboard stalls at 8 warps
// per SM, ncu profiles/r02): thread 0 stages them with the tensor memory
// accelerator, cp.async.bulk.tensor.2d over the work array viewed as a
// (rows = B*M*(N+1)*6, cols = ld) fp32 matrix, box 6 rows x 32 columns = one
// node-stage block of one 32-column chunk.  Per item only the chunks holding
// live Gamma_u columns and the Gamma_x column are loaded, once per UNIQUE
// node of the item's closed neighbourhood (host tables per SC-node chunk:
// a chain chunk of 8 nodes reads 10 node rows instead of 24 per-edge rows),
// into a double-buffered shared ring completed on an mbarrier
// (complete_tx).  Within a stage the next item's tiles are in flight while
// the current item computes; the first item of a stage waits for them.
// Ordering: generic stores of Gamma (own CTA: after a CTA barrier; other
// CTAs: their release + our acquire of the stage flag) are made visible to
// the async proxy by fence.proxy.async.global before each issue.
// The recursion then runs from shared memory: one thread per (node, 4
// columns), float4 tile reads (conflict free), A blocks broadcast.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* tm, int c0, int c1, uint64_t* mbar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          umma::smem_u32(dst)),
      "l"(tm), "r"(c0), "r"(c1), "r"(umma::smem_u32(mbar))
      : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* mbar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(umma::smem_u32(mbar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

constexpr int kTileBytes = 6 * 32 * 4;  // one (node, stage, 32-column chunk) box

template <int SC, int CPS, int GW, bool DB>
__global__ void __launch_bounds__(256, 1) k_condense_tma(const FusedArgs a, const __grid_constant__ CUtensorMap tm) {
  constexpr int NX = 6, NU = 6;
  extern __shared__ __align__(128) unsigned char smraw[];
  const int N = a.N, ld = a.ld, M = a.M;
  const int n0 = N * NU, XC = N * NU;
  const int NCH = ld / 32;  // 32-column chunks per row
  const int tid = threadIdx.x, nt = blockDim.x;
  const int64_t bi = blockIdx.x / a.splits;
  const int split = (int)(blockIdx.x % a.splits);
  const int nb = split * a.per, ne = min(M, nb + a.per);
  const int nn = ne - nb;
  const int nsub = (nn + SC - 1) / SC;
  const int chunk0 = nb / SC;  // per is a multiple of SC
  const int emax = SC * (a.dslot - 1) > 0 ? SC * (a.dslot - 1) : 1;
  int* flags = a.flags + bi * a.splits;
  const int64_t stage_stride = (int64_t)NX * ld;
  const int64_t node_stride = (int64_t)(N + 1) * stage_stride;
  float* Wb = a.W + bi * (int64_t)M * node_stride;

  // shared memory: neighbour tile ring (2 x umax x NCH tiles) | 2 block
  // stages | Gc | QGc | Qs | wv | gs | nptr | mbarriers
  // passes of CPS 32-column chunks: slot p holds chunks [CPS p, CPS p + CPS)
  // of an item's unique neighbour rows; slot p's k-th fill is item k.  DB
  // (one pass): two slots alternating by item instead, the next item's tiles
  // issued as the current item starts
  const int npass = (NCH + CPS - 1) / CPS;
  const size_t ring = (size_t)a.umax * CPS * kTileBytes;
  const int nslot = DB ? 2 : npass;
  float* nbuf0 = reinterpret_cast<float*>(smraw);
  float* nbuf1 = reinterpret_cast<float*>(smraw + ring);
  unsigned char* sbase = smraw + nslot * ring;
  const size_t sbytes = stage_bytes<NX, NU>(SC, emax);
  float* Gc = (float*)(sbase + 2 * sbytes);
  float* QGc = Gc + (int64_t)SC * NX * ld;
  float* Qs = QGc + (int64_t)SC * NX * ld;
  double* wv = (double*)(((uintptr_t)(Qs + SC * NX * NX) + 15) & ~(uintptr_t)15);
  double* gs = wv + SC * NX;
  int* nptr = (int*)(gs + n0);
  // the CTA's chunk tables, staged once: unique-node offsets / ids and the
  // (node, slot) -> unique index map (no dependent global loads per item)
  const int nchk = (a.per + SC - 1) / SC;
  int* cptr = nptr + a.per + 1;                 // nchk + 1
  int* cnod = cptr + nchk + 1;                  // nchk * umax
  unsigned char* cslot = (unsigned char*)(cnod + nchk * a.umax);  // nchk * SC * dslot
  // H accumulator of the CTA (block pairs x 36, fp32): stage partials are
  // folded in once per stage
  float* Hacc = (float*)(((uintptr_t)(cslot + nchk * SC * a.dslot) + 15) & ~(uintptr_t)15);
  uint64_t* mb = (uint64_t*)(Hacc + a.npairs * NU * NU);

  for (int t = tid; t <= nn; t += nt) nptr[t] = a.ptr[nb + t];
  {
    const int c0p = a.cu_ptr[chunk0];
    for (int t = tid; t <= nsub; t += nt) cptr[t] = a.cu_ptr[chunk0 + t] - c0p;
    for (int t = tid; t < a.cu_ptr[chunk0 + nsub] - c0p; t += nt) cnod[t] = a.cu_nodes[c0p + t];
    for (int t = tid; t < nsub * SC * a.dslot; t += nt) cslot[t] = a.cu_slot[(int64_t)chunk0 * SC * a.dslot + t];
  }
  // H work of a stage is balanced over all threads: at stage k the
  // npk = k(k+1)/2 live block pairs get R = 256 / npk threads each, thread
  // (pair pp = tid % npk, slice sl = tid / npk) summing the rows
  // sl, sl + R, ... of every item of the stage in registers; the slices are
  // folded into Hacc in a fixed order at the end of the stage
  int bq = 0, bp = 0, pp = 0, sl = 0, R = 1;
  bool hact = false;
  const bool balance = nsub >= 4;  // (a CTA with 1-3 items per stage folds too often)
  float acc[NU][NU];
#pragma unroll
  for (int u = 0; u < NU; ++u)
#pragma unroll
    for (int v = 0; v < NU; ++v) acc[u][v] = 0.f;
  for (int t = tid; t < n0; t += nt) gs[t] = 0.0;
  for (int t = tid; t < a.npairs * NU * NU; t += nt) Hacc[t] = 0.f;
  if (tid == 0) {
    umma::mbar_init(&mb[0], 1);
    umma::mbar_init(&mb[1], 1);
  }
  __syncthreads();

  auto prefetch = [&](int j) {  // A / B / c / Q / x_ref blocks of item j (cp.async)
    const int n = j / nsub, s0 = nb + (j % nsub) * SC;
    const int sc = min(SC, ne - s0), k = n + 1;
    const Stage<NX, NU> S = stage_at<NX, NU>(sbase + (j & 1) * sbytes, SC, emax);
    const int64_t pstage = bi * N + n;
    const int eb = nptr[s0 - nb], ee = nptr[s0 - nb + sc];
    const int nE = ee - eb;
    const float* gas = a.a_self + (pstage * M + s0) * NX * NX;
    for (int t = tid; t < sc * NX * NX; t += nt) cp_async4(S.as + t, gas + t);
    if (nE > 0) {
      const float* gan = a.a_nbr + (pstage * a.E + eb) * NX * NX;
      for (int t = tid; t < nE * NX * NX; t += nt) cp_async4(S.an + t, gan + t);
    }
    const float* gb = a.b + (pstage * M + s0) * NX * NU;
    for (int t = tid; t < sc * NX * NU; t += nt) cp_async4(S.bb + t, gb + t);
    const double* gc = a.c + (pstage * M + s0) * NX;
    for (int t = tid; t < sc * NX; t += nt) cp_async8(S.cc + t, gc + t);
    for (int t = tid; t < sc * NX * NX; t += nt) {
      const int li = t / (NX * NX), e = t - li * NX * NX;
      cp_async8(S.qd + t, a.q + bi * a.q_stride + ((int64_t)(s0 + li) * (N + 1) + k) * NX * NX + e);
    }
    for (int t = tid; t < sc * NX; t += nt) {
      const int li = t / NX, e = t - li * NX;
      cp_async8(S.xd + t, a.xref + bi * a.xref_stride + ((int64_t)(s0 + li) * (N + 1) + k) * NX + e);
    }
    cp_async_commit();
  };
  // warp 0: TMA tiles of half h of item j (stage n rows of its unique
  // neighbours, the live chunks among {2h, 2h+1}), one lane per unique node;
  // a half without live chunks still completes its phase (expect_tx 0)
  const int lane = tid & 31;
  auto issue_half = [&](int j, int h) {
    const int n = j / nsub, sub = j % nsub;
    const int u0 = cptr[sub], U = cptr[sub + 1] - u0;
    const int nlive = (NU * n + 31) / 32, xch = XC / 32;
    const int cb = CPS * h, ceo = min(CPS * h + CPS, NCH);
    int cnt = 0;
    for (int ch = cb; ch < ceo; ++ch) cnt += (ch < nlive || ch == xch) ? 1 : 0;
    const int slotw = DB ? (j & 1) : h;
    float* dst = slotw ? nbuf1 : nbuf0;
    uint64_t* bar = &mb[slotw];
    if (lane == 0) mbar_expect_tx(bar, (uint32_t)(U * cnt * kTileBytes));
    __syncwarp();
    if (cnt == 0) return;
    for (int u = lane; u < U; u += 32) {
      const int row = (int)(((bi * M + cnod[u0 + u]) * (N + 1) + n) * NX);
      fence_proxy_async_global();
      for (int ch = cb; ch < ceo; ++ch)
        if (ch < nlive || ch == xch)
          tma_load_2d(dst + (u * CPS + (ch - cb)) * (kTileBytes / 4), &tm, ch * 32, row, bar);
    }
  };
  const int items = N * nsub;
  if (items > 0) prefetch(0);

  // stage 0: Gamma_u = 0, Gamma_x = x0 (condensing.py:205-206)
  for (int t = tid; t < nn * NX * ld; t += nt) {
    const int li = t / (NX * ld), rem = t - li * NX * ld, r = rem / ld, col = rem - r * ld;
    Wb[(int64_t)(nb + li) * node_stride + rem] = (col == XC) ? (float)a.x0[(bi * M + nb + li) * NX + r] : 0.f;
  }
  const int d0 = a.dep_ptr[split], d1 = a.dep_ptr[split + 1];
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    st_release(&flags[split], 1);
  }

  for (int j = 0; j < items; ++j) {
    const int n = j / nsub, sub = j % nsub;
    const int s0 = nb + sub * SC, sc = min(SC, ne - s0);
    const int k = n + 1;
    const int live = n * NU;
    const Stage<NX, NU> S = stage_at<NX, NU>(sbase + (j & 1) * sbytes, SC, emax);
    if (sub == 0) {
      for (int d = d0 + tid; d < d1; d += nt) {
        const int* f = &flags[a.dep[d]];
        while (ld_acquire(f) < k) __nanosleep(32);
      }
      const int npk = k * (k + 1) / 2;
      if (balance) {
        R = max(1, min(SC * NX, nt / npk));
        pp = tid % npk;
        sl = tid / npk;
        hact = sl < R;
      } else {  // few items per stage: fixed pair ownership, no folds
        R = 1;
        pp = tid;
        sl = 0;
        hact = tid < npk;
      }
      bq = (int)((sqrtf(8.f * pp + 1.f) - 1.f) * 0.5f);
      while ((bq + 1) * (bq + 2) / 2 <= pp) ++bq;
      while (bq * (bq + 1) / 2 > pp) --bq;
      bp = pp - bq * (bq + 1) / 2;
    }
    cp_async_wait_all();
    __syncthreads();
    if (tid < 32) {
      if (sub == 0) issue_half(j, 0);  // first item of a stage: its rows just became final
      if (DB) {
        if (j + 1 < items && (j + 1) / nsub == n) issue_half(j + 1, 0);  // in flight under item j
      } else {
        for (int h = 1; h < npass; ++h) issue_half(j, h);
      }
    }
    if (j + 1 < items) prefetch(j + 1);
    for (int t = tid; t < sc * NX * NX; t += nt) {
      const int li = t / (NX * NX), e = t - li * NX * NX, r = e / NX, cc = e - r * NX;
      const double* Qk = S.qd + li * NX * NX;
      Qs[t] = (float)(0.5 * (Qk[r * NX + cc] + Qk[cc * NX + r]));
    }
    const int ebase = nptr[s0 - nb];
    const unsigned char* slot = cslot + sub * SC * a.dslot;
    // Gamma rows of stage k, one half (64 columns) at a time: one thread per
    // (node, 2 columns); per column the FMA order of K-REC (closed
    // neighbourhood in slot order, rows, then the 6 products), then c on
    // Gamma_x, B on block n, zeros elsewhere
#pragma unroll 1
    for (int h = 0; h < npass; ++h) {
      const int cb0 = 32 * CPS * h, ncol = min(32 * CPS, ld - cb0);
      const int slotr = DB ? (j & 1) : h;
      umma::mbar_wait(&mb[slotr], (uint32_t)(DB ? ((j >> 1) & 1) : (j & 1)));
      const float* nbuf = slotr ? nbuf1 : nbuf0;
      const int G2 = ncol / GW;
      for (int t = tid; t < sc * G2; t += nt) {
        const int li = t / G2, c0 = cb0 + (t - li * G2) * GW;
        const int i = s0 + li;
        float r6[NX][GW];
#pragma unroll
        for (int r = 0; r < NX; ++r)
#pragma unroll
          for (int e = 0; e < GW; ++e) r6[r][e] = 0.f;
        const bool xin = c0 <= XC && XC < c0 + GW;
        if (c0 < live || xin) {
          const int el0 = nptr[i - nb] - ebase, deg = nptr[i - nb + 1] - nptr[i - nb];
          for (int ss = 0; ss <= deg; ++ss) {
            const int u = slot[li * a.dslot + ss];
            const float* g = nbuf + (u * CPS + ((c0 >> 5) - CPS * h)) * (kTileBytes / 4) + (c0 & 31);
            float w[NX][GW];
#pragma unroll
            for (int qq = 0; qq < NX; ++qq) {
              if (GW == 4) {
                const float4 v = *reinterpret_cast<const float4*>(g + qq * 32);
                w[qq][0] = v.x;
                w[qq][GW > 1 ? 1 : 0] = v.y;
                w[qq][GW > 2 ? 2 : 0] = v.z;
                w[qq][GW > 3 ? 3 : 0] = v.w;
              } else {
                const float2 v = *reinterpret_cast<const float2*>(g + qq * 32);
                w[qq][0] = v.x;
                w[qq][GW > 1 ? 1 : 0] = v.y;
              }
            }
            const float4* A4 = reinterpret_cast<const float4*>(ss == 0 ? S.as + li * NX * NX
                                                                      : S.an + (el0 + ss - 1) * NX * NX);
            float av[NX * NX];
#pragma unroll
            for (int q4 = 0; q4 < NX * NX / 4; ++q4) {
              const float4 v4 = A4[q4];
              av[4 * q4] = v4.x;
              av[4 * q4 + 1] = v4.y;
              av[4 * q4 + 2] = v4.z;
              av[4 * q4 + 3] = v4.w;
            }
#pragma unroll
            for (int r = 0; r < NX; ++r)
#pragma unroll
              for (int qq = 0; qq < NX; ++qq)
#pragma unroll
                for (int e = 0; e < GW; ++e) r6[r][e] = fmaf(av[r * NX + qq], w[qq][e], r6[r][e]);
          }
          if (xin) {
#pragma unroll
            for (int r = 0; r < NX; ++r)
#pragma unroll
              for (int e = 0; e < GW; ++e)
                if (c0 + e == XC) r6[r][e] += (float)S.cc[li * NX + r];
          }
        }
#pragma unroll
        for (int e = 0; e < GW; ++e) {
          const int col = c0 + e;
          const bool rec_col = col < live || col == XC;
          const bool b_col = col >= live && col < live + NU;
#pragma unroll
          for (int r = 0; r < NX; ++r)
            r6[r][e] = rec_col ? r6[r][e] : (b_col ? S.bb[(li * NX + r) * NU + (col - live)] : 0.f);
        }
        float* Wo = Wb + (int64_t)i * node_stride + (int64_t)k * stage_stride + c0;
        float* Gs = Gc + (int64_t)li * NX * ld + c0;
#pragma unroll
        for (int r = 0; r < NX; ++r) {
          if (GW == 4) {
            const float4 v = make_float4(r6[r][0], r6[r][GW > 1 ? 1 : 0], r6[r][GW > 2 ? 2 : 0],
                                         r6[r][GW > 3 ? 3 : 0]);
            *reinterpret_cast<float4*>(Wo + (int64_t)r * ld) = v;
            *reinterpret_cast<float4*>(Gs + (int64_t)r * ld) = v;
          } else {
            const float2 v = make_float2(r6[r][0], r6[r][GW > 1 ? 1 : 0]);
            *reinterpret_cast<float2*>(Wo + (int64_t)r * ld) = v;
            *reinterpret_cast<float2*>(Gs + (int64_t)r * ld) = v;
          }
        }
      }
      __syncthreads();  // the slot of pass h is free again
      if (!DB && h == 0 && tid < 32 && j + 1 < items && (j + 1) / nsub == n)
        issue_half(j + 1, 0);  // the next item's first pass, in flight under this item
    }
    if (sub == nsub - 1 && tid == 0) {
      __threadfence();
      st_release(&flags[split], k + 1);
    }
    // Qs G on the live columns of stage k, and w = 2 Q Gamma_x - 2 Q x_ref
    const int lk = k * NU;
    for (int t = tid; t < sc * lk; t += nt) {
      const int li = t / lk, col = t - li * lk;
      const float* Gs = Gc + (int64_t)li * NX * ld + col;
      float gcol[NX];
#pragma unroll
      for (int qq = 0; qq < NX; ++qq) gcol[qq] = Gs[(int64_t)qq * ld];
      const float* Qn = Qs + li * NX * NX;
      float* Os = QGc + (int64_t)li * NX * ld + col;
#pragma unroll
      for (int r = 0; r < NX; ++r) {
        float sacc = 0.f;
#pragma unroll
        for (int qq = 0; qq < NX; ++qq) sacc = fmaf(Qn[r * NX + qq], gcol[qq], sacc);
        Os[(int64_t)r * ld] = sacc;
      }
    }
    for (int t = tid; t < sc * NX; t += nt) {
      const int li = t / NX, r = t - li * NX;
      const double* Qk = S.qd + li * NX * NX + r * NX;
      const double* xr = S.xd + li * NX;
      const float* gx = Gc + (int64_t)li * NX * ld + XC;
      double qg = 0.0, qx = 0.0;
#pragma unroll
      for (int qq = 0; qq < NX; ++qq) {
        qg += Qk[qq] * (double)gx[(int64_t)qq * ld];
        qx += Qk[qq] * xr[qq];
      }
      wv[t] = 2.0 * qg + (-2.0 * qx);
    }
    __syncthreads();
    if (hact) {
      for (int row = sl; row < sc * NX; row += R) {
        {
          const float* gp = Gc + (int64_t)row * ld + bp * NU;
          const float* gq = QGc + (int64_t)row * ld + bq * NU;
          const float2 x01 = *reinterpret_cast<const float2*>(gp), x23 = *reinterpret_cast<const float2*>(gp + 2),
                       x45 = *reinterpret_cast<const float2*>(gp + 4);
          const float2 y01 = *reinterpret_cast<const float2*>(gq), y23 = *reinterpret_cast<const float2*>(gq + 2),
                       y45 = *reinterpret_cast<const float2*>(gq + 4);
          const float x[NU] = {x01.x, x01.y, x23.x, x23.y, x45.x, x45.y};
          const float y[NU] = {y01.x, y01.y, y23.x, y23.y, y45.x, y45.y};
#pragma unroll
          for (int u = 0; u < NU; ++u)
#pragma unroll
            for (int v = 0; v < NU; ++v) acc[u][v] = fmaf(x[u], y[v], acc[u][v]);
        }
      }
    }
    for (int cidx = tid; cidx < lk; cidx += nt) {
      double sg = gs[cidx];
      for (int li = 0; li < sc; ++li)
#pragma unroll
        for (int r = 0; r < NX; ++r) sg += (double)Gc[((int64_t)li * NX + r) * ld + cidx] * wv[li * NX + r];
      gs[cidx] = sg;
    }
    // (no barrier here: the next item's loop-top barrier orders these reads
    // of Gc / QGc before its recursion overwrites them)
    if (balance && sub == nsub - 1) {
      // fold the stage's slices into Hacc (Gc / QGc are free until the
      // next item's recursion): stage in shared memory, then each pair's
      // owner adds its R slices in slice order
      __syncthreads();
      float* stg = Gc;
      if (hact) {
#pragma unroll
        for (int u = 0; u < NU; ++u)
#pragma unroll
          for (int v = 0; v < NU; ++v) {
            stg[tid * NU * NU + u * NU + v] = acc[u][v];
            acc[u][v] = 0.f;
          }
      }
      __syncthreads();
      const int npk = k * (k + 1) / 2;
      for (int t = tid; t < npk * NU * NU; t += nt) {
        const int p2 = t / (NU * NU), e = t - p2 * NU * NU;
        float hs = Hacc[t];
        for (int s2 = 0; s2 < R; ++s2) hs += stg[(p2 + s2 * npk) * NU * NU + e];
        Hacc[t] = hs;
      }
      __syncthreads();
    }
  }

  const int PU = a.npairs * NU * NU;
  float* P = a.partH + (bi * a.splits + split) * (int64_t)PU;
  if (balance) {
    for (int t = tid; t < PU; t += nt) P[t] = Hacc[t];
  } else if (tid < a.npairs) {
#pragma unroll
    for (int u = 0; u < NU; ++u)
#pragma unroll
      for (int v = 0; v < NU; ++v) P[tid * NU * NU + u * NU + v] = acc[u][v];
  }
  for (int t = tid; t < n0; t += nt) a.partg[(bi * a.splits + split) * n0 + t] = gs[t];
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    int* done = a.flags + (int64_t)gridDim.x;
    if (atomicAdd(done, 1) == (int)gridDim.x - 1) {
      for (int s2 = 0; s2 < (int)gridDim.x; ++s2) a.flags[s2] = 0;
      *done = 0;
      __threadfence();
    }
  }
}

__device__ __forceinline__ void qpb_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void qpb_arrive(int id, int n) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// ---------------------------------------------------------------------------
// K-COND, warp-specialised pipeline (the default TMA kernel).  Per item the
// round-1/2 kernels run recursion -> QG -> H/g back to back on all warps
// with CTA barriers between them (ncu: ~40 % of warp samples at barriers,
// more warps per SM gave nothing).  Here warps 0-3 (group R) produce item j
// -- TMA tiles, recursion (Gamma rows to W and to the double-buffered Gc),
// Qs, QG, w -- while warps 4-7 (group H) fold item j-1 into H and g.  The
// groups hand items over through named barriers per Gc/QGc buffer
// (FULL: R arrives, H syncs; EMPTY: H arrives, R syncs two items later);
// each group syncs internally on its own named barrier.  Numerics are those
// of k_condense_tma (same per-column FMA order, fp32 H accumulation folded
// into the CTA accumulator once per stage in a fixed order, fp64 g).
// ---------------------------------------------------------------------------
// optional per-stage cycle accounting of k_condense_tmap (CTA 0; one thread
// per group): per stage k (< 32) 8 counters -- [0] group R item time, [1] R
// waiting for buffer EMPTY, [2] R waiting on neighbour stage flags, [3] R
// waiting for its TMA tiles, [4] group H waiting for FULL, [5] H busy, [6] H
// stage fold, [7] items; [8..11] R: blocks-in barrier + issue, Qs, recursion
// passes, flag + w; [12..15] H: Qs*G + barrier, H rows, g, rest;
// [16..21] finer R / H splits (scripts/cond_stages.py).  Compiled in only
// with -DGM_COND_PROF (make NVFLAGS+=-DGM_COND_PROF); gm_cond_profile(1)
// enables + zeroes.  (Caveat: clock reads may be scheduled across a
// bar.sync, so a barrier wait can show up in the following segment.)
__device__ unsigned long long g_cond_prof[32 * 24];
__device__ int g_cond_prof_on;
#ifdef GM_COND_PROF
constexpr bool kCondProf = true;
#else
constexpr bool kCondProf = false;
#endif
__device__ __forceinline__ long long cprof_clock(bool on) { return (kCondProf && on) ? clock64() : 0; }
__device__ __forceinline__ void cprof_add(bool on, int k, int slot, long long v) {
  if (kCondProf && on && k < 32) atomicAdd(&g_cond_prof[k * 24 + slot], (unsigned long long)v);
}

template <int SC, int CPS, int GW, bool DB, int GH, int GR = 128>
__global__ void __launch_bounds__(GR + GH, 1) k_condense_tmap(const FusedArgs a, const __grid_constant__ CUtensorMap tm) {
  constexpr int NX = 6, NU = 6;
  constexpr int GT = GR;        // group R threads (group H: GH)
  constexpr int NT = GT + GH;
  constexpr int BAR_R = 1, BAR_H = 2, BAR_FULL = 3, BAR_EMPTY = 5;  // FULL / EMPTY: + buffer
  extern __shared__ __align__(128) unsigned char smraw[];
  const int N = a.N, ld = a.ld, M = a.M;
  const int n0 = N * NU, XC = N * NU;
  const int NCH = ld / 32;
  const int tid = threadIdx.x;
  const bool grpR = tid < GT;
  const int gt = grpR ? tid : tid - GT;  // thread index within the group
  const int64_t bi = blockIdx.x / a.splits;
  const int split = (int)(blockIdx.x % a.splits);
  const int nb = split * a.per, ne = min(M, nb + a.per);
  const int nn = ne - nb;
  const int nsub = (nn + SC - 1) / SC;
  const int chunk0 = nb / SC;
  const int emax = SC * (a.dslot - 1) > 0 ? SC * (a.dslot - 1) : 1;
  int* flags = a.flags + bi * a.splits;
  const int64_t stage_stride = (int64_t)NX * ld;
  const int64_t node_stride = (int64_t)(N + 1) * stage_stride;
  float* Wb = a.W + bi * (int64_t)M * node_stride;

  // shared memory: tile ring | 2 block stages | 2 x (Gc, QGc) | Qs | 2 x wv |
  // gs | nptr | chunk tables | Hacc | mbarriers.  When shared memory is
  // short (meshes), Hacc is the CTA's fp32 partial in global memory instead
  // (folded once per stage, L2-resident)
  const int npass = (NCH + CPS - 1) / CPS;
  const size_t ring = (size_t)a.umax * CPS * kTileBytes;
  const int nslot = DB ? 2 : npass;
  float* nbuf0 = reinterpret_cast<float*>(smraw);
  float* nbuf1 = reinterpret_cast<float*>(smraw + ring);
  unsigned char* sbase = smraw + nslot * ring;
  const size_t sbytes = stage_bytes<NX, NU>(SC, emax);
  const int64_t gsz = (int64_t)SC * NX * ld;
  float* Gc2 = (float*)(sbase + 2 * sbytes);  // buffer b: Gc = Gc2 + 2 b gsz, QGc = Gc + gsz
  float* Qs2 = Gc2 + 4 * gsz;  // 2 x SC*NX*NX
  double* wv2 = (double*)(((uintptr_t)(Qs2 + 2 * SC * NX * NX) + 15) & ~(uintptr_t)15);  // 2 x SC*NX
  double* gs = wv2 + 2 * SC * NX;
  int* nptr = (int*)(gs + n0);
  const int nchk = (a.per + SC - 1) / SC;
  int* cptr = nptr + a.per + 1;
  int* cnod = cptr + nchk + 1;
  unsigned char* cslot = (unsigned char*)(cnod + nchk * a.umax);
  float* Hs = (float*)(((uintptr_t)(cslot + nchk * SC * a.dslot) + 15) & ~(uintptr_t)15);
  uint64_t* mb = (uint64_t*)(a.hacc_gl ? Hs : Hs + a.npairs * NU * NU);
  float* const P = a.partH + (bi * a.splits + split) * (int64_t)(a.npairs * NU * NU);
  float* Hacc = a.hacc_gl ? P : Hs;

  for (int t = tid; t <= nn; t += NT) nptr[t] = a.ptr[nb + t];
  {
    const int c0p = a.cu_ptr[chunk0];
    for (int t = tid; t <= nsub; t += NT) cptr[t] = a.cu_ptr[chunk0 + t] - c0p;
    for (int t = tid; t < a.cu_ptr[chunk0 + nsub] - c0p; t += NT) cnod[t] = a.cu_nodes[c0p + t];
    for (int t = tid; t < nsub * SC * a.dslot; t += NT) cslot[t] = a.cu_slot[(int64_t)chunk0 * SC * a.dslot + t];
  }
  for (int t = tid; t < n0; t += NT) gs[t] = 0.0;
  for (int t = tid; t < a.npairs * NU * NU; t += NT) Hacc[t] = 0.f;
  if (tid == 0) {
    umma::mbar_init(&mb[0], 1);
    umma::mbar_init(&mb[1], 1);
  }
  const int items = N * nsub;
  // stage 0: Gamma_u = 0, Gamma_x = x0 (condensing.py:205-206)
  for (int t = tid; t < nn * NX * ld; t += NT) {
    const int li = t / (NX * ld), rem = t - li * NX * ld, r = rem / ld, col = rem - r * ld;
    Wb[(int64_t)(nb + li) * node_stride + rem] = (col == XC) ? (float)a.x0[(bi * M + nb + li) * NX + r] : 0.f;
  }
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    st_release(&flags[split], 1);
  }

  // QGc = Qs Gc on flattened (node, column) indices [t0, t1) of the live columns
  auto qg_cols = [&](const float* Gc, const float* Qs, float* QGc, int lk, int t0, int t1) {
    for (int t = t0 + gt; t < t1; t += (grpR ? GT : GH)) {
      const int li = t / lk, col = t - li * lk;
      const float* Gs = Gc + (int64_t)li * NX * ld + col;
      float gcol[NX];
#pragma unroll
      for (int qq = 0; qq < NX; ++qq) gcol[qq] = Gs[(int64_t)qq * ld];
      const float* Qn = Qs + li * NX * NX;
      float* Os = QGc + (int64_t)li * NX * ld + col;
#pragma unroll
      for (int r = 0; r < NX; ++r) {
        float sacc = 0.f;
#pragma unroll
        for (int qq = 0; qq < NX; ++qq) sacc = fmaf(Qn[r * NX + qq], gcol[qq], sacc);
        Os[(int64_t)r * ld] = sacc;
      }
    }
  };

  if (grpR) {
    // ===================== group R: tiles, recursion, part of QG =====================
    const int lane = tid & 31;
    const bool pf = kCondProf && g_cond_prof_on && blockIdx.x == 0 && gt == 0;
    auto prefetch = [&](int j) {
      const int n = j / nsub, s0 = nb + (j % nsub) * SC;
      const int sc = min(SC, ne - s0), k = n + 1;
      const Stage<NX, NU> S = stage_at<NX, NU>(sbase + (j & 1) * sbytes, SC, emax);
      const int64_t pstage = bi * N + n;
      const int eb = nptr[s0 - nb], ee = nptr[s0 - nb + sc];
      const int nE = ee - eb;
      if (a.al16) {  // 16-byte units: A 9 per node / edge, B 9, c 3, Q 18, x_ref 3
        const char* gas = (const char*)(a.a_self + (pstage * M + s0) * NX * NX);
        for (int t = gt; t < sc * 9; t += GT) cp_async16((char*)S.as + 16 * t, gas + 16 * t);
        const char* gan = (const char*)(a.a_nbr + (pstage * a.E + eb) * NX * NX);
        for (int t = gt; t < nE * 9; t += GT) cp_async16((char*)S.an + 16 * t, gan + 16 * t);
        const char* gb = (const char*)(a.b + (pstage * M + s0) * NX * NU);
        for (int t = gt; t < sc * 9; t += GT) cp_async16((char*)S.bb + 16 * t, gb + 16 * t);
        const char* gc = (const char*)(a.c + (pstage * M + s0) * NX);
        for (int t = gt; t < sc * 3; t += GT) cp_async16((char*)S.cc + 16 * t, gc + 16 * t);
        for (int t = gt; t < sc * 18; t += GT) {
          const int li = t / 18, e = t - li * 18;
          cp_async16((char*)(S.qd + li * NX * NX) + 16 * e,
                     (const char*)(a.q + bi * a.q_stride + ((int64_t)(s0 + li) * (N + 1) + k) * NX * NX) + 16 * e);
        }
        for (int t = gt; t < sc * 3; t += GT) {
          const int li = t / 3, e = t - li * 3;
          cp_async16((char*)(S.xd + li * NX) + 16 * e,
                     (const char*)(a.xref + bi * a.xref_stride + ((int64_t)(s0 + li) * (N + 1) + k) * NX) + 16 * e);
        }
        cp_async_commit();
        return;
      }
      const float* gas = a.a_self + (pstage * M + s0) * NX * NX;
      for (int t = gt; t < sc * NX * NX; t += GT) cp_async4(S.as + t, gas + t);
      if (nE > 0) {
        const float* gan = a.a_nbr + (pstage * a.E + eb) * NX * NX;
        for (int t = gt; t < nE * NX * NX; t += GT) cp_async4(S.an + t, gan + t);
      }
      const float* gb = a.b + (pstage * M + s0) * NX * NU;
      for (int t = gt; t < sc * NX * NU; t += GT) cp_async4(S.bb + t, gb + t);
      const double* gc = a.c + (pstage * M + s0) * NX;
      for (int t = gt; t < sc * NX; t += GT) cp_async8(S.cc + t, gc + t);
      for (int t = gt; t < sc * NX * NX; t += GT) {
        const int li = t / (NX * NX), e = t - li * NX * NX;
        cp_async8(S.qd + t, a.q + bi * a.q_stride + ((int64_t)(s0 + li) * (N + 1) + k) * NX * NX + e);
      }
      for (int t = gt; t < sc * NX; t += GT) {
        const int li = t / NX, e = t - li * NX;
        cp_async8(S.xd + t, a.xref + bi * a.xref_stride + ((int64_t)(s0 + li) * (N + 1) + k) * NX + e);
      }
      cp_async_commit();
    };
    // tiles of item j, pass h: called by every group-R thread; unique node u
    // goes to warp u % (GR/32), so the group's warps issue in parallel
    auto issue_half = [&](int j, int h) {
      const int n = j / nsub, sub = j % nsub;
      const int u0 = cptr[sub], U = cptr[sub + 1] - u0;
      const int nlive = (NU * n + 31) / 32, xch = XC / 32;
      const int cb = CPS * h, ceo = min(CPS * h + CPS, NCH);
      int cnt = 0;
      for (int ch = cb; ch < ceo; ++ch) cnt += (ch < nlive || ch == xch) ? 1 : 0;
      const int slotw = DB ? (j & 1) : h;
      float* dst = slotw ? nbuf1 : nbuf0;
      uint64_t* bar = &mb[slotw];
      // one box of 6 rows x 32*CPS columns per unique node (the tensor map
      // of this kernel): dead columns ride along (zeros in W)
      // (complete_tx may precede the expect: the tx-count goes transiently
      // negative, the phase still needs gt 0's single arrival)
      if (gt == 0) mbar_expect_tx(bar, cnt ? (uint32_t)(U * CPS * kTileBytes) : 0u);
      if (cnt == 0) return;
      const int ub = (gt & 31) * (GT / 32) + (gt >> 5);
      if (ub < U) fence_proxy_async_global();
      for (int u = ub; u < U; u += GT) {
        const int row = (int)(((bi * M + cnod[u0 + u]) * (N + 1) + n) * NX);
        tma_load_2d(dst + u * CPS * (kTileBytes / 4), &tm, cb * 32, row, bar);
      }
    };
    const int d0 = a.dep_ptr[split], d1 = a.dep_ptr[split + 1];
    if (items > 0) prefetch(0);
    for (int j = 0; j < items; ++j) {
      const int n = j / nsub, sub = j % nsub;
      const int s0 = nb + sub * SC, sc = min(SC, ne - s0);
      const int k = n + 1, live = n * NU, b = j & 1;
      const Stage<NX, NU> S = stage_at<NX, NU>(sbase + (j & 1) * sbytes, SC, emax);
      float* Gc = Gc2 + 2 * b * gsz;
      double* wv = wv2 + b * SC * NX;
      const long long pt0 = cprof_clock(pf);
      if (sub == 0)
        for (int d = d0 + gt; d < d1; d += GT) {
          const int* f = &flags[a.dep[d]];
          while (ld_acquire(f) < k) __nanosleep(32);
        }
      cprof_add(pf, k, 2, cprof_clock(pf) - pt0);
      const long long pq0 = cprof_clock(pf);
      cp_async_wait_all();
      const long long pq1 = cprof_clock(pf);
      cprof_add(pf, k, 16, pq1 - pq0);
      qpb_sync(BAR_R, GT);  // blocks of item j in; the previous recursion left the tile slots
      const long long pq2 = cprof_clock(pf);
      cprof_add(pf, k, 17, pq2 - pq1);
      {
        if (sub == 0) issue_half(j, 0);
        if (DB) {
          if (j + 1 < items && (j + 1) / nsub == n) issue_half(j + 1, 0);
        } else {
          for (int h = 1; h < npass; ++h) issue_half(j, h);
        }
      }
      const long long pq3 = cprof_clock(pf);
      cprof_add(pf, k, 18, pq3 - pq2);
      if (j + 1 < items) prefetch(j + 1);
      const long long pt1 = cprof_clock(pf);
      cprof_add(pf, k, 19, pt1 - pq3);
      cprof_add(pf, k, 8, pt1 - pt0);
      if (j >= 2) qpb_sync(BAR_EMPTY + b, NT);  // group H is done with buffer b (item j-2)
      cprof_add(pf, k, 1, cprof_clock(pf) - pt1);
      float* Qs = Qs2 + b * SC * NX * NX;
      for (int t = gt; t < sc * NX * NX; t += GT) {
        const int li = t / (NX * NX), e = t - li * NX * NX, r = e / NX, cc = e - r * NX;
        const double* Qk = S.qd + li * NX * NX;
        Qs[t] = (float)(0.5 * (Qk[r * NX + cc] + Qk[cc * NX + r]));
      }
      const int ebase = nptr[s0 - nb];
      const unsigned char* slot = cslot + sub * SC * a.dslot;
      const long long pt3 = cprof_clock(pf);
      cprof_add(pf, k, 9, pt3 - pt1);
#pragma unroll 1
      for (int h = 0; h < npass; ++h) {
        const int cb0 = 32 * CPS * h, ncol = min(32 * CPS, ld - cb0);
        const int slotr = DB ? (j & 1) : h;
        const long long pt2 = cprof_clock(pf);
        umma::mbar_wait(&mb[slotr], (uint32_t)(DB ? ((j >> 1) & 1) : (j & 1)));
        cprof_add(pf, k, 3, cprof_clock(pf) - pt2);
        const float* nbuf = slotr ? nbuf1 : nbuf0;
        const int G2 = ncol / GW;
        for (int t = gt; t < sc * G2; t += GT) {
          const int li = t / G2, c0 = cb0 + (t - li * G2) * GW;
          const int i = s0 + li;
          float r6[NX][GW];
#pragma unroll
          for (int r = 0; r < NX; ++r)
#pragma unroll
            for (int e = 0; e < GW; ++e) r6[r][e] = 0.f;
          const bool xin = c0 <= XC && XC < c0 + GW;
          if (c0 < live || xin) {
            const int el0 = nptr[i - nb] - ebase, deg = nptr[i - nb + 1] - nptr[i - nb];
            for (int ss = 0; ss <= deg; ++ss) {
              const int u = slot[li * a.dslot + ss];
              const float* g = nbuf + u * CPS * (kTileBytes / 4) + (c0 - 32 * CPS * h);
              float w[NX][GW];
#pragma unroll
              for (int qq = 0; qq < NX; ++qq) {
                if (GW == 4) {
                  const float4 v = *reinterpret_cast<const float4*>(g + qq * 32 * CPS);
                  w[qq][0] = v.x;
                  w[qq][GW > 1 ? 1 : 0] = v.y;
                  w[qq][GW > 2 ? 2 : 0] = v.z;
                  w[qq][GW > 3 ? 3 : 0] = v.w;
                } else {
                  const float2 v = *reinterpret_cast<const float2*>(g + qq * 32 * CPS);
                  w[qq][0] = v.x;
                  w[qq][GW > 1 ? 1 : 0] = v.y;
                }
              }
              const float4* A4 = reinterpret_cast<const float4*>(ss == 0 ? S.as + li * NX * NX
                                                                        : S.an + (el0 + ss - 1) * NX * NX);
              float av[NX * NX];
#pragma unroll
              for (int q4 = 0; q4 < NX * NX / 4; ++q4) {
                const float4 v4 = A4[q4];
                av[4 * q4] = v4.x;
                av[4 * q4 + 1] = v4.y;
                av[4 * q4 + 2] = v4.z;
                av[4 * q4 + 3] = v4.w;
              }
#pragma unroll
              for (int r = 0; r < NX; ++r)
#pragma unroll
                for (int qq = 0; qq < NX; ++qq)
#pragma unroll
                  for (int e = 0; e < GW; ++e) r6[r][e] = fmaf(av[r * NX + qq], w[qq][e], r6[r][e]);
            }
            if (xin) {
#pragma unroll
              for (int r = 0; r < NX; ++r)
#pragma unroll
                for (int e = 0; e < GW; ++e)
                  if (c0 + e == XC) r6[r][e] += (float)S.cc[li * NX + r];
            }
          }
#pragma unroll
          for (int e = 0; e < GW; ++e) {
            const int col = c0 + e;
            const bool rec_col = col < live || col == XC;
            const bool b_col = col >= live && col < live + NU;
#pragma unroll
            for (int r = 0; r < NX; ++r)
              r6[r][e] = rec_col ? r6[r][e] : (b_col ? S.bb[(li * NX + r) * NU + (col - live)] : 0.f);
          }
          float* Wo = Wb + (int64_t)i * node_stride + (int64_t)k * stage_stride + c0;
          float* Gs = Gc + (int64_t)li * NX * ld + c0;
#pragma unroll
          for (int r = 0; r < NX; ++r) {
            if (GW == 4) {
              const float4 v = make_float4(r6[r][0], r6[r][GW > 1 ? 1 : 0], r6[r][GW > 2 ? 2 : 0],
                                           r6[r][GW > 3 ? 3 : 0]);
              *reinterpret_cast<float4*>(Wo + (int64_t)r * ld) = v;
              *reinterpret_cast<float4*>(Gs + (int64_t)r * ld) = v;
            } else {
              const float2 v = make_float2(r6[r][0], r6[r][GW > 1 ? 1 : 0]);
              *reinterpret_cast<float2*>(Wo + (int64_t)r * ld) = v;
              *reinterpret_cast<float2*>(Gs + (int64_t)r * ld) = v;
            }
          }
        }
        qpb_sync(BAR_R, GT);  // Gamma rows of the pass written; its tile slot is free again
        if (!DB && h == 0 && j + 1 < items && (j + 1) / nsub == n) issue_half(j + 1, 0);
      }
      const long long pt4 = cprof_clock(pf);
      cprof_add(pf, k, 10, pt4 - pt3);
      if (sub == nsub - 1 && gt == 0) {
        __threadfence();
        st_release(&flags[split], k + 1);
      }
      {
        const int nq = sc * k * NU;
        qg_cols(Gc, Qs, Gc + gsz, k * NU, 0, nq * a.qg_r8 / 8);
      }
      for (int t = gt; t < sc * NX; t += GT) {
        const int li = t / NX, r = t - li * NX;
        const double* Qk = S.qd + li * NX * NX + r * NX;
        const double* xr = S.xd + li * NX;
        const float* gx = Gc + (int64_t)li * NX * ld + XC;
        double qg = 0.0, qx = 0.0;
#pragma unroll
        for (int qq = 0; qq < NX; ++qq) {
          qg += Qk[qq] * (double)gx[(int64_t)qq * ld];
          qx += Qk[qq] * xr[qq];
        }
        wv[t] = 2.0 * qg + (-2.0 * qx);
      }
      __threadfence_block();
      qpb_arrive(BAR_FULL + b, NT);  // item j -> group H
      cprof_add(pf, k, 11, cprof_clock(pf) - pt4);
      cprof_add(pf, k, 0, cprof_clock(pf) - pt0);
      cprof_add(pf, k, 7, 1);
    }
    // consume group H's last EMPTY arrivals (balanced barrier phases)
    for (int j = max(items, 2); j < items + 2; ++j) qpb_sync(BAR_EMPTY + (j & 1), NT);
  } else {
    // ===================== group H: H and g =====================
    // stage k: npk = k(k+1)/2 live block pairs over 128 threads: npk <= 128
    // -> R = 128 / npk row slices per pair; npk > 128 -> two pairs per thread
    float acc0[NU][NU], acc1[NU][NU];
#pragma unroll
    for (int u = 0; u < NU; ++u)
#pragma unroll
      for (int v = 0; v < NU; ++v) acc0[u][v] = acc1[u][v] = 0.f;
    int R = 1, sl = 0, bp0 = 0, bq0 = 0, bp1 = 0, bq1 = 0;
    bool h0 = false, h1 = false;
    auto pair_of = [](int p, int& bp, int& bq) {
      bq = (int)((sqrtf(8.f * p + 1.f) - 1.f) * 0.5f);
      while ((bq + 1) * (bq + 2) / 2 <= p) ++bq;
      while (bq * (bq + 1) / 2 > p) --bq;
      bp = p - bq * (bq + 1) / 2;
    };
    for (int j = 0; j < items; ++j) {
      const int n = j / nsub, sub = j % nsub;
      const int s0 = nb + sub * SC, sc = min(SC, ne - s0);
      const int k = n + 1, b = j & 1, npk = k * (k + 1) / 2;
      float* Gc = Gc2 + 2 * b * gsz;
      float* QGc = Gc + gsz;
      const double* wv = wv2 + b * SC * NX;
      if (sub == 0) {
        if (npk <= GH) {
          // one item per stage (cfg3-like): at most 4 row slices, so the
          // staged fold sums few slices (A/B: cfg3 K-COND -2 %; with several
          // items per stage the fold is amortised and wide slicing wins)
          R = max(1, min(nsub == 1 ? 4 : SC * NX, GH / npk));
          sl = gt / npk;
          h0 = sl < R;
          h1 = false;
          pair_of(gt % npk, bp0, bq0);
        } else {
          R = 1;
          sl = 0;
          h0 = true;
          h1 = gt + GH < npk;
          pair_of(gt, bp0, bq0);
          pair_of(min(gt + GH, npk - 1), bp1, bq1);
        }
      }
      const bool pf = kCondProf && g_cond_prof_on && blockIdx.x == 0 && gt == 0;
      const long long ph0 = cprof_clock(pf);
      qpb_sync(BAR_FULL + b, NT);  // item j from group R
      const long long ph1 = cprof_clock(pf);
      cprof_add(pf, k, 4, ph1 - ph0);
      // Qs G on the live columns of stage k (group H: balances the groups)
      {
        const int nq = sc * k * NU;
        qg_cols(Gc, Qs2 + b * SC * NX * NX, QGc, k * NU, nq * a.qg_r8 / 8, nq);
        cprof_add(pf, k, 21, cprof_clock(pf) - ph1);
        qpb_sync(BAR_H, GH);
      }
      const long long ph3 = cprof_clock(pf);
      cprof_add(pf, k, 12, ph3 - ph1);
      auto hrow = [&](int bp, int bq, float (&acc)[NU][NU]) {
        for (int row = sl; row < sc * NX; row += R) {
          const float* gp = Gc + (int64_t)row * ld + bp * NU;
          const float* gq = QGc + (int64_t)row * ld + bq * NU;
          const float2 x01 = *reinterpret_cast<const float2*>(gp), x23 = *reinterpret_cast<const float2*>(gp + 2),
                       x45 = *reinterpret_cast<const float2*>(gp + 4);
          const float2 y01 = *reinterpret_cast<const float2*>(gq), y23 = *reinterpret_cast<const float2*>(gq + 2),
                       y45 = *reinterpret_cast<const float2*>(gq + 4);
          const float x[NU] = {x01.x, x01.y, x23.x, x23.y, x45.x, x45.y};
          const float y[NU] = {y01.x, y01.y, y23.x, y23.y, y45.x, y45.y};
#pragma unroll
          for (int u = 0; u < NU; ++u)
#pragma unroll
            for (int v = 0; v < NU; ++v) acc[u][v] = fmaf(x[u], y[v], acc[u][v]);
        }
      };
      if (h0) hrow(bp0, bq0, acc0);
      if (h1) hrow(bp1, bq1, acc1);
      const long long ph4 = cprof_clock(pf);
      cprof_add(pf, k, 13, ph4 - ph3);
      const int lk = k * NU;
      for (int cidx = gt; cidx < lk; cidx += GH) {
        // three fp64 chains (rows r, r + 3 of each node) instead of one
        // 6 sc-long chain, folded in a fixed order
        double s0 = gs[cidx], s1 = 0.0, s2 = 0.0;
#pragma unroll
        for (int li = 0; li < SC; ++li) {
          if (li >= sc) break;
          const float* gcol = Gc + (int64_t)li * NX * ld + cidx;
          const double* w = wv + li * NX;
#pragma unroll
          for (int r = 0; r < NX; r += 3) {
            s0 = fma((double)gcol[(int64_t)r * ld], w[r], s0);
            s1 = fma((double)gcol[(int64_t)(r + 1) * ld], w[r + 1], s1);
            s2 = fma((double)gcol[(int64_t)(r + 2) * ld], w[r + 2], s2);
          }
        }
        gs[cidx] = s0 + (s1 + s2);
      }
      const long long ph2 = cprof_clock(pf);
      cprof_add(pf, k, 14, ph2 - ph4);
      if (sub == nsub - 1 && R == 1) {
        // one owner per pair (pair gt, and gt + GH): fold in place, no
        // staging and no barriers (same sums as the staged fold with R = 1)
        if (h0) {
          float* hp = Hacc + (int64_t)gt * NU * NU;
#pragma unroll
          for (int u = 0; u < NU; ++u)
#pragma unroll
            for (int v = 0; v < NU; ++v) {
              hp[u * NU + v] += acc0[u][v];
              acc0[u][v] = 0.f;
            }
        }
        if (h1) {
          float* hp = Hacc + (int64_t)(gt + GH) * NU * NU;
#pragma unroll
          for (int u = 0; u < NU; ++u)
#pragma unroll
            for (int v = 0; v < NU; ++v) {
              hp[u * NU + v] += acc1[u][v];
              acc1[u][v] = 0.f;
            }
        }
      } else if (sub == nsub - 1) {
        // fold the stage into Hacc through this buffer (group R does not
        // touch it before our EMPTY arrival): slot gt <- acc0, gt + 128 <- acc1
        float* stg = Gc;
        qpb_sync(BAR_H, GH);  // every H thread is done reading buffer b
        if (h0)
#pragma unroll
          for (int u = 0; u < NU; ++u)
#pragma unroll
            for (int v = 0; v < NU; ++v) {
              stg[gt * NU * NU + u * NU + v] = acc0[u][v];
              acc0[u][v] = 0.f;
            }
        if (h1)
#pragma unroll
          for (int u = 0; u < NU; ++u)
#pragma unroll
            for (int v = 0; v < NU; ++v) {
              stg[(gt + GH) * NU * NU + u * NU + v] = acc1[u][v];
              acc1[u][v] = 0.f;
            }
        qpb_sync(BAR_H, GH);
#pragma unroll 4
        for (int t = gt; t < npk * NU * NU; t += GH) {
          const int p2 = t / (NU * NU), e = t - p2 * NU * NU;
          float hs = Hacc[t];
          for (int s2 = 0; s2 < R; ++s2) hs += stg[(p2 + s2 * npk) * NU * NU + e];
          Hacc[t] = hs;
        }
        qpb_sync(BAR_H, GH);
      }
      qpb_arrive(BAR_EMPTY + b, NT);  // buffer b back to group R
      cprof_add(pf, k, 5, cprof_clock(pf) - ph1);
      cprof_add(pf, k, 6, cprof_clock(pf) - ph2);
    }
  }
  __syncthreads();
  if (!a.hacc_gl)
    for (int t = tid; t < a.npairs * NU * NU; t += NT) P[t] = Hacc[t];
  for (int t = tid; t < n0; t += NT) a.partg[(bi * a.splits + split) * n0 + t] = gs[t];
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    int* done = a.flags + (int64_t)gridDim.x;
    if (atomicAdd(done, 1) == (int)gridDim.x - 1) {
      for (int s2 = 0; s2 < (int)gridDim.x; ++s2) a.flags[s2] = 0;
      *done = 0;
      __threadfence();
    }
  }
}

// ---------------------------------------------------------------------------
// K-COND on the tensor cores (n0 = N*nu <= 128): the same persistent stage
// wavefront and the same fp32 Gamma recursion as k_condense_fused, but the
// node reduction of H -- per work item of SC nodes a rank-(SC*nx) update
//     H += G' (Qs G),   G = stage-k Gamma_u rows of the item (SC*nx x n0)
// -- runs as tcgen05.mma kind::tf32 in 3xTF32 form (umma.cuh) into one
// 128 x 128 fp32 accumulator in TMEM per CTA.  The recursion writes its rows
// straight into the K-major operand buffers (hi/lo split), one elected thread
// issues 3 * KC/8 MMAs of N = round16(k*nu) columns (causality: only the first
// k*nu columns are live at stage k) and commits to an mbarrier.  g rides on
// the tensor core too: a 16-row B operand whose row 0 is w = 2 Q Gamma_x -
// 2 Q x_ref accumulates sum G' w into TMEM column 128 (fp32 per CTA, fp64
// fixed-order reduction).  Latency hiding: within a stage the next item's
// first neighbour rows are loaded into registers while the current item's
// operands are built, and each thread waits for the previous item's MMAs
// only right before it overwrites an operand buffer.  At the end the accumulator
// is read back with tcgen05.ld into the same per-CTA pair-ordered partials
// the SIMT kernel writes, so the fixed-order fp64 reduction is shared.
// ---------------------------------------------------------------------------
// Division by a per-item runtime divisor d >= 1 through its fp32 reciprocal
// and one correction step: exact for 0 <= t < 2^22 (every dividend below is
// a (node, column) index of one item, < 16 x 129).  ~6 instructions instead
// of the ~20 of an integer division; the item loops issue several per item.
struct FDiv {
  int d;
  float r;
};
__device__ __forceinline__ FDiv fdiv_make(int d) { return FDiv{d, d > 0 ? __frcp_rn((float)d) : 0.f}; }
__device__ __forceinline__ int fdiv(const FDiv& f, int t, int& rem) {
  int q = __float2int_rz(__int2float_rn(t) * f.r);
  int r = t - q * f.d;
  if (r < 0) {
    --q;
    r += f.d;
  } else if (r >= f.d) {
    ++q;
    r -= f.d;
  }
  rem = r;
  return q;
}

template <int NX, int NU>
__global__ void __launch_bounds__(kTcThreads, 1) k_condense_tc(const FusedArgs a) {
  extern __shared__ __align__(16) unsigned char smraw[];
  const int N = a.N, ld = a.ld, SC = a.sc, M = a.M;
  const int n0 = N * NU, XC = N * NU;
  const int tid = threadIdx.x, nt = blockDim.x, warp = tid >> 5;
  const int64_t bi = blockIdx.x / a.splits;
  const int split = (int)(blockIdx.x % a.splits);
  const int nb = a.lo + split * a.per, ne = min(a.hi, nb + a.per);
  const bool rec = a.rec != 0;
  const int nn = ne - nb;
  const int nsub = (nn + SC - 1) / SC;
  const int emax = SC * (a.dslot - 1) > 0 ? SC * (a.dslot - 1) : 1;
  const int KC = ((SC * NX + 7) / 8) * 8;               // K rows per item, MMA-padded
  const uint32_t sbo = (uint32_t)(KC / 4) * 128u;        // 8-row group stride
  const size_t bufb = 16 * (size_t)sbo;                  // 128-row operand buffer
  int* flags = rec ? a.flags + bi * a.splits : nullptr;
  const int64_t stage_stride = (int64_t)NX * ld;
  const int64_t node_stride = (int64_t)(N + 1) * stage_stride;
  float* Wb = a.W + bi * (int64_t)M * node_stride;

  const size_t sbytes = stage_bytes<NX, NU>(SC, emax);
  unsigned char* ops = smraw + ((2 * sbytes + 127) & ~size_t(127));
  unsigned char* g_hi = ops;
  unsigned char* g_lo = ops + bufb;
  unsigned char* q_hi = ops + 2 * bufb;
  unsigned char* q_lo = ops + 3 * bufb;
  unsigned char* w_hi = ops + 4 * bufb;                  // 16-row B operand: row 0 = g weights
  unsigned char* w_lo = w_hi + 2 * sbo;
  float* Qs = (float*)(w_lo + 2 * sbo);                  // SC x NX*NX  (Q + Q')/2
  float* gx = Qs + SC * NX * NX;                         // SC x NX     Gamma_x rows
  double* wv = (double*)(((uintptr_t)(gx + SC * NX) + 15) & ~(uintptr_t)15);  // SC x NX
  double* gs = wv + SC * NX;                             // n0
  uint64_t* mbar = (uint64_t*)(gs + n0);
  uint32_t* tslot = (uint32_t*)(mbar + 1);
  int* nptr = (int*)(tslot + 2);                         // nn + 1

  if (warp == 0) umma::tmem_alloc<256>(tslot);  // H in columns [0, 128), g in column 128
  if (tid == 32) umma::mbar_init(mbar, 1);
  for (int t = tid; t <= nn; t += nt) nptr[t] = a.ptr[nb + t];
  for (int t = tid; t < (int)((4 * bufb + 4 * sbo) / 16); t += nt) ((float4*)ops)[t] = make_float4(0.f, 0.f, 0.f, 0.f);
  umma::fence_before();
  __syncthreads();
  umma::fence_after();
  const uint32_t tmem = *tslot;
  uint32_t phase = 0;
  bool pending = false, issued = false;
  float wpre[5][NX];
  bool pre_ok = false;
  // per-thread wait for the previous item's MMAs (they read the operand
  // buffers) just before this thread first overwrites them, so the tensor
  // core overlaps the neighbour loads and FMAs of the next item
  auto operands_free = [&]() {
    if (pending) {
      umma::mbar_wait(mbar, phase);
      phase ^= 1;
      pending = false;
      umma::fence_after();
    }
  };

  // stage operands of item j: 16-byte cp.async for every contiguous segment
  // (a_self, a_nbr, b, c of the chunk; Q and x_ref per node), 4-byte for the
  // edge sources
  auto prefetch = [&](int j, int n, int sub) {
    const int s0 = nb + sub * SC;
    const int sc = min(SC, ne - s0), k = n + 1;
    const Stage<NX, NU> S = stage_at<NX, NU>(smraw + (j & 1) * sbytes, SC, emax);
    const int64_t pstage = bi * N + n;
    const int eb = nptr[s0 - nb], ee = nptr[s0 - nb + sc];
    const int nE = ee - eb;
    constexpr int A4 = NX * NX / 4, C2 = NX / 2;  // 16-byte units per node / edge
    static_assert((NX * NX) % 4 == 0 && NX % 2 == 0, "16-byte staging");
    if (rec) {
    const float4* gas = (const float4*)(a.a_self + (pstage * M + s0) * NX * NX);
    for (int t = tid; t < sc * A4; t += nt) cp_async16((float4*)S.as + t, gas + t);
    if (nE > 0) {
      const float4* gan = (const float4*)(a.a_nbr + (pstage * a.E + eb) * NX * NX);
      for (int t = tid; t < nE * A4; t += nt) cp_async16((float4*)S.an + t, gan + t);
      for (int t = tid; t < nE; t += nt) cp_async4(S.src + t, a.src + eb + t);
    }
    if constexpr ((NX * NU) % 4 == 0) {
      const float4* gb = (const float4*)(a.b + (pstage * M + s0) * NX * NU);
      for (int t = tid; t < sc * (NX * NU / 4); t += nt) cp_async16((float4*)S.bb + t, gb + t);
    } else {
      const float* gb = a.b + (pstage * M + s0) * NX * NU;
      for (int t = tid; t < sc * NX * NU; t += nt) cp_async4(S.bb + t, gb + t);
    }
    const double2* gc = (const double2*)(a.c + (pstage * M + s0) * NX);
    for (int t = tid; t < sc * C2; t += nt) cp_async16((double2*)S.cc + t, gc + t);
    }
    constexpr int Q2 = NX * NX / 2;
    for (int t = tid; t < sc * Q2; t += nt) {
      const int li = t / Q2, e = t - li * Q2;
      const double2* gq = (const double2*)(a.q + bi * a.q_stride + ((int64_t)(s0 + li) * (N + 1) + k) * NX * NX);
      cp_async16((double2*)S.qd + t, gq + e);
    }
    for (int t = tid; t < sc * C2; t += nt) {
      const int li = t / C2, e = t - li * C2;
      const double2* gx = (const double2*)(a.xref + bi * a.xref_stride + ((int64_t)(s0 + li) * (N + 1) + k) * NX);
      cp_async16((double2*)S.xd + t, gx + e);
    }
    cp_async_commit();
  };
  const int items = N * nsub;
  if (items > 0) prefetch(0, 0, 0);

  // stage 0: Gamma_u = 0, Gamma_x = x0 (condensing.py:205-206)
  for (int row = warp; rec && row < nn * NX; row += nt >> 5) {
    const int li = row / NX, r = row - li * NX;
    float* Wr0 = Wb + (int64_t)(nb + li) * node_stride + (int64_t)r * ld;
    const float x0v = (float)a.x0[(bi * M + nb + li) * NX + r];
    for (int col = tid & 31; col < ld; col += 32) Wr0[col] = (col == XC) ? x0v : 0.f;
  }
  const int d0 = rec ? a.dep_ptr[split] : 0, d1 = rec ? a.dep_ptr[split + 1] : 0;
  __syncthreads();
  if (rec && tid == 0) {
    __threadfence();
    st_release(&flags[split], 1);
  }

  for (int j = 0, n = 0, sub = 0; j < items; ++j, n += (sub + 1 == nsub), sub = (sub + 1 == nsub) ? 0 : sub + 1) {
    const int s0 = nb + sub * SC, sc = min(SC, ne - s0);
    const int k = n + 1;
    const int live = n * NU;
    const Stage<NX, NU> S = stage_at<NX, NU>(smraw + (j & 1) * sbytes, SC, emax);
    if (rec && sub == 0) {
      for (int d = d0 + tid; d < d1; d += nt) {
        const int* f = &flags[a.dep[d]];
        while (ld_acquire(f) < k) __nanosleep(32);
      }
    }
    cp_async_wait_all();
    __syncthreads();
    if (j + 1 < items) prefetch(j + 1, sub + 1 == nsub ? n + 1 : n, sub + 1 == nsub ? 0 : sub + 1);
    for (int t = tid; t < sc * NX * NX; t += nt) {
      const int li = t / (NX * NX), e = t - li * NX * NX, r = e / NX, cc = e - r * NX;
      const double* Qk = S.qd + li * NX * NX;
      Qs[t] = (float)(0.5 * (Qk[r * NX + cc] + Qk[cc * NX + r]));
    }
    const int ebase = nptr[s0 - nb];
    // (R1) the live Gamma_u columns and Gamma_x of stage k (condensing.py:213-
    // 224): one (node, column) per thread over the closed neighbourhood, all
    // neighbour loads of a node issued before the FMAs (one L2/DRAM round
    // trip for deg < 5); work spread over live columns only
    // without the recursion (K-HG on tcgen05) the rows are read from Gamma:
    // the live columns, the B block and Gamma_x of stage k
    const int nlive = rec ? live : live + NU;
    const int lw = nlive + 1;
    const FDiv flw = fdiv_make(lw);
    for (int t = tid, it = 0; t < sc * lw; t += nt, ++it) {
      int cc;
      const int li = fdiv(flw, t, cc);
      const int col = cc < nlive ? cc : XC;
      const int i = s0 + li;
      float r6[NX];
#pragma unroll
      for (int r = 0; r < NX; ++r) r6[r] = 0.f;
      if (!rec) {
        const float* Wr = Wb + (int64_t)i * node_stride + (int64_t)k * stage_stride + col;
#pragma unroll
        for (int r = 0; r < NX; ++r) r6[r] = __ldcg(Wr + (int64_t)r * ld);
      } else {
      const int el0 = nptr[i - nb] - ebase, deg = nptr[i - nb + 1] - nptr[i - nb];
      const float* Wn = Wb + (int64_t)n * stage_stride + col;
      for (int s = 0; s <= deg; s += 5) {
        float w[5][NX];
        if (s == 0 && it == 0 && pre_ok) {  // loaded during the previous item
#pragma unroll
          for (int u = 0; u < 5; ++u)
#pragma unroll
            for (int qq = 0; qq < NX; ++qq) w[u][qq] = wpre[u][qq];
        } else {
#pragma unroll
          for (int u = 0; u < 5; ++u) {
            const int ss = s + u;
            if (ss <= deg) {
              const int jn = ss == 0 ? i : S.src[el0 + ss - 1];
              const float* Wj = Wn + (int64_t)jn * node_stride;
#pragma unroll
              for (int qq = 0; qq < NX; ++qq) w[u][qq] = __ldcg(Wj + (int64_t)qq * ld);
            }
          }
        }
#pragma unroll
        for (int u = 0; u < 5; ++u) {
          const int ss = s + u;
          if (ss <= deg) {
            // block as 16-byte shared loads (broadcast within the warp),
            // consumed two rows at a time to bound register pressure
            const float4* A4 =
                (const float4*)(ss == 0 ? S.as + li * NX * NX : S.an + (el0 + ss - 1) * NX * NX);
            if constexpr ((2 * NX) % 4 == 0) {
#pragma unroll
              for (int r = 0; r < NX; r += 2) {
                float ab[2 * NX];
#pragma unroll
                for (int e = 0; e < 2 * NX / 4; ++e) {
                  const float4 v = A4[(r * NX) / 4 + e];
                  ab[4 * e] = v.x;
                  ab[4 * e + 1] = v.y;
                  ab[4 * e + 2] = v.z;
                  ab[4 * e + 3] = v.w;
                }
#pragma unroll
                for (int qq = 0; qq < NX; ++qq) {
                  r6[r] = fmaf(ab[qq], w[u][qq], r6[r]);
                  r6[r + 1] = fmaf(ab[NX + qq], w[u][qq], r6[r + 1]);
                }
              }
            } else {
              const float* Af = (const float*)A4;
#pragma unroll
              for (int r = 0; r < NX; ++r)
#pragma unroll
                for (int qq = 0; qq < NX; ++qq) r6[r] = fmaf(Af[r * NX + qq], w[u][qq], r6[r]);
            }
          }
        }
      }
      if (col == XC) {
#pragma unroll
        for (int r = 0; r < NX; ++r) r6[r] += (float)S.cc[li * NX + r];
      }
      float* Wo = Wb + (int64_t)i * node_stride + (int64_t)k * stage_stride + col;
#pragma unroll
      for (int r = 0; r < NX; ++r) Wo[(int64_t)r * ld] = r6[r];
      }
      operands_free();
      if (col < n0) {
        umma::putn_split<NX>(g_hi, g_lo, col, li * NX, sbo, r6);
      } else {
#pragma unroll
        for (int r = 0; r < NX; ++r) gx[li * NX + r] = r6[r];
      }
    }
    // (R2) block n <- B_n, every other column zero (global rows only: the
    // operand buffers hold zeros beyond the live columns already)
    operands_free();
    const int nz = rec ? ld - lw : 0;
    const FDiv fnz = fdiv_make(nz);
    for (int t = tid; t < sc * nz; t += nt) {
      int cc;
      const int li = fdiv(fnz, t, cc);
      int col = live + cc;
      if (col >= XC) ++col;
      const int i = s0 + li;
      float r6[NX];
      const bool isb = col < live + NU;
#pragma unroll
      for (int r = 0; r < NX; ++r) r6[r] = isb ? S.bb[(li * NX + r) * NU + (col - live)] : 0.f;
      float* Wo = Wb + (int64_t)i * node_stride + (int64_t)k * stage_stride + col;
#pragma unroll
      for (int r = 0; r < NX; ++r) Wo[(int64_t)r * ld] = r6[r];
      if (isb) umma::putn_split<NX>(g_hi, g_lo, col, li * NX, sbo, r6);
    }
    // padding nodes of a short last chunk: zero K rows
    for (int t = tid; t < (SC - sc) * live; t += nt) {
      const int li = sc + t / live, col = t - (t / live) * live;
      float z[NX];
#pragma unroll
      for (int r = 0; r < NX; ++r) z[r] = 0.f;
      umma::putn_split<NX>(g_hi, g_lo, col, li * NX, sbo, z);
    }
    if (sc < SC) {
      for (int t = tid; t < (SC - sc) * NU; t += nt) {
        const int li = sc + t / NU, col = live + t % NU;
        float z[NX];
#pragma unroll
        for (int r = 0; r < NX; ++r) z[r] = 0.f;
        umma::putn_split<NX>(g_hi, g_lo, col, li * NX, sbo, z);
      }
    }
    __syncthreads();
    if (rec && sub == nsub - 1 && tid == 0) {  // all of this CTA's stage-k rows are out
      __threadfence();
      st_release(&flags[split], k + 1);
    }
    // register prefetch of the next item's first (node, column) neighbour
    // rows (same stage: its dependencies are already met), in flight while
    // this item's B operand is built and its MMAs run
    pre_ok = false;
    if (rec && a.reg_prefetch && sub + 1 < nsub) {
      const int s0n = s0 + SC, scn = min(SC, ne - s0n);
      if (tid < scn * lw) {
        int cc;
        const int li = fdiv(flw, tid, cc);
        const int col = cc < live ? cc : XC;
        const int i = s0n + li;
        const int e0 = nptr[i - nb], deg = nptr[i - nb + 1] - e0;
        const float* Wn = Wb + (int64_t)n * stage_stride + col;
#pragma unroll
        for (int u = 0; u < 5; ++u) {
          if (u <= deg) {
            const int jn = u == 0 ? i : __ldg(a.src + e0 + u - 1);
            const float* Wj = Wn + (int64_t)jn * node_stride;
#pragma unroll
            for (int qq = 0; qq < NX; ++qq) wpre[u][qq] = __ldcg(Wj + (int64_t)qq * ld);
          }
        }
        pre_ok = true;
      }
    }
    // Qs G on the live columns of stage k -> B operand; w = 2 Q Gamma_x - 2 Q x_ref
    const int lk = k * NU;
    const FDiv flk = fdiv_make(lk);
    for (int t = tid; t < SC * lk; t += nt) {
      int col;
      const int li = fdiv(flk, t, col);
      float gcol[NX], o[NX];
      umma::getn<NX>(g_hi, g_lo, col, li * NX, sbo, gcol);
      const float4* Qn4 = (const float4*)(Qs + li * NX * NX);
#pragma unroll
      for (int r = 0; r < NX; ++r) o[r] = 0.f;
      if (li < sc) {
#pragma unroll
        for (int e = 0; e < NX * NX / 4; ++e) {
          const float4 q4 = Qn4[e];
          const float qv[4] = {q4.x, q4.y, q4.z, q4.w};
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int idx = 4 * e + u, r = idx / NX, qq = idx % NX;
            o[r] = fmaf(qv[u], gcol[qq], o[r]);
          }
        }
      }
      umma::putn_split<NX>(q_hi, q_lo, col, li * NX, sbo, o);
    }
    // g weights w = 2 Q Gamma_x - 2 Q x_ref (fp64, condensing.py:388) as row 0
    // of the 16-row B operand: a second MMA chain accumulates g = sum G' w
    for (int t = tid; t < SC * NX; t += nt) {
      const int li = t / NX, r = t - li * NX;
      double wr = 0.0;
      if (li < sc) {
        const double* Qk = S.qd + li * NX * NX + r * NX;
        const double* xr = S.xd + li * NX;
        double qg = 0.0, qx = 0.0;
#pragma unroll
        for (int qq = 0; qq < NX; ++qq) {
          qg += Qk[qq] * (double)gx[li * NX + qq];
          qx += Qk[qq] * xr[qq];
        }
        wr = 2.0 * qg + (-2.0 * qx);
      }
      umma::put_split(w_hi, w_lo, 0, t, sbo, (float)wr);
    }
    umma::fence_async_smem();
    __syncthreads();
    if (tid == 0) {
      umma::fence_after();
      // H: N = the live columns of stage k (TMEM is not zeroed by
      // tcgen05.alloc: the first MMA, accumulate = 0, spans every column
      // used later); g: N = 16 from the w operand into TMEM column 128
      const int Nm = max(16, (((issued ? lk : n0) + 15) / 16) * 16);
      umma::gram_3xtf32(tmem, g_hi, g_lo, sbo, q_hi, q_lo, sbo, KC / 8, umma::idesc_tf32(128, Nm), issued);
      umma::gram_3xtf32(tmem + 128, g_hi, g_lo, sbo, w_hi, w_lo, sbo, KC / 8, umma::idesc_tf32(128, 16),
                        issued);
      umma::commit(mbar);
    }
    pending = true;
    issued = true;
    // no barrier here: the next item's loop-top barrier orders the MMA issue
    // before any operand rewrite (each thread also waits on the mbarrier)
  }
  if (pending) {
    umma::mbar_wait(mbar, phase);
    umma::fence_after();
  }

  // partials: TMEM row m = p*nu + u, column c = q*nu + v -> pair (p, q), p <= q
  const int PU = a.npairs * NU * NU;
  float* P = a.partH + (bi * a.splits + split) * (int64_t)PU;
  {
    const int m = (warp & 3) * 32 + (tid & 31);
    const int cw = 128 / (nt / 128);  // columns per warp quadruple
    const int cbeg = (warp >> 2) * cw;
    const int p = m / NU, u = m - p * NU;
    for (int c0 = cbeg; c0 < cbeg + cw; c0 += 16) {
      float v[16];
      umma::tmem_ld16(tmem + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)c0, v);
      if (m < n0) {
#pragma unroll
        for (int jj = 0; jj < 16; ++jj) {
          const int c = c0 + jj;
          const int q = c / NU, vv = c - q * NU;
          if (c < n0 && p <= q) P[(q * (q + 1) / 2 + p) * NU * NU + u * NU + vv] = issued ? v[jj] : 0.f;
        }
      }
    }
  }
  if (warp < 4) {
    float v[16];
    const int m = warp * 32 + (tid & 31);
    umma::tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + 128u, v);
    if (m < n0) a.partg[(bi * a.splits + split) * n0 + m] = issued ? (double)v[0] : 0.0;
  }
  umma::fence_before();
  __syncthreads();
  if (warp == 0) umma::tmem_free<256>(tmem);
  if (rec && tid == 0) {
    __threadfence();
    int* done = a.flags + (int64_t)gridDim.x;
    if (atomicAdd(done, 1) == (int)gridDim.x - 1) {
      for (int s = 0; s < (int)gridDim.x; ++s) a.flags[s] = 0;
      *done = 0;
      __threadfence();
    }
  }
}

struct PairReduceArgs {
  int nu, n0, npairs, splits, groups;
  const float* partH;
  const double* partg;
  double* tmpH;  // (B, groups, npairs*nu*nu)
  double* tmpg;  // (B, groups, n0)
  const double* r;
  int64_t r_stride;
  const double* uref;
  int64_t uref_stride;
  double* H;
  double* g;
};

// pass 1: fixed-order sum of one group of CTA partials, coalesced
__global__ void k_pair_reduce1(const PairReduceArgs a) {
  const int PU = a.npairs * a.nu * a.nu;
  const int64_t bi = blockIdx.z;
  const int grp = blockIdx.y;
  const int per = (a.splits + a.groups - 1) / a.groups;
  const int s0 = grp * per, s1 = min(a.splits, s0 + per);
  const int u = blockIdx.x * blockDim.x + threadIdx.x;
  if (u < PU) {
    const float* P = a.partH + bi * a.splits * (int64_t)PU + u;
    double s = 0.0;
#pragma unroll 4
    for (int sp = s0; sp < s1; ++sp) s += (double)P[(int64_t)sp * PU];
    a.tmpH[(bi * a.groups + grp) * (int64_t)PU + u] = s;
  }
  if (u < a.n0) {
    double s = 0.0;
    for (int sp = s0; sp < s1; ++sp) s += a.partg[(bi * a.splits + sp) * a.n0 + u];
    a.tmpg[(bi * a.groups + grp) * a.n0 + u] = s;
  }
}

// pass 2: H = S + R-bar, mirrored (diagonal blocks averaged so H is exactly
// symmetric), g = sum + r_lin (condensing.py:154, :380-381, :388, :403)
__global__ void k_pair_reduce2(const PairReduceArgs a) {
  const int nu = a.nu, nn = nu * nu, n0 = a.n0;
  const int PU = a.npairs * nn;
  const int64_t bi = blockIdx.y;
  const int u = blockIdx.x * blockDim.x + threadIdx.x;
  const double* T = a.tmpH + bi * a.groups * (int64_t)PU;
  auto S = [&](int idx) {
    double s = 0.0;
    for (int grp = 0; grp < a.groups; ++grp) s += T[(int64_t)grp * PU + idx];
    return s;
  };
  if (u < PU) {
    const int t = u / nn, e = u - t * nn, ea = e / nu, eb = e - ea * nu;
    int q = (int)((sqrtf(8.f * t + 1.f) - 1.f) * 0.5f);
    while ((q + 1) * (q + 2) / 2 <= t) ++q;
    while (q * (q + 1) / 2 > t) --q;
    const int p = t - q * (q + 1) / 2;
    const int c1 = p * nu + ea, c2 = q * nu + eb;
    double* Hb = a.H + bi * (int64_t)n0 * n0;
    if (p < q) {
      const double h = S(u);
      Hb[(int64_t)c1 * n0 + c2] = h;
      Hb[(int64_t)c2 * n0 + c1] = h;
    } else if (ea <= eb) {
      double h = 0.5 * (S(u) + S(t * nn + eb * nu + ea));
      if (a.r) {
        const double* Rk = a.r + bi * a.r_stride + (int64_t)p * nn;
        h += 0.5 * (Rk[ea * nu + eb] + Rk[eb * nu + ea]);
      }
      Hb[(int64_t)c1 * n0 + c2] = h;
      Hb[(int64_t)c2 * n0 + c1] = h;
    }
  }
  if (u < n0) {
    double s = 0.0;
    for (int grp = 0; grp < a.groups; ++grp) s += a.tmpg[(bi * a.groups + grp) * n0 + u];
    if (a.r) {
      const int k = u / nu, row = u % nu;
      const double* Rk = a.r + bi * a.r_stride + (int64_t)k * nn + row * nu;
      const double* uk = a.uref + bi * a.uref_stride + (int64_t)k * nu;
      double ru = 0.0;
      for (int j = 0; j < nu; ++j) ru += Rk[j] * uk[j];
      s = -2.0 * ru + s;
    }
    a.g[bi * n0 + u] = s;
  }
}

using FusedKernel = void (*)(const FusedArgs);

FusedKernel pick_tc_kernel(int nx, int nu) {
  if (nx == 6 && nu == 6) return k_condense_tc<6, 6>;
  if (nx == 6 && nu == 3) return k_condense_tc<6, 3>;
  if (nx == 6 && nu == 2) return k_condense_tc<6, 2>;
  if (nx == 6 && nu == 1) return k_condense_tc<6, 1>;
  if (nx == 4 && nu == 2) return k_condense_tc<4, 2>;
  if (nx == 2 && nu == 1) return k_condense_tc<2, 1>;
  return nullptr;
}

// shared memory of k_condense_tc (same carve-up as the kernel)
size_t tc_smem(int SC, int nx, int nu, int dslot, int n0, int64_t per) {
  const int emax = SC * (dslot - 1) > 0 ? SC * (dslot - 1) : 1;
  size_t st = sizeof(double) * ((size_t)SC * nx * 2 + (size_t)SC * nx * nx) +
              sizeof(float) * ((size_t)SC * nx * nx + (size_t)emax * nx * nx + (size_t)SC * nx * nu) +
              sizeof(int) * (size_t)emax;
  st = (st + 15) & ~size_t(15);
  const int KC = ((SC * nx + 7) / 8) * 8;
  const size_t bufb = 16 * (size_t)(KC / 4) * 128;
  size_t b = ((2 * st + 127) & ~size_t(127)) + 4 * bufb + 4 * (size_t)(KC / 4) * 128;
  b += sizeof(float) * ((size_t)SC * nx * nx + (size_t)SC * nx);
  b = (b + 15) & ~size_t(15);
  b += sizeof(double) * ((size_t)SC * nx + n0) + 8 + 8;
  return b + sizeof(int) * (size_t)(per + 1) + 16;
}

FusedKernel pick_kernel(int nx, int nu) {
  if (nx == 6 && nu == 6) return k_condense_fused<6, 6>;
  if (nx == 6 && nu == 3) return k_condense_fused<6, 3>;
  if (nx == 6 && nu == 2) return k_condense_fused<6, 2>;
  if (nx == 6 && nu == 1) return k_condense_fused<6, 1>;
  if (nx == 4 && nu == 2) return k_condense_fused<4, 2>;
  if (nx == 2 && nu == 1) return k_condense_fused<2, 1>;
  return nullptr;
}

size_t fused_smem(int SC, int nx, int nu, int ld, int dslot, int n0, int64_t per) {
  const int emax = SC * (dslot - 1) > 0 ? SC * (dslot - 1) : 1;
  size_t st = sizeof(double) * ((size_t)SC * nx * 2 + (size_t)SC * nx * nx) +
              sizeof(float) * ((size_t)SC * nx * nx + (size_t)emax * nx * nx + (size_t)SC * nx * nu) +
              sizeof(int) * (size_t)emax;
  st = (st + 15) & ~size_t(15);
  size_t f = (size_t)SC * nx * ld * 2 + (size_t)SC * nx * nx;
  size_t b = 2 * st + ((f * sizeof(float) + 15) & ~size_t(15)) + sizeof(double) * ((size_t)SC * nx + n0);
  return b + sizeof(int) * (size_t)(per + 1) + 16;
}

// CTA dependency lists for node partition `per`: CTA s waits on the owners of
// every in-neighbour of its nodes (graph.py CSR), itself excluded.
int ensure_deps(gm_ctx* ctx, int64_t per, int splits) {
  if (ctx->dep_per == per && ctx->d_dep_ptr) return GM_OK;
  std::vector<int> dptr(splits + 1, 0), dl;
  for (int s = 0; s < splits; ++s) {
    std::vector<int> mine;
    const int64_t lo = s * per, hi = std::min<int64_t>(ctx->M, lo + per);
    for (int64_t i = lo; i < hi; ++i)
      for (int64_t e = ctx->h_ptr[i]; e < ctx->h_ptr[i + 1]; ++e) {
        const int o = (int)(ctx->h_src[e] / per);
        if (o != s) mine.push_back(o);
      }
    std::sort(mine.begin(), mine.end());
    mine.erase(std::unique(mine.begin(), mine.end()), mine.end());
    dl.insert(dl.end(), mine.begin(), mine.end());
    dptr[s + 1] = (int)dl.size();
  }
  if (dl.empty()) dl.push_back(0);
  if (ctx->d_dep_ptr) ctx->retired.push_back(ctx->d_dep_ptr);  // captured graphs may hold them
  if (ctx->d_dep) ctx->retired.push_back(ctx->d_dep);
  ctx->d_dep_ptr = ctx->d_dep = nullptr;
  GM_CUDA(ctx, cudaMalloc(&ctx->d_dep_ptr, sizeof(int) * dptr.size()));
  GM_CUDA(ctx, cudaMalloc(&ctx->d_dep, sizeof(int) * dl.size()));
  GM_CUDA(ctx, cudaMemcpy(ctx->d_dep_ptr, dptr.data(), sizeof(int) * dptr.size(), cudaMemcpyHostToDevice));
  GM_CUDA(ctx, cudaMemcpy(ctx->d_dep, dl.data(), sizeof(int) * dl.size(), cudaMemcpyHostToDevice));
  ctx->dep_per = per;
  return GM_OK;
}

int ensure_flags(gm_ctx* ctx, int64_t n) {
  if (n <= ctx->flag_cap) return GM_OK;
  if (ctx->d_flags) ctx->retired.push_back(ctx->d_flags);
  ctx->d_flags = nullptr;
  const int64_t cap = std::max<int64_t>(n, 1024);
  GM_CUDA(ctx, cudaMalloc(&ctx->d_flags, sizeof(int) * cap));
  GM_CUDA(ctx, cudaMemset(ctx->d_flags, 0, sizeof(int) * cap));
  ctx->flag_cap = cap;
  return GM_OK;
}

// ---- K-COND TMA variant: host side -----------------------------------------
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_tiled() {
  static EncodeTiledFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return (EncodeTiledFn) nullptr;
    return (EncodeTiledFn)p;
  }();
  return fn;
}

// unique closed-neighbourhood nodes of every SC-node chunk (ascending ids)
// and each (node, slot)'s index into them; slot 0 = self, then the in-edges
// in CSR (edge) order
int ensure_chunks(gm_ctx* ctx, int SC) {
  if (ctx->cu_sc == SC && ctx->d_cu_ptr) return GM_OK;
  const int64_t M = ctx->M;
  const int dslot = (int)ctx->dmax + 1;
  if (dslot > 255) return 1;
  const int64_t nch = (M + SC - 1) / SC;
  std::vector<int> cptr(nch + 1, 0), cnodes;
  std::vector<unsigned char> slot((size_t)nch * SC * dslot, 255);
  int umax = 0;
  std::vector<int> u;
  for (int64_t c = 0; c < nch; ++c) {
    const int64_t lo = c * SC, hi = std::min<int64_t>(M, lo + SC);
    u.clear();
    for (int64_t i = lo; i < hi; ++i) {
      u.push_back((int)i);
      for (int64_t e = ctx->h_ptr[i]; e < ctx->h_ptr[i + 1]; ++e) u.push_back((int)ctx->h_src[e]);
    }
    std::sort(u.begin(), u.end());
    u.erase(std::unique(u.begin(), u.end()), u.end());
    if ((int)u.size() > 255) return 1;
    umax = std::max(umax, (int)u.size());
    auto idx = [&](int node) { return (unsigned char)(std::lower_bound(u.begin(), u.end(), node) - u.begin()); };
    for (int64_t i = lo; i < hi; ++i) {
      unsigned char* sl = slot.data() + ((size_t)c * SC + (i - lo)) * dslot;
      sl[0] = idx((int)i);
      for (int64_t e = ctx->h_ptr[i]; e < ctx->h_ptr[i + 1]; ++e) sl[1 + (e - ctx->h_ptr[i])] = idx((int)ctx->h_src[e]);
    }
    cnodes.insert(cnodes.end(), u.begin(), u.end());
    cptr[c + 1] = (int)cnodes.size();
  }
  if (ctx->d_cu_ptr) ctx->retired.push_back(ctx->d_cu_ptr);
  if (ctx->d_cu_nodes) ctx->retired.push_back(ctx->d_cu_nodes);
  if (ctx->d_cu_slot) ctx->retired.push_back(ctx->d_cu_slot);
  ctx->d_cu_ptr = ctx->d_cu_nodes = nullptr;
  ctx->d_cu_slot = nullptr;
  GM_CUDA(ctx, cudaMalloc(&ctx->d_cu_ptr, sizeof(int) * cptr.size()));
  GM_CUDA(ctx, cudaMalloc(&ctx->d_cu_nodes, sizeof(int) * cnodes.size()));
  GM_CUDA(ctx, cudaMalloc(&ctx->d_cu_slot, slot.size()));
  GM_CUDA(ctx, cudaMemcpy(ctx->d_cu_ptr, cptr.data(), sizeof(int) * cptr.size(), cudaMemcpyHostToDevice));
  GM_CUDA(ctx, cudaMemcpy(ctx->d_cu_nodes, cnodes.data(), sizeof(int) * cnodes.size(), cudaMemcpyHostToDevice));
  GM_CUDA(ctx, cudaMemcpy(ctx->d_cu_slot, slot.data(), slot.size(), cudaMemcpyHostToDevice));
  ctx->cu_sc = SC;
  ctx->cu_umax = umax;
  return GM_OK;
}

size_t tma_smem(int SC, int CPS, bool DB, int umax, int ld, int dslot, int n0, int64_t per, bool pipe = false,
                bool hacc_smem = true) {
  const int emax = SC * (dslot - 1) > 0 ? SC * (dslot - 1) : 1;
  const int npass = (ld / 32 + CPS - 1) / CPS;
  size_t b = (size_t)(DB ? 2 : npass) * umax * CPS * kTileBytes;
  b += 2 * stage_bytes<6, 6>(SC, emax);
  b += sizeof(float) * ((size_t)(pipe ? 4 : 2) * SC * 6 * ld + (size_t)(pipe ? 2 : 1) * SC * 36);
  b = (b + 15) & ~size_t(15);
  b += sizeof(double) * ((size_t)(pipe ? 2 : 1) * SC * 6 + n0);
  b += sizeof(int) * (size_t)(per + 1);
  const size_t nchk = (size_t)((per + SC - 1) / SC);
  b += sizeof(int) * (nchk + 1 + nchk * umax) + nchk * SC * dslot;
  b = (b + 15) & ~size_t(15);
  const int N = n0 / 6;
  if (hacc_smem) b += sizeof(float) * (size_t)(N * (N + 1) / 2) * 36;  // Hacc
  return b + 2 * sizeof(uint64_t) + 16;
}

int launch_pair_reduce(gm_ctx* ctx, int B, int nu, int n0, int npairs, int splits, int groups, float* partH,
                       double* partg, double* tmpH, double* tmpg, const double* r, int64_t r_stride,
                       const double* u_ref, int64_t uref_stride, double* H, double* g, cudaStream_t st);

// 1 = not applicable (shape, tables, smem), else a GM_ code
int condense_tma(gm_ctx* ctx, int B, int N, const float* a_self, const float* a_nbr, const float* b,
                 const double* c, const double* x0, float* gamma, int ld, const double* q, int64_t q_stride,
                 const double* x_ref, int64_t xref_stride, const double* r, int64_t r_stride,
                 const double* u_ref, int64_t uref_stride, double* H, double* g, void* stream) {
  const int nu = 6, n0 = N * nu, npairs = N * (N + 1) / 2;
  // ld >= 96: the per-stage H fold stages 256 x 36 floats in the Gc / QGc
  // buffers (2 x 8 nodes x 6 rows x ld floats)
  if (ctx->nx != 6 || ctx->n_u != 6 || npairs > 256 || ld % 32 != 0 || ld < 96 || n0 >= ld ||
      ((uintptr_t)gamma & 15))
    return 1;
  EncodeTiledFn enc = encode_tiled();
  if (!enc) return 1;
  const int64_t M = ctx->M;
  const int dslot = (int)ctx->dmax + 1;
  const size_t budget = std::min<size_t>(ctx->smem_optin, 227 * 1024) - 2048;
  // 8-node items (with 4-node items the per-item overheads outweigh the
  // staging: cfg5 30 ms vs 21 ms for the per-thread-load kernel).  Tile
  // passes: all 4 chunks of an item in one pass (4-column thread groups) when
  // that fits shared memory, else two passes of 2 chunks (2-column groups):
  // a chain item has 10 unique rows (1 pass, 31 KB of tiles), a mesh item 26
  // (80 KB in 1 pass).  GM_TMA_CPS=14|4|2 forces a variant (measurement
  // override: 14 = one pass double-buffered).
  constexpr int SC = 8;
  int64_t per = M;
  if (B < ctx->sm_count) {
    const int64_t want = std::max<int64_t>(1, ctx->sm_count / B);
    per = (M + want - 1) / want;
  }
  per = (per + SC - 1) / SC * SC;
  int rc0 = ensure_chunks(ctx, SC);
  if (rc0) return rc0;
  static const int cps_env = [] {
    const char* v = std::getenv("GM_TMA_CPS");
    return v ? std::atoi(v) : 0;
  }();
  // variants in order of preference: one pass double-buffered by item
  // (chains), one pass single-buffered (meshes), two passes of 2 chunks
  struct Var {
    int cps;
    bool db;
    bool pipe;
    void (*fn)(const FusedArgs, const CUtensorMap);
    int threads;
    int gr = 128;  // pipeline: recursion group size
  };
  // the warp-specialised pipeline first (GM_TMA_PIPE=0 skips it)
  static const int pipe_env = [] {
    const char* v = std::getenv("GM_TMA_PIPE");
    return v ? std::atoi(v) : 1;
  }();
  // pipeline group H size: 256 threads (GM_TMA_GH=128: 128); the fold of a
  // stage stages max(GH, npk) 6x6 pairs in the 2 * SC*6*ld floats of a buffer
  // group sizes: R 128 + H 256 (384 threads, 168 registers) for chains;
  // R 256 + H 256 (512 threads, 128 registers) where the recursion has more
  // neighbour blocks (degree >= 3: meshes; cfg5 11.2 -> 10.7 ms, cfg4 and
  // cfg3 even).  Measured and dropped: R 256 + H 128 (cfg4 22.9 vs 20.8 ms).
  static const int gh_env = [] {
    const char* v = std::getenv("GM_TMA_GH");
    return v ? std::atoi(v) : 256;
  }();
  static const int gr_env = [] {
    const char* v = std::getenv("GM_TMA_GR");
    return v ? std::atoi(v) : 0;
  }();
  // group R: 256 threads (the 512-thread pipeline) unless GM_TMA_GR says
  // otherwise; 128 when the 512-thread variant does not fit.  Chains took 128
  // until group H's in-place fold and three-chain gradient shifted the balance
  // (same-box A/B after those: cfg3 K-COND -2 %, cfg4 -4.5 %, M = 10^4 -4 %)
  const int gr_pref[2] = {gr_env ? gr_env : 256, gr_env ? gr_env : 128};
  const Var vars[12] = {{4, true, true, k_condense_tmap<8, 4, 4, true, 256, 256>, 512, 256},
                       {4, false, true, k_condense_tmap<8, 4, 4, false, 256, 256>, 512, 256},
                       {2, false, true, k_condense_tmap<8, 2, 2, false, 256, 256>, 512, 256},
                       {4, true, true, k_condense_tmap<8, 4, 4, true, 256>, 384},
                       {4, false, true, k_condense_tmap<8, 4, 4, false, 256>, 384},
                       {2, false, true, k_condense_tmap<8, 2, 2, false, 256>, 384},
                       {4, true, true, k_condense_tmap<8, 4, 4, true, 128>, 256},
                       {4, false, true, k_condense_tmap<8, 4, 4, false, 128>, 256},
                       {2, false, true, k_condense_tmap<8, 2, 2, false, 128>, 256},
                       {4, true, false, k_condense_tma<8, 4, 4, true>, 256},
                       {4, false, false, k_condense_tma<8, 4, 4, false>, 256},
                       {2, false, false, k_condense_tma<8, 2, 2, false>, 256}};
  const int npk_max = N * (N + 1) / 2;
  const Var* var = nullptr;
  for (int pass = 0; pass < 2 && !var && pipe_env != 0; ++pass)
    for (const Var& v : vars)
      if (v.pipe && (cps_env == 0 || cps_env == v.cps + (v.db ? 10 : 0)) && v.gr == gr_pref[pass] &&
          v.threads - v.gr == gh_env && npk_max <= 2 * (v.threads - v.gr) &&
          36 * std::max(v.threads - v.gr, npk_max) <= 2 * SC * 6 * ld &&
          tma_smem(SC, v.cps, v.db, ctx->cu_umax, ld, dslot, n0, per, true, false) <= budget) {
        var = &v;
        break;
      }
  if (!var)  // neither pipeline size fits: the single-group TMA kernel
    for (const Var& v : vars)
      if (!v.pipe && (cps_env == 0 || cps_env == v.cps + (v.db ? 10 : 0)) &&
          tma_smem(SC, v.cps, v.db, ctx->cu_umax, ld, dslot, n0, per, false, true) <= budget) {
        var = &v;
        break;
      }
  if (!var) return 1;
  // the pipeline keeps its H accumulator on chip when that fits (chains),
  // else in its global partial (meshes: 26-row tile ring)
  const bool hacc_smem =
      !var->pipe || tma_smem(SC, var->cps, var->db, ctx->cu_umax, ld, dslot, n0, per, true, true) <= budget;
  const size_t sm = tma_smem(SC, var->cps, var->db, ctx->cu_umax, ld, dslot, n0, per, var->pipe, hacc_smem);
  auto kfn = var->fn;
  GM_CUDA(ctx, cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  int occ = 0;
  GM_CUDA(ctx, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kfn, var->threads, sm));
  if (occ < 1) return 1;
  const int splits = (int)((M + per - 1) / per);
  const int64_t grid = (int64_t)B * splits;
  if (splits > 1 && grid > (int64_t)ctx->sm_count * occ) return 1;
  int rc = ensure_deps(ctx, per, splits);
  if (rc) return rc;
  rc = ensure_flags(ctx, grid + 1);
  if (rc) return rc;
  // the work array as a (B*M*(N+1)*6, ld) fp32 matrix, 6 x 32 boxes
  CUtensorMap tm;
  const cuuint64_t dims[2] = {(cuuint64_t)ld, (cuuint64_t)B * M * (N + 1) * 6};
  const cuuint64_t strides[1] = {(cuuint64_t)ld * 4};
  // box: one 32-column chunk (k_condense_tma), or the whole pass of 32*CPS
  // columns (k_condense_tmap: one TMA per unique node and pass)
  const cuuint32_t box[2] = {var->pipe ? (cuuint32_t)(32 * var->cps) : 32u, 6};
  const cuuint32_t estr[2] = {1, 1};
  if (enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void*)gamma, dims, strides, box, estr,
          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return 1;
  const int groups = std::min(splits, 16);
  const int PU = npairs * nu * nu;
  auto up = [](size_t x) { return (x + 255) & ~size_t(255); };
  const size_t pH = sizeof(float) * (size_t)grid * PU, pg = sizeof(double) * (size_t)grid * n0;
  const size_t tH = sizeof(double) * (size_t)B * groups * PU, tg = sizeof(double) * (size_t)B * groups * n0;
  char* scr = (char*)gm_scratch(ctx, up(pH) + up(pg) + up(tH) + tg + 256);
  if (!scr) return gm_fail(ctx, GM_ERR_CUDA, "scratch allocation failed");
  FusedArgs a{};
  a.M = (int)M;
  a.E = (int)ctx->E;
  a.N = N;
  a.ld = ld;
  a.per = (int)per;
  a.splits = splits;
  a.sc = SC;
  a.npairs = npairs;
  a.dslot = dslot;
  a.ptr = ctx->d_ptr;
  a.src = ctx->d_src;
  a.dep_ptr = ctx->d_dep_ptr;
  a.dep = ctx->d_dep;
  a.a_self = a_self;
  a.a_nbr = a_nbr;
  a.b = b;
  a.c = c;
  a.x0 = x0;
  a.W = gamma;
  a.q = q;
  a.q_stride = q_stride;
  a.xref = x_ref;
  a.xref_stride = xref_stride;
  a.partH = (float*)scr;
  a.partg = (double*)(scr + up(pH));
  a.flags = ctx->d_flags;
  a.rec = 1;
  a.lo = 0;
  a.hi = (int)M;
  a.cu_ptr = ctx->d_cu_ptr;
  a.cu_nodes = ctx->d_cu_nodes;
  a.cu_slot = ctx->d_cu_slot;
  a.umax = ctx->cu_umax;
  // Qs*Gamma split between the pipeline's groups (measured: all in group H, 0/8, is fastest)
  static const int qg_env = [] {
    const char* v = std::getenv("GM_TMA_QGR");
    return v ? std::max(0, std::min(8, std::atoi(v))) : 0;
  }();
  a.qg_r8 = qg_env;
  a.hacc_gl = hacc_smem ? 0 : 1;
  a.al16 = ((((uintptr_t)a_self | (uintptr_t)a_nbr | (uintptr_t)b | (uintptr_t)c | (uintptr_t)q |
              (uintptr_t)x_ref) & 15) == 0 && (q_stride % 2) == 0 && (xref_stride % 2) == 0)
               ? 1
               : 0;
  cudaStream_t st = (cudaStream_t)stream;
  cudaLaunchConfig_t lc{};
  lc.gridDim = dim3((unsigned)grid);
  lc.blockDim = dim3((unsigned)var->threads);
  lc.dynamicSmemBytes = sm;
  lc.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  lc.attrs = attr;
  lc.numAttrs = splits > 1 ? 1 : 0;  // stage waits across CTAs need co-residency
  GM_CUDA(ctx, cudaLaunchKernelEx(&lc, kfn, a, tm));
  GM_LAUNCH_CHECK(ctx, "k_condense_tma");
  ctx->last_cond_kernel = !var->pipe ? 3 : (var->threads == 512 ? 5 : 4);
  return launch_pair_reduce(ctx, B, nu, n0, npairs, splits, groups, a.partH, a.partg,
                            (double*)(scr + up(pH) + up(pg)), (double*)(scr + up(pH) + up(pg) + up(tH)), r,
                            r_stride, u_ref, uref_stride, H, g, st);
}

int launch_pair_reduce(gm_ctx* ctx, int B, int nu, int n0, int npairs, int splits, int groups, float* partH,
                       double* partg, double* tmpH, double* tmpg, const double* r, int64_t r_stride,
                       const double* u_ref, int64_t uref_stride, double* H, double* g, cudaStream_t st) {
  PairReduceArgs ra{};
  ra.nu = nu;
  ra.n0 = n0;
  ra.npairs = npairs;
  ra.splits = splits;
  ra.groups = groups;
  ra.partH = partH;
  ra.partg = partg;
  ra.tmpH = tmpH;
  ra.tmpg = tmpg;
  ra.r = r;
  ra.r_stride = r_stride;
  ra.uref = u_ref;
  ra.uref_stride = uref_stride;
  ra.H = H;
  ra.g = g;
  const int PU = npairs * nu * nu;
  const unsigned eb = (unsigned)gm_ceil_div(std::max(PU, n0), 256);
  k_pair_reduce1<<<dim3(eb, (unsigned)groups, (unsigned)B), 256, 0, st>>>(ra);
  GM_LAUNCH_CHECK(ctx, "k_pair_reduce1");
  k_pair_reduce2<<<dim3(eb, (unsigned)B), 256, 0, st>>>(ra);
  GM_LAUNCH_CHECK(ctx, "k_pair_reduce2");
  return GM_OK;
}

}  // namespace

// K-HG: the cost part of condense_ocp over the node range [node_lo, node_hi)
// from a Gamma produced elsewhere (per-stage K-REC, the partitioned driver):
// the fused kernel without the recursion (a.rec = 0), split-K over node
// ranges (no co-residency requirement), then the shared fixed-order fp64
// reduction.  tc != 0 selects k_condense_tc (tcgen05 3xTF32 H), else the SIMT
// k_condense_fused (fp32 FMA with round-to-nearest accumulation: the tensor
// core accumulator truncates).  partial != 0 leaves out
// R-bar / r_lin (added by one rank only).  Returns 1 (not handled) when the
// shape has no instantiation.
int gm_fused_cost(gm_ctx* ctx, int tc, int B, int N, const float* gamma, int ld, const double* q,
                  int64_t q_stride, const double* x_ref, int64_t xref_stride, const double* r,
                  int64_t r_stride, const double* u_ref, int64_t uref_stride, double* H, double* g,
                  int partial, void* stream) {
  const int nx = ctx->nx, nu = ctx->n_u, n0 = N * nu;
  const int npairs = N * (N + 1) / 2;
  const int64_t lo = ctx->node_lo, hi = gm_node_hi(ctx), nodes = hi - lo;
  FusedKernel kern = tc ? ((n0 <= 128) ? pick_tc_kernel(nx, nu) : nullptr)
                        : (npairs <= 256 ? pick_kernel(nx, nu) : nullptr);
  if (!kern || nodes < 1 || (ld % 4) != 0 || ((uintptr_t)gamma & 15) || ((uintptr_t)q & 15) ||
      ((uintptr_t)x_ref & 15) || (q_stride % 2) != 0 || (xref_stride % 2) != 0)
    return 1;
  const int dslot = (int)ctx->dmax + 1;
  int SC = tc ? 8 : 16;
  const int threads = tc ? kTcThreads : 256;
  const int64_t want = std::max<int64_t>(1, (2 * (int64_t)ctx->sm_count + B - 1) / B);
  const int64_t per = std::max<int64_t>(SC, (nodes + want - 1) / want);
  auto smem_of = [&](int sc_) {
    return tc ? tc_smem(sc_, nx, nu, dslot, n0, per) : fused_smem(sc_, nx, nu, ld, dslot, n0, per);
  };
  while (!tc && SC > 1 && smem_of(SC) > kFusedSmemBudget) SC >>= 1;
  const int splits = (int)((nodes + per - 1) / per);
  const size_t sm = smem_of(SC);
  if (sm > kFusedSmemBudget) return 1;
  cudaStream_t st = (cudaStream_t)stream;
  GM_CUDA(ctx, cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  const int64_t grid = (int64_t)B * splits;
  const int groups = std::min(splits, 16);
  const int PU = npairs * nu * nu;
  auto up = [](size_t x) { return (x + 255) & ~size_t(255); };
  const size_t pH = sizeof(float) * (size_t)grid * PU, pg = sizeof(double) * (size_t)grid * n0;
  const size_t tH = sizeof(double) * (size_t)B * groups * PU, tg = sizeof(double) * (size_t)B * groups * n0;
  char* scr = (char*)gm_scratch(ctx, up(pH) + up(pg) + up(tH) + tg + 256);
  if (!scr) return gm_fail(ctx, GM_ERR_CUDA, "scratch allocation failed");
  FusedArgs a{};
  a.M = (int)ctx->M;
  a.E = (int)ctx->E;
  a.N = N;
  a.ld = ld;
  a.per = (int)per;
  a.splits = splits;
  a.sc = SC;
  a.npairs = npairs;
  a.dslot = dslot;
  a.ptr = ctx->d_ptr;
  a.src = ctx->d_src;
  a.W = const_cast<float*>(gamma);
  a.q = q;
  a.q_stride = q_stride;
  a.xref = x_ref;
  a.xref_stride = xref_stride;
  a.partH = (float*)scr;
  a.partg = (double*)(scr + up(pH));
  a.rec = 0;
  a.lo = (int)lo;
  a.hi = (int)hi;
  kern<<<(unsigned)grid, (unsigned)threads, sm, st>>>(a);
  GM_LAUNCH_CHECK(ctx, tc ? "k_condense_tc(cost)" : "k_condense_fused(cost)");
  PairReduceArgs ra{};
  ra.nu = nu;
  ra.n0 = n0;
  ra.npairs = npairs;
  ra.splits = splits;
  ra.groups = groups;
  ra.partH = a.partH;
  ra.partg = a.partg;
  ra.tmpH = (double*)(scr + up(pH) + up(pg));
  ra.tmpg = (double*)(scr + up(pH) + up(pg) + up(tH));
  ra.r = partial ? nullptr : r;
  ra.r_stride = r_stride;
  ra.uref = u_ref;
  ra.uref_stride = uref_stride;
  ra.H = H;
  ra.g = g;
  const unsigned eb = (unsigned)gm_ceil_div(std::max(PU, n0), 256);
  k_pair_reduce1<<<dim3(eb, (unsigned)groups, (unsigned)B), 256, 0, st>>>(ra);
  GM_LAUNCH_CHECK(ctx, "k_pair_reduce1");
  k_pair_reduce2<<<dim3(eb, (unsigned)B), 256, 0, st>>>(ra);
  GM_LAUNCH_CHECK(ctx, "k_pair_reduce2");
  return GM_OK;
}

extern "C" {

int gm_set_condense_mode(gm_ctx* ctx, int mode) {
  if (!ctx) return GM_ERR_CONFIG;
  if (mode < 0 || mode > 3) return gm_fail(ctx, GM_ERR_CONFIG, "condense mode must be 0, 1, 2 or 3");
  ctx->cond_mode = mode;
  return GM_OK;
}

int gm_condense_fused(gm_ctx* ctx, int B, int N, const float* a_self, const float* a_nbr,
                      const float* b, const double* c, const double* x0, float* gamma, int ld,
                      const double* q, int64_t q_stride, const double* x_ref, int64_t xref_stride,
                      const double* r, int64_t r_stride, const double* u_ref, int64_t uref_stride,
                      double* H, double* g, void* stream) {
  int rc = gm_need_device(ctx);
  if (rc) return rc;
  if (ctx->M < 1) return gm_fail(ctx, GM_ERR_CONFIG, "graph not set");
  if (ctx->nx < 1 || ctx->n_u < 1) return gm_fail(ctx, GM_ERR_CONFIG, "dimensions not set");
  if (B < 0 || N < 1) return gm_fail(ctx, GM_ERR_CONFIG, "need B >= 0 and horizon >= 1");
  if (ld < N * ctx->n_u + 1) return gm_fail(ctx, GM_ERR_CONFIG, "gamma leading dimension too small");
  ctx->last_cond_kernel = 0;
  if (B == 0) return GM_OK;
  // default (mode 0): the TMA-staged kernel for the reference architecture
  // from 512 node rows (below, e.g. cfg2 at M = 100, the per-stage tile
  // issue / wait latency of a one-item-per-stage CTA costs more than the
  // staging saves: 0.20 vs 0.10 ms)
  if (ctx->cond_mode == 0 && ctx->node_lo == 0 && gm_node_hi(ctx) == ctx->M && (int64_t)B * ctx->M >= 512) {
    static const bool no_tma = std::getenv("GM_NO_TMA") != nullptr;  // measurement override
    if (!no_tma) {
      rc = condense_tma(ctx, B, N, a_self, a_nbr, b, c, x0, gamma, ld, q, q_stride, x_ref, xref_stride, r,
                        r_stride, u_ref, uref_stride, H, g, stream);
      if (rc != 1) return rc;
    }
  }
  const int nx = ctx->nx, nu = ctx->n_u, n0 = N * nu;
  const int npairs = N * (N + 1) / 2;
  const int dslot = (int)ctx->dmax + 1;
  // tensor-core H (k_condense_tc) whenever the H accumulator fits one
  // 128 x 128 TMEM tile; gm_set_condense_mode forces either kernel
  // (auto mode: from ~512 node rows up; below that, the per-item MMA issue /
  // commit / wait round trip costs more than the SIMT products it replaces:
  // cfg2, M = 100, 0.18 ms tc vs 0.10 ms SIMT; cfg3, M = 1000, equal)
  // Auto mode keeps H on the SIMT kernel: the tcgen05 accumulator truncates
  // on every add, so at 10^4 nodes the 3xTF32 H drifts to ~7e-5 relative
  // (u to ~1.5e-4) where the fp32 FMA kernel stays at ~2e-6 (DESIGN.md 4,
  // scripts/diag_precision.py); gm_set_condense_mode(3) selects tcgen05
  const bool tc_ok = ctx->cond_mode == 3;
  FusedKernel tck = (n0 <= 128 && tc_ok) ? pick_tc_kernel(nx, nu) : nullptr;
  FusedKernel kern = tck ? tck : pick_kernel(nx, nu);
  const bool whole = ctx->node_lo == 0 && gm_node_hi(ctx) == ctx->M;
  // node partition: cps CTAs per SM, all co-resident (the stage waits need
  // it).  k_condense_tc: threads x SC (nodes per item) x CTAs per SM,
  // default 512 x 8 x 1; GM_TC_CFG="threads,sc,cps" overrides (the
  // occupancy query decides how many CTAs per SM are really co-resident)
  int tc_threads = kTcThreads, tc_sc = 8, cps = 1;
  if (tck) {
    if (const char* v = getenv("GM_TC_CFG")) {
      int t0 = 0, s0 = 0, c0 = 0;
      if (sscanf(v, "%d,%d,%d", &t0, &s0, &c0) == 3 && t0 >= 128 && t0 <= kTcThreads && t0 % 128 == 0 &&
          s0 >= 2 && s0 <= 16 && c0 >= 1 && c0 <= 4) {
        tc_threads = t0;
        tc_sc = s0;
        cps = c0;
      }
    }
  }
  const int64_t M = ctx->M;
  const int threads = tck ? tc_threads : 256;
  int64_t per = M;
  int SC = 16;
  size_t sm = 0;
  int occ = 0;
  // partition for `cps` co-resident CTAs per SM; if the occupancy query
  // grants fewer, repartition for what it grants (nptr, and so the shared
  // memory size, depends on the partition)
  for (int attempt = 0; attempt < 2; ++attempt) {
    const int64_t slots = (int64_t)ctx->sm_count * cps;
    per = M;
    if (B < slots) {
      const int64_t want = std::max<int64_t>(1, slots / B);
      per = (M + want - 1) / want;
    }
    SC = tck ? tc_sc : 16;
    auto smem_of = [&](int sc_) {
      return tck ? tc_smem(sc_, nx, nu, dslot, n0, per) : fused_smem(sc_, nx, nu, ld, dslot, n0, per);
    };
    while (SC > 1 && smem_of(SC) > kFusedSmemBudget) SC >>= 1;
    sm = smem_of(SC);
    if (!kern || !whole || npairs > 256 || sm > kFusedSmemBudget || ctx->cond_mode == 2) break;
    GM_CUDA(ctx, cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    GM_CUDA(ctx, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, threads, sm));
    if (occ < 1) return gm_fail(ctx, GM_ERR_CONFIG, "fused condensing kernel does not fit an SM");
    if (occ >= cps) break;
    cps = occ;
  }
  if (!kern || !whole || npairs > 256 || sm > kFusedSmemBudget || ctx->cond_mode == 2) {
    // shapes outside the fused kernel's instantiations: the two-kernel path
    rc = gm_condense_gammas(ctx, B, N, a_self, a_nbr, b, c, x0, gamma, ld, stream);
    if (rc) return rc;
    ctx->last_cond_kernel = 6;
    return gm_condense_cost(ctx, B, N, gamma, ld, q, q_stride, x_ref, xref_stride, r, r_stride,
                            u_ref, uref_stride, H, g, 0, stream);
  }
  cudaStream_t st = (cudaStream_t)stream;
  const int splits = (int)((M + per - 1) / per);
  rc = ensure_deps(ctx, per, splits);
  if (rc) return rc;
  const int64_t grid = (int64_t)B * splits;
  if (splits > 1 && grid > (int64_t)ctx->sm_count * occ)
    return gm_fail(ctx, GM_ERR_CONFIG,
                   "fused condensing grid not co-resident (" + std::to_string(grid) + " CTAs, " +
                       std::to_string(occ) + " per SM, " + std::to_string(sm) + " B shared)");
  rc = ensure_flags(ctx, grid + 1);
  if (rc) return rc;
  const int groups = std::min(splits, 16);
  const int PU = npairs * nu * nu;
  auto up = [](size_t x) { return (x + 255) & ~size_t(255); };
  const size_t pH = sizeof(float) * (size_t)grid * PU, pg = sizeof(double) * (size_t)grid * n0;
  const size_t tH = sizeof(double) * (size_t)B * groups * PU, tg = sizeof(double) * (size_t)B * groups * n0;
  char* scr = (char*)gm_scratch(ctx, up(pH) + up(pg) + up(tH) + tg + 256);
  if (!scr) return gm_fail(ctx, GM_ERR_CUDA, "scratch allocation failed");
  FusedArgs a{};
  a.M = (int)M;
  a.E = (int)ctx->E;
  a.N = N;
  a.ld = ld;
  a.per = (int)per;
  a.splits = splits;
  a.sc = SC;
  a.npairs = npairs;
  a.dslot = dslot;
  a.ptr = ctx->d_ptr;
  a.src = ctx->d_src;
  a.dep_ptr = ctx->d_dep_ptr;
  a.dep = ctx->d_dep;
  a.a_self = a_self;
  a.a_nbr = a_nbr;
  a.b = b;
  a.c = c;
  a.x0 = x0;
  a.W = gamma;
  a.q = q;
  a.q_stride = q_stride;
  a.xref = x_ref;
  a.xref_stride = xref_stride;
  a.partH = (float*)scr;
  a.partg = (double*)(scr + up(pH));
  a.flags = ctx->d_flags;
  a.rec = 1;
  a.lo = 0;
  a.hi = (int)M;
  {
    const char* v = getenv("GM_TC_PREFETCH");
    a.reg_prefetch = v ? atoi(v) : 1;
  }
  if (getenv("GM_TC_DEBUG")) {
    cudaFuncAttributes fa{};
    cudaFuncGetAttributes(&fa, kern);
    fprintf(stderr,
            "k_condense: tc=%d threads=%d SC=%d per=%lld splits=%d grid=%lld occ=%d smem=%zu regs=%d static=%zu "
            "maxthr=%d\n",
            tck != nullptr, threads, SC, (long long)per, splits, (long long)grid, occ, sm, fa.numRegs,
            fa.sharedSizeBytes, fa.maxThreadsPerBlock);
  }
  if (splits > 1) {
    // CTAs of one instance spin on each other's stage flags: launch
    // cooperatively so the driver guarantees co-residency (or fails the
    // launch loudly) even when other work shares the SMs
    cudaLaunchConfig_t lc{};
    lc.gridDim = dim3((unsigned)grid);
    lc.blockDim = dim3((unsigned)threads);
    lc.dynamicSmemBytes = sm;
    lc.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    lc.attrs = attr;
    lc.numAttrs = 1;
    GM_CUDA(ctx, cudaLaunchKernelEx(&lc, kern, a));
  } else {
    // one CTA per instance: no inter-CTA waits, any grid size
    kern<<<(unsigned)grid, (unsigned)threads, sm, st>>>(a);
  }
  GM_LAUNCH_CHECK(ctx, "k_condense_fused");
  ctx->last_cond_kernel = tck != nullptr ? 2 : 1;
  PairReduceArgs ra{};
  ra.nu = nu;
  ra.n0 = n0;
  ra.npairs = npairs;
  ra.splits = splits;
  ra.groups = groups;
  ra.partH = a.partH;
  ra.partg = a.partg;
  ra.tmpH = (double*)(scr + up(pH) + up(pg));
  ra.tmpg = (double*)(scr + up(pH) + up(pg) + up(tH));
  ra.r = r;
  ra.r_stride = r_stride;
  ra.uref = u_ref;
  ra.uref_stride = uref_stride;
  ra.H = H;
  ra.g = g;
  const unsigned eb = (unsigned)gm_ceil_div(std::max(PU, n0), 256);
  k_pair_reduce1<<<dim3(eb, (unsigned)groups, (unsigned)B), 256, 0, st>>>(ra);
  GM_LAUNCH_CHECK(ctx, "k_pair_reduce1");
  k_pair_reduce2<<<dim3(eb, (unsigned)B), 256, 0, st>>>(ra);
  GM_LAUNCH_CHECK(ctx, "k_pair_reduce2");
  return GM_OK;
}

}  // extern "C"

extern "C" int gm_cond_profile(int on) {
  if (!kCondProf) return GM_ERR_CONFIG;  // built without -DGM_COND_PROF
  on = on != 0 ? 1 : 0;
  cudaMemcpyToSymbol(g_cond_prof_on, &on, sizeof(int));
  static const unsigned long long z[32 * 24] = {0};
  cudaMemcpyToSymbol(g_cond_prof, z, sizeof(z));
  return GM_OK;
}

extern "C" int gm_cond_phase_cycles(unsigned long long* out) {
  return cudaMemcpyFromSymbol(out, g_cond_prof, sizeof(unsigned long long) * 32 * 24) == cudaSuccess ? GM_OK
                                                                                                    : GM_ERR_CUDA;
}

extern "C" int gm_last_condense_kernel(gm_ctx* ctx) { return ctx ? ctx->last_cond_kernel : 0; }
