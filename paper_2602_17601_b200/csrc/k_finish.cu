// K-RS: state reconstruction and the device-side RTI epilogue.
//
// reconstruct_states (condensing.py:409-416): x^i = Gamma_u^i u + Gamma_x^i.
// gm_mpc_finish: mpc.py:151-200 without a host round trip -- the QP status is
// read on the device, the damped update / fallback policy / shift are applied
// and the successor trajectory is written in one elementwise pass.
#include <algorithm>
#include <cstdlib>

#include "common.cuh"

namespace {

// Planned-state rows of node gi at stage k, (Gamma_u u + Gamma_x)[a] for
// a < nx, by one warp: lane l reads the 16-byte column chunks l*4 + 128 j of
// each row (coalesced 512-B rows; only chunks holding causal columns
// [0, k*nu) or the Gamma_x column), the loads of up to 8 rows are issued
// before any arithmetic, and each row's partial sums meet in a fixed-order
// butterfly (bitwise reproducible).  Lane a < nx returns row a.
__device__ __forceinline__ double warp_rows(const float* W, int ld, int N, int nx, int nu, int64_t gi, int k,
                                            const double* u, int lane) {
  const float* rows = W + ((gi * (N + 1) + k) * nx) * (int64_t)ld;
  const int live = k * nu, xc = N * nu;
  double mine = 0.0;
  for (int a0 = 0; a0 < nx; a0 += 8) {
    double s[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) s[q] = 0.0;
    for (int c0 = lane * 4; c0 < ld; c0 += 128) {
      if (c0 >= live && (xc < c0 || xc >= c0 + 4)) continue;
      double coef[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int c = c0 + j;
        coef[j] = c < live ? u[c] : (c == xc ? 1.0 : 0.0);
      }
      float4 v[8];
#pragma unroll
      for (int q = 0; q < 8; ++q)
        if (a0 + q < nx) v[q] = __ldcs(reinterpret_cast<const float4*>(rows + (int64_t)(a0 + q) * ld + c0));
#pragma unroll
      for (int q = 0; q < 8; ++q)
        if (a0 + q < nx) {
          s[q] = fma((double)v[q].x, coef[0], s[q]);
          s[q] = fma((double)v[q].y, coef[1], s[q]);
          s[q] = fma((double)v[q].z, coef[2], s[q]);
          s[q] = fma((double)v[q].w, coef[3], s[q]);
        }
    }
    // reduce-scatter butterfly: after the xor-16/8/4 levels lane l holds a
    // partial of row 4*b4 + 2*b3 + b2 (b = bits of l) summed over 8 lanes,
    // the xor-2/1 levels finish it: lane 4a holds row a (9 exchanges for 8
    // rows instead of 40)
    const bool h4 = lane & 16, h3 = lane & 8, h2 = lane & 4;
    double t4[4], t2[2];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const double send = h4 ? s[q] : s[q + 4];
      const double keep = h4 ? s[q + 4] : s[q];
      t4[q] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
    }
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const double send = h3 ? t4[q] : t4[q + 2];
      const double keep = h3 ? t4[q + 2] : t4[q];
      t2[q] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
    }
    double v;
    {
      const double send = h2 ? t2[0] : t2[1];
      const double keep = h2 ? t2[1] : t2[0];
      v = keep + __shfl_xor_sync(0xffffffffu, send, 4);
    }
    v += __shfl_xor_sync(0xffffffffu, v, 2);
    v += __shfl_xor_sync(0xffffffffu, v, 1);
    const double got = __shfl_sync(0xffffffffu, v, (4 * (lane - a0)) & 31);
    if (lane >= a0 && lane < a0 + 8) mine = got;
  }
  return mine;
}

// one warp per (node, stage) item, items in Gamma's memory order
__global__ void __launch_bounds__(256, 3) k_reconstruct(const float* W, int ld, int M, int N, int nx, int nu,
                              const double* u, int ldu, double* x, int64_t items) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t w = w0; w < items; w += nw) {
    const int k = (int)(w % (N + 1));
    const int64_t gi = w / (N + 1);
    const int64_t bi = gi / M;
    const double v = warp_rows(W, ld, N, nx, nu, gi, k, u + bi * ldu, lane);
    if (lane < nx) x[(gi * (N + 1) + k) * nx + lane] = v;
  }
}

struct FinishArgs {
  int M, N, nx, nu, ld, ldu, fallback, has_prev;
  double damp;
  const float* W;
  const double* u;
  const int* status;
  const int* iters;
  const double* lin_states;
  const double* lin_inputs;
  const double* fb_states;
  const double* fb_inputs;
  const double* u_prev;
  double* cur_states;
  double* planned_states;
  double* planned_inputs;
  double* next_states;
  double* next_inputs;
  double* u_applied;
  double* summary;
};

__device__ __forceinline__ bool solved(int st) {
  return st == GM_QP_OPTIMAL || st == GM_QP_MAX_ITERATIONS;
}

// state entries: (1-a) lin + a planned (mpc.py:396-398), or the fallback plan
// when the solve failed (mpc.py:415-418).
__global__ void __launch_bounds__(256, 3) k_finish_states(const FinishArgs A, int64_t items) {
  const int M = A.M, N = A.N, nx = A.nx;
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t w = w0; w < items; w += nw) {  // (bi, i, k): Gamma's memory order
    const int k = (int)(w % (N + 1));
    const int64_t gi = w / (N + 1);
    const int i = (int)(gi % M);
    const int64_t bi = gi / M;
    const bool ok = solved(A.status[bi]);
    double p = 0.0;
    if (ok) p = warp_rows(A.W, A.ld, N, nx, A.nu, gi, k, A.u + bi * A.ldu, lane);
    if (lane < nx) {
      const int a = lane;
      const int64_t t = ((bi * (N + 1) + k) * M + i) * nx + a;
      const double v = ok ? (1.0 - A.damp) * A.lin_states[t] + A.damp * p : A.fb_states[t];
      if (A.cur_states) A.cur_states[t] = v;
      // planned_states (M, N+1, nx) = lin_states.transpose(1, 0, 2)   (mpc.py:407)
      A.planned_states[((bi * M + i) * (N + 1) + k) * nx + a] = v;
      // _shift (mpc.py:90-99): s[k-1] = s[k] for k >= 1, s[N] = s[N]
      const int64_t base = bi * (int64_t)(N + 1) * M * nx;
      if (k >= 1) A.next_states[base + ((int64_t)(k - 1) * M + i) * nx + a] = v;
      if (k == N) A.next_states[base + ((int64_t)N * M + i) * nx + a] = v;
    }
  }
}

// Fixed-order butterfly of warp_rows for 8 row partials: lane a < 8 returns
// row a (bitwise the same sums as warp_rows' single-chunk case).
__device__ __forceinline__ double butterfly8(const double (&s)[8], int lane) {
  const bool h4 = lane & 16, h3 = lane & 8, h2 = lane & 4;
  double t4[4], t2[2];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const double send = h4 ? s[q] : s[q + 4];
    const double keep = h4 ? s[q + 4] : s[q];
    t4[q] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
  }
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const double send = h3 ? t4[q] : t4[q + 2];
    const double keep = h3 ? t4[q + 2] : t4[q];
    t2[q] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
  }
  double v;
  {
    const double send = h2 ? t2[0] : t2[1];
    const double keep = h2 ? t2[1] : t2[0];
    v = keep + __shfl_xor_sync(0xffffffffu, send, 4);
  }
  v += __shfl_xor_sync(0xffffffffu, v, 2);
  v += __shfl_xor_sync(0xffffffffu, v, 1);
  return __shfl_sync(0xffffffffu, v, (4 * lane) & 31);
}

// k_finish_states for nx = NX <= 8 and ld <= 128 (one 16-byte column chunk
// per lane and row): software-pipelined, the Gamma rows (and u coefficients)
// of the warp's next item are loaded before the current item is reduced, so
// two items' rows are in flight per warp.  Same sums in the same order as
// warp_rows (bitwise identical results).
template <int NX>
__global__ void __launch_bounds__(256, 3) k_finish_states_pipe(const FinishArgs A, int64_t items) {
  const int M = A.M, N = A.N, ld = A.ld, nu = A.nu;
  const int lane = threadIdx.x & 31, c0 = lane * 4, xc = N * nu;
  const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  float4 v[NX];
  double coef[4];
  // item -> (instance, node, stage) in 32-bit unsigned arithmetic (the host
  // launches this kernel only for items < 2^31): the 64-bit divisions they
  // replace were ~100 instructions each and bounded the kernel on issue
  const unsigned N1 = (unsigned)(N + 1), Mu = (unsigned)M;
  unsigned fk = 0, fgi = 0;
  auto fetch = [&](int64_t w) {
    const unsigned wu = (unsigned)w;
    fgi = wu / N1;
    fk = wu - fgi * N1;
    const int k = (int)fk;
    const int64_t gi = fgi;
    const int64_t bi = fgi / Mu;
    const int live = k * nu;
    const bool act = solved(A.status[bi]) && c0 < ld && (c0 < live || (xc >= c0 && xc < c0 + 4));
    const float* rows = A.W + ((gi * (N + 1) + k) * NX) * (int64_t)ld + c0;
    const double* u = A.u + bi * A.ldu;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int c = c0 + j;
      coef[j] = !act ? 0.0 : (c < live ? u[c] : (c == xc ? 1.0 : 0.0));
    }
#pragma unroll
    for (int q = 0; q < NX; ++q)
      v[q] = act ? __ldcs(reinterpret_cast<const float4*>(rows + (int64_t)q * ld)) : make_float4(0.f, 0.f, 0.f, 0.f);
  };
  if (w0 < items) fetch(w0);
  for (int64_t w = w0; w < items; w += nw) {
    double s[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) s[q] = 0.0;
#pragma unroll
    for (int q = 0; q < NX; ++q) {
      s[q] = fma((double)v[q].x, coef[0], s[q]);
      s[q] = fma((double)v[q].y, coef[1], s[q]);
      s[q] = fma((double)v[q].z, coef[2], s[q]);
      s[q] = fma((double)v[q].w, coef[3], s[q]);
    }
    const int k = (int)fk;
    const unsigned gu = fgi, bu = gu / Mu;
    const int64_t gi = gu, bi = bu;
    const int i = (int)(gu - bu * Mu);
    if (w + nw < items) fetch(w + nw);
    const double p = butterfly8(s, lane);
    if (lane < NX) {
      const bool ok = solved(A.status[bi]);
      const int a = lane;
      const int64_t t = ((bi * (N + 1) + k) * M + i) * NX + a;
      const double x = ok ? (1.0 - A.damp) * A.lin_states[t] + A.damp * p : A.fb_states[t];
      if (A.cur_states) A.cur_states[t] = x;
      A.planned_states[((bi * M + i) * (N + 1) + k) * NX + a] = x;
      const int64_t base = bi * (int64_t)(N + 1) * M * NX;
      if (k >= 1) A.next_states[base + ((int64_t)(k - 1) * M + i) * NX + a] = x;
      if (k == N) A.next_states[base + ((int64_t)N * M + i) * NX + a] = x;
    }
  }
}

// K-RS by linear rollout (large batches).  The planned trajectory of
// reconstruct_states, x = Gamma_u u + Gamma_x (condensing.py:409-416), is the
// Gamma recursion (condensing.py:182-228) applied to u:
//     p_0 = x0,  p_{n+1}(i) = A_self p_n(i) + sum_{e in in(i)} A_e p_n(src e)
//                             + B_n(i) u_n + c_n(i)
// (reference tests/test_condensing.py:120-135 checks exactly this identity),
// so it needs the stage blocks (36 (deg + 2) fp32 + 6 fp64 per node-stage)
// instead of Gamma's 6 x ld fp32 rows.  One thread per (instance, node, row);
// p ping-pongs through global scratch (L2-resident), stages separated by a
// grid barrier (cooperative launch: co-residency guaranteed); the epilogue of
// k_finish_states is applied to every p_k as it is formed.
struct RolloutArgs {
  const float* a_self;
  const float* a_nbr;
  const float* b;
  const double* c;
  const double* x0;
  const int* ptr;
  const int* src;
  double* p0;
  double* p1;
  unsigned* bar;  // [count, generation]
};

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u32(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// grid-wide barrier: self-resetting count, monotone generation
__device__ __forceinline__ void grid_barrier(unsigned* bar, unsigned& gen) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(&bar[0], 1u) == gridDim.x - 1) {
      atomicExch(&bar[0], 0u);
      st_release_u32(&bar[1], gen + 1);
    } else {
      while (ld_acquire_u32(&bar[1]) == gen) __nanosleep(64);
    }
  }
  ++gen;
  __syncthreads();
}

template <int NX, int NU>
__global__ void __launch_bounds__(256) k_rollout(const FinishArgs A, const RolloutArgs R, int B) {
  const int M = A.M, N = A.N;
  const int64_t rows = (int64_t)B * M * NX;
  const int64_t t0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x, nt = (int64_t)gridDim.x * blockDim.x;
  __shared__ unsigned gen_s;
  if (threadIdx.x == 0) gen_s = ld_acquire_u32(&R.bar[1]);
  __syncthreads();
  unsigned gen = gen_s;
  auto finish = [&](int64_t bi, int i, int a, int k, double p) {
    const bool ok = solved(A.status[bi]);
    const int64_t t = ((bi * (N + 1) + k) * M + i) * NX + a;
    const double x = ok ? (1.0 - A.damp) * A.lin_states[t] + A.damp * p : A.fb_states[t];
    if (A.cur_states) A.cur_states[t] = x;
    A.planned_states[((bi * M + i) * (N + 1) + k) * NX + a] = x;
    const int64_t base = bi * (int64_t)(N + 1) * M * NX;
    if (k >= 1) A.next_states[base + ((int64_t)(k - 1) * M + i) * NX + a] = x;
    if (k == N) A.next_states[base + ((int64_t)N * M + i) * NX + a] = x;
  };
  for (int64_t r = t0; r < rows; r += nt) {  // stage 0: p_0 = x0
    const double v = R.x0[r];
    R.p0[r] = v;
    const int64_t gi = r / NX;
    finish(gi / M, (int)(gi % M), (int)(r % NX), 0, v);
  }
  for (int n = 0; n < N; ++n) {
    grid_barrier(R.bar, gen);
    const double* pin = (n & 1) ? R.p1 : R.p0;
    double* pout = (n & 1) ? R.p0 : R.p1;
    for (int64_t r = t0; r < rows; r += nt) {
      const int a = (int)(r % NX);
      const int64_t gi = r / NX, bi = gi / M;
      const int i = (int)(gi - bi * M);
      const int64_t ps = (bi * N + n) * (int64_t)M + i;  // (instance, stage, node) block index
      const float* as = R.a_self + ps * NX * NX + a * NX;
      const double* pi = pin + gi * NX;
      double acc = R.c[ps * NX + a];
#pragma unroll
      for (int q = 0; q < NX; ++q) acc = fma((double)as[q], pi[q], acc);
      const int e0 = R.ptr[i], e1 = R.ptr[i + 1];
      const int64_t eb = (bi * N + n) * (int64_t)R.ptr[M];
      for (int e = e0; e < e1; ++e) {
        const float* an = R.a_nbr + (eb + e) * NX * NX + a * NX;
        const double* pj = pin + (bi * M + R.src[e]) * NX;
#pragma unroll
        for (int q = 0; q < NX; ++q) acc = fma((double)an[q], pj[q], acc);
      }
      const float* bb = R.b + ps * NX * NU + a * NU;
      const double* un = A.u + bi * A.ldu + n * NU;
#pragma unroll
      for (int j = 0; j < NU; ++j) acc = fma((double)bb[j], un[j], acc);
      pout[r] = acc;
      finish(bi, i, a, n + 1, acc);
    }
  }
}

__global__ void k_finish_inputs(const FinishArgs A, int B) {
  const int N = A.N, nu = A.nu;
  const int64_t total = (int64_t)B * N * nu;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int j = (int)(t % nu);
    const int k = (int)((t / nu) % N);
    const int64_t bi = t / ((int64_t)N * nu);
    const int st = A.status[bi];
    const bool ok = solved(st);
    const double v = ok ? (1.0 - A.damp) * A.lin_inputs[t] + A.damp * A.u[bi * A.ldu + k * nu + j]
                        : A.fb_inputs[t];
    A.planned_inputs[t] = v;
    if (k >= 1) A.next_inputs[bi * N * nu + (k - 1) * nu + j] = v;
    if (k == N - 1) A.next_inputs[bi * N * nu + (int64_t)(N - 1) * nu + j] = v;
    if (k == 0) {
      double ua;
      if (ok)
        ua = v;  // lin_inputs[0] after the update (mpc.py:406)
      else if (A.fallback == 0 && A.has_prev)
        ua = A.u_prev[bi * nu + j];  // hold-previous-input (mpc.py:410-411)
      else
        ua = 0.0;  // zero-input (mpc.py:413)
      A.u_applied[bi * nu + j] = ua;
      if (A.summary) {
        double* sm = A.summary + bi * (nu + 2);
        sm[j] = ua;
        if (j == 0) {
          sm[nu] = (double)st;
          sm[nu + 1] = A.iters ? (double)A.iters[bi] : 0.0;
        }
      }
    }
  }
}

}  // namespace

extern "C" {

int gm_reconstruct_states(gm_ctx* ctx, int B, int N, const float* gamma, int ld, const double* u,
                          int ldu, double* x, void* stream) {
  int rc = gm_need_device(ctx);
  if (rc) return rc;
  if (ctx->M < 1 || ctx->nx < 1) return gm_fail(ctx, GM_ERR_CONFIG, "graph/dimensions not set");
  if (ld % 4 != 0 || ((uintptr_t)gamma & 15)) return gm_fail(ctx, GM_ERR_CONFIG, "gamma rows must be 16-byte aligned (ld % 4 == 0)");
  const int64_t items = (int64_t)B * ctx->M * (N + 1);
  if (items == 0) return GM_OK;
  const int blocks = (int)std::min<int64_t>((items + 7) / 8, 16 * ctx->sm_count);
  k_reconstruct<<<blocks, 256, 0, (cudaStream_t)stream>>>(gamma, ld, (int)ctx->M, N, ctx->nx,
                                                          ctx->n_u, u, ldu, x, items);
  GM_LAUNCH_CHECK(ctx, "k_reconstruct");
  return GM_OK;
}

int gm_mpc_finish(gm_ctx* ctx, int B, int N, const float* gamma, int ld, const double* u, int ldu,
                  const int32_t* status, const int32_t* iterations, const double* lin_states,
                  const double* lin_inputs, const double* fb_states, const double* fb_inputs,
                  double sqp_damping, int fallback, const double* u_prev, int has_prev,
                  double* cur_states, double* planned_states, double* planned_inputs,
                  double* next_states, double* next_inputs, double* u_applied, double* summary,
                  void* stream) {
  int rc = gm_need_device(ctx);
  if (rc) return rc;
  if (ctx->M < 1 || ctx->nx < 1) return gm_fail(ctx, GM_ERR_CONFIG, "graph/dimensions not set");
  if (B == 0) return GM_OK;
  if (ld % 4 != 0 || ((uintptr_t)gamma & 15)) return gm_fail(ctx, GM_ERR_CONFIG, "gamma rows must be 16-byte aligned (ld % 4 == 0)");
  FinishArgs a{};
  a.M = (int)ctx->M;
  a.N = N;
  a.nx = ctx->nx;
  a.nu = ctx->n_u;
  a.ld = ld;
  a.ldu = ldu;
  a.fallback = fallback;
  a.has_prev = has_prev;
  a.damp = sqp_damping;
  a.W = gamma;
  a.u = u;
  a.status = status;
  a.iters = iterations;
  a.lin_states = lin_states;
  a.lin_inputs = lin_inputs;
  a.fb_states = fb_states ? fb_states : lin_states;
  a.fb_inputs = fb_inputs ? fb_inputs : lin_inputs;
  a.u_prev = u_prev;
  a.cur_states = cur_states;
  a.planned_states = planned_states;
  a.planned_inputs = planned_inputs;
  a.next_states = next_states;
  a.next_inputs = next_inputs;
  a.u_applied = u_applied;
  a.summary = summary;
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t items = (int64_t)B * (N + 1) * ctx->M;
  const int blocks = (int)std::min<int64_t>((items + 7) / 8, 16 * ctx->sm_count);
  // nx = 6, ld <= 128: the pipelined kernel (B200, ncu: cfg5 2.15 -> 1.46 ms,
  // cfg4 4.38 -> 2.97 ms per launch; batching 2 or 4 items per warp at lower
  // occupancy measured slower, 2.93 / 5.18 ms at cfg5).  GM_FIN_MODE=0 forces
  // the generic kernel (measurement override).
  static const int fin_mode = [] {
    const char* e = std::getenv("GM_FIN_MODE");
    return e ? std::atoi(e) : -1;
  }();
  if (ctx->nx == 6 && ld <= 128 && fin_mode != 0 && items < (int64_t(1) << 31))
    k_finish_states_pipe<6><<<blocks, 256, 0, st>>>(a, items);
  else
    k_finish_states<<<blocks, 256, 0, st>>>(a, items);
  GM_LAUNCH_CHECK(ctx, "k_finish_states");
  const int64_t ti = (int64_t)B * N * ctx->n_u;
  k_finish_inputs<<<(int)std::max<int64_t>(1, std::min<int64_t>((ti + 255) / 256, 1024)), 256, 0, st>>>(a, B);
  GM_LAUNCH_CHECK(ctx, "k_finish_inputs");
  return GM_OK;
}

int gm_mpc_finish_rollout(gm_ctx* ctx, int B, int N, const float* a_self, const float* a_nbr, const float* b,
                          const double* c, const double* x0, const double* u, int ldu, const int32_t* status,
                          const int32_t* iterations, const double* lin_states, const double* lin_inputs,
                          const double* fb_states, const double* fb_inputs, double sqp_damping, int fallback,
                          const double* u_prev, int has_prev, double* cur_states, double* planned_states,
                          double* planned_inputs, double* next_states, double* next_inputs, double* u_applied,
                          double* summary, void* stream) {
  int rc = gm_need_device(ctx);
  if (rc) return rc;
  if (ctx->M < 1 || ctx->nx < 1) return gm_fail(ctx, GM_ERR_CONFIG, "graph/dimensions not set");
  if (ctx->nx != 6 || ctx->n_u != 6) return gm_fail(ctx, GM_ERR_CONFIG, "rollout epilogue: nx = nu = 6 only");
  if (ctx->node_hi >= 0 && (ctx->node_lo != 0 || ctx->node_hi != ctx->M))
    return gm_fail(ctx, GM_ERR_CONFIG, "rollout epilogue needs the whole graph (no node range)");
  if (!a_self || !b || !c || !x0 || (ctx->E > 0 && !a_nbr)) return gm_fail(ctx, GM_ERR_CONFIG, "missing stage blocks");
  if (B == 0) return GM_OK;
  FinishArgs a{};
  a.M = (int)ctx->M;
  a.N = N;
  a.nx = ctx->nx;
  a.nu = ctx->n_u;
  a.ld = 0;
  a.ldu = ldu;
  a.fallback = fallback;
  a.has_prev = has_prev;
  a.damp = sqp_damping;
  a.W = nullptr;
  a.u = u;
  a.status = status;
  a.iters = iterations;
  a.lin_states = lin_states;
  a.lin_inputs = lin_inputs;
  a.fb_states = fb_states ? fb_states : lin_states;
  a.fb_inputs = fb_inputs ? fb_inputs : lin_inputs;
  a.u_prev = u_prev;
  a.cur_states = cur_states;
  a.planned_states = planned_states;
  a.planned_inputs = planned_inputs;
  a.next_states = next_states;
  a.next_inputs = next_inputs;
  a.u_applied = u_applied;
  a.summary = summary;
  const int64_t rows = (int64_t)B * ctx->M * 6;
  if (!ctx->d_gbar) {
    GM_CUDA(ctx, cudaMalloc(&ctx->d_gbar, 2 * sizeof(unsigned)));
    GM_CUDA(ctx, cudaMemset(ctx->d_gbar, 0, 2 * sizeof(unsigned)));
  }
  double* pp = (double*)gm_scratch(ctx, 2 * sizeof(double) * (size_t)rows);
  if (!pp) return gm_fail(ctx, GM_ERR_CUDA, "scratch allocation failed");
  RolloutArgs r{};
  r.a_self = a_self;
  r.a_nbr = a_nbr;
  r.b = b;
  r.c = c;
  r.x0 = x0;
  r.ptr = ctx->d_ptr;
  r.src = ctx->d_src;
  r.p0 = pp;
  r.p1 = pp + rows;
  r.bar = ctx->d_gbar;
  int occ = 0;
  GM_CUDA(ctx, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_rollout<6, 6>, 256, 0));
  if (occ < 1) return gm_fail(ctx, GM_ERR_CUDA, "k_rollout does not fit an SM");
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((rows + 255) / 256, (int64_t)ctx->sm_count * occ));
  cudaStream_t st = (cudaStream_t)stream;
  cudaLaunchConfig_t lc{};
  lc.gridDim = dim3((unsigned)grid);
  lc.blockDim = dim3(256);
  lc.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  lc.attrs = attr;
  lc.numAttrs = 1;  // stage barriers need every CTA resident
  GM_CUDA(ctx, cudaLaunchKernelEx(&lc, k_rollout<6, 6>, a, r, B));
  GM_LAUNCH_CHECK(ctx, "k_rollout");
  const int64_t ti = (int64_t)B * N * ctx->n_u;
  k_finish_inputs<<<(int)std::max<int64_t>(1, std::min<int64_t>((ti + 255) / 256, 1024)), 256, 0, st>>>(a, B);
  GM_LAUNCH_CHECK(ctx, "k_finish_inputs");
  return GM_OK;
}

}  // extern "C"
