// K-RS: state reconstruction and the device-side RTI epilogue.
//
// reconstruct_states (condensing.py:409-416): x^i = Gamma_u^i u + Gamma_x^i.
// gm_mpc_finish: mpc.py:151-200 without a host round trip -- the QP status is
// read on the device, the damped update / fallback policy / shift are applied
// and the successor trajectory is written in one elementwise pass.
#include <algorithm>

#include "common.cuh"

namespace {

__device__ __forceinline__ double planned_entry(const float* W, int ld, int N, int nx, int nu,
                                                int64_t gi, int k, int a, const double* u) {
  const float* row = W + ((gi * (N + 1) + k) * nx + a) * (int64_t)ld;
  // only the causal columns [0, k*nu) can be non-zero
  double s = 0.0;
  const int live = k * nu;
  for (int c = 0; c < live; ++c) s = fma((double)row[c], u[c], s);
  return s + (double)row[N * nu];
}

__global__ void k_reconstruct(const float* W, int ld, int M, int N, int nx, int nu,
                              const double* u, int ldu, double* x, int64_t total) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int a = (int)(t % nx);
    const int k = (int)((t / nx) % (N + 1));
    const int64_t gi = t / ((int64_t)nx * (N + 1));
    const int64_t bi = gi / M;
    x[t] = planned_entry(W, ld, N, nx, nu, gi, k, a, u + bi * ldu);
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
__global__ void k_finish_states(const FinishArgs A, int64_t total) {
  const int M = A.M, N = A.N, nx = A.nx;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int a = (int)(t % nx);
    const int i = (int)((t / nx) % M);
    const int k = (int)((t / ((int64_t)nx * M)) % (N + 1));
    const int64_t bi = t / ((int64_t)nx * M * (N + 1));
    double v;
    if (solved(A.status[bi])) {
      const double p = planned_entry(A.W, A.ld, N, nx, A.nu, bi * M + i, k, a, A.u + bi * A.ldu);
      v = (1.0 - A.damp) * A.lin_states[t] + A.damp * p;
    } else {
      v = A.fb_states[t];
    }
    if (A.cur_states) A.cur_states[t] = v;
    // planned_states (M, N+1, nx) = lin_states.transpose(1, 0, 2)   (mpc.py:407)
    A.planned_states[((bi * M + i) * (N + 1) + k) * nx + a] = v;
    // _shift (mpc.py:90-99): s[k-1] = s[k] for k >= 1, s[N] = s[N]
    const int64_t base = bi * (int64_t)(N + 1) * M * nx;
    if (k >= 1) A.next_states[base + ((int64_t)(k - 1) * M + i) * nx + a] = v;
    if (k == N) A.next_states[base + ((int64_t)N * M + i) * nx + a] = v;
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
  const int64_t total = (int64_t)B * ctx->M * (N + 1) * ctx->nx;
  if (total == 0) return GM_OK;
  const int blocks = (int)std::min<int64_t>((total + 255) / 256, 8 * ctx->sm_count);
  k_reconstruct<<<blocks, 256, 0, (cudaStream_t)stream>>>(gamma, ld, (int)ctx->M, N, ctx->nx,
                                                          ctx->n_u, u, ldu, x, total);
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
  const int64_t total = (int64_t)B * (N + 1) * ctx->M * ctx->nx;
  const int blocks = (int)std::min<int64_t>((total + 255) / 256, 8 * ctx->sm_count);
  k_finish_states<<<blocks, 256, 0, st>>>(a, total);
  GM_LAUNCH_CHECK(ctx, "k_finish_states");
  const int64_t ti = (int64_t)B * N * ctx->n_u;
  k_finish_inputs<<<(int)std::max<int64_t>(1, std::min<int64_t>((ti + 255) / 256, 1024)), 256, 0, st>>>(a, B);
  GM_LAUNCH_CHECK(ctx, "k_finish_inputs");
  return GM_OK;
}

}  // extern "C"
