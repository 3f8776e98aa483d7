// Shared definitions for the B200 GNN-MPC library (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <string>
#include <vector>

#include "../../include/gnnmpc_b200.h"

#define GM_MAX_LAYERS 12
#define GM_MAX_NX 16

// ---------------------------------------------------------------------------
// device views of the model (gnn.py:44-84).  Per layer l (dims[l] -> dims[l+1]):
//   wt64[l]  (dims[l], dims[l+1]) fp64, transposed: forward pass, coalesced over outputs
//   w32[l]   (dims[l+1], dims[l]) fp32, reference layout: input-Jacobian chain
//   b64[l]   (dims[l+1]) fp64
// ---------------------------------------------------------------------------
struct MlpView {
  int L;
  int dims[GM_MAX_LAYERS + 1];
  const double* wt64[GM_MAX_LAYERS];
  const float* w32[GM_MAX_LAYERS];
  const double* b64[GM_MAX_LAYERS];
};

struct MlpHost {
  int L = 0;
  std::vector<int> dims;
  double* d_wt64 = nullptr;
  float* d_w32 = nullptr;
  double* d_b64 = nullptr;
  std::vector<int64_t> w_off, b_off;
  MlpView view() const {
    MlpView v{};
    v.L = L;
    for (int l = 0; l <= L && l <= GM_MAX_LAYERS; ++l) v.dims[l] = dims[l];
    for (int l = 0; l < L; ++l) {
      v.wt64[l] = d_wt64 + w_off[l];
      v.w32[l] = d_w32 + w_off[l];
      v.b64[l] = d_b64 + b_off[l];
    }
    return v;
  }
  int max_width() const {
    int w = 0;
    for (int d : dims) w = d > w ? d : w;
    return w;
  }
  int hidden_sum() const {  // mask bytes per sample
    int s = 0;
    for (int l = 1; l < L; ++l) s += dims[l];
    return s;
  }
};

struct gm_ctx {
  int device = -1;
  std::string err;
  // graph (graph.py:25-63) as in-edge CSR in canonical edge order
  int64_t M = 0, E = 0, dmax = 0, bound = 0;
  std::vector<int64_t> h_ptr, h_src;
  int* d_ptr = nullptr;
  int* d_src = nullptr;
  int* d_dst = nullptr;
  int64_t node_lo = 0, node_hi = -1;
  int lin_mode = 0;  // gm_set_linearize_mode
  int cond_mode = 0;  // gm_set_condense_mode
  // K-COND variant of the last gm_condense_fused launch (gm_last_condense_kernel):
  // 1 SIMT k_condense_fused, 2 tcgen05 k_condense_tc, 3 k_condense_tma,
  // 4 k_condense_tmap 384 threads, 5 k_condense_tmap 512 threads, 6 two-kernel path
  int last_cond_kernel = 0;
  // model
  bool has_model = false;
  int n_p = 0, n_m = 0;
  int m_nx = 0, m_nu = 0;  // model dims (gm_linearize)
  int nx = 0, n_u = 0;     // condensing dims (gm_set_dims / gm_set_model)
  double dt = 0;
  MlpHost psi, phi;
  double* d_norm = nullptr;  // state_mean(nx) state_scale(nx) input_mean(nu) input_scale(nu)
  int64_t norm_len = 0;
  int64_t model_gen = 0;  // bumped when weight buffers / baked scalars change (gm_model_generation)
  // scratch (grown on demand, stream-ordered use only)
  void* scratch = nullptr;
  size_t scratch_bytes = 0;
  std::vector<void*> retired;  // outgrown scratch kept alive: captured CUDA graphs may use it
  int sm_count = 148;
  size_t smem_optin = 227 * 1024;
  // fused condensing (k_condense_fused.cu): per-CTA stage flags (self-resetting,
  // zero between launches) and the CTA dependency lists of the node partition
  int* d_flags = nullptr;
  int64_t flag_cap = 0;
  unsigned* d_gbar = nullptr;  // grid barrier of the rollout epilogue (count, generation)
  // native data plane (k_comm.cu): NCCL communicator of the partitioned step
  void* nccl_comm = nullptr;
  int comm_rank = 0, comm_world = 1;
  int64_t dep_per = -1;
  int* d_dep_ptr = nullptr;
  int* d_dep = nullptr;
  // K-COND TMA variant: per node chunk of `cu_sc` nodes, its unique
  // closed-neighbourhood nodes (cu_ptr / cu_nodes) and each (node, slot)'s
  // index into them (cu_slot, 255 = none)
  int cu_sc = 0, cu_umax = 0;
  int* d_cu_ptr = nullptr;
  int* d_cu_nodes = nullptr;
  unsigned char* d_cu_slot = nullptr;
};

// error helpers -------------------------------------------------------------
int gm_fail(gm_ctx* ctx, int code, const std::string& msg);
int gm_cuda_check(gm_ctx* ctx, cudaError_t e, const char* what);
int gm_need_device(gm_ctx* ctx);
void* gm_scratch(gm_ctx* ctx, size_t bytes);
void gm_comm_release(gm_ctx* ctx);  // k_comm.cu: destroys the context's communicator

#define GM_CUDA(ctx, expr)                                          \
  do {                                                              \
    cudaError_t _e = (expr);                                        \
    if (_e != cudaSuccess) return gm_cuda_check((ctx), _e, #expr); \
  } while (0)

void gm_count_launch();

#define GM_LAUNCH_CHECK(ctx, what)                                 \
  do {                                                             \
    gm_count_launch();                                             \
    cudaError_t _e = cudaGetLastError();                           \
    if (_e != cudaSuccess) return gm_cuda_check((ctx), _e, what); \
  } while (0)

// the fused per-row MLP chains of the layer-wise linearisation apply
// (k_linearize_layers.cu)
bool gm_lin_chains(const gm_ctx* ctx);

// K-HG through the fused kernels without the recursion (k_condense_fused.cu):
// tc != 0 tcgen05, else SIMT; returns 1 when the shape is not handled
int gm_fused_cost(gm_ctx* ctx, int tc, int B, int N, const float* gamma, int ld, const double* q,
                  int64_t q_stride, const double* x_ref, int64_t xref_stride, const double* r,
                  int64_t r_stride, const double* u_ref, int64_t uref_stride, double* H, double* g,
                  int partial, void* stream);

static inline int64_t gm_node_hi(const gm_ctx* c) { return c->node_hi < 0 ? c->M : c->node_hi; }

static inline int gm_ceil_div(int64_t a, int64_t b) { return (int)((a + b - 1) / b); }
