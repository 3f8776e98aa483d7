#include <cstdlib>
// Context, graph index construction and model upload.
//
// Graph: GraphTopology validation (graph.py:35-54) and the index tables of
// _edge_index (gnn.py:107-126) / _padded_neighborhood (condensing.py:158-172)
// are rebuilt here on the host from the in-neighbour CSR, bit-exact with the
// reference (tests/test_graph_tables.py).  The device keeps only the CSR
// (ptr, src) plus dst: slot s>0 of node i is edge ptr[i]+s-1, so the padded
// ELL table of the reference is never materialised on the GPU.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>

#include "common.cuh"

#include <atomic>

static std::atomic<int64_t> g_launches{0};
void gm_count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

int gm_fail(gm_ctx* ctx, int code, const std::string& msg) {
  if (ctx) ctx->err = msg;
  return code;
}

int gm_cuda_check(gm_ctx* ctx, cudaError_t e, const char* what) {
  std::string m = std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e);
  return gm_fail(ctx, GM_ERR_CUDA, m);
}

int gm_need_device(gm_ctx* ctx) {
  if (!ctx) return GM_ERR_CONFIG;
  if (ctx->device < 0) return gm_fail(ctx, GM_ERR_CONFIG, "host-only context has no device");
  cudaError_t e = cudaSetDevice(ctx->device);
  if (e != cudaSuccess) return gm_cuda_check(ctx, e, "cudaSetDevice");
  return GM_OK;
}

void* gm_scratch(gm_ctx* ctx, size_t bytes) {
  if (bytes <= ctx->scratch_bytes) return ctx->scratch;
  // grow; the old buffer is retired, not freed, so CUDA graphs captured with
  // it stay valid until the context is destroyed
  if (ctx->scratch) ctx->retired.push_back(ctx->scratch);
  size_t want = bytes + bytes / 4 + (1 << 20);
  if (cudaMalloc(&ctx->scratch, want) != cudaSuccess) {
    ctx->scratch = nullptr;
    ctx->scratch_bytes = 0;
    return nullptr;
  }
  ctx->scratch_bytes = want;
  return ctx->scratch;
}

static void free_mlp(MlpHost& m) {
  cudaFree(m.d_wt64);
  cudaFree(m.d_w32);
  cudaFree(m.d_b64);
  m.d_wt64 = nullptr;
  m.d_w32 = nullptr;
  m.d_b64 = nullptr;
}

extern "C" {

int gm_abi_version(void) { return 1; }

int64_t gm_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }

// elapsed times between consecutive recorded events (ms): out[i] = t(ev[i+1]) -
// t(ev[i]), i < n - 1; the events must have completed.  One call for a step's
// stage times (StepTiming) instead of one host round trip per pair.
int gm_event_times(int n, void* const* events, float* out) {
  if (n < 2 || !events || !out) return GM_ERR_CONFIG;
  for (int i = 0; i + 1 < n; ++i)
    if (cudaEventElapsedTime(&out[i], (cudaEvent_t)events[i], (cudaEvent_t)events[i + 1]) != cudaSuccess)
      return GM_ERR_CUDA;
  return GM_OK;
}

int gm_create(gm_ctx** out, int device) {
  if (!out) return GM_ERR_CONFIG;
  gm_ctx* c = new gm_ctx();
  c->device = device;
  if (device >= 0) {
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess || device >= n) {
      delete c;
      return GM_ERR_CUDA;
    }
    cudaSetDevice(device);
    cudaDeviceGetAttribute(&c->sm_count, cudaDevAttrMultiProcessorCount, device);
    int optin = 0;
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
    c->smem_optin = (size_t)optin;
  }
  // benchmark/profiling overrides of the kernel-variant switches
  if (const char* v = getenv("GM_CONDENSE_MODE")) {
    const int m = atoi(v);
    c->cond_mode = (m >= 0 && m <= 3) ? m : 0;
  }
  if (const char* v = getenv("GM_LINEARIZE_MODE")) {
    const int m = atoi(v);
    c->lin_mode = (m >= 0 && m <= 4) ? m : 0;
  }
  *out = c;
  return GM_OK;
}

void gm_destroy(gm_ctx* ctx) {
  if (!ctx) return;
  if (ctx->device >= 0) {
    cudaSetDevice(ctx->device);
    cudaFree(ctx->d_ptr);
    cudaFree(ctx->d_src);
    cudaFree(ctx->d_dst);
    cudaFree(ctx->d_norm);
    cudaFree(ctx->scratch);
    cudaFree(ctx->d_flags);
    cudaFree(ctx->d_gbar);
    gm_comm_release(ctx);
    cudaFree(ctx->d_dep_ptr);
    cudaFree(ctx->d_dep);
    cudaFree(ctx->d_cu_ptr);
    cudaFree(ctx->d_cu_nodes);
    cudaFree(ctx->d_cu_slot);
    for (void* p : ctx->retired) cudaFree(p);
    free_mlp(ctx->psi);
    free_mlp(ctx->phi);
  }
  delete ctx;
}

const char* gm_last_error(const gm_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

int gm_set_graph(gm_ctx* ctx, int64_t node_count, int64_t neighbor_bound, const int64_t* nbr_ptr,
                 const int64_t* nbr_list) {
  if (!ctx) return GM_ERR_CONFIG;
  // validation, graph.py:35-54 (same checks, same order)
  if (node_count < 1) return gm_fail(ctx, GM_ERR_CONFIG, "node_count must be >= 1");
  if (neighbor_bound < 1) return gm_fail(ctx, GM_ERR_CONFIG, "neighbor_bound must be >= 1");
  if (!nbr_ptr || nbr_ptr[0] != 0) return gm_fail(ctx, GM_ERR_CONFIG, "nbr_ptr must start at 0");
  int64_t E = nbr_ptr[node_count];
  if (E > 0 && !nbr_list) return gm_fail(ctx, GM_ERR_CONFIG, "missing neighbour list");
  if (E >= (int64_t(1) << 31) || node_count >= (int64_t(1) << 31))
    return gm_fail(ctx, GM_ERR_CONFIG, "graph too large for 32-bit device indices");
  int64_t dmax = 0;
  std::vector<int64_t> sorted;
  for (int64_t i = 0; i < node_count; ++i) {
    int64_t a = nbr_ptr[i], b = nbr_ptr[i + 1];
    if (b < a) return gm_fail(ctx, GM_ERR_CONFIG, "nbr_ptr must be non-decreasing");
    int64_t deg = b - a;
    if (deg > neighbor_bound)
      return gm_fail(ctx, GM_ERR_CONFIG, "node " + std::to_string(i) + " has " +
                                             std::to_string(deg) + " neighbors > bound " +
                                             std::to_string(neighbor_bound));
    sorted.assign(nbr_list + a, nbr_list + b);
    std::sort(sorted.begin(), sorted.end());
    for (size_t k = 1; k < sorted.size(); ++k)
      if (sorted[k] == sorted[k - 1])
        return gm_fail(ctx, GM_ERR_CONFIG, "node " + std::to_string(i) + " has duplicate neighbors");
    for (int64_t k = a; k < b; ++k) {
      int64_t j = nbr_list[k];
      if (j < 0 || j >= node_count)
        return gm_fail(ctx, GM_ERR_CONFIG, "node " + std::to_string(i) +
                                               " references out-of-range neighbor " +
                                               std::to_string(j));
      if (j == i)
        return gm_fail(ctx, GM_ERR_CONFIG, "node " + std::to_string(i) +
                                               " lists itself as neighbor; self-coupling is implicit");
    }
    dmax = deg > dmax ? deg : dmax;
  }
  ctx->M = node_count;
  ctx->E = E;
  ctx->dmax = dmax;
  ctx->bound = neighbor_bound;
  ctx->h_ptr.assign(nbr_ptr, nbr_ptr + node_count + 1);
  ctx->h_src.assign(nbr_list, nbr_list + E);
  ctx->node_lo = 0;
  ctx->node_hi = -1;
  if (ctx->device < 0) return GM_OK;
  int rc = gm_need_device(ctx);
  if (rc) return rc;
  std::vector<int> ptr32(node_count + 1), src32(E > 0 ? E : 1), dst32(E > 0 ? E : 1);
  for (int64_t i = 0; i <= node_count; ++i) ptr32[i] = (int)nbr_ptr[i];
  for (int64_t i = 0; i < node_count; ++i)
    for (int64_t k = nbr_ptr[i]; k < nbr_ptr[i + 1]; ++k) {
      src32[k] = (int)nbr_list[k];
      dst32[k] = (int)i;
    }
  cudaFree(ctx->d_ptr);
  cudaFree(ctx->d_src);
  cudaFree(ctx->d_dst);
  ctx->d_ptr = ctx->d_src = ctx->d_dst = nullptr;
  if (ctx->d_dep_ptr) ctx->retired.push_back(ctx->d_dep_ptr);
  if (ctx->d_dep) ctx->retired.push_back(ctx->d_dep);
  ctx->d_dep_ptr = ctx->d_dep = nullptr;
  ctx->dep_per = -1;
  if (ctx->d_cu_ptr) ctx->retired.push_back(ctx->d_cu_ptr);
  if (ctx->d_cu_nodes) ctx->retired.push_back(ctx->d_cu_nodes);
  if (ctx->d_cu_slot) ctx->retired.push_back(ctx->d_cu_slot);
  ctx->d_cu_ptr = ctx->d_cu_nodes = nullptr;
  ctx->d_cu_slot = nullptr;
  ctx->cu_sc = 0;
  GM_CUDA(ctx, cudaMalloc(&ctx->d_ptr, sizeof(int) * (node_count + 1)));
  GM_CUDA(ctx, cudaMalloc(&ctx->d_src, sizeof(int) * src32.size()));
  GM_CUDA(ctx, cudaMalloc(&ctx->d_dst, sizeof(int) * dst32.size()));
  GM_CUDA(ctx, cudaMemcpy(ctx->d_ptr, ptr32.data(), sizeof(int) * ptr32.size(), cudaMemcpyHostToDevice));
  GM_CUDA(ctx, cudaMemcpy(ctx->d_src, src32.data(), sizeof(int) * src32.size(), cudaMemcpyHostToDevice));
  GM_CUDA(ctx, cudaMemcpy(ctx->d_dst, dst32.data(), sizeof(int) * dst32.size(), cudaMemcpyHostToDevice));
  return GM_OK;
}

int64_t gm_edge_count(const gm_ctx* ctx) { return ctx ? ctx->E : -1; }
int64_t gm_max_degree(const gm_ctx* ctx) { return ctx ? ctx->dmax : -1; }

int gm_graph_tables(const gm_ctx* ctx, int64_t* dst, int64_t* src, int64_t* gather,
                    int64_t* nbr_slots, int64_t* edge_slot) {
  if (!ctx || ctx->M < 1) return GM_ERR_CONFIG;
  const int64_t M = ctx->M, E = ctx->E, d = ctx->dmax;
  const int64_t gw = d > 1 ? d : 1;  // gnn.py:120: max(d_max, 1) columns
  const int64_t S = 1 + d;           // condensing.py:163
  if (gather)
    for (int64_t k = 0; k < M * gw; ++k) gather[k] = E;  // pad = E (phantom message row)
  if (nbr_slots)
    for (int64_t i = 0; i < M; ++i) {
      nbr_slots[i * S] = i;
      for (int64_t s = 1; s < S; ++s) nbr_slots[i * S + s] = M;  // pad = phantom node M
    }
  for (int64_t i = 0; i < M; ++i) {
    for (int64_t e = ctx->h_ptr[i]; e < ctx->h_ptr[i + 1]; ++e) {
      int64_t s = e - ctx->h_ptr[i];
      if (dst) dst[e] = i;
      if (src) src[e] = ctx->h_src[e];
      if (gather) gather[i * gw + s] = e;
      if (nbr_slots) nbr_slots[i * S + 1 + s] = ctx->h_src[e];
      if (edge_slot) edge_slot[e] = s + 1;
    }
  }
  return GM_OK;
}

int gm_set_node_range(gm_ctx* ctx, int64_t lo, int64_t hi) {
  if (!ctx) return GM_ERR_CONFIG;
  if (lo < 0 || hi > ctx->M || lo > hi) return gm_fail(ctx, GM_ERR_CONFIG, "bad node range");
  ctx->node_lo = lo;
  ctx->node_hi = hi;
  return GM_OK;
}

// Upload one MLP.  When the layer dims are unchanged the new parameters are
// copied into the existing device buffers, so CUDA graphs captured with these
// pointers (mpc.py StepPlan) read the new weights.  Otherwise the old buffers
// are retired (kept alive until gm_destroy, never freed under a captured
// graph) and *realloc is set: the caller bumps the model generation so the
// host drops every captured graph.
static int upload_mlp(gm_ctx* ctx, MlpHost& m, int L, const int32_t* dims, const double* w,
                      const double* b, bool* realloc) {
  if (L < 1 || L > GM_MAX_LAYERS)
    return gm_fail(ctx, GM_ERR_CONFIG, "MLP needs 1.." + std::to_string(GM_MAX_LAYERS) + " layers");
  for (int l = 0; l < L; ++l)
    if (dims[l] < 1 || dims[l + 1] < 1) return gm_fail(ctx, GM_ERR_CONFIG, "layer dims must be >= 1");
  const bool same = m.d_wt64 && m.L == L && (int)m.dims.size() == L + 1 &&
                    std::equal(m.dims.begin(), m.dims.end(), dims);
  std::vector<int64_t> w_off(L, 0), b_off(L, 0);
  int64_t wn = 0, bn = 0;
  for (int l = 0; l < L; ++l) {
    w_off[l] = wn;
    b_off[l] = bn;
    wn += (int64_t)dims[l] * dims[l + 1];
    bn += dims[l + 1];
  }
  std::vector<double> wt(wn);
  std::vector<float> w32(wn);
  for (int l = 0; l < L; ++l) {
    const int in = dims[l], out = dims[l + 1];
    const double* Wl = w + w_off[l];  // (out, in) row-major
    for (int o = 0; o < out; ++o)
      for (int k = 0; k < in; ++k) {
        double v = Wl[(int64_t)o * in + k];
        if (!std::isfinite(v)) return gm_fail(ctx, GM_ERR_CONFIG, "parameters must be finite");
        wt[w_off[l] + (int64_t)k * out + o] = v;
        w32[w_off[l] + (int64_t)o * in + k] = (float)v;
      }
  }
  if (!same) {
    if (m.d_wt64) {
      ctx->retired.push_back(m.d_wt64);
      ctx->retired.push_back(m.d_w32);
      ctx->retired.push_back(m.d_b64);
    }
    m.d_wt64 = nullptr;
    m.d_w32 = nullptr;
    m.d_b64 = nullptr;
    m.L = L;
    m.dims.assign(dims, dims + L + 1);
    m.w_off = w_off;
    m.b_off = b_off;
    GM_CUDA(ctx, cudaMalloc(&m.d_wt64, sizeof(double) * wn));
    GM_CUDA(ctx, cudaMalloc(&m.d_w32, sizeof(float) * wn));
    GM_CUDA(ctx, cudaMalloc(&m.d_b64, sizeof(double) * bn));
    *realloc = true;
  }
  GM_CUDA(ctx, cudaMemcpy(m.d_wt64, wt.data(), sizeof(double) * wn, cudaMemcpyHostToDevice));
  GM_CUDA(ctx, cudaMemcpy(m.d_w32, w32.data(), sizeof(float) * wn, cudaMemcpyHostToDevice));
  GM_CUDA(ctx, cudaMemcpy(m.d_b64, b, sizeof(double) * bn, cudaMemcpyHostToDevice));
  return GM_OK;
}

int gm_set_model(gm_ctx* ctx, int n_p, int n_u, int n_m, double dt, int psi_layers,
                 const int32_t* psi_dims, const double* psi_w, const double* psi_b, int phi_layers,
                 const int32_t* phi_dims, const double* phi_w, const double* phi_b,
                 const double* state_mean, const double* state_scale, const double* input_mean,
                 const double* input_scale) {
  int rc = gm_need_device(ctx);
  if (rc) return rc;
  // GnnModel.__post_init__ checks (gnn.py:56-71)
  const int nx = 2 * n_p;
  if (n_p < 1 || n_u < 1 || n_m < 1) return gm_fail(ctx, GM_ERR_CONFIG, "model dims must be >= 1");
  if (nx > GM_MAX_NX) return gm_fail(ctx, GM_ERR_CONFIG, "node state dim too large for this build");
  if (!(dt > 0)) return gm_fail(ctx, GM_ERR_CONFIG, "dt must be positive");
  if (psi_dims[0] != nx) return gm_fail(ctx, GM_ERR_CONFIG, "psi input dim != node state dim");
  if (psi_dims[psi_layers] != n_m) return gm_fail(ctx, GM_ERR_CONFIG, "psi output dim != n_m");
  if (phi_dims[0] != nx + n_m + n_u) return gm_fail(ctx, GM_ERR_CONFIG, "phi input dim != n_state + n_m + n_u");
  if (phi_dims[phi_layers] != n_p) return gm_fail(ctx, GM_ERR_CONFIG, "phi output dim != n_p");
  for (int k = 0; k < nx; ++k)
    if (!(state_scale[k] > 0)) return gm_fail(ctx, GM_ERR_CONFIG, "normalization scales must be positive");
  for (int k = 0; k < n_u; ++k)
    if (!(input_scale[k] > 0)) return gm_fail(ctx, GM_ERR_CONFIG, "normalization scales must be positive");
  // kernels of captured graphs may still read the buffers updated in place
  GM_CUDA(ctx, cudaDeviceSynchronize());
  // scalars are kernel arguments baked into captured graphs: any change
  // invalidates them like a reallocation does
  bool realloc = !ctx->has_model || ctx->n_p != n_p || ctx->n_m != n_m || ctx->m_nu != n_u ||
                 ctx->dt != dt;
  rc = upload_mlp(ctx, ctx->psi, psi_layers, psi_dims, psi_w, psi_b, &realloc);
  if (rc) return rc;
  rc = upload_mlp(ctx, ctx->phi, phi_layers, phi_dims, phi_w, phi_b, &realloc);
  if (rc) return rc;
  std::vector<double> norm(2 * nx + 2 * n_u);
  std::memcpy(norm.data(), state_mean, sizeof(double) * nx);
  std::memcpy(norm.data() + nx, state_scale, sizeof(double) * nx);
  std::memcpy(norm.data() + 2 * nx, input_mean, sizeof(double) * n_u);
  std::memcpy(norm.data() + 2 * nx + n_u, input_scale, sizeof(double) * n_u);
  if (!ctx->d_norm || ctx->norm_len != (int64_t)norm.size()) {
    if (ctx->d_norm) ctx->retired.push_back(ctx->d_norm);
    ctx->d_norm = nullptr;
    GM_CUDA(ctx, cudaMalloc(&ctx->d_norm, sizeof(double) * norm.size()));
    ctx->norm_len = (int64_t)norm.size();
    realloc = true;
  }
  GM_CUDA(ctx, cudaMemcpy(ctx->d_norm, norm.data(), sizeof(double) * norm.size(), cudaMemcpyHostToDevice));
  if (realloc) ++ctx->model_gen;
  ctx->n_p = n_p;
  ctx->n_m = n_m;
  ctx->m_nx = nx;
  ctx->m_nu = n_u;
  ctx->nx = nx;
  ctx->n_u = n_u;
  ctx->dt = dt;
  ctx->has_model = true;
  return GM_OK;
}

int64_t gm_model_generation(const gm_ctx* ctx) { return ctx ? ctx->model_gen : -1; }

int gm_set_dims(gm_ctx* ctx, int nx, int nu) {
  if (!ctx) return GM_ERR_CONFIG;
  if (nx < 1 || nu < 1) return gm_fail(ctx, GM_ERR_CONFIG, "dimensions must be >= 1");
  if (nx > GM_MAX_NX) return gm_fail(ctx, GM_ERR_CONFIG, "node state dim too large for this build");
  ctx->nx = nx;
  ctx->n_u = nu;
  return GM_OK;
}

int gm_gamma_ld(int N, int nu) {
  int need = N * nu + 2;
  return ((need + 31) / 32) * 32;
}

}  // extern "C"
