/*
 * gnnmpc_b200.h -- C ABI of the B200-native GNN-MPC hot path.
 *
 * One shared library (libgnnmpc_b200.so, sm_100a) exports the per-step hot
 * path of the reference package ``gnnmpc`` (arXiv 2602.17601) as plain
 * C entry points: pointers + sizes, no torch types.  The reference is pure
 * Python; the functions below are what its Python API
 * for this path would bind through an FFI (ctypes stub in INTEGRATION.md).
 * Each entry point names the reference function it replaces
 * (paths relative to /root/reference/pkg/src/gnnmpc/).
 *
 * Conventions
 *   - M nodes per instance, N horizon stages, nx = 2*n_p state, nu inputs,
 *     E directed edges in the canonical node-major order of
 *     GraphTopology.edges (graph.py:60-63).
 *   - B independent instances (scenarios) share one model and one topology;
 *     every per-instance array is instance-major.  B = 1 reproduces the
 *     reference call exactly.
 *   - "device" pointers are CUDA device memory on the context's device and
 *     are owned by the caller; the context owns weights, graph tables and
 *     scratch.  All device work is stream-ordered on `stream` (a
 *     cudaStream_t passed as void*); no entry point synchronises the host
 *     unless stated.
 *   - Gamma work array ("gamma"): fp32 (B*M, N+1, nx, ld) with
 *     Gamma_u (condensing.py:187) in columns [0, N*nu) and Gamma_x in
 *     column N*nu; ld = gm_gamma_ld(N, nu) (>= N*nu+2, multiple of 32).
 *   - Return codes: GM_OK, GM_ERR_CONFIG (the reference raises ValueError /
 *     ConfigurationError, condensing.py:36-37), GM_ERR_NUMERIC (numerical
 *     abort, cli.py:332-338 exit 3), GM_ERR_CUDA (CUDA / NCCL failure).
 *     The message is available from gm_last_error().  QP failures are
 *     statuses, not errors (qpsolver.py:24-28).
 */
#ifndef GNNMPC_B200_H
#define GNNMPC_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GM_OK 0
#define GM_ERR_CONFIG 2
#define GM_ERR_NUMERIC 3
#define GM_ERR_CUDA 4

/* QpStatus, declaration order of qpsolver.py:24-28 */
#define GM_QP_OPTIMAL 0
#define GM_QP_MAX_ITERATIONS 1
#define GM_QP_PRIMAL_INFEASIBLE 2
#define GM_QP_NUMERICAL_FAILURE 3

typedef struct gm_ctx gm_ctx;

/* SolverSettings (qpsolver.py:66-76); warm_start is a separate pointer. */
typedef struct gm_qp_settings {
  double tolerance;            /* 1e-8 */
  int32_t max_iterations;      /* 50 */
  double regularization;       /* 1e-9 */
  double fraction_to_boundary; /* 0.995 */
} gm_qp_settings;

int gm_abi_version(void);

/* Number of kernels this library has launched in the process (all
 * contexts); bench.py reports the per-step delta as gpu_launches. */
int64_t gm_launch_count(void);
/* Elapsed ms between consecutive completed CUDA events: out[i] = ev[i] ->
 * ev[i+1], i < n - 1 (the step's stage times in one call). */
int gm_event_times(int n, void* const* events, float* out);

/* Context.  device < 0 creates a host-only context: graph index
 * construction works, every device entry point returns GM_ERR_CONFIG. */
int gm_create(gm_ctx** out, int device);
void gm_destroy(gm_ctx* ctx);
const char* gm_last_error(const gm_ctx* ctx);

/* ---- graph (graph.py:25-74) ------------------------------------------- */
/* Replaces GraphTopology validation (graph.py:35-54) + the index tables of
 * _edge_index (gnn.py:107-126) and _padded_neighborhood
 * (condensing.py:158-172).  Host inputs: in-neighbour lists as CSR,
 * nbr_ptr (node_count+1), nbr_list (nbr_ptr[node_count]). */
int gm_set_graph(gm_ctx* ctx, int64_t node_count, int64_t neighbor_bound,
                 const int64_t* nbr_ptr, const int64_t* nbr_list);
int64_t gm_edge_count(const gm_ctx* ctx);
int64_t gm_max_degree(const gm_ctx* ctx);
/* Host outputs, bit-exact with the reference tables:
 *   dst, src   (E)                   gnn.py:116-117
 *   gather     (M, max(d,1)) pad E   gnn.py:120-125
 *   nbr_slots  (M, 1+d)      pad M   condensing.py:163-171
 *   edge_slot  (E)                   condensing.py:166-172
 * Any pointer may be NULL to skip that table. */
int gm_graph_tables(const gm_ctx* ctx, int64_t* dst, int64_t* src, int64_t* gather,
                    int64_t* nbr_slots, int64_t* edge_slot);

/* ---- model (gnn.py:44-104, mlp.py:15-64) ------------------------------- */
/* Host inputs.  psi_w / phi_w: the row-major (out, in) weight matrices of
 * each layer concatenated; *_b: biases concatenated; dims arrays have
 * n_layers+1 entries. */
int gm_set_model(gm_ctx* ctx, int n_p, int n_u, int n_m, double dt,
                 int psi_layers, const int32_t* psi_dims, const double* psi_w, const double* psi_b,
                 int phi_layers, const int32_t* phi_dims, const double* phi_w, const double* phi_b,
                 const double* state_mean, const double* state_scale,
                 const double* input_mean, const double* input_scale);

/* Model generation: incremented by gm_set_model whenever the device weight
 * buffers are reallocated (layer dims changed) or a scalar baked into kernel
 * arguments (n_p, n_u, n_m, dt) changed.  Parameter edits with unchanged dims
 * are copied into the existing buffers and keep the generation, so captured
 * CUDA graphs stay valid and read the new weights; a host that captured
 * graphs must drop them when the generation moves.  Buffers are never freed
 * under a captured graph (retired until gm_destroy). */
int64_t gm_model_generation(const gm_ctx* ctx);

/* State / input dimensions used by the condensing entry points when the
 * linearisation was not produced by gm_linearize (set_model sets both). */
int gm_set_dims(gm_ctx* ctx, int nx, int nu);

/* Restrict node-wise work to owned nodes [lo, hi) of every instance (graph
 * partition for multi-GPU; default = all nodes). */
int gm_set_node_range(gm_ctx* ctx, int64_t lo, int64_t hi);

/* ---- stage 1: linearize_trajectory (gnn.py:308-321 -> :237-298) ------- */
/* P = B*K linearisation points.  Device inputs X (P, M, nx) fp64,
 * U (P, nu) fp64.  Device outputs: a_self (P, M, nx, nx), a_nbr (P, E, nx,
 * nx) in edge order, b (P, M, nx, nu) in fp32 and the offset c (P, M, nx) in
 * fp64, evaluated from the stored fp32 blocks so the affine model is exact at
 * the linearisation point to fp64 round-off (gnn.py:290-297).
 * f_next (P, M, nx) fp64 = step_array(X, U) (gnn.py:153-159), may be NULL. */
int gm_linearize(gm_ctx* ctx, int64_t P, const double* X, const double* U, float* a_self,
                 float* a_nbr, float* b, double* c, double* f_next, void* stream);

/* Linearisation kernel selection: 0 = automatic (fused per-tile kernel for
 * fewer than 8k node points with the reference architecture, layer-wise
 * chain above), 1 = always the fused kernel, 2 = always the layer-wise chain
 * (forward and Jacobian chains fused per row for the reference
 * architecture: forward passes on fp64 DMMA, Jacobian chains on tcgen05),
 * 3 = layer-wise with one launch per layer, 4 = as 2 with every chain as a
 * per-row SIMT kernel.  All compute the
 * same formulas; the switch exists for tests and benchmarks. */
int gm_set_linearize_mode(gm_ctx* ctx, int mode);

/* step_array only (gnn.py:153-159): f (P, M, nx) fp64. */
int gm_step(gm_ctx* ctx, int64_t P, const double* X, const double* U, double* f, void* stream);

/* ---- stage 2: condense_gammas (condensing.py:182-228) ------------------ */
int gm_gamma_ld(int N, int nu);
/* lin blocks as produced by gm_linearize with P = B*N; x0 (B, M, nx) fp64. */
int gm_condense_gammas(gm_ctx* ctx, int B, int N, const float* a_self, const float* a_nbr,
                       const float* b, const double* c, const double* x0, float* gamma, int ld,
                       void* stream);
/* One stage n -> n+1 only (for the node-partitioned recursion whose halo
 * rows are exchanged between stages).  Stage 0 is written by n = -1. */
int gm_condense_gammas_stage(gm_ctx* ctx, int B, int N, int n, const float* a_self,
                             const float* a_nbr, const float* b, const double* c,
                             const double* x0, float* gamma, int ld, void* stream);

/* ---- stage 3: condense_ocp cost part (condensing.py:363-389, :402-403) -- */
/* H (B, n0, n0) fp64 symmetrised, g (B, n0) fp64, n0 = N*nu.
 * q (B, M, N+1, nx, nx), x_ref (B, M, N+1, nx), r (B, N, nu, nu),
 * u_ref (B, N, nu): fp64 device; a per-instance stride of 0 broadcasts
 * one array to all instances (strides in elements).
 * partial != 0 writes only the (symmetrised) node sums over the owned node
 * range, without R-bar and r_lin: the multi-GPU partial that is all-reduced
 * (rank 0 passes partial = 0, so the sum over ranks is the full H, g). */
int gm_condense_cost(gm_ctx* ctx, int B, int N, const float* gamma, int ld, const double* q,
                     int64_t q_stride, const double* x_ref, int64_t xref_stride, const double* r,
                     int64_t r_stride, const double* u_ref, int64_t uref_stride, double* H,
                     double* g, int partial, void* stream);

/* Fused condensing: gm_condense_gammas followed by gm_condense_cost (partial
 * = 0) in one persistent kernel plus a two-pass fixed-order reduction
 * (condense_gammas condensing.py:182-228 + the cost part of condense_ocp
 * :376-389, :402-403).  Same arguments and outputs as the two calls; gamma is
 * fully written.  Requires the whole node range (gm_set_node_range unset);
 * shapes outside the fused kernel's instantiations run the two-kernel path.
 * One launch per context at a time (per-context stage counters). */
/* Kernel selection of gm_condense_fused: 0 = auto (nx = nu = 6 with 8-node
 * items fitting shared memory: the TMA-staged kernel k_condense_tma, else the
 * SIMT fused kernel; H and g always in fp32 FMA with round-to-nearest
 * accumulation), 1 = always the SIMT fused kernel (per-thread neighbour
 * loads), 2 = the two-kernel path (per-stage K-REC launches + K-HG),
 * 3 = the tcgen05 3xTF32 H kernel (opt-in: the tensor-core accumulator
 * truncates on every add, ~7e-5 relative H error at 10^4 nodes).  The same
 * switch selects K-HG in gm_condense_cost (3: tcgen05, else SIMT).
 * For tests and benchmarks. */
int gm_set_condense_mode(gm_ctx* ctx, int mode);
int gm_condense_fused(gm_ctx* ctx, int B, int N, const float* a_self, const float* a_nbr,
                      const float* b, const double* c, const double* x0, float* gamma, int ld,
                      const double* q, int64_t q_stride, const double* x_ref, int64_t xref_stride,
                      const double* r, int64_t r_stride, const double* u_ref, int64_t uref_stride,
                      double* H, double* g, void* stream);

/* ---- per-node condensing (condensing.py:231-243, :285-295, :334-360) --- */
/* local_hessian_gradient for every node of the node range [lo, hi) of every
 * instance: H (B, nodes, n0, n0) = sum_k Gu_k' Qs_k Gu_k (Qs = (Q + Q')/2,
 * i.e. the reference's symmetrised 0.5 (h + h')) and g (B, nodes, n0) =
 * sum_k Gu_k' (2 Q_k Gx_k + q_lin_k), fp64, from the fp32 work array (all
 * N+1 stages, all n0 columns).  q (B, M, N+1, nx, nx), q_lin (B, M, N+1, nx)
 * fp64 device, per-instance strides in elements (0 broadcasts). */
int gm_node_hessians(gm_ctx* ctx, int B, int N, const float* gamma, int ld, const double* q,
                     int64_t q_stride, const double* q_lin, int64_t qlin_stride, double* H,
                     double* g, void* stream);
/* assemble_qp's node sum (condensing.py:344-355): dst (B, len) = base (B,
 * len, may be NULL) + sum_{i < count} src (B, count, len), ascending i, fp64;
 * sym_n > 0 (len = sym_n^2) returns the symmetrised 0.5 (S + S'). */
int gm_sum_nodes(gm_ctx* ctx, int B, int count, int len, int sym_n, const double* src,
                 const double* base, double* dst, void* stream);

/* Constraint rows (condensing.py:263-282, :312-323), per instance:
 * rows [0, n_in) are input rows: row k has coefficients in_c (nu) at
 * column block in_stage[k]; rows [n_in, n_in+n_st) are state rows:
 * C = st_c . Gamma_u[node, stage], d = st_d - st_c . Gamma_x[node, stage].
 * Row data shared by all instances; outputs C (B, m0, n0), d (B, m0) fp64. */
int gm_constraint_rows(gm_ctx* ctx, int B, int N, const float* gamma, int ld, int n_in,
                       const int32_t* in_stage, const double* in_c, const double* in_d, int n_st,
                       const int32_t* st_node, const int32_t* st_stage, const double* st_c,
                       const double* st_d, double* C, double* d, void* stream);

/* expand_soft_constraints (condensing.py:419-439), batched.  soft_idx (ns)
 * row indices into the m0 rows; rho1/rho2 (ns).  Outputs H (B, n, n),
 * g (B, n), C (B, m, n), d (B, m) with n = n0+ns, m = m0+ns. */
int gm_expand_soft(gm_ctx* ctx, int B, int n0, int m0, const double* H0, const double* g0,
                   const double* C0, const double* d0, int ns, const int32_t* soft_idx,
                   const double* rho1, const double* rho2, double* H, double* g, double* C,
                   double* d, void* stream);

/* ---- stage 4: solve_qp (qpsolver.py:112-243), batched ------------------ */
/* One QP per instance: H (B, n, n), g (B, n), C (B, m, n), d (B, m),
 * warm (B, n) or NULL.  Outputs u (B, n), lam (B, m), status (B),
 * iterations (B), resid (B, 3) = stationarity, primal_infeas,
 * complementarity of the returned iterate. */
int gm_solve_qp(gm_ctx* ctx, int B, int n, int m, const double* H, const double* g,
                const double* C, const double* d, const double* warm,
                const gm_qp_settings* settings, double* u, double* lam, int32_t* status,
                int32_t* iterations, double* resid, void* stream);

/* Diagnostics: per-phase cycle accounting of K-QP (block 0).  gm_qp_profile(1)
 * enables and zeroes the counters (2: counters 13-15 account the Cholesky
 * pivot chain instead of the Schur build); gm_qp_phase_cycles copies 16
 * counters (synchronous).  The counters are compiled in only with
 * -DGM_QP_PROF; otherwise gm_qp_profile(on != 0) returns GM_ERR_CONFIG. */
int gm_qp_profile(int on);
int gm_qp_phase_cycles(unsigned long long* out);
/* Diagnostics: per-stage cycle accounting of the pipelined K-COND (CTA 0):
 * 32 stages x 8 counters (group R item / empty-wait / flag-wait / tile-wait,
 * group H full-wait / busy / fold, items).  gm_cond_profile(1) enables and
 * zeroes; gm_cond_phase_cycles copies 256 counters (synchronous). */
int gm_cond_profile(int on);
int gm_cond_phase_cycles(unsigned long long* out);
/* Diagnostics: the K-COND variant of the context's last gm_condense_fused
 * call: 0 none, 1 SIMT k_condense_fused, 2 tcgen05 k_condense_tc, 3
 * k_condense_tma, 4 / 5 k_condense_tmap with 384 / 512 threads, 6 the
 * two-kernel path. */
int gm_last_condense_kernel(gm_ctx* ctx);
/* Diagnostics: factor a dense SPD matrix A (n x n, row-major, device) with
 * K-QP's own Cholesky and solve A x = b; L (n x n) lower, ok = 0 when a pivot
 * failed.  Used by the tests to check the factorisation in isolation. */
int gm_chol_check(gm_ctx* ctx, int n, const double* A, const double* b, double* L, double* x,
                  int32_t* ok, void* stream);
/* Diagnostics: known-answer check of the tcgen05 3xTF32 Gram product used by
 * K-COND's H accumulation: S (P, P) = G' Q for G, Q (K, P) fp32 row-major,
 * P <= 128 (one CTA, TMEM accumulator). */
int gm_gram_check(gm_ctx* ctx, int K, int P, const float* G, const float* Q, float* S, void* stream);

/* ---- reconstruct_states (condensing.py:409-416) ------------------------ */
/* u (B, ldu) fp64 (first N*nu used); x (B, M, N+1, nx) fp64. */
int gm_reconstruct_states(gm_ctx* ctx, int B, int N, const float* gamma, int ld,
                          const double* u, int ldu, double* x, void* stream);

/* ---- mpc_step tail (mpc.py:151-200) ------------------------------------ */
/* Device-side RTI epilogue, no host sync.  Per instance, when status is
 * OPTIMAL or MAX_ITERATIONS: planned = reconstruct(u) and the trajectory
 * becomes (1-a) lin + a planned (a = sqp_damping), u_applied = its input 0;
 * otherwise the trajectory falls back to fb_states / fb_inputs (the
 * previous plan with x_measured at stage 0) and u_applied follows the
 * fallback policy (0 hold-previous-input using u_prev when has_prev != 0,
 * 1 zero-input).  Outputs: cur_states (B, N+1, M, nx) unshifted (may be
 * NULL), planned_states (B, M, N+1, nx), planned_inputs (B, N, nu), the
 * shifted successor next_states (B, N+1, M, nx) / next_inputs (B, N, nu)
 * (mpc.py:90-99), u_applied (B, nu) and summary (B, nu+2) = [u_applied,
 * status, iterations] for a single small device->host read (may be NULL). */
int gm_mpc_finish(gm_ctx* ctx, int B, int N, const float* gamma, int ld, const double* u,
                  int ldu, const int32_t* status, const int32_t* iterations,
                  const double* lin_states, const double* lin_inputs, const double* fb_states,
                  const double* fb_inputs, double sqp_damping, int fallback,
                  const double* u_prev, int has_prev, double* cur_states,
                  double* planned_states, double* planned_inputs, double* next_states,
                  double* next_inputs, double* u_applied, double* summary, void* stream);
/* Same epilogue with the planned states formed by linear rollout instead of
 * from Gamma: p_0 = x0, p_{n+1}(i) = A_self p_n(i) + sum_e A_e p_n(src e) +
 * B_n(i) u_n + c_n(i), which equals Gamma_u u + Gamma_x (reference
 * condensing.py:182-228, 409-416; tests/test_condensing.py:120-135) while
 * reading the stage blocks (a_self / a_nbr / b as written by gm_linearize,
 * c, x0 (B, M, nx)) instead of Gamma's rows; for large batches (cfg4, cfg5).
 * nx = nu = 6, whole graph (no node range). */
int gm_mpc_finish_rollout(gm_ctx* ctx, int B, int N, const float* a_self, const float* a_nbr,
                          const float* b, const double* c, const double* x0, const double* u,
                          int ldu, const int32_t* status, const int32_t* iterations,
                          const double* lin_states, const double* lin_inputs,
                          const double* fb_states, const double* fb_inputs, double sqp_damping,
                          int fallback, const double* u_prev, int has_prev, double* cur_states,
                          double* planned_states, double* planned_inputs, double* next_states,
                          double* next_inputs, double* u_applied, double* summary, void* stream);

/* ---- native data plane of the partitioned step (multi-GPU) ------------- */
/* SURVEY 8b gm_init_comm.  An NCCL communicator owned by the context
 * (NCCL resolved at run time: libnccl.so.2, the copy torch loaded when
 * present).  Everything is stream-ordered with no host synchronisation, so
 * a rank's step (kernels + exchanges + all-reduce) can be captured in one
 * CUDA graph.  The reference has no counterpart (single process; the
 * node-chunk pool condensing.py:208-227 is what the partition generalises).
 *   gm_comm_available   1 when libnccl.so.2 and its symbols resolved
 *   gm_comm_unique_id   rank 0 creates the 128-byte id, the host broadcasts it
 *   gm_init_comm        ncclCommInitRank on the context's device (collective)
 *   gm_allreduce_sum    in-place fp64 sum over the ranks ([H | g | C | d])
 *   gm_sendrecv         one grouped batch of byte sends / receives (halo rows) */
int gm_comm_available(void);
int gm_comm_unique_id(void* out128);
int gm_init_comm(gm_ctx* ctx, const void* unique_id128, int rank, int world);
int gm_comm_destroy(gm_ctx* ctx);
int gm_allreduce_sum(gm_ctx* ctx, double* buf, int64_t count, void* stream);
int gm_sendrecv(gm_ctx* ctx, int nsend, const int* send_peers, void* const* send_bufs,
                const int64_t* send_bytes, int nrecv, const int* recv_peers, void* const* recv_bufs,
                const int64_t* recv_bytes, void* stream);

/* ---- node-partitioned recursion: halo pack / unpack (multi-GPU) ------- */
/* Strided row gather / scatter for the per-stage halo exchange of the
 * node-partitioned Gamma recursion (the reference's node-chunk pool,
 * condensing.py:208-227, generalised to row slabs over devices).
 * gather: dst (n_outer, n_idx, row_bytes) contiguous <- src rows at
 *   src + o*outer_stride_bytes + idx[i]*row_stride_bytes;
 * scatter: the inverse.  idx (n_idx) int32 device; all sizes and addresses
 * multiples of 8 bytes. */
int gm_gather_rows(gm_ctx* ctx, const void* src, void* dst, const int32_t* idx, int n_idx,
                   int64_t row_bytes, int64_t row_stride_bytes, int n_outer,
                   int64_t outer_stride_bytes, void* stream);
int gm_scatter_rows(gm_ctx* ctx, const void* src, void* dst, const int32_t* idx, int n_idx,
                    int64_t row_bytes, int64_t row_stride_bytes, int n_outer,
                    int64_t outer_stride_bytes, void* stream);

/* ---- batched training gradients (training.py:99-150) ------------------ */
/* Number of model parameters (psi weights, psi biases, phi weights, phi
 * biases), the length of gm_loss_gradients' grads; -1 without a model. */
int gm_param_count(const gm_ctx* ctx);
/* loss_gradients for a batch of B records with the context's model and
 * graph, fp64: X, Xn (B, M, nx), U (B, nu), weights (M, nx) (the diagonal of
 * O per node, training.py:_weight_grid) device.  loss (1) device receives
 * sum(W r^2)/B + l2 |p|^2; grads (gm_param_count) device, in the order of
 * training.py:_params: every psi weight matrix (out, in) row-major, psi
 * biases, phi weights, phi biases.  Deterministic (fixed-order sums). */
int gm_loss_gradients(gm_ctx* ctx, int B, const double* X, const double* U, const double* Xn,
                      const double* weights, double l2_lambda, double* loss, double* grads,
                      void* stream);

/* ---- cfg2 plant: trunk.py chain (trunk.py:116-160) ------------------------ */
/* One controller period (substeps semi-implicit Euler substeps of dt_sim) of B
 * chain plants with M nodes: X, Xout (B, M, 6) fp64 [p | v], U (B, nu) fp64
 * tendon tensions (clipped to [0, u_max] when clip != 0, trunk.py:152),
 * rest (M, 3) rest positions, fmap (M, 3, nu) tendon force map (device);
 * gravity (3) is a HOST array.
 * *bad (device int) is set to 1 when a state becomes non-finite (the
 * reference raises FloatingPointError, trunk.py:158-159). */
int gm_trunk_step(gm_ctx* ctx, int B, int M, int nu, int substeps, double dt_sim, double mass,
                  double k, double c, double kb, double rest_len, const double* gravity,
                  const double* rest, const double* fmap, double u_max, int clip, const double* X,
                  const double* U, double* Xout, int32_t* bad, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* GNNMPC_B200_H */
