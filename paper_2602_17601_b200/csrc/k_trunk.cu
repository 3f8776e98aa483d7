// Chain plant of the closed-loop tracking configuration (BASELINE cfg2):
// gravity-loaded point masses with neighbour spring-dampers, a restoring
// force toward the rest shape and tendon inputs, integrated by semi-implicit
// Euler substeps (reference: trunk.py:116-160, _accelerations /
// sim_substep / step_state_array).
//
// One CTA per instance, one thread per node; every substep is force ->
// barrier -> velocity/position update -> barrier, all in fp64 with the
// reference's operation order per term, so the device plant tracks the numpy
// plant to round-off.  Keeping the plant on the device makes the closed loop
// device resident: only the applied input leaves the GPU each step.
#include "common.cuh"

namespace {

struct TrunkArgs {
  int B, M, nu, substeps, clip, fm_sparse;
  double dt_sim, mass, k, c, kb, rest_len, u_max;
  double g[3];
  const double* rest;  // (M, 3)
  const double* fmap;  // (M, 3, nu) tendon force map
  const double* X;     // (B, M, 6)
  const double* U;     // (B, nu)
  double* Xout;        // (B, M, 6)
  int* bad;            // set when a state becomes non-finite
};

__global__ void k_trunk_step(const TrunkArgs a) {
  extern __shared__ double sh[];
  const int M = a.M;
  double* P = sh;          // M x 3
  double* V = sh + 3 * M;  // M x 3
  double* u = sh + 6 * M;  // nu
  const int64_t b = blockIdx.x;
  const double* X = a.X + b * (int64_t)M * 6;
  for (int t = threadIdx.x; t < M * 3; t += blockDim.x) {
    const int i = t / 3, d = t - 3 * i;
    P[t] = X[i * 6 + d];
    V[t] = X[i * 6 + 3 + d];
  }
  for (int j = threadIdx.x; j < a.nu; j += blockDim.x) {
    double v = a.U[b * a.nu + j];
    if (a.clip) v = fmin(fmax(v, 0.0), a.u_max);  // np.clip(u, 0, u_max) (trunk.py:152)
    u[j] = v;
  }
  __syncthreads();
  for (int s = 0; s < a.substeps; ++s) {
    double acc[3] = {0.0, 0.0, 0.0};
    const int i = threadIdx.x;
    if (i < M) {
      // f = m g (trunk.py:118-119)
      double f[3] = {a.mass * a.g[0], a.mass * a.g[1], a.mass * a.g[2]};
      // segment terms: f[1:] -= axial + damp, f[:-1] += axial + damp (:121-127)
      auto seg = [&](int lo, double sign) {
        double dl[3], len2 = 0.0;
#pragma unroll
        for (int d = 0; d < 3; ++d) {
          dl[d] = P[(lo + 1) * 3 + d] - P[lo * 3 + d];
          len2 += dl[d] * dl[d];
        }
        const double len = fmax(sqrt(len2), 1e-12);
#pragma unroll
        for (int d = 0; d < 3; ++d) {
          const double axial = a.k * (len - a.rest_len) * (dl[d] / len);
          const double damp = a.c * (V[(lo + 1) * 3 + d] - V[lo * 3 + d]);
          f[d] += sign * (axial + damp);
        }
      };
      if (i >= 1) seg(i - 1, -1.0);
      if (i + 1 < M) seg(i, 1.0);
      if (i >= 1) {  // rest-shape restoring force, moving nodes (:129-130)
#pragma unroll
        for (int d = 0; d < 3; ++d) f[d] -= a.kb * (P[i * 3 + d] - a.rest[i * 3 + d]);
      }
      // tendon forces fm @ u (:132-133)
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        double t = 0.0;
        for (int j = 0; j < a.nu; ++j) t += a.fmap[(i * 3 + d) * a.nu + j] * u[j];
        f[d] += t;
      }
#pragma unroll
      for (int d = 0; d < 3; ++d) acc[d] = f[d] / a.mass;
    }
    __syncthreads();
    if (i < M) {  // v += dt a, base pinned; p += dt v, base at rest (:138-144)
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        const double v = i == 0 ? 0.0 : V[i * 3 + d] + a.dt_sim * acc[d];
        V[i * 3 + d] = v;
        P[i * 3 + d] = i == 0 ? a.rest[d] : P[i * 3 + d] + a.dt_sim * v;
      }
    }
    __syncthreads();
  }
  double* O = a.Xout + b * (int64_t)M * 6;
  bool finite = true;
  for (int t = threadIdx.x; t < M * 3; t += blockDim.x) {
    const int i = t / 3, d = t - 3 * i;
    O[i * 6 + d] = P[t];
    O[i * 6 + 3 + d] = V[t];
    finite = finite && isfinite(P[t]) && isfinite(V[t]);
  }
  if (!finite) atomicExch(a.bad, 1);
}

}  // namespace

extern "C" int gm_trunk_step(gm_ctx* ctx, int B, int M, int nu, int substeps, double dt_sim, double mass,
                             double k, double c, double kb, double rest_len, const double* gravity,
                             const double* rest, const double* fmap, double u_max, int clip, const double* X,
                             const double* U, double* Xout, int32_t* bad, void* stream) {
  int rc = gm_need_device(ctx);
  if (rc) return rc;
  if (B < 0 || M < 2 || nu < 0 || substeps < 1) return gm_fail(ctx, GM_ERR_CONFIG, "bad plant dimensions");
  if (M > 1024) return gm_fail(ctx, GM_ERR_CONFIG, "plant kernel supports up to 1024 nodes");
  if (B == 0) return GM_OK;
  TrunkArgs a{};
  a.B = B;
  a.M = M;
  a.nu = nu;
  a.substeps = substeps;
  a.clip = clip;
  a.dt_sim = dt_sim;
  a.mass = mass;
  a.k = k;
  a.c = c;
  a.kb = kb;
  a.rest_len = rest_len;
  a.u_max = u_max;
  a.g[0] = gravity[0];
  a.g[1] = gravity[1];
  a.g[2] = gravity[2];
  a.rest = rest;
  a.fmap = fmap;
  a.X = X;
  a.U = U;
  a.Xout = Xout;
  a.bad = bad;
  const int threads = ((M + 31) / 32) * 32;
  const size_t smem = sizeof(double) * (6 * (size_t)M + nu);
  k_trunk_step<<<B, threads, smem, (cudaStream_t)stream>>>(a);
  GM_LAUNCH_CHECK(ctx, "k_trunk_step");
  return GM_OK;
}
