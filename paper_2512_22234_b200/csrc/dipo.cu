// DiPO token-level objective at the stop-gradient behaviour policy.
//   A_i = r_i - mean_{j in g(i)} r_j
//   rho_k = exp(logp_k - logp_old_k)                          (Eq. 7: pi_old = sg(pi_theta))
//   C_eps(rho, A) = min(rho A, clip(rho, 1-eps, 1+eps) A)
//   loss = -(1/n_groups) sum_g (1/N_g) sum_{k in g} C_eps(rho_k, A_{i(k)})   (Eq. 8, P:206-225;
//          N_g = token count of the group, readings c10/c11)
// Step 1 accumulates per-group (sum r, count, sum |tau|) so that a caller can
// all-reduce them when a group straddles ranks; step 2 produces dloss/dlogp
// per token and the (loss, tokens, clipped) partial sums that the caller
// all-reduces over NCCL -- the only cross-GPU exchange of the hot path.
#include "abi_common.h"

namespace bd {
namespace {

__global__ void group_stats_kernel(int n_traj, const float* __restrict__ rewards, const int32_t* __restrict__ gid,
                                   const int32_t* __restrict__ len, int n_groups, double* __restrict__ stats) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n_traj; i += gridDim.x * blockDim.x) {
    const int g = gid[i];
    if (g < 0 || g >= n_groups) continue;
    atomicAdd(&stats[3 * g + 0], (double)rewards[i]);
    atomicAdd(&stats[3 * g + 1], 1.0);
    atomicAdd(&stats[3 * g + 2], (double)len[i]);
  }
}

__global__ void __launch_bounds__(256) token_loss_kernel(int64_t n, const float* __restrict__ logp,
                                                         const float* __restrict__ logp_old,
                                                         const int32_t* __restrict__ traj,
                                                         const float* __restrict__ rewards,
                                                         const int32_t* __restrict__ gid,
                                                         const double* __restrict__ stats, int n_groups_global,
                                                         float eps, float* __restrict__ dlogp,
                                                         double* __restrict__ partials) {
  double loss = 0.0, toks = 0.0, clipped = 0.0;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
    const int i = traj[k];
    const int g = gid[i];
    const double mean_r = stats[3 * g + 0] / stats[3 * g + 1];
    const double A = (double)rewards[i] - mean_r;
    const double Ng = stats[3 * g + 2];
    // logp == NULL: behaviour policy = sg(current policy) (Eq. 7), rho == 1
    const double rho = logp ? exp((double)logp[k] - (double)logp_old[k]) : 1.0;
    const double lo = 1.0 - eps, hi = 1.0 + eps;
    const double rc = rho < lo ? lo : (rho > hi ? hi : rho);
    const double un = rho * A, cl = rc * A;
    const double val = un <= cl ? un : cl;
    const bool inside = rho > lo && rho < hi;
    const double dc = un <= cl ? A : (inside ? A : 0.0);
    const double norm = 1.0 / (Ng * (double)n_groups_global);
    dlogp[k] = (float)(-rho * dc * norm);
    loss -= val * norm;
    toks += 1.0;
    clipped += (!inside && rho != 1.0) ? 1.0 : 0.0;
  }
  // block reduction then one fp64 atomic per block per partial
  __shared__ double sh[3][8];
  for (int off = 16; off; off >>= 1) {
    loss += __shfl_xor_sync(0xffffffffu, loss, off);
    toks += __shfl_xor_sync(0xffffffffu, toks, off);
    clipped += __shfl_xor_sync(0xffffffffu, clipped, off);
  }
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) {
    sh[0][w] = loss;
    sh[1][w] = toks;
    sh[2][w] = clipped;
  }
  __syncthreads();
  if (threadIdx.x < 3) {
    double acc = 0.0;
    for (int j = 0; j < (int)(blockDim.x >> 5); ++j) acc += sh[threadIdx.x][j];
    atomicAdd(&partials[threadIdx.x], acc);
  }
}

}  // namespace
}  // namespace bd

extern "C" int bd_dipo_group_stats(int32_t n_traj, const float* rewards, const int32_t* group_of_traj,
                                   const int32_t* traj_len, int32_t n_groups, double* group_stats, void* stream_) {
  using namespace bd;
  if (n_traj < 0 || n_groups <= 0) return set_error(BD_ERR_INVALID_ARG, "bad sizes");
  if (n_traj == 0) return BD_OK;
  if (!rewards || !group_of_traj || !traj_len || !group_stats) return set_error(BD_ERR_INVALID_ARG, "null pointer");
  const int blocks = (n_traj + 255) / 256;
  group_stats_kernel<<<blocks, 256, 0, static_cast<cudaStream_t>(stream_)>>>(n_traj, rewards, group_of_traj,
                                                                             traj_len, n_groups, group_stats);
  note_launches(1);
  return check_cuda(cudaGetLastError(), "group_stats_kernel launch");
}

extern "C" int bd_dipo_token_loss(int64_t n_tokens, const float* logp, const float* logp_old,
                                  const int32_t* traj_of_token, const float* rewards, const int32_t* group_of_traj,
                                  const double* group_stats, int32_t n_groups_global, float eps, float* dlogp,
                                  double* partials, void* stream_) {
  using namespace bd;
  if (n_tokens < 0 || n_groups_global <= 0 || !(eps >= 0.f)) return set_error(BD_ERR_INVALID_ARG, "bad sizes");
  if (n_tokens == 0) return BD_OK;
  if ((!logp) != (!logp_old) || !traj_of_token || !rewards || !group_of_traj || !group_stats || !dlogp || !partials)
    return set_error(BD_ERR_INVALID_ARG, "null pointer");
  long long blocks = (n_tokens + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  token_loss_kernel<<<(unsigned)blocks, 256, 0, static_cast<cudaStream_t>(stream_)>>>(
      n_tokens, logp, logp_old, traj_of_token, rewards, group_of_traj, group_stats, n_groups_global, eps, dlogp,
      partials);
  note_launches(1);
  return check_cuda(cudaGetLastError(), "token_loss_kernel launch");
}
