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
//
// Both steps are deterministic (no floating-point atomics): group statistics
// are summed by one thread per group in trajectory order, the token partials
// by one CTA in a fixed-order tree.  Out-of-range trajectory / group ids and
// empty groups give NaN (dlogp of the token, and the loss partial), which the
// DiPO step treats as "abort".
#include "abi_common.h"

#include <cmath>

namespace bd {
namespace {

__global__ void group_stats_kernel(int n_traj, const float* __restrict__ rewards, const int32_t* __restrict__ gid,
                                   const int32_t* __restrict__ len, int n_groups, double* __restrict__ stats) {
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= n_groups) return;
  double sr = 0.0, cnt = 0.0, sl = 0.0;
  for (int i = 0; i < n_traj; ++i) {
    if (gid[i] != g) continue;
    sr += (double)rewards[i];
    cnt += 1.0;
    sl += (double)len[i];
  }
  stats[3 * g + 0] += sr;
  stats[3 * g + 1] += cnt;
  stats[3 * g + 2] += sl;
}

struct TokTerm {
  double val, dlogp;
  bool inside, ok;
};

__device__ __forceinline__ TokTerm token_term(int64_t k, const float* logp, const float* logp_old,
                                              const int32_t* traj, int n_traj, const float* rewards,
                                              const int32_t* gid, int n_groups, const double* stats,
                                              int n_groups_global, float eps) {
  TokTerm t{0.0, 0.0, true, false};
  const int i = traj[k];
  if (i < 0 || i >= n_traj) return t;
  const int g = gid[i];
  if (g < 0 || g >= n_groups) return t;
  const double cnt = stats[3 * g + 1], Ng = stats[3 * g + 2];
  if (!(cnt > 0.0) || !(Ng > 0.0)) return t;
  const double A = (double)rewards[i] - stats[3 * g + 0] / cnt;
  // logp == NULL: behaviour policy = sg(current policy) (Eq. 7), rho == 1
  const double rho = logp ? exp((double)logp[k] - (double)logp_old[k]) : 1.0;
  const double lo = 1.0 - eps, hi = 1.0 + eps;
  const double rc = rho < lo ? lo : (rho > hi ? hi : rho);
  const double un = rho * A, cl = rc * A;
  t.inside = rho > lo && rho < hi;
  const double dc = un <= cl ? A : (t.inside ? A : 0.0);
  const double norm = 1.0 / (Ng * (double)n_groups_global);
  t.val = -(un <= cl ? un : cl) * norm;
  t.dlogp = -rho * dc * norm;
  t.inside = t.inside || rho == 1.0;
  t.ok = true;
  return t;
}

__global__ void __launch_bounds__(256) token_grad_kernel(int64_t n, const float* __restrict__ logp,
                                                         const float* __restrict__ logp_old,
                                                         const int32_t* __restrict__ traj, int n_traj,
                                                         const float* __restrict__ rewards,
                                                         const int32_t* __restrict__ gid, int n_groups,
                                                         const double* __restrict__ stats, int n_groups_global,
                                                         float eps, float* __restrict__ dlogp) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
    const TokTerm t = token_term(k, logp, logp_old, traj, n_traj, rewards, gid, n_groups, stats, n_groups_global, eps);
    dlogp[k] = t.ok ? (float)t.dlogp : __int_as_float(0x7fc00000);
  }
}

// One CTA, fixed order: thread t sums tokens t, t + 1024, ...; then a shared
// tree.  partials += (loss, tokens, clipped); NaN loss if any token is invalid.
constexpr int kRedThreads = 1024;
__global__ void __launch_bounds__(kRedThreads) token_loss_reduce_kernel(
    int64_t n, const float* __restrict__ logp, const float* __restrict__ logp_old, const int32_t* __restrict__ traj,
    int n_traj, const float* __restrict__ rewards, const int32_t* __restrict__ gid, int n_groups,
    const double* __restrict__ stats, int n_groups_global, float eps, double* __restrict__ partials) {
  __shared__ double sh[3][kRedThreads];
  double loss = 0.0, toks = 0.0, clipped = 0.0;
  for (int64_t k = threadIdx.x; k < n; k += kRedThreads) {
    const TokTerm t = token_term(k, logp, logp_old, traj, n_traj, rewards, gid, n_groups, stats, n_groups_global, eps);
    loss += t.ok ? t.val : (double)NAN;
    toks += 1.0;
    clipped += t.inside ? 0.0 : 1.0;
  }
  sh[0][threadIdx.x] = loss;
  sh[1][threadIdx.x] = toks;
  sh[2][threadIdx.x] = clipped;
  __syncthreads();
  for (int s = kRedThreads / 2; s > 0; s >>= 1) {
    if ((int)threadIdx.x < s)
      for (int c = 0; c < 3; ++c) sh[c][threadIdx.x] += sh[c][threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x < 3) partials[threadIdx.x] += sh[threadIdx.x][0];
}

}  // namespace
}  // namespace bd

extern "C" int bd_dipo_group_stats(int32_t n_traj, const float* rewards, const int32_t* group_of_traj,
                                   const int32_t* traj_len, int32_t n_groups, double* group_stats, void* stream_) {
  using namespace bd;
  if (n_traj < 0 || n_groups <= 0) return set_error(BD_ERR_INVALID_ARG, "bad sizes");
  if (n_traj == 0) return BD_OK;
  if (!rewards || !group_of_traj || !traj_len || !group_stats) return set_error(BD_ERR_INVALID_ARG, "null pointer");
  const int blocks = (n_groups + 127) / 128;
  group_stats_kernel<<<blocks, 128, 0, static_cast<cudaStream_t>(stream_)>>>(n_traj, rewards, group_of_traj,
                                                                             traj_len, n_groups, group_stats);
  note_launches(1);
  return check_cuda(cudaGetLastError(), "group_stats_kernel launch");
}

extern "C" int bd_dipo_token_loss(int64_t n_tokens, const float* logp, const float* logp_old,
                                  const int32_t* traj_of_token, int32_t n_traj, const float* rewards,
                                  const int32_t* group_of_traj, const double* group_stats, int32_t n_groups,
                                  int32_t n_groups_global, float eps, float* dlogp, double* partials,
                                  void* stream_) {
  using namespace bd;
  if (n_tokens < 0 || n_traj < 0 || n_groups <= 0 || n_groups_global <= 0 || !(eps >= 0.f))
    return set_error(BD_ERR_INVALID_ARG, "bad sizes");
  if (n_tokens == 0) return BD_OK;
  if ((!logp) != (!logp_old) || !traj_of_token || !rewards || !group_of_traj || !group_stats || !dlogp || !partials)
    return set_error(BD_ERR_INVALID_ARG, "null pointer");
  cudaStream_t stream = static_cast<cudaStream_t>(stream_);
  long long blocks = (n_tokens + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  token_grad_kernel<<<(unsigned)blocks, 256, 0, stream>>>(n_tokens, logp, logp_old, traj_of_token, n_traj, rewards,
                                                          group_of_traj, n_groups, group_stats, n_groups_global, eps,
                                                          dlogp);
  token_loss_reduce_kernel<<<1, kRedThreads, 0, stream>>>(n_tokens, logp, logp_old, traj_of_token, n_traj, rewards,
                                                          group_of_traj, n_groups, group_stats, n_groups_global, eps,
                                                          partials);
  note_launches(2);
  return check_cuda(cudaGetLastError(), "token_loss kernels launch");
}
