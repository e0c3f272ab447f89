// env_crypto.cu -- crypto VecEnv kernels: reset, single step (K2), state get/set.
// All envs of the lockstep C3 workload read the same LOB row; a block stages the
// two rows it needs in shared memory when its envs agree on the row (the common
// case), otherwise threads read their rows through L1.
#include "env_crypto.cuh"

namespace {

constexpr int kThreads = 256;

__global__ void k_crypto_reset(EnvDev e, const uint8_t* __restrict__ mask) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= e.N) return;
  if (mask && !mask[i]) return;
  e.cash[i] = e.cash0;
  e.hold[i] = 0;
  e.tau[i] = 0;
  e.t_ep[i] = 0;
  e.window[i] = 0;
  e.m_v0[i] = e.cash0; e.m_vprev[i] = e.cash0; e.m_peak[i] = e.cash0; e.m_mdd[i] = 0.0;
  e.m_mean[i] = 0.0; e.m_m2[i] = 0.0; e.m_n[i] = 0;
}

__global__ void __launch_bounds__(kThreads) k_crypto_step(EnvDev e, const int16_t* __restrict__ actions, TrajDev o) {
  __shared__ __align__(16) float rows_s[2 * FIN_C_ROW];
  __shared__ int t_first;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const bool live = i < e.N;
  int t = live ? e.t_ep[i] : 0;
  if (threadIdx.x == 0) t_first = t;
  __syncthreads();
  const bool uniform = __syncthreads_and(!live || t == t_first);
  const int tb = t_first;
  if (uniform && tb + 1 < e.rows) {
    for (int j = threadIdx.x; j < 2 * FIN_C_ROW; j += blockDim.x) rows_s[j] = e.market[(size_t)tb * FIN_C_ROW + j];
  }
  __syncthreads();
  if (!live) return;
  if (t >= e.L) {
    set_flag(e, FIN_FLAG_EPISODE_DONE);
    if (o.reward) o.reward[i] = 0.f;
    if (o.done) o.done[i] = 1;
    return;
  }
  if (t + 1 >= e.rows) { set_flag(e, FIN_FLAG_BAD_INDEX); return; }
  const float* row = (uniform ? rows_s : e.market + (size_t)t * FIN_C_ROW);
  const float* rown = row + FIN_C_ROW;
  double b = e.cash[i];
  int h = e.hold[i], tau = e.tau[i];
  int a = actions[i];
  if (a > 1 || a < -1) { set_flag(e, FIN_FLAG_ACTION_RANGE); a = a > 1 ? 1 : -1; }
  double v, vn;
  int delta;
  crypto_transition(e, b, h, tau, row, rown, a, v, vn, delta);
  t += 1;
  const bool done = t == e.L;
  if (o.reward) o.reward[i] = (float)fmul64(fsub64(vn, v), e.scale);
  if (o.done) o.done[i] = done;
  if (o.cash) o.cash[i] = b;
  if (o.asset) o.asset[i] = vn;
  if (o.hold) o.hold[i] = (int16_t)h;
  if (o.actions) o.actions[i] = (int16_t)delta;
  if (done && e.autoreset) { b = e.cash0; h = 0; tau = 0; t = 0; }
  e.cash[i] = b;
  e.hold[i] = (int16_t)h;
  e.tau[i] = tau;
  e.t_ep[i] = t;
}

__global__ void k_crypto_get_state(EnvDev e, double* cash, int16_t* hold, double* asset, int32_t* t_ep) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= e.N) return;
  double b = e.cash[i];
  int t = e.t_ep[i];
  if (cash) cash[i] = b;
  if (hold) hold[i] = e.hold[i];
  if (t_ep) t_ep[i] = t;
  if (asset) {
    if (t >= e.rows) t = e.rows - 1;
    asset[i] = fadd64(b, fmul64((double)e.hold[i], (double)e.market[(size_t)t * FIN_C_ROW + FIN_C_MID]));
  }
}

__global__ void k_crypto_set_state(EnvDev e, const double* cash, const int16_t* hold, const int32_t* t_ep,
                                   const int32_t* tau) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= e.N) return;
  if (cash) e.cash[i] = cash[i];
  if (hold) e.hold[i] = hold[i];
  if (t_ep) e.t_ep[i] = t_ep[i];
  e.tau[i] = tau ? tau[i] : 0;
  int t = e.t_ep[i];
  if (t >= e.rows) t = e.rows - 1;
  double v = fadd64(e.cash[i], fmul64((double)e.hold[i], (double)e.market[(size_t)t * FIN_C_ROW + FIN_C_MID]));
  e.m_v0[i] = v; e.m_vprev[i] = v; e.m_peak[i] = v; e.m_mdd[i] = 0.0;
  e.m_mean[i] = 0.0; e.m_m2[i] = 0.0; e.m_n[i] = 0;
}

inline int blocks_for(int n) { return (n + kThreads - 1) / kThreads; }

}  // namespace

namespace fin {

cudaError_t launch_crypto_reset(const EnvDev& e, const uint8_t* mask, cudaStream_t s) {
  k_crypto_reset<<<blocks_for(e.N), kThreads, 0, s>>>(e, mask);
  return cudaGetLastError();
}
cudaError_t launch_crypto_step(const EnvDev& e, const int16_t* actions, const TrajDev& o, cudaStream_t s) {
  k_crypto_step<<<blocks_for(e.N), kThreads, 0, s>>>(e, actions, o);
  return cudaGetLastError();
}
cudaError_t launch_crypto_get_state(const EnvDev& e, double* cash, int16_t* hold, double* asset, int32_t* t_ep,
                                    cudaStream_t s) {
  k_crypto_get_state<<<blocks_for(e.N), kThreads, 0, s>>>(e, cash, hold, asset, t_ep);
  return cudaGetLastError();
}
cudaError_t launch_crypto_set_state(const EnvDev& e, const double* cash, const int16_t* hold, const int32_t* t_ep,
                                    const int32_t* tau, cudaStream_t s) {
  k_crypto_set_state<<<blocks_for(e.N), kThreads, 0, s>>>(e, cash, hold, t_ep, tau);
  return cudaGetLastError();
}

}  // namespace fin
