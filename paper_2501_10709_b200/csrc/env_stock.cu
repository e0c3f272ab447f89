// env_stock.cu -- stock VecEnv kernels: reset, single step (K1), replay rollout
// (K4), state get/set.  PAPER.md §4.2: reset / step / reward over
// all SubEnvs; the paper vmaps them in PyTorch on an A100, here each is
// one hand-written sm_100a kernel over the SoA state.
#include "env_stock.cuh"

namespace {

constexpr int kThreads = 256;

__device__ __forceinline__ MetricAcc load_metric(const EnvDev& e, int i) {
  MetricAcc m;
  m.v0 = e.m_v0[i]; m.vprev = e.m_vprev[i]; m.peak = e.m_peak[i]; m.mdd = e.m_mdd[i];
  m.mean = e.m_mean[i]; m.m2 = e.m_m2[i]; m.n = e.m_n[i];
  return m;
}
__device__ __forceinline__ void store_metric(const EnvDev& e, int i, const MetricAcc& m) {
  e.m_v0[i] = m.v0; e.m_vprev[i] = m.vprev; e.m_peak[i] = m.peak; e.m_mdd[i] = m.mdd;
  e.m_mean[i] = m.mean; e.m_m2[i] = m.m2; e.m_n[i] = m.n;
}

__global__ void k_stock_reset(EnvDev e, const uint8_t* __restrict__ mask) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= e.N) return;
  if (mask && !mask[i]) return;
  e.cash[i] = e.cash0;
  for (int k = 0; k < e.K; ++k) e.hold[(size_t)k * e.N + i] = 0;
  e.t_ep[i] = 0;
  e.window[i] = window_of(e, e.env_offset + i);
  for (int m = 0; m < FIN_MAX_MEMBERS; ++m)
    for (int k = 0; k < e.K; ++k) e.ou[((size_t)m * e.K + k) * e.N + i] = 0.f;
  MetricAcc a;
  metric_start(a, e.cash0);
  store_metric(e, i, a);
}

// K1: one step of every env with supplied actions [N][K].  One env per thread;
// state SoA loads are coalesced; the two market rows are read through L1 (the
// whole C1 market is 1.2 MB and stays L2-resident; envs of a warp share a row).
template <int KP>
__global__ void __launch_bounds__(kThreads) k_stock_step(EnvDev e, const int16_t* __restrict__ actions, TrajDev o) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= e.N) return;
  const int K = e.K, N = e.N;
  int t = e.t_ep[i];
  const int w = e.window[i];
  double b = e.cash[i];
  int h[KP], a[KP], ex[KP];
#pragma unroll
  for (int k = 0; k < KP; ++k) {
    h[k] = (k < K) ? (int)e.hold[(size_t)k * N + i] : 0;
    a[k] = (k < K) ? (int)actions[(size_t)i * K + k] : 0;
  }
  if (t >= e.L) {  // done env, autoreset = 0: ignored
    set_flag(e, FIN_FLAG_EPISODE_DONE);
    if (o.reward) o.reward[i] = 0.f;
    if (o.done) o.done[i] = 1;
    return;
  }
  const int d = day_of(e, w, t);
  if (d < 0 || d + 1 >= e.rows) {
    set_flag(e, FIN_FLAG_BAD_INDEX);
    return;
  }
  const float* p = e.market + (size_t)d * e.row_floats;  // channel 0 = close
  const float* pn = p + e.row_floats;
  double v, vn;
  bool oor = false;
  stock_transition<KP>(e, b, h, p, pn, a, v, vn, ex, oor);
  if (oor) set_flag(e, FIN_FLAG_ACTION_RANGE);
  t += 1;
  const bool done = (t == e.L);
  if (o.reward) o.reward[i] = stock_reward(e, v, vn);
  if (o.done) o.done[i] = done ? 1 : 0;
  if (o.cash) o.cash[i] = b;
  if (o.asset) o.asset[i] = vn;
#pragma unroll
  for (int k = 0; k < KP; ++k) {
    if (k < K) {
      if (o.hold) o.hold[(size_t)i * K + k] = (int16_t)h[k];
      if (o.actions) o.actions[(size_t)i * K + k] = (int16_t)ex[k];
    }
  }
  if (done && e.autoreset) {
    b = e.cash0;
#pragma unroll
    for (int k = 0; k < KP; ++k) h[k] = 0;
    t = 0;
    if (e.wadv) e.window[i] = (w + 1) % e.W;
  }
  e.cash[i] = b;
#pragma unroll
  for (int k = 0; k < KP; ++k)
    if (k < K) e.hold[(size_t)k * N + i] = (int16_t)h[k];
  e.t_ep[i] = t;
}

// K4: T steps with supplied actions [T][N][K]; the env state (cash, holdings,
// episode clock, window, metric accumulators) lives in registers for all T.
template <int KP>
__global__ void __launch_bounds__(kThreads) k_stock_replay(EnvDev e, const int16_t* __restrict__ actions, int T,
                                                           TrajDev o) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const bool live = i < e.N;
  const int K = e.K, N = e.N;
  AggAcc agg;
  agg_init(agg);
  if (live) {
    int t = e.t_ep[i];
    int w = e.window[i];
    double b = e.cash[i];
    int h[KP], a[KP], ex[KP];
#pragma unroll
    for (int k = 0; k < KP; ++k) h[k] = (k < K) ? (int)e.hold[(size_t)k * N + i] : 0;
    MetricAcc m = load_metric(e, i);
    int cnt = 0;
    double rsum = 0.0;
    bool oor = false, bad = false;
    for (int s = 0; s < T; ++s) {
      const int16_t* ar = actions + ((size_t)s * N + i) * K;
#pragma unroll
      for (int k = 0; k < KP; ++k) a[k] = (k < K) ? (int)ar[k] : 0;
      const size_t ti = (size_t)s * N + i;
      if (t >= e.L) {
        set_flag(e, FIN_FLAG_EPISODE_DONE);
        if (o.reward) o.reward[ti] = 0.f;
        if (o.done) o.done[ti] = 1;
        continue;
      }
      const int d = day_of(e, w, t);
      if (d < 0 || d + 1 >= e.rows) { bad = true; break; }
      const float* p = e.market + (size_t)d * e.row_floats;
      double v, vn;
      stock_transition<KP>(e, b, h, p, p + e.row_floats, a, v, vn, ex, oor);
      t += 1;
      const bool done = (t == e.L);
      const float r = stock_reward(e, v, vn);
      rsum += (double)r;
      if (o.reward) o.reward[ti] = r;
      if (o.done) o.done[ti] = done ? 1 : 0;
      if (o.cash) o.cash[ti] = b;
      if (o.asset) o.asset[ti] = vn;
      if (o.hold || o.actions) {
#pragma unroll
        for (int k = 0; k < KP; ++k) {
          if (k < K) {
            if (o.hold) o.hold[ti * K + k] = (int16_t)h[k];
            if (o.actions) o.actions[ti * K + k] = (int16_t)ex[k];
          }
        }
      }
      metric_push(m, vn);
      if (done) {
        double em[3];
        metric_finish(m, 252.0, 0.0, em);
        if (o.ep_metrics && cnt < o.ep_capacity) {
          double* dst = o.ep_metrics + ((size_t)cnt * N + i) * 3;
          dst[0] = em[0]; dst[1] = em[1]; dst[2] = em[2];
        }
        ++cnt;
        agg_episode(agg, em);
        if (e.autoreset) {
          b = e.cash0;
#pragma unroll
          for (int k = 0; k < KP; ++k) h[k] = 0;
          t = 0;
          if (e.wadv) w = (w + 1) % e.W;
          metric_start(m, e.cash0);
        }
      }
    }
    if (oor) set_flag(e, FIN_FLAG_ACTION_RANGE);
    if (bad) set_flag(e, FIN_FLAG_BAD_INDEX);
    agg.s[FIN_AGG_SUM_REWARD] = rsum;
    e.cash[i] = b;
#pragma unroll
    for (int k = 0; k < KP; ++k)
      if (k < K) e.hold[(size_t)k * N + i] = (int16_t)h[k];
    e.t_ep[i] = t;
    e.window[i] = w;
    store_metric(e, i, m);
    if (o.ep_count) o.ep_count[i] = cnt;
  }
  if (o.agg_partial) agg_block_write(agg, o.agg_partial + (size_t)blockIdx.x * FIN_AGG_LEN);
}

__global__ void k_stock_get_state(EnvDev e, double* cash, int16_t* hold, double* asset, int32_t* t_ep,
                                  int32_t* window) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= e.N) return;
  const int K = e.K;
  double b = e.cash[i];
  if (cash) cash[i] = b;
  if (t_ep) t_ep[i] = e.t_ep[i];
  if (window) window[i] = e.window[i];
  if (hold)
    for (int k = 0; k < K; ++k) hold[(size_t)i * K + k] = e.hold[(size_t)k * e.N + i];
  if (asset) {
    int t = e.t_ep[i];
    int d = day_of(e, e.window[i], t);
    if (d >= e.rows) d = e.rows - 1;
    const float* p = e.market + (size_t)d * e.row_floats;
    double v = b;
    for (int k = 0; k < K; ++k) v = fadd64(v, fmul64((double)e.hold[(size_t)k * e.N + i], (double)p[k]));
    asset[i] = v;
  }
}

__global__ void k_stock_set_state(EnvDev e, const double* cash, const int16_t* hold, const int32_t* t_ep,
                                  const int32_t* window) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= e.N) return;
  const int K = e.K;
  if (cash) e.cash[i] = cash[i];
  if (hold)
    for (int k = 0; k < K; ++k) e.hold[(size_t)k * e.N + i] = hold[(size_t)i * K + k];
  if (t_ep) e.t_ep[i] = t_ep[i];
  if (window) e.window[i] = window[i];
  // online metrics restart at the current equity
  int d = day_of(e, e.window[i], e.t_ep[i]);
  if (d >= e.rows) d = e.rows - 1;
  const float* p = e.market + (size_t)d * e.row_floats;
  double v = e.cash[i];
  for (int k = 0; k < K; ++k) v = fadd64(v, fmul64((double)e.hold[(size_t)k * e.N + i], (double)p[k]));
  MetricAcc m;
  metric_start(m, v);
  store_metric(e, i, m);
}

__global__ void k_agg_finalize(const double* __restrict__ partial, int n_blocks, double* agg) {
  const int j = threadIdx.x;
  if (j >= FIN_AGG_LEN) return;
  double s = (j < FIN_AGG_NSUM) ? 0.0 : __longlong_as_double(0x7ff0000000000000ULL);
  for (int b = 0; b < n_blocks; ++b) {
    double x = partial[(size_t)b * FIN_AGG_LEN + j];
    s = (j < FIN_AGG_NSUM) ? s + x : fmin(s, x);
  }
  agg[j] = s;
}

inline int blocks_for(int n) { return (n + kThreads - 1) / kThreads; }

}  // namespace

namespace fin {

#define FIN_DISPATCH_KP(K, KERNEL, GRID, BLOCK, STREAM, ...)                    \
  do {                                                                          \
    if ((K) <= 4) KERNEL<4><<<GRID, BLOCK, 0, STREAM>>>(__VA_ARGS__);           \
    else if ((K) <= 8) KERNEL<8><<<GRID, BLOCK, 0, STREAM>>>(__VA_ARGS__);      \
    else if ((K) <= 16) KERNEL<16><<<GRID, BLOCK, 0, STREAM>>>(__VA_ARGS__);    \
    else KERNEL<32><<<GRID, BLOCK, 0, STREAM>>>(__VA_ARGS__);                   \
  } while (0)

cudaError_t launch_stock_reset(const EnvDev& e, const uint8_t* mask, cudaStream_t s) {
  k_stock_reset<<<blocks_for(e.N), kThreads, 0, s>>>(e, mask);
  return cudaGetLastError();
}

cudaError_t launch_stock_step(const EnvDev& e, const int16_t* actions, const TrajDev& o, cudaStream_t s) {
  FIN_DISPATCH_KP(e.K, k_stock_step, blocks_for(e.N), kThreads, s, e, actions, o);
  return cudaGetLastError();
}

cudaError_t launch_stock_replay(const EnvDev& e, const int16_t* actions, int T, const TrajDev& o, int* n_blocks,
                                cudaStream_t s) {
  *n_blocks = blocks_for(e.N);
  FIN_DISPATCH_KP(e.K, k_stock_replay, blocks_for(e.N), kThreads, s, e, actions, T, o);
  return cudaGetLastError();
}

cudaError_t launch_stock_get_state(const EnvDev& e, double* cash, int16_t* hold, double* asset, int32_t* t_ep,
                                   int32_t* window, cudaStream_t s) {
  k_stock_get_state<<<blocks_for(e.N), kThreads, 0, s>>>(e, cash, hold, asset, t_ep, window);
  return cudaGetLastError();
}

cudaError_t launch_stock_set_state(const EnvDev& e, const double* cash, const int16_t* hold, const int32_t* t_ep,
                                   const int32_t* window, cudaStream_t s) {
  k_stock_set_state<<<blocks_for(e.N), kThreads, 0, s>>>(e, cash, hold, t_ep, window);
  return cudaGetLastError();
}

cudaError_t launch_agg_finalize(const double* partial, int n_blocks, double* agg, cudaStream_t s) {
  k_agg_finalize<<<1, 32, 0, s>>>(partial, n_blocks, agg);
  return cudaGetLastError();
}

}  // namespace fin
