// rollout_crypto.cu -- fused crypto Q-network rollout (BASELINE configs[3]).
// Per step and env: observation [h, tau/max_hold, f_1..f_101] (reading R24) ->
// Q = MLP(q(obs)) on tcgen05 with the 60 KB Q-net resident in shared memory ->
// argmax (lowest index on ties) with epsilon-greedy exploration ->
// a in {-1, 0, 1} -> LOB-walk execution, reward, done / reset (env_crypto.cuh) ->
// online episode metrics.
#include <cuda_bf16.h>

#include "env_crypto.cuh"
#include "philox.cuh"
#include "rollout_tc.cuh"

namespace {

using tc::TcParams;

struct CryptoOps {
  static constexpr int IN = 2 + FIN_C_FACTORS;  // 103
  struct State {
    bool live;
    double b;
    int h, tau, t_ep;
    int act;
    MetricAcc m;
    AggAcc agg;
    int cnt;
    double rsum;
    bool bad, nonfinite;
  };

  __device__ __forceinline__ static void init(State& st, const TcParams& p, int env, int row) {
    const EnvDev& e = p.e;
    st.live = env < e.N;
    st.cnt = 0;
    st.rsum = 0.0;
    st.bad = st.nonfinite = false;
    st.act = 0;
    agg_init(st.agg);
    if (st.live) {
      st.b = e.cash[env];
      st.h = e.hold[env];
      st.tau = e.tau[env];
      st.t_ep = e.t_ep[env];
      st.m.v0 = e.m_v0[env]; st.m.vprev = e.m_vprev[env]; st.m.peak = e.m_peak[env]; st.m.mdd = e.m_mdd[env];
      st.m.mean = e.m_mean[env]; st.m.m2 = e.m_m2[env]; st.m.n = e.m_n[env];
    } else {
      st.b = 0.0; st.h = 0; st.tau = 0; st.t_ep = 0;
      metric_start(st.m, 0.0);
    }
  }

  __device__ __forceinline__ static uint32_t obs_bits(int idx, const State& st, const float* row, float inv_hold_den) {
    float v;
    if (idx == 0) v = (float)st.h;
    else if (idx == 1) v = __fdiv_rn((float)st.tau, inv_hold_den);
    else if (idx < IN) v = __ldg(row + FIN_C_F0 + (idx - 2));
    else v = 0.f;
    return (uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(v));
  }

  __device__ __forceinline__ static void build_obs(State& st, const TcParams& p, int env, int row, int t,
                                                   uint32_t xa) {
    constexpr int KT8 = PlanCrypto::kIn / 8;
    const EnvDev& e = p.e;
    if (!st.live) {
#pragma unroll
      for (int c = 0; c < KT8; ++c) sm100::st_shared_v4(xa + tc::cm_off(row, c, KT8), 0u, 0u, 0u, 0u);
      return;
    }
    int tr = st.t_ep;
    if (tr + 1 >= e.rows) { st.bad = true; tr = 0; }
    const float* mrow = e.market + (size_t)tr * FIN_C_ROW;
    const float den = (float)e.max_hold;
#pragma unroll
    for (int c = 0; c < KT8; ++c) {
      uint32_t w4[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int i0 = 8 * c + 2 * j;
        w4[j] = obs_bits(i0, st, mrow, den) | (obs_bits(i0 + 1, st, mrow, den) << 16);
      }
      sm100::st_shared_v4(xa + tc::cm_off(row, c, KT8), w4[0], w4[1], w4[2], w4[3]);
    }
  }

  __device__ __forceinline__ static uint16_t* hidden_ptr(State& st, const TcParams& p, int env, int t, int m, int l,
                                                         int hid) {
    if (!st.live || !p.o.mlp_hidden) return nullptr;
    return p.o.mlp_hidden + (((size_t)t * p.e.N + env) * 2 + l) * hid;
  }

  __device__ __forceinline__ static void consume(State& st, const TcParams& p, int env, int t, int m, const float* z) {
    if (!st.live) return;
    const EnvDev& e = p.e;
    if (p.o.mlp_out) {
      float* dst = p.o.mlp_out + ((size_t)t * e.N + env) * 3;
      dst[0] = z[0]; dst[1] = z[1]; dst[2] = z[2];
    }
    int best = 0;
    if (z[1] > z[best]) best = 1;
    if (z[2] > z[best]) best = 2;
    if (!(isfinite(z[0]) && isfinite(z[1]) && isfinite(z[2]))) { st.nonfinite = true; best = 1; }
    float u0 = 1.f, u1 = 0.f;
    if (p.noise_mode == FIN_NOISE_SUPPLIED) {
      const float* nz = p.noise + ((size_t)t * e.N + env) * 2;
      u0 = __ldg(nz); u1 = __ldg(nz + 1);
    } else if (p.noise_mode == FIN_NOISE_PHILOX) {
      float u[2];
      philox_uniform2((uint64_t)(e.env_offset + env), (uint32_t)(e.t_global + t), p.noise_seed, u);
      u0 = u[0]; u1 = u[1];
    }
    if (u0 < e.eps) best = min((int)((double)u1 * 3.0), 2);   // exact product, as the oracle
    st.act = best - 1;
  }

  __device__ __forceinline__ static void finish_step(State& st, const TcParams& p, int env, int t) {
    if (!st.live) return;
    const EnvDev& e = p.e;
    const size_t ti = (size_t)t * e.N + env;
    if (st.t_ep >= e.L || st.t_ep + 1 >= e.rows) {
      st.bad = true;
      if (p.o.reward) p.o.reward[ti] = 0.f;
      if (p.o.done) p.o.done[ti] = 1;
      return;
    }
    const float* row = e.market + (size_t)st.t_ep * FIN_C_ROW;
    double v, vn;
    int delta;
    crypto_transition(e, st.b, st.h, st.tau, row, row + FIN_C_ROW, st.act, v, vn, delta);
    st.t_ep += 1;
    const bool done = st.t_ep == e.L;
    const float r = (float)fmul64(fsub64(vn, v), e.scale);
    st.rsum += (double)r;
    if (p.o.reward) p.o.reward[ti] = r;
    if (p.o.done) p.o.done[ti] = done ? 1 : 0;
    if (p.o.cash) p.o.cash[ti] = st.b;
    if (p.o.asset) p.o.asset[ti] = vn;
    if (p.o.actions) p.o.actions[ti] = (int16_t)st.act;
    if (p.o.hold) p.o.hold[ti] = (int16_t)st.h;
    metric_push(st.m, vn);
    if (done) {
      double em[3];
      metric_finish(st.m, 252.0, 0.0, em);
      if (p.o.ep_metrics && st.cnt < p.o.ep_capacity) {
        double* dst = p.o.ep_metrics + ((size_t)st.cnt * e.N + env) * 3;
        dst[0] = em[0]; dst[1] = em[1]; dst[2] = em[2];
      }
      ++st.cnt;
      agg_episode(st.agg, em);
      if (e.autoreset) {
        st.b = e.cash0; st.h = 0; st.tau = 0; st.t_ep = 0;
        metric_start(st.m, e.cash0);
      }
    }
  }

  __device__ __forceinline__ static void finalize(State& st, const TcParams& p, int env) {
    const EnvDev& e = p.e;
    if (st.live) {
      e.cash[env] = st.b;
      e.hold[env] = (int16_t)st.h;
      e.tau[env] = st.tau;
      e.t_ep[env] = st.t_ep;
      e.m_v0[env] = st.m.v0; e.m_vprev[env] = st.m.vprev; e.m_peak[env] = st.m.peak; e.m_mdd[env] = st.m.mdd;
      e.m_mean[env] = st.m.mean; e.m_m2[env] = st.m.m2; e.m_n[env] = st.m.n;
      if (p.o.ep_count) p.o.ep_count[env] = st.cnt;
      if (st.bad) set_flag(e, FIN_FLAG_BAD_INDEX);
      if (st.nonfinite) set_flag(e, FIN_FLAG_NONFINITE);
    }
    st.agg.s[FIN_AGG_SUM_REWARD] = st.rsum;
    if (p.o.agg_partial) agg_group_write(st.agg, p.o.agg_partial + (size_t)blockIdx.x * FIN_AGG_LEN,
                                         threadIdx.x - tc::kEnvWarp0 * 32, 1);
  }
};

}  // namespace

namespace fin {

cudaError_t launch_crypto_rollout(const tc::TcParams& p, int n_tiles, cudaStream_t s) {
  using S = tc::Smem<PlanCrypto, true>;
  auto kern = tc::k_tc_rollout<PlanCrypto, true, CryptoOps>;
  cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, S::kTotal);
  if (err != cudaSuccess) return err;
  kern<<<n_tiles, tc::kThreads, S::kTotal, s>>>(p);
  return cudaGetLastError();
}

}  // namespace fin
