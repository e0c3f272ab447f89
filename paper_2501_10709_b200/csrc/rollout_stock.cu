// rollout_stock.cu -- fused stock policy rollout (K3, with the C2 ensemble K5 inside)
// and the standalone MLP probe (K7), instantiated from rollout_tc.cuh.
//
// Per step and env (thread r of the env warpgroup):
//   observation s_t = [b/b0, close_norm_t, h/max_trade, f_t]  (readings R13, R14)
//   -> per member m: z_m = MLP_m(q(s_t)) on tcgen05 (BASELINE configs[1,2])
//   -> member action (R17, R19): PPO clip(tanh z + std eps), SAC tanh(z + std eps),
//      DDPG OU x <- x + theta(0 - x) + sigma eps, clip(tanh z + x)
//   -> ensemble mean (R20) -> shares = rha(max_trade * abar)  (R18)
//   -> trade, reward, done / reset (env_stock.cuh), online episode metrics.
#include <cuda_bf16.h>

#include "env_stock.cuh"
#include "philox.cuh"
#include "rollout_tc.cuh"

namespace {

using tc::TcParams;

template <int KA, int IA>
struct StockOps {
  static constexpr int KP4 = (KA + 3) / 4 * 4;
  static constexpr int IN = 1 + 2 * KA + IA * KA;

  struct State {
    bool live;
    double b;
    int h[KA];
    int t_ep, w, d;
    float asum[KA];
    float ou[KA];
    MetricAcc m;
    AggAcc agg;
    int cnt;
    double rsum;
    bool oor, bad, nonfinite;
  };

  __device__ __forceinline__ static void init(State& st, const TcParams& p, int env, int row) {
    const EnvDev& e = p.e;
    st.live = env < e.N;
    st.cnt = 0;
    st.rsum = 0.0;
    st.oor = st.bad = st.nonfinite = false;
    agg_init(st.agg);
    if (st.live) {
      st.b = e.cash[env];
#pragma unroll
      for (int k = 0; k < KA; ++k) st.h[k] = e.hold[(size_t)k * e.N + env];
      st.t_ep = e.t_ep[env];
      st.w = e.window[env];
      st.m.v0 = e.m_v0[env]; st.m.vprev = e.m_vprev[env]; st.m.peak = e.m_peak[env]; st.m.mdd = e.m_mdd[env];
      st.m.mean = e.m_mean[env]; st.m.m2 = e.m_m2[env]; st.m.n = e.m_n[env];
      // OU state of the (single) DDPG member, slot = member index
      int slot = -1;
      for (int m = 0; m < p.M; ++m)
        if (p.kinds[m] == FIN_DDPG_OU) slot = m;
#pragma unroll
      for (int k = 0; k < KA; ++k) st.ou[k] = slot >= 0 ? e.ou[((size_t)slot * e.K + k) * e.N + env] : 0.f;
    } else {
      st.b = 0.0;
#pragma unroll
      for (int k = 0; k < KA; ++k) { st.h[k] = 0; st.ou[k] = 0.f; }
      st.t_ep = 0; st.w = 0;
      metric_start(st.m, 0.0);
    }
  }

  // q(x) of one observation element; idx is a compile-time constant after unrolling
  __device__ __forceinline__ static uint32_t obs_bits(int idx, const State& st, const float* mrow, uint32_t b0bits,
                                                      float inv_trade_den) {
    float v;
    if (idx == 0) return b0bits;
    if (idx <= KA) v = __ldg(mrow + KP4 + (idx - 1));                      // close_norm_t[k]
    else if (idx <= 2 * KA) v = __fdiv_rn((float)st.h[idx - KA - 1], inv_trade_den);  // h_k / max_trade
    else if (idx < IN) {
      const int j = idx - (2 * KA + 1);
      v = __ldg(mrow + (2 + j / KA) * KP4 + (j % KA));                     // feature, indicator-major
    } else v = 0.f;
    return (uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(v));
  }

  template <class Plan>
  __device__ __forceinline__ static void build_obs_t(State& st, const TcParams& p, int env, int row, int t,
                                                     uint32_t xa) {
    const EnvDev& e = p.e;
    constexpr int KT8 = Plan::kIn / 8;
    if (!st.live) {
#pragma unroll
      for (int c = 0; c < KT8; ++c) sm100::st_shared_v4(xa + tc::cm_off(row, c, KT8), 0u, 0u, 0u, 0u);
      return;
    }
    st.d = day_of(e, st.w, st.t_ep);
    if (st.d < 0 || st.d + 1 >= e.rows) { st.bad = true; st.d = 0; }
    const float* mrow = e.market + (size_t)st.d * e.row_floats;
    const uint32_t b0 = (uint32_t)__bfloat16_as_ushort(__double2bfloat16(fdiv64(st.b, e.cash0)));
    const float den = (float)e.max_trade;
#pragma unroll
    for (int c = 0; c < KT8; ++c) {
      uint32_t w4[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int i0 = 8 * c + 2 * j;
        w4[j] = obs_bits(i0, st, mrow, b0, den) | (obs_bits(i0 + 1, st, mrow, b0, den) << 16);
      }
      sm100::st_shared_v4(xa + tc::cm_off(row, c, KT8), w4[0], w4[1], w4[2], w4[3]);
    }
#pragma unroll
    for (int k = 0; k < KA; ++k) st.asum[k] = 0.f;
  }

  __device__ __forceinline__ static uint16_t* hidden_ptr(State& st, const TcParams& p, int env, int t, int m, int l,
                                                         int hid) {
    if (!st.live || !p.o.mlp_hidden) return nullptr;
    return p.o.mlp_hidden + ((((size_t)t * p.M + m) * p.e.N + env) * 2 + l) * hid;
  }

  __device__ __forceinline__ static void consume(State& st, const TcParams& p, int env, int t, int m, const float* z) {
    if (!st.live) return;
    const EnvDev& e = p.e;
    const int kind = p.kinds[m];
    float eps[KA];
    if (p.noise_mode == FIN_NOISE_SUPPLIED) {
      const float* nz = p.noise + (((size_t)t * p.M + m) * e.N + env) * KA;
#pragma unroll
      for (int k = 0; k < KA; ++k) eps[k] = __ldg(nz + k);
    } else if (p.noise_mode == FIN_NOISE_PHILOX) {
#pragma unroll
      for (int blk = 0; blk < (KA + 3) / 4; ++blk) {
        float zz[4];
        philox_normals4((uint64_t)(e.env_offset + env), (uint32_t)(e.t_global + t), ((uint32_t)m << 16) | blk,
                        p.noise_seed, zz);
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if (blk * 4 + j < KA) eps[blk * 4 + j] = zz[j];
      }
    } else {
#pragma unroll
      for (int k = 0; k < KA; ++k) eps[k] = 0.f;
    }
    if (p.o.mlp_out) {
      float* dst = p.o.mlp_out + (((size_t)t * p.M + m) * e.N + env) * KA;
#pragma unroll
      for (int k = 0; k < KA; ++k) dst[k] = z[k];
    }
    const float wm = p.weighted ? p.mw[m] : 1.f;
#pragma unroll
    for (int k = 0; k < KA; ++k) {
      float a;
      const float zk = z[k];
      if (kind == FIN_SAC_SQUASH) {
        a = tanhf(__fadd_rn(zk, __fmul_rn(e.noise_std, eps[k])));
      } else if (kind == FIN_DDPG_OU) {
        const float x = __fadd_rn(__fadd_rn(st.ou[k], __fmul_rn(e.ou_theta, __fsub_rn(0.f, st.ou[k]))),
                                  __fmul_rn(e.ou_sigma, eps[k]));
        st.ou[k] = x;
        a = fminf(fmaxf(__fadd_rn(tanhf(zk), x), -1.f), 1.f);
      } else {  // PPO Gaussian (also C1's single policy)
        a = fminf(fmaxf(__fadd_rn(tanhf(zk), __fmul_rn(e.noise_std, eps[k])), -1.f), 1.f);
      }
      if (!isfinite(a)) { st.nonfinite = true; a = 0.f; }
      st.asum[k] = p.weighted ? __fadd_rn(st.asum[k], __fmul_rn(wm, a)) : __fadd_rn(st.asum[k], a);
    }
  }

  __device__ __forceinline__ static void finish_step(State& st, const TcParams& p, int env, int t) {
    if (!st.live) return;
    const EnvDev& e = p.e;
    const size_t ti = (size_t)t * e.N + env;
    if (st.t_ep >= e.L) {  // done env without autoreset
      st.bad = true;
      if (p.o.reward) p.o.reward[ti] = 0.f;
      if (p.o.done) p.o.done[ti] = 1;
      return;
    }
    int a[KA], ex[KA];
#pragma unroll
    for (int k = 0; k < KA; ++k) {
      const float abar = (p.M == 1 || p.weighted) ? st.asum[k] : __fdiv_rn(st.asum[k], (float)p.M);
      a[k] = rha_f32(__fmul_rn((float)e.max_trade, abar));
      if (p.act_only && p.mean_out) p.mean_out[(size_t)env * KA + k] = abar;
    }
    if (p.act_only) {  // fin_ensemble_act: report the action, leave the env untouched
      if (p.o.actions) {
#pragma unroll
        for (int k = 0; k < KA; ++k) p.o.actions[(size_t)env * KA + k] = (int16_t)a[k];
      }
      return;
    }
    const float* mrow = e.market + (size_t)st.d * e.row_floats;
    double v, vn;
    stock_transition<KA>(e, st.b, st.h, mrow, mrow + e.row_floats, a, v, vn, ex, st.oor);
    st.t_ep += 1;
    const bool done = st.t_ep == e.L;
    const float r = stock_reward(e, v, vn);
    st.rsum += (double)r;
    if (p.o.reward) p.o.reward[ti] = r;
    if (p.o.done) p.o.done[ti] = done ? 1 : 0;
    if (p.o.cash) p.o.cash[ti] = st.b;
    if (p.o.asset) p.o.asset[ti] = vn;
    if (p.o.actions || p.o.hold) {
#pragma unroll
      for (int k = 0; k < KA; ++k) {
        if (p.o.actions) p.o.actions[ti * KA + k] = (int16_t)ex[k];
        if (p.o.hold) p.o.hold[ti * KA + k] = (int16_t)st.h[k];
      }
    }
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
        st.b = e.cash0;
#pragma unroll
        for (int k = 0; k < KA; ++k) { st.h[k] = 0; st.ou[k] = 0.f; }
        st.t_ep = 0;
        if (e.wadv) st.w = (st.w + 1) % e.W;
        metric_start(st.m, e.cash0);
      }
    }
  }

  __device__ __forceinline__ static void finalize(State& st, const TcParams& p, int env) {
    const EnvDev& e = p.e;
    if (p.act_only) return;
    if (st.live) {
      e.cash[env] = st.b;
#pragma unroll
      for (int k = 0; k < KA; ++k) e.hold[(size_t)k * e.N + env] = (int16_t)st.h[k];
      e.t_ep[env] = st.t_ep;
      e.window[env] = st.w;
      e.m_v0[env] = st.m.v0; e.m_vprev[env] = st.m.vprev; e.m_peak[env] = st.m.peak; e.m_mdd[env] = st.m.mdd;
      e.m_mean[env] = st.m.mean; e.m_m2[env] = st.m.m2; e.m_n[env] = st.m.n;
      int slot = -1;
      for (int m = 0; m < p.M; ++m)
        if (p.kinds[m] == FIN_DDPG_OU) slot = m;
      if (slot >= 0) {
#pragma unroll
        for (int k = 0; k < KA; ++k) e.ou[((size_t)slot * e.K + k) * e.N + env] = st.ou[k];
      }
      if (p.o.ep_count) p.o.ep_count[env] = st.cnt;
      if (st.oor) set_flag(e, FIN_FLAG_ACTION_RANGE);
      if (st.bad) set_flag(e, FIN_FLAG_BAD_INDEX);
      if (st.nonfinite) set_flag(e, FIN_FLAG_NONFINITE);
    }
    st.agg.s[FIN_AGG_SUM_REWARD] = st.rsum;
    if (p.o.agg_partial) agg_group_write(st.agg, p.o.agg_partial + (size_t)blockIdx.x * FIN_AGG_LEN,
                                         threadIdx.x - tc::kEnvWarp0 * 32, 1);
  }
};

// Binds the env ops to one network plan (build_obs needs the plan's padded width).
template <int KA, int IA, class Plan>
struct StockOpsP : StockOps<KA, IA> {
  using Base = StockOps<KA, IA>;
  static_assert(Base::IN <= Plan::kIn, "observation wider than the network input");
  __device__ __forceinline__ static void build_obs(typename Base::State& st, const TcParams& p, int env, int row,
                                                   int t, uint32_t xa) {
    Base::template build_obs_t<Plan>(st, p, env, row, t, xa);
  }
};

// ---------------------------------------------------------------- K7 probe
template <class Plan>
struct ProbeOps {
  struct State {
    int b;
  };
  __device__ __forceinline__ static void init(State& st, const TcParams& p, int env, int row) { st.b = env; }
  __device__ __forceinline__ static void build_obs(State& st, const TcParams& p, int env, int row, int t,
                                                   uint32_t xa) {
    constexpr int KT8 = Plan::kIn / 8;
    const bool live = st.b < p.B;
    const uint16_t* x = p.x_in + (size_t)st.b * p.in_dim;
#pragma unroll 1
    for (int c = 0; c < KT8; ++c) {
      uint32_t w4[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int i0 = 8 * c + 2 * j;
        const uint32_t lo = (live && i0 < p.in_dim) ? x[i0] : 0u;
        const uint32_t hi = (live && i0 + 1 < p.in_dim) ? x[i0 + 1] : 0u;
        w4[j] = lo | (hi << 16);
      }
      sm100::st_shared_v4(xa + tc::cm_off(row, c, KT8), w4[0], w4[1], w4[2], w4[3]);
    }
  }
  __device__ __forceinline__ static uint16_t* hidden_ptr(State& st, const TcParams& p, int env, int t, int m, int l,
                                                         int hid) {
    if (st.b >= p.B || !p.hid_out) return nullptr;
    return p.hid_out + ((size_t)st.b * 2 + l) * hid;
  }
  __device__ __forceinline__ static void consume(State& st, const TcParams& p, int env, int t, int m,
                                                 const float* z) {
    if (st.b >= p.B) return;
    for (int k = 0; k < p.out_dim; ++k) p.z_out[(size_t)st.b * p.out_dim + k] = z[k];
  }
  __device__ __forceinline__ static void finish_step(State&, const TcParams&, int, int) {}
  __device__ __forceinline__ static void finalize(State&, const TcParams&, int) {}
};

template <class Plan, bool RES, class Ops>
cudaError_t launch_tc(const TcParams& p, int n_tiles, cudaStream_t s) {
  using S = tc::Smem<Plan, RES>;
  auto kern = tc::k_tc_rollout<Plan, RES, Ops>;
  cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, S::kTotal);
  if (err != cudaSuccess) return err;
  kern<<<n_tiles, tc::kThreads, S::kTotal, s>>>(p);
  return cudaGetLastError();
}

}  // namespace

namespace fin {

// net: 0 = PlanStockC1 (K=30, I=8), 1 = PlanStockSmall (K=4, I=4)
cudaError_t launch_stock_rollout(int net, const tc::TcParams& p, int n_tiles, cudaStream_t s) {
  if (net == 0) return launch_tc<PlanStockC1, false, StockOpsP<30, 8, PlanStockC1>>(p, n_tiles, s);
  if (net == 1) return launch_tc<PlanStockSmall, true, StockOpsP<4, 4, PlanStockSmall>>(p, n_tiles, s);
  return cudaErrorInvalidValue;
}

// net: 0 = PlanStockC1, 1 = PlanStockSmall, 2 = PlanCrypto
cudaError_t launch_mlp_probe(int net, const tc::TcParams& p, int n_tiles, cudaStream_t s) {
  if (net == 0) return launch_tc<PlanStockC1, false, ProbeOps<PlanStockC1>>(p, n_tiles, s);
  if (net == 1) return launch_tc<PlanStockSmall, true, ProbeOps<PlanStockSmall>>(p, n_tiles, s);
  if (net == 2) return launch_tc<PlanCrypto, true, ProbeOps<PlanCrypto>>(p, n_tiles, s);
  return cudaErrorInvalidValue;
}

}  // namespace fin
