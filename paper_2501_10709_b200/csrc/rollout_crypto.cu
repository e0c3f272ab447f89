// rollout_crypto.cu -- fused crypto Q-network rollout (BASELINE configs[3]).
// Per step and env: observation [h, tau/max_hold, f_1..f_101] (reading R24) ->
// Q = MLP(q(obs)) on tcgen05 with the 60 KB Q-net resident in shared memory ->
// argmax (lowest index on ties) with epsilon-greedy exploration ->
// a in {-1, 0, 1} -> LOB-walk execution, reward, done / reset (env_crypto.cuh) ->
// online episode metrics.  All envs of the C3 workload read the same row t
// (lockstep, reading R27).  With several members (DQN / Double DQN / Dueling DQN,
// PAPER.md §5.2.2) each member's greedy action is one vote and the
// executed action is the plurality winner, ties to hold, then to the lowest index
// (reading R-VOTE); a dueling member's greedy action is the argmax of its advantage
// head (outputs 0..2; Q = V + A - mean A has the same argmax).  Once per step a tile stages the bf16 factor part of the
// observation and the two book rows in shared memory; a tile whose envs sit on
// different rows takes the per-env path.  The market rows live in a 3-slot ring
// (row k in slot k mod 3): during step t the tile cp.asyncs row t+2, so the C3 loop
// never waits on HBM for its next row (276 MB series, streamed once).
#include <cuda_bf16.h>

#include "env_crypto.cuh"
#include "philox.cuh"
#include "rollout_tc.cuh"
#include "sm100.cuh"

namespace {

using tc::TcParams;

__device__ __forceinline__ uint32_t bf16_bits(float v) {
  return (uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(v));
}
__device__ __forceinline__ bool bar_red_and(int bar_id, bool pred) {
  uint32_t r;
  asm volatile(
      "{\n\t.reg .pred p, q;\n\t"
      "setp.ne.u32 p, %1, 0;\n\t"
      "bar.red.and.pred q, %2, 128, p;\n\t"
      "selp.u32 %0, 1, 0, q;\n\t}"
      : "=r"(r)
      : "r"((uint32_t)pred), "r"(bar_id)
      : "memory");
  return r != 0;
}
__device__ __forceinline__ void bar_sync128(int bar_id) {
  asm volatile("bar.sync %0, 128;" ::"r"(bar_id) : "memory");
}

// Plan: PlanCrypto (BASELINE configs[3]: 103-128-128-3/-4) or PlanCryptoPaper (the
// paper's three 128-unit hidden layers); both take the same 112-wide input.
template <class Plan>
struct CryptoOps {
  static constexpr int IN = 2 + FIN_C_FACTORS;  // 103
  static constexpr int KT8 = Plan::kIn / 8;
  static constexpr bool kSplitOK = true;        // column-split epilogues (no layer-1 addend)
  static constexpr bool kSplitAddend = false;
  static constexpr bool kSegments = false;
  static constexpr bool kL1Init = false;
  static constexpr int kOffImgT = 0;
  static constexpr bool kEpiPipe = true;        // double-buffered TMEM loads in the epilogues
  static constexpr bool kStageBias = true;
  static constexpr bool kL1Bcast = true;        // uniform tiles: shared layer-1 inputs read with SBO = 0
  static constexpr int kBcastKG = KT8 - 2;      // k-groups 2.. (columns 16..) of the observation
  static constexpr int kOffX = 0;                               // bf16 obs row (112)
  static constexpr int kOffB = 256;                             // kBcastKG core matrices of 8 equal rows
  static constexpr int kOffR = kOffB + kBcastKG * 128;          // ring of 3 rows (3 x 144 floats)
  static constexpr int kOffT = kOffR + 3 * FIN_C_ROW * 4;
  static constexpr int kStageBytes = kOffT + 16;

  struct State {
    bool live, uniform;
    int k0, k1, k2;    // market row held by ring slot 0 / 1 / 2 (-1: none); same in every thread
    int pend;          // row being prefetched (-1: none)
    int slot_t;        // ring slot of this step's row (uniform case)
    int tprev;         // the last uniform step's row (-1: none); same in every thread
    double b;
    int h, tau, t_ep;
    int act;
    int vote0, vote1, vote2;   // (scalars: a dynamically indexed array would live in local memory)
    float u0, u1;      // the step's epsilon-greedy uniforms (drawn in prepare(), under layer 2)
    MetricAcc m;
    AggAcc agg;
    int cnt;
    double rsum;
    bool bad, nonfinite;
  };

  __device__ __forceinline__ static void init(State& st, const TcParams& p, int env, int row) {
    const EnvDev& e = p.e;
    st.live = env < e.N;
    st.uniform = false;
    st.cnt = 0;
    st.rsum = 0.0;
    st.bad = st.nonfinite = false;
    st.act = 0;
    st.k0 = st.k1 = st.k2 = -1;
    st.pend = -1;
    st.slot_t = 0;
    st.tprev = -1;
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

  __device__ __forceinline__ static void stage(State& st, const TcParams& p, int env, int gtid, int t, uint8_t* stg,
                                               int bar_id) {
    const EnvDev& e = p.e;
    int* sr = reinterpret_cast<int*>(stg + kOffT);
    int tr = st.t_ep;
    if (st.live && (tr + 1 >= e.rows)) { st.bad = true; tr = 0; }
    sm100::cp_async_wait<0>();      // this thread's part of the last prefetch ...
    // Lockstep prediction: the row after the last uniform step's.  One barrier-reduction both
    // checks it and publishes everyone's part of the prefetch; otherwise thread 0's row is
    // exchanged through shared memory and checked.
    const int tp = st.tprev >= 0 && st.tprev + 2 < e.rows ? st.tprev + 1 : -1;   // same in every thread
    int t0 = tp;
    bool uni = tp >= 0 && bar_red_and(bar_id, !st.live || tr == tp);
    if (!uni) {
      if (gtid == 0) sr[0] = st.live ? tr : -1;
      bar_sync128(bar_id);            // ... and everyone else's
      t0 = sr[0];
      uni = bar_red_and(bar_id, !st.live || tr == t0) && t0 >= 0;
    }
    FIN_TR(gtid == 0, t, 20);
    st.pend = -1;
    st.uniform = uni;
    st.tprev = uni ? t0 : -1;
    FIN_TR(gtid == 0, t, 21);
    if (uni) {
      float* ring = reinterpret_cast<float*>(stg + kOffR);
      // rows t0 and t0 + 1 must be in the ring; load whichever is missing
      const bool have0 = held(st, t0), have1 = held(st, t0 + 1);
      if (!have0 || !have1) {
        for (int j = gtid; j < 2 * FIN_C_ROW; j += 128) {
          const int r = t0 + (j >= FIN_C_ROW ? 1 : 0);
          if ((r == t0 && !have0) || (r == t0 + 1 && !have1))
            ring[(r % 3) * FIN_C_ROW + (j % FIN_C_ROW)] = __ldg(e.market + (size_t)r * FIN_C_ROW + (j % FIN_C_ROW));
        }
        set_held(st, t0);
        set_held(st, t0 + 1);
        bar_sync128(bar_id);   // ring rows visible (prefetched rows: since the barrier above)
      }
      st.slot_t = t0 % 3;
      const float* mrow = ring + st.slot_t * FIN_C_ROW;
      uint16_t* xs = reinterpret_cast<uint16_t*>(stg + kOffX);
      FIN_TR(gtid == 0, t, 22);
      for (int idx = gtid; idx < Plan::kIn; idx += 128)
        xs[idx] = (idx >= 2 && idx < IN) ? (uint16_t)bf16_bits(mrow[FIN_C_F0 + idx - 2]) : (uint16_t)0;
      // the same columns 16.. as core matrices of 8 identical rows (the broadcast layer-1 operand)
      if (gtid < kBcastKG * 8) {
        const int c0 = 8 * (2 + (gtid >> 3));
        uint32_t w4[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int i0 = c0 + 2 * j;
          const uint32_t lo = i0 < IN ? bf16_bits(mrow[FIN_C_F0 + i0 - 2]) : 0u;
          const uint32_t hi = i0 + 1 < IN ? bf16_bits(mrow[FIN_C_F0 + i0 - 1]) : 0u;
          w4[j] = lo | (hi << 16);
        }
        reinterpret_cast<uint4*>(stg + kOffB)[gtid] = make_uint4(w4[0], w4[1], w4[2], w4[3]);
      }
      FIN_TR(gtid == 0, t, 27);
      // prefetch row t0 + 2 (the next step's marking row) into the third slot
      const int r2 = t0 + 2;
      if (r2 < e.rows && t + 1 < p.T && !held(st, r2)) {
        const float* src = e.market + (size_t)r2 * FIN_C_ROW;
        float* dst = ring + (r2 % 3) * FIN_C_ROW;
        for (int j = gtid; j < FIN_C_ROW / 4; j += 128) sm100::cp_async16(dst + 4 * j, src + 4 * j);
        sm100::cp_async_commit();
        set_held(st, r2);
        st.pend = r2;
      }
      FIN_TR(gtid == 0, t, 23);
      bar_sync128(bar_id);   // xs visible
      FIN_TR(gtid == 0, t, 24);
    }
  }

  __device__ __forceinline__ static bool held(const State& st, int r) {
    const int s = r % 3;
    return (s == 0 ? st.k0 : (s == 1 ? st.k1 : st.k2)) == r;
  }
  __device__ __forceinline__ static void set_held(State& st, int r) {
    const int s = r % 3;
    if (s == 0) st.k0 = r;
    else if (s == 1) st.k1 = r;
    else st.k2 = r;
  }

  __device__ __forceinline__ static void build_obs(State& st, const TcParams& p, int env, int row, int t, int m,
                                                   uint32_t xa, uint8_t* stg) {
    const EnvDev& e = p.e;
    if (!st.live) {
#pragma unroll
      for (int c = 0; c < KT8; ++c) tc::sts128(xa + tc::cm_off(row, c, KT8), 0u, 0u, 0u, 0u);
      return;
    }
    const float den = (float)e.max_hold;
    const uint32_t priv = bf16_bits((float)st.h) | (bf16_bits(div_int_f32(st.tau, den, e.rmax_hold)) << 16);
    if (st.uniform) {
      const uint4* xs = reinterpret_cast<const uint4*>(stg + kOffX);
#pragma unroll
      for (int c = 0; c < KT8; ++c) {
        const uint4 v = xs[c];
        tc::sts128(xa + tc::cm_off(row, c, KT8), c == 0 ? priv : v.x, v.y, v.z, v.w);
      }
    } else {
      const float* mrow = e.market + (size_t)(st.t_ep + 1 < e.rows ? st.t_ep : 0) * FIN_C_ROW;
#pragma unroll
      for (int c = 0; c < KT8; ++c) {
        uint32_t w4[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int i0 = 8 * c + 2 * j;
          const uint32_t lo = (i0 >= 2 && i0 < IN) ? bf16_bits(__ldg(mrow + FIN_C_F0 + i0 - 2)) : 0u;
          const uint32_t hi = (i0 + 1 >= 2 && i0 + 1 < IN) ? bf16_bits(__ldg(mrow + FIN_C_F0 + i0 - 1)) : 0u;
          w4[j] = lo | (hi << 16);
        }
        if (c == 0) w4[0] = priv;
        tc::sts128(xa + tc::cm_off(row, c, KT8), w4[0], w4[1], w4[2], w4[3]);
      }
    }
  }

  // resident (env-issued) layer 1: a uniform tile writes only its private k-groups 0 and 1;
  // the MMA reads columns 16.. from the broadcast core matrices (l1_bcast)
  __device__ __forceinline__ static void build_obs_bcast(State& st, const TcParams& p, int env, int row, int t,
                                                         int m, uint32_t xa, uint8_t* stg) {
    if (!st.uniform) {
      build_obs(st, p, env, row, t, m, xa, stg);
      return;
    }
    const EnvDev& e = p.e;
    const uint4* xs = reinterpret_cast<const uint4*>(stg + kOffX);
    const uint4 v0 = xs[0], v1 = xs[1];
    uint32_t priv = 0u;
    if (st.live) {
      const float den = (float)e.max_hold;
      priv = bf16_bits((float)st.h) | (bf16_bits(div_int_f32(st.tau, den, e.rmax_hold)) << 16);
    }
    tc::sts128(xa + tc::cm_off(row, 0, KT8), priv, v0.y, v0.z, v0.w);
    tc::sts128(xa + tc::cm_off(row, 1, KT8), v1.x, v1.y, v1.z, v1.w);
  }
  __device__ __forceinline__ static uint32_t l1_bcast(const State& st, uint8_t* stg) {
    return st.uniform ? sm100::smem_u32(stg + kOffB) : 0u;
  }

  __device__ __forceinline__ static const float* l1_addend(State&, const TcParams&, int, uint8_t*) { return nullptr; }

  __device__ __forceinline__ static uint16_t* hidden_ptr(State& st, const TcParams& p, int env, int t, int m, int l,
                                                         int hid) {
    if (!st.live || !p.o.mlp_hidden) return nullptr;
    return p.o.mlp_hidden + ((((size_t)t * p.M + m) * p.e.N + env) * Plan::kNH + l) * hid;
  }

  // the hidden-activation log row of env ``env`` for an epilogue helper warpgroup
  __device__ __forceinline__ static uint16_t* helper_hidden_ptr(const TcParams& p, int env, int t, int m, int l,
                                                                int hid) {
    if (env >= p.e.N || !p.o.mlp_hidden) return nullptr;
    return p.o.mlp_hidden + ((((size_t)t * p.M + m) * p.e.N + env) * Plan::kNH + l) * hid;
  }

  // the step's epsilon-greedy uniforms do not depend on the network: drawn while layer 2 runs
  __device__ __forceinline__ static void prepare(State& st, const TcParams& p, int env, int t, int m) {
    if (!st.live || m != 0) return;
    const EnvDev& e = p.e;
    st.u0 = 1.f;
    st.u1 = 0.f;
    if (p.noise_mode == FIN_NOISE_SUPPLIED) {
      const float* nz = p.noise + ((size_t)t * e.N + env) * 2;
      st.u0 = __ldg(nz); st.u1 = __ldg(nz + 1);
    } else if (p.noise_mode == FIN_NOISE_PHILOX) {
      float u[2];
      philox_uniform2((uint64_t)(e.env_offset + env), (uint32_t)(e.t_global + t), p.noise_seed, u);
      st.u0 = u[0]; st.u1 = u[1];
    }
  }
  __device__ __forceinline__ static void consume(State& st, const TcParams& p, int env, int t, int m, const float* z) {
    if (!st.live) return;
    const EnvDev& e = p.e;
    if (p.o.mlp_out) {
      float* dst = p.o.mlp_out + (((size_t)t * p.M + m) * e.N + env) * 3;
      dst[0] = z[0]; dst[1] = z[1]; dst[2] = z[2];
    }
    // argmax, lowest index on ties (no dynamic indexing of z: it would go to local memory)
    const float z0 = z[0], z1 = z[1], z2 = z[2];
    int best = 0;
    float bv = z0;
    if (z1 > bv) { best = 1; bv = z1; }
    if (z2 > bv) best = 2;
    if (!(isfinite(z0) && isfinite(z1) && isfinite(z2))) { st.nonfinite = true; best = 1; }
    if (m == 0) st.vote0 = st.vote1 = st.vote2 = 0;
    st.vote0 += best == 0;
    st.vote1 += best == 1;
    st.vote2 += best == 2;
    if (m + 1 < p.M) return;
    // plurality; ties to hold (index 1), then to the lowest index
    best = 1;
    int bc = st.vote1;
    if (st.vote0 > bc) { best = 0; bc = st.vote0; }
    if (st.vote2 > bc) best = 2;
    if (st.u0 < e.eps) best = min((int)((double)st.u1 * 3.0), 2);   // exact product, as the oracle
    st.act = best - 1;
  }

  __device__ __forceinline__ static void finish_step(State& st, const TcParams& p, int env, int t, uint8_t* stg,
                                                     uint8_t*) {
    if (!st.live) return;
    const EnvDev& e = p.e;
    const size_t ti = (size_t)t * e.N + env;
    FIN_CHECK(t >= 0 && t < p.T && env >= 0 && env < e.N);
    if (st.t_ep >= e.L || st.t_ep + 1 >= e.rows) {
      st.bad = true;
      if (p.o.reward) p.o.reward[ti] = 0.f;
      if (p.o.done) p.o.done[ti] = 1;
      return;
    }
    const float* ring = reinterpret_cast<const float*>(stg + kOffR);
    const float* row = st.uniform ? ring + st.slot_t * FIN_C_ROW : e.market + (size_t)st.t_ep * FIN_C_ROW;
    const float* row_next = st.uniform ? ring + ((st.slot_t + 1) % 3) * FIN_C_ROW : row + FIN_C_ROW;
    double v, vn;
    int delta;
    crypto_transition(e, st.b, st.h, st.tau, row, row_next, st.act, v, vn, delta);
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

  __device__ __forceinline__ static void finalize(State& st, const TcParams& p, int env, int gtid, int bar_id,
                                                  int tile) {
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
    if (p.o.agg_partial)
      agg_group_write(st.agg, p.o.agg_partial + ((size_t)blockIdx.x * p.tiles_per_cta + tile) * FIN_AGG_LEN, gtid,
                      bar_id, tile);
  }
};

}  // namespace

namespace fin {

int num_sms();

// The C3 loop is latency-bound (one lockstep step at a time): spread tiles over the
// SMs first (one tile per CTA); pair tiles per CTA only when tiles outnumber SMs.
#ifndef FIN_CRYPTO_SPLIT
#define FIN_CRYPTO_SPLIT 2   // warpgroups sharing each hidden-layer epilogue (one tile per CTA)
#endif
constexpr int kCryptoSplit = FIN_CRYPTO_SPLIT;

template <class Plan>
cudaError_t launch_crypto_plan(const tc::TcParams& p, int n_envs, int* tiles, cudaStream_t s) {
  using Ops = CryptoOps<Plan>;
  const int n_tiles = (n_envs + tc::kTileM - 1) / tc::kTileM;
  const bool two = n_tiles > num_sms();
  *tiles = two ? 2 : 1;
  // the Q-nets stay resident in shared memory while they fit (60 KB each, 92 KB for the
  // paper's 3 x 128 net); a larger voting ensemble (9 or 30 members)
  // streams them like the stock nets
  if (two) {
    if (p.M <= tc::Smem<Plan, true, 2, Ops>::max_members()) return tc::launch<Plan, true, 2, Ops>(p, n_envs, s);
    return tc::launch<Plan, false, 2, Ops>(p, n_envs, s);
  }
  if (p.M <= tc::Smem<Plan, true, 1, Ops>::max_members())
    return tc::launch<Plan, true, 1, Ops, tc::kRing, 1, kCryptoSplit>(p, n_envs, s);
  return tc::launch<Plan, false, 1, Ops>(p, n_envs, s);
}

// net: 2 = PlanCrypto, 4 = PlanCryptoPaper
cudaError_t launch_crypto_rollout(int net, const tc::TcParams& p, int n_envs, int* tiles, cudaStream_t s) {
  if (net == 2) return launch_crypto_plan<PlanCrypto>(p, n_envs, tiles, s);
  if (net == 4) return launch_crypto_plan<PlanCryptoPaper>(p, n_envs, tiles, s);
  return cudaErrorInvalidValue;
}

}  // namespace fin
