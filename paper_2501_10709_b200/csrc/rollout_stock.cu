// rollout_stock.cu -- fused stock policy rollout (K3, with the C2 ensemble K5 inside)
// and the standalone MLP probe (K7), instantiated from rollout_tc.cuh.
//
// Per step and env (thread r of a tile's env warpgroup):
//   observation s_t = [b/b0, close_norm_t, h/max_trade, f_t]  (readings R13, R14)
//   -> per member m: z_m = MLP_m(q(s_t)) on tcgen05 (BASELINE configs[1,2])
//   -> member action (R17, R19): PPO clip(tanh z + std eps), SAC tanh(z + std eps),
//      DDPG OU x <- x + theta(0 - x) + sigma eps, clip(tanh z + x)
//   -> ensemble mean (R20) -> shares = rha(max_trade * abar)  (R18)
//   -> trade, reward, done / reset (env_stock.cuh), online episode metrics.
//
// Staging: the market part of the observation (close_norm, indicators; 270 of 301
// inputs for C1) and the two close-price rows are the same for every env of a
// tile that sits on the same day d (tile-aligned windows, lockstep clocks: the
// normal case).  group_apply (group_stage.cuh) converts that row once per tile into
// shared memory (bf16 observation part, fp64 prices); each env copies it into its
// observation row, patches in its private entries (cash, holdings) and reads its
// execution / marking prices from it.  Tiles whose envs sit on several days are
// served one day at a time by the same code path.
#include <cuda_bf16.h>

#include <type_traits>

// the fused rollout forms the -2^52 x product operands with a DMUL (FIN_MROWS=1, staged rows,
// raises the spills of every K3 variant: its env warps run under the MMA warps' register budget)
#ifndef FIN_MROWS
#define FIN_MROWS 0
#endif
#ifndef FIN_KCHUNK
#define FIN_KCHUNK 10  // assets per row chunk (A/B on the headline: 3 / 6 / 8 / 10 / 15 / 30 -> 10 best, +0.7% over 6)
#endif
#include "env_stock.cuh"
#include "group_stage.cuh"
#include "philox.cuh"
#include "rollout_tc.cuh"

namespace {

using tc::TcParams;

__device__ __forceinline__ uint32_t bf16_bits(float v) {
  return (uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(v));
}

#ifndef FIN_PHILOX16
#define FIN_PHILOX16 0   // 1: consume draws 16 normals per Philox call (4 counters interleaved)
#endif
#ifndef FIN_STREAM_EARLY
#define FIN_STREAM_EARLY 1   // 1: the small-N kernel's own Philox draws (mode 4) under layer 2 (StockOps EARLY)
#endif
#ifndef FIN_NOISE_LATE
#define FIN_NOISE_LATE 1   // 1: noise in consume for the single policy, under layer 2 for ensembles
#endif

// Supplied normals [T][M][N][K].  Streamed (p.noise_ready != null, small N):
// k_stream_noise writes them on the idle SMs while this kernel runs; each of its blocks finishes
// the steps in order and counts each group of FIN_NOISE_GROUP steps in noise_ready[t / G]
// (release), so a full count at group g publishes every step before its end.  A consumer that
// has not yet seen step t complete (avail < t) first checks the last group (once the producer is
// done: no further waits in the call), else waits for t's group (acquire).  The data are then
// read by weak loads, ordered after the acquire by the memory model (never the non-coherent
// path, whose lines may predate the producer's stores), from a pointer laundered after the
// wait so the compiler cannot hoist them above it.  The wait is bounded (~8 s): past it the
// sticky FIN_FLAG_NOISE_WAIT is raised and later waits return at once.
__device__ __forceinline__ uint32_t ld_acquire_u32(const uint32_t* f) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
  return v;
}
// the step's noise pointer, laundered through a volatile asm after the wait: the loads depend
// on it, so the compiler cannot hoist them above the wait (they stay free to batch)
__device__ __forceinline__ const float* noise_after_wait(const float* a) {
  const float* q;
  asm volatile("mov.b64 %0, %1;" : "=l"(q) : "l"(a));
  return q;
}
template <bool STREAM>
__device__ __forceinline__ float noise_ld(const float* a) {
  if constexpr (STREAM) return *noise_after_wait(a);   // a weak load ordered after the acquire
  else return __ldg(a);
}
__device__ __forceinline__ void noise_wait(const TcParams& p, const EnvDev& e, int t, int& avail) {
  if (t <= avail) return;   // (the laundered loads follow the wait)
  const uint32_t tgt = p.noise_ready_target;
  const int last = (p.T - 1) / FIN_NOISE_GROUP, g = t / FIN_NOISE_GROUP;
  if (g < last && ld_acquire_u32(p.noise_ready + last) >= tgt) {
    avail = p.T - 1;
    return;
  }
  for (uint32_t spin = 0;; ++spin) {
    if (ld_acquire_u32(p.noise_ready + g) >= tgt) {
      avail = g * FIN_NOISE_GROUP + FIN_NOISE_GROUP - 1;
      return;
    }
    if (spin == 0 && (*(const volatile uint32_t*)e.flags & FIN_FLAG_NOISE_WAIT)) return;   // sticky: wait once
    if (spin > (1u << 26)) {
      set_flag(e, FIN_FLAG_NOISE_WAIT);
      return;
    }
    __nanosleep(128);
  }
}

// tanh(x) = sign(x) (1 - 2 / (exp(2|x|) + 1)) with the fast exp / reciprocal: absolute
// error ~1e-7 (the sampled share count 100 a moves by ~1e-5, well inside the 1e-4
// rounding-boundary allowance of the parity check); ~8 instructions instead of the
// ~35 of tanhf, which the rollout inlines once per asset.
__device__ __forceinline__ float tanh_f32(float x) {
  const float e2 = __expf(2.f * fabsf(x));
  const float t = 1.f - __fdividef(2.f, e2 + 1.f);
  return copysignf(t, x);
}

// ENS = false: the single-policy (C1) specialisation -- one non-DDPG member, no OU
// state kept in registers.  LOG = false: no optional trajectory logs (actions, cash,
// asset, holdings, network outputs / hidden activations) and no fin_ensemble_act mode
// -- the production rollout (reward, done, episode metrics, aggregate) carries none of
// their per-step branches.
// STREAM = true: the small-N instantiation that reads streamed pre-drawn noise (p.noise_ready,
// DESIGN.md §4.3); the others carry none of its code (A/B: the wait code alone in the large-N
// kernel cost 3% of the headline).
template <int KA, int IA, class Plan, bool ENS = true, bool LOG = true, bool STREAM = false, bool EARLY = false>
struct StockOps {
  static constexpr bool kStream = STREAM;
  static constexpr int KOU = ENS ? KA : 1;
  // the streamed-noise (small-N) instantiation of the streamed-weight plan also splits the
  // hidden epilogues over two warpgroups; layer 1's z1s addend pointer is
  // handed to the helper through shared memory
  static constexpr bool kSplitOK = STREAM;
  static constexpr bool kSplitAddend = true;
  static constexpr bool kSegments = true;   // balanced persistent schedule (init_seg / finalize_seg)
  static constexpr bool kL1Bcast = false;   // (crypto only: broadcast layer-1 A operand)
#ifndef FIN_STOCK_EPIPIPE
#define FIN_STOCK_EPIPIPE 0
#endif
  static constexpr bool kEpiPipe = FIN_STOCK_EPIPIPE;
  // ensembles read biases from L2 (no staged copy): the C2 ensemble then fits the dual layout
  // (two CTAs per SM), 6.1e8 -> 6.8e8 env-steps/s; the single policy keeps its staged copy
  static constexpr bool kStageBias = !ENS;
  // where the step's noise is drawn: inside consume for the single policy (+3.6%: no noise
  // registers live across the layer-2 epilogue), under layer 2 for ensembles (FIN_NOISE_LATE
  // overrides: 0 never late, 2 always late)
  // EARLY (the small-N production kernel drawing Philox itself, api.cu's mode 4: 99-148 tiles): its
  // env threads idle through the layer-2 MMA (one tile per SM), so the draws are made in prepare()
  // under layer 2 instead of on the chain in consume (A/B, scripts/early_ab.py: +3.4% at 16,384 x
  // 256).  A separate instantiation: supplied / pre-drawn normals taken early were 9% slower, and
  // one kernel holding both paths lost the whole small-N gain (register pressure).
  static constexpr bool kNoiseLate = !EARLY && (FIN_NOISE_LATE == 2 || (FIN_NOISE_LATE == 1 && !ENS));
  static constexpr int KP4 = (KA + 3) / 4 * 4;
  static constexpr int IN = 1 + 2 * KA + IA * KA;
  static constexpr int KT8 = Plan::kIn / 8;
  using Obs = StockObs<KA, IA>;
  static_assert(Obs::kEnvPad == Plan::kIn, "factored layer 1: the network input is the private part");
  // staging, two buffers: [price rows of a day (f64, fin_internal.cuh) | z1s rows of that
  // day per member (f32)] x 2 | slots | broadcast.  The current step uses buffer sb;
  // the other one receives, by cp.async under the step's work, the rows of the day
  // predicted for the next step (the tile's first env: next day, or the first day of
  // its window after a reset -- envs of a tile step in lockstep).
  static constexpr int kOffP = 0;
  static constexpr int kOffZ = kPriceRows * KP4 * 8;
  // FIN_L1_INIT=1 (A/B, off by default): the layer-1 accumulator starts at z1s[d] (+ b1),
  // stored into each env's TMEM row with tcgen05.st before the layer-1 MMAs, instead of
  // the epilogue adding it (same values for uniform and mixed tiles, same bits): measured
  // neutral (7.49 vs 7.37 ms at 65,536 envs).  Also measured and not kept: a tcgen05.cp of
  // a broadcast image of the row (SBO = 0): 32 copies of 8 columns cost ~2.3 k cycles on
  // the tile's critical path (scripts/micro/tmem_cp_rate.cu).
#ifndef FIN_L1_INIT
#define FIN_L1_INIT 0
#endif
  static constexpr bool kL1Init = FIN_L1_INIT && !ENS;
  // z1s rows staged (the epilogue addend of up to kStageM ensemble members; kL1Init: 1)
  static constexpr int kStageM = ENS ? FIN_STAGE_MEMBERS : 1;
  static constexpr int kRegion = kOffZ + kStageM * Plan::kH1 * 4;
  static constexpr int kOffS = 2 * kRegion;
  static constexpr int kOffB = kOffS + 16;      // int[4]: d0, predicted day, -, -
  static constexpr int kOffImgT = 0;
  // single policy: the episode-metric accumulators live in shared memory between steps ([6][row]
  // doubles, episode count n in a register) -- 12 shared accesses per step instead of ~12 registers
  // held across it, whose pressure made ptxas spill ~47 values per warp-step (FIN_METRIC_SM=0: A/B)
#ifndef FIN_METRIC_SM
#define FIN_METRIC_SM 1
#endif
  static constexpr bool kMetricSm = FIN_METRIC_SM && !ENS;
  static constexpr int kOffM = kOffB + 16;
  static constexpr int kStageBytes = kOffM + (kMetricSm ? 6 * tc::kTileM * 8 : 0);
  static constexpr int kSaveOff = tc::kTileM * Plan::kIn * 2;   // exact-redo scratch in the A operand
  static_assert(kSaveOff + (KA + 7) / 8 * tc::kTileM * 16 <= tc::kTileM * Plan::kHidMax * 2, "save fits the A operand");

  struct State {
    bool live;
    int gtid, bar_id, round;
    double b;
    double vc;         // pre-trade asset of the next step (cached v, then the last post-trade v)
    int h[KA];
    int t_ep, w, d;
    uint32_t b0bits;
    bool zsm;          // every live env of the tile is on day d0, whose rows are staged
    int d0;
    int sb;            // current staging buffer
    int kcur, koth;    // day held by buffer sb / by buffer sb ^ 1 (-1: none)
    int pend;          // day being prefetched into buffer sb ^ 1 (-1: none)
    float asum[KA];
    float eps[KA];     // this member's noise of the step (prepare(), while layer 2 runs)
    float ou[KOU];
    MetricAcc m;       // (the aggregate partials live in e.agg_env: touched once per episode); kMetricSm:
                       // only m.n (and m until the first stage(), which moves it to shared memory)
    uint32_t msa;      // kMetricSm: shared address of this row's accumulators (field f at + f * 128 * 8)
    int cnt;
    double rsum;
    int t_begin, t_end;   // steps of this segment (whole call: 0, T)
    int navail;           // streamed noise: last step known complete (noise_wait)
    bool oor, bad, nonfinite;
  };

  __device__ __forceinline__ static void init(State& st, const TcParams& p, int env, int row) {
    init_seg(st, p, env, row, 0, p.T);
  }
  // steps [t0, t1) of the call; a tail (t0 > 0) continues the episode count and reward sum
  // its head left in seg_cnt / seg_rsum and the aggregate partials in agg_env
  __device__ __forceinline__ static void init_seg(State& st, const TcParams& p, int env, int row, int t0, int t1) {
    const EnvDev& e = p.e;
    st.live = env < e.N;
    if constexpr (STREAM) st.navail = -1;
    st.t_begin = t0;
    st.t_end = t1;
    st.round = 0;
    st.cnt = (t0 > 0 && st.live) ? e.seg_cnt[env] : 0;
    st.rsum = (t0 > 0 && st.live) ? e.seg_rsum[env] : 0.0;
    st.oor = st.bad = st.nonfinite = false;
    st.d = 0;
    st.vc = 0.0;
    st.sb = 0;
    st.kcur = st.koth = -1;
    st.pend = -1;
    if (st.live && t0 == 0) agg_init_g(e.agg_env + env, (size_t)e.N);
    if (st.live) {
      st.b = e.cash[env];
      st.vc = e.vcur[env];
      load_hold<KA>(e, env, st.h);
      st.t_ep = e.t_ep[env];
      st.w = e.window[env];
      st.m.v0 = e.m_v0[env]; st.m.vprev = e.m_vprev[env]; st.m.peak = e.m_peak[env]; st.m.mdd = e.m_mdd[env];
      st.m.mean = e.m_mean[env]; st.m.m2 = e.m_m2[env]; st.m.n = e.m_n[env];
      // OU state of a single DDPG member lives in registers (slot 0); with several DDPG
      // members every slot is read and written in global memory (L2) at its use
#pragma unroll
      for (int k = 0; k < KOU; ++k) st.ou[k] = (ENS && p.n_ddpg == 1) ? e.ou[(size_t)k * e.N + env] : 0.f;
    } else {
      st.b = 0.0;
#pragma unroll
      for (int k = 0; k < KA; ++k) st.h[k] = 0;
#pragma unroll
      for (int k = 0; k < KOU; ++k) st.ou[k] = 0.f;
      st.t_ep = 0; st.w = 0;
      metric_start(st.m, 0.0);
    }
  }

  // stage day k into buffer region reg: f64 price rows of day k and the members' z1s rows
  __device__ __forceinline__ static void stage_row(const TcParams& p, int k, int gtid, uint8_t* reg) {
    const EnvDev& e = p.e;
    FIN_CHECK(k >= 0 && k < e.rows && k < p.z1s_rows);
    stage_price_rows(e, reinterpret_cast<double*>(reg + kOffP), k, gtid, 128);
    float* zs = reinterpret_cast<float*>(reg + kOffZ);
    for (int j = gtid; j < min(p.M, kStageM) * Plan::kH1; j += 128) {
      const int m = j / Plan::kH1, n = j % Plan::kH1;
      zs[j] = __ldg(p.z1s + ((size_t)m * p.z1s_rows + k) * Plan::kH1 + n);
    }
  }
  // the same rows by cp.async (16-byte chunks, no wait): completed by the next stage()
  __device__ __forceinline__ static void prefetch_row(const TcParams& p, int k, int gtid, uint8_t* reg) {
    const EnvDev& e = p.e;
    FIN_CHECK(k >= 0 && k < e.rows && k < p.z1s_rows);
    const int np = kPriceRows * e.kp / 2;                 // 16-B chunks of the price rows
    const uint8_t* src = reinterpret_cast<const uint8_t*>(e.px + (size_t)k * kPriceRows * e.kp);
    for (int j = gtid; j < np; j += 128) sm100::cp_async16(reg + kOffP + 16 * j, src + 16 * j);
    constexpr int nz = Plan::kH1 / 4;                   // chunks per member z1s row
    for (int j = gtid; j < min(p.M, kStageM) * nz; j += 128) {
      const int m = j / nz, c = j % nz;
      sm100::cp_async16(reg + kOffZ + (m * Plan::kH1 + 4 * c) * 4,
                        p.z1s + ((size_t)m * p.z1s_rows + k) * Plan::kH1 + 4 * c);
    }
    sm100::cp_async_commit();
  }
  __device__ __forceinline__ static uint8_t* region(uint8_t* stg, int b) { return stg + b * kRegion; }

  __device__ __forceinline__ static void m_put(State& st, const MetricAcc& m) {
    if constexpr (kMetricSm) {
      const double f[6] = {m.v0, m.vprev, m.peak, m.mdd, m.mean, m.m2};
#pragma unroll
      for (int i = 0; i < 6; ++i)
        asm volatile("st.shared.f64 [%0], %1;" ::"r"(st.msa + (uint32_t)(i * tc::kTileM * 8)), "d"(f[i]) : "memory");
      st.m.n = m.n;
    } else {
      st.m = m;
    }
  }
  __device__ __forceinline__ static MetricAcc m_get(const State& st) {
    if constexpr (kMetricSm) {
      double f[6];
#pragma unroll
      for (int i = 0; i < 6; ++i)
        asm volatile("ld.shared.f64 %0, [%1];" : "=d"(f[i]) : "r"(st.msa + (uint32_t)(i * tc::kTileM * 8)) : "memory");
      MetricAcc m;
      m.v0 = f[0]; m.vprev = f[1]; m.peak = f[2]; m.mdd = f[3]; m.mean = f[4]; m.m2 = f[5];
      m.n = st.m.n;
      return m;
    } else {
      return st.m;
    }
  }

  // kL1Init: this env's row of the layer-1 accumulator <- z1s[d] (+ b1) of its day
  __device__ __forceinline__ static void l1_init_rows(State& st, const TcParams& p, uint32_t t_lane, uint8_t* stg) {
    if constexpr (kL1Init) {
      const float* src = st.zsm ? reinterpret_cast<const float*>(region(stg, st.sb) + kOffZ)
                                : p.z1s + (size_t)(st.live ? st.d : 0) * Plan::kH1;
#pragma unroll 1
      for (int c = 0; c < Plan::kH1 / 16; ++c) {
        uint32_t v[16];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float4 x = reinterpret_cast<const float4*>(src + 16 * c)[q];
          v[4 * q] = __float_as_uint(x.x); v[4 * q + 1] = __float_as_uint(x.y);
          v[4 * q + 2] = __float_as_uint(x.z); v[4 * q + 3] = __float_as_uint(x.w);
        }
        sm100::tmem_st16(t_lane + (uint32_t)(16 * c), v);
      }
      sm100::tmem_wait_st();
    }
  }


  // once per step, all 128 threads of the tile: day of every env; if the tile sits on
  // one day, stage that day once (prices, z1s rows) for the whole step
  __device__ __forceinline__ static void stage(State& st, const TcParams& p, int env, int gtid, int t, uint8_t* stg,
                                               int bar_id) {
    const EnvDev& e = p.e;
    st.gtid = gtid;
    st.bar_id = bar_id;
    GroupSlots* gs = reinterpret_cast<GroupSlots*>(stg + kOffS);
    int* bc = reinterpret_cast<int*>(stg + kOffB);
    if (t == st.t_begin) {
      gs_init(gs, gtid, bar_id);
      if constexpr (kMetricSm) {
        st.msa = sm100::smem_u32(stg + kOffM) + (uint32_t)gtid * 8u;
        const MetricAcc m0 = st.m;
        m_put(st, m0);
      }
    }
    if (st.live) {
      st.d = day_of(e, st.w, st.t_ep);
      if (st.d < 0 || st.d + 1 >= e.rows) { st.bad = true; st.d = 0; }
      st.b0bits = (uint32_t)__bfloat16_as_ushort(__double2bfloat16(fdiv64_rcp(st.b, e.cash0, e.rcash0)));
    }
    if (gtid == 0) {
      bc[0] = st.live ? st.d : -1;
      // predicted day of the next step (lockstep envs): from this thread's env
      int dn = -1;
      if (st.live && !st.bad) {
        if (st.t_ep + 1 < e.L) dn = st.d + 1;
        else if (e.autoreset) dn = day_of(e, e.wadv ? (st.w + 1) % e.W : st.w, 0);
      }
      bc[1] = (dn >= 0 && dn + 1 < e.rows) ? dn : -1;
    }
    sm100::cp_async_wait<0>();                 // this thread's part of the last prefetch
    gs_bar(bar_id);                            // ... and everyone else's
    FIN_TR(threadIdx.x == 128, t, 23);
    if (st.pend >= 0) {                        // the prefetched buffer becomes current
      st.sb ^= 1;
      const int k = st.kcur;
      st.kcur = st.koth;
      st.koth = k;
      st.pend = -1;
    }
    const int d0 = bc[0], dn = bc[1];
    const bool uni = !gs_bar_or(bar_id, st.live && st.d != d0) && d0 >= 0;
    FIN_TR(threadIdx.x == 128, t, 24);
    st.zsm = uni;
    st.d0 = d0;
    if (uni && d0 != st.kcur) {
      stage_row(p, d0, gtid, region(stg, st.sb));
      st.kcur = d0;
      gs_bar(bar_id);
    }
    if (gtid == 0) gs->staged = st.kcur;   // for group_apply in finish_step (after its barrier)

    // rows of the predicted next day into the other buffer, under this step's work
    // (that buffer was last read in the previous step, before this step's barriers)
    if (dn >= 0 && t + 1 < st.t_end && dn != st.kcur) {
      prefetch_row(p, dn, gtid, region(stg, st.sb ^ 1));
      st.koth = dn;
      st.pend = dn;
    }
    FIN_TR(threadIdx.x == 128, t, 25);
  }

  // factored layer 1: the shared-input term of this env's day, member m
  __device__ __forceinline__ static const float* l1_addend(State& st, const TcParams& p, int m, uint8_t* stg) {
    if constexpr (kL1Init) return nullptr;   // the accumulator started at z1s[d] + b1
    if (st.zsm && m < kStageM) return reinterpret_cast<const float*>(region(stg, st.sb) + kOffZ) + m * Plan::kH1;
    return p.z1s + ((size_t)m * p.z1s_rows + st.d) * Plan::kH1;
  }

  // the env-private observation entries [b/b0, h_k/max_trade, 0 pad] -> X (bf16)
  __device__ __forceinline__ static void build_obs(State& st, const TcParams& p, int env, int row, int t, int m,
                                                   uint32_t xa, uint8_t* stg) {
    const EnvDev& e = p.e;
    if (m == 0) {
#pragma unroll
      for (int k = 0; k < KA; ++k) st.asum[k] = 0.f;
    }
    const float den = (float)e.max_trade;
    const float inv_den = e.rmax_trade;   // = __frcp_rn(den), computed on the host
#pragma unroll
    for (int c = 0; c < KT8; ++c) {
      uint32_t w4[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        uint32_t lohi[2];
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const int idx = 8 * c + 2 * j + q;
          lohi[q] = !st.live ? 0u
                    : idx == 0 ? st.b0bits
                    : idx <= KA ? bf16_bits(div_int_f32(st.h[idx - 1], den, inv_den))
                                : 0u;
        }
        w4[j] = lohi[0] | (lohi[1] << 16);
      }
      tc::sts128(xa + tc::cm_off(row, c, KT8), w4[0], w4[1], w4[2], w4[3]);
      if (LOG && m == 0 && st.live && p.o.obs_private)
        reinterpret_cast<uint4*>(p.o.obs_private + ((size_t)t * e.N + env) * Plan::kIn)[c] =
            make_uint4(w4[0], w4[1], w4[2], w4[3]);
    }
    if (LOG && m == 0 && st.live && p.o.day) p.o.day[(size_t)t * e.N + env] = st.d;
  }

  // the column-split helper's rows of the same log (no env state)
  __device__ __forceinline__ static uint16_t* helper_hidden_ptr(const TcParams& p, int env, int t, int m, int l,
                                                                int hid) {
    if (!LOG || env >= p.e.N || !p.o.mlp_hidden) return nullptr;
    return p.o.mlp_hidden + ((((size_t)t * p.M + m) * p.e.N + env) * Plan::kNH + l) * hid;
  }
  __device__ __forceinline__ static uint16_t* hidden_ptr(State& st, const TcParams& p, int env, int t, int m, int l,
                                                         int hid) {
    if (!LOG || !st.live || !p.o.mlp_hidden) return nullptr;
    return p.o.mlp_hidden + ((((size_t)t * p.M + m) * p.e.N + env) * Plan::kNH + l) * hid;
  }

  // the member's noise for this step: Philox4x32-10 + Box-Muller (R-NOISE) or the
  // supplied normals; independent of the network output, so it runs while layer 2 does
  __device__ __forceinline__ static void prepare(State& st, const TcParams& p, int env, int t, int m) {
    if constexpr (kNoiseLate) return;   // drawn inside consume (no noise registers live across epilogues)
    if (!st.live) return;
    const EnvDev& e = p.e;
    const float* nz = p.noise + (((size_t)t * p.M + m) * e.N + env) * KA;
    // noise in blocks of 8 assets: two Philox counters (blocks 2q, 2q+1) per call
#pragma unroll
    for (int pb = 0; pb < (KA + 7) / 8; ++pb) {
      float eps[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
      if (p.noise_mode == FIN_NOISE_PHILOX) {
        const Normals8 nv =
            philox_normals8_v((uint64_t)(e.env_offset + env), (uint32_t)(e.t_global + t),
                              ((uint32_t)m << 16) | (uint32_t)(2 * pb), ((uint32_t)m << 16) | (uint32_t)(2 * pb + 1),
                              p.noise_seed);
        eps[0] = nv.a.x; eps[1] = nv.a.y; eps[2] = nv.a.z; eps[3] = nv.a.w;
        eps[4] = nv.b.x; eps[5] = nv.b.y; eps[6] = nv.b.z; eps[7] = nv.b.w;
        if (pb == 0) FIN_TR(threadIdx.x == 128 && m == 0, t, 16);
      } else if (p.noise_mode == FIN_NOISE_SUPPLIED) {
        if constexpr (STREAM) if (pb == 0) noise_wait(p, e, t, st.navail);
#pragma unroll
        for (int j = 0; j < 8; ++j)
          if (pb * 8 + j < KA) eps[j] = noise_ld<STREAM>(nz + pb * 8 + j);
      }
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (pb * 8 + j < KA) st.eps[pb * 8 + j] = eps[j];
    }
  }

  __device__ __forceinline__ static void consume(State& st, const TcParams& p, int env, int t, int m, const float* z) {
    if (!st.live) return;
    const EnvDev& e = p.e;
    const int kind = p.kinds[m];
    const bool sac = kind == FIN_SAC_SQUASH, ddpg = kind == FIN_DDPG_OU;
    if (LOG && p.o.mlp_out) {
      float* dst = p.o.mlp_out + (((size_t)t * p.M + m) * e.N + env) * KA;
#pragma unroll
      for (int k = 0; k < KA; ++k) dst[k] = z[k];
    }
    const float wm = p.weighted ? p.mw[m] : 1.f;
#if FIN_PHILOX16
    // in-kernel Philox noise: four counters per call (16 normals), twice the interleave
    Normals16 n16;
#endif
#pragma unroll
    for (int pb = 0; pb < (KA + 7) / 8; ++pb) {
      float eps[8];
#if FIN_PHILOX16
      if constexpr (kNoiseLate) {
        if (p.noise_mode == FIN_NOISE_PHILOX) {
          if ((pb & 1) == 0) {
            const uint32_t mb = (uint32_t)m << 16;
            const uint32_t w2[4] = {mb | (uint32_t)(2 * pb), mb | (uint32_t)(2 * pb + 1), mb | (uint32_t)(2 * pb + 2),
                                    mb | (uint32_t)(2 * pb + 3)};
            n16 = philox_normals16_v((uint64_t)(e.env_offset + env), (uint32_t)(e.t_global + t), w2, p.noise_seed);
          }
#pragma unroll
          for (int j = 0; j < 8; ++j) eps[j] = n16.v[8 * (pb & 1) + j];
        } else {
          const float* nz = p.noise + (((size_t)t * p.M + m) * e.N + env) * KA;
#pragma unroll
          for (int j = 0; j < 8; ++j) eps[j] = 0.f;
          if (p.noise_mode == FIN_NOISE_SUPPLIED) {
            if constexpr (STREAM) if (pb == 0) noise_wait(p, e, t, st.navail);
#pragma unroll
            for (int j = 0; j < 8; ++j)
              if (pb * 8 + j < KA) eps[j] = noise_ld<STREAM>(nz + pb * 8 + j);
          }
        }
      } else
#endif
      if constexpr (kNoiseLate) {
        const float* nz = p.noise + (((size_t)t * p.M + m) * e.N + env) * KA;
#pragma unroll
        for (int j = 0; j < 8; ++j) eps[j] = 0.f;
        if (p.noise_mode == FIN_NOISE_PHILOX) {
          const Normals8 nv =
              philox_normals8_v((uint64_t)(e.env_offset + env), (uint32_t)(e.t_global + t),
                                ((uint32_t)m << 16) | (uint32_t)(2 * pb), ((uint32_t)m << 16) | (uint32_t)(2 * pb + 1),
                                p.noise_seed);
          eps[0] = nv.a.x; eps[1] = nv.a.y; eps[2] = nv.a.z; eps[3] = nv.a.w;
          eps[4] = nv.b.x; eps[5] = nv.b.y; eps[6] = nv.b.z; eps[7] = nv.b.w;
        } else if (p.noise_mode == FIN_NOISE_SUPPLIED) {
          if constexpr (STREAM) if (pb == 0) noise_wait(p, e, t, st.navail);
#pragma unroll
          for (int j = 0; j < 8; ++j)
            if (pb * 8 + j < KA) eps[j] = noise_ld<STREAM>(nz + pb * 8 + j);
        }
      } else {
#pragma unroll
        for (int j = 0; j < 8; ++j) eps[j] = pb * 8 + j < KA ? st.eps[pb * 8 + j] : 0.f;
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int k = pb * 8 + j;
        if (k >= KA) break;
        // one tanh per asset for every member kind:
        //   SAC   a = tanh(z + std eps)
        //   PPO   a = clip(tanh(z) + std eps)
        //   DDPG  x = x + theta (0 - x) + sigma eps;  a = clip(tanh(z) + x)
        const float se = __fmul_rn(e.noise_std, eps[j]);
        const float pre = sac ? __fadd_rn(z[k], se) : z[k];
        float post = se;
        if (ENS && ddpg) {
          const int ko = ENS ? k : 0;
          float* gx = e.ou + ((size_t)p.ou_slot[m] * e.K + k) * e.N + env;
          const float x = p.n_ddpg == 1 ? st.ou[ko] : *gx;
          post = __fadd_rn(__fadd_rn(x, __fmul_rn(e.ou_theta, __fsub_rn(0.f, x))), __fmul_rn(e.ou_sigma, eps[j]));
          if (p.n_ddpg == 1) st.ou[ko] = post;
          else if (!(LOG && p.act_only) || p.commit_ou) *gx = post;   // act-only: commit on request
        }
        const float th = tanh_f32(pre);
        float a = sac ? th : fminf(fmaxf(__fadd_rn(th, post), -1.f), 1.f);
        if (!isfinite(a)) { st.nonfinite = true; a = 0.f; }
        st.asum[k] = p.weighted ? __fadd_rn(st.asum[k], __fmul_rn(wm, a)) : __fadd_rn(st.asum[k], a);
      }
    }
  }

  __device__ __forceinline__ static void finish_step(State& st, const TcParams& p, int env, int t, uint8_t* stg,
                                                     uint8_t* a_tile) {
    const EnvDev& e = p.e;
    const size_t ti = (size_t)t * e.N + env;
    FIN_CHECK(!st.live || (t >= 0 && t < p.T && env >= 0 && env < e.N));
    FIN_CHECK(!st.live || st.bad || (st.d >= 0 && st.d + 1 < e.rows));
    int a[KA];
    FIN_TR(threadIdx.x == 128, t, 17);
    const float inv_m = p.inv_m;   // fl(1 / M) (host): uniform mean (R20); the weighted sum is already scaled
#pragma unroll
    for (int k = 0; k < KA; ++k) {
      const float abar = (!ENS || p.M == 1 || p.weighted) ? st.asum[k] : __fmul_rn(st.asum[k], inv_m);
      a[k] = rha_f32(__fmul_rn((float)e.max_trade, abar));
      if (LOG && st.live && p.act_only && p.mean_out) p.mean_out[(size_t)env * KA + k] = abar;
    }
    if (LOG && p.act_only) {  // fin_ensemble_act: report the action, leave the env untouched
      if (st.live && p.o.actions) {
#pragma unroll
        for (int k = 0; k < KA; ++k) p.o.actions[(size_t)env * KA + k] = (int16_t)a[k];
      }
      return;
    }
    const bool stepping = st.live && st.t_ep < e.L;
    if (st.live && !stepping) {  // done env without autoreset: ignored
      st.bad = true;
      if (p.o.reward) p.o.reward[ti] = 0.f;
      if (p.o.done) p.o.done[ti] = 1;
    }
    GroupSlots* gs = reinterpret_cast<GroupSlots*>(stg + kOffS);
    group_apply(
        gs, st.round, st.d, stepping, st.gtid, st.bar_id,
        [&](int k) {
          stage_row(p, k, st.gtid, region(stg, st.sb));
          st.kcur = k;
        },
        [&]() {
          const double* pd = reinterpret_cast<const double*>(region(stg, st.sb) + kOffP);
          FIN_TR(threadIdx.x == 128, t, 19);
          const double v = st.vc;
          // post-sell holdings for the rare exact buy redo: [octet][row] in the tile's A operand
          // past the observation columns (free while the env steps: the layer-3 MMAs have completed
          // and the next observation only fills the first kTileM x kIn bf16)
          uint4* save = reinterpret_cast<uint4*>(a_tile + kSaveOff) + st.gtid;
          clamp_actions<KA>(e, a, st.oor, (LOG && p.o.actions) ? p.o.actions + ti * KA : nullptr);
          stock_trade<KA>(e, st.b, st.h, pd, KP4, pack_acts<KA>(a), save, tc::kTileM);
          const double vn = stock_mark<KA>(st.b, st.h, pd + kRowPN * KP4, KP4);
          st.vc = vn;
          FIN_TR(threadIdx.x == 128, t, 20);
          st.t_ep += 1;
          const bool done = st.t_ep == e.L;
          const float r = stock_reward(e, v, vn);
          st.rsum += (double)r;
          if (p.o.reward) p.o.reward[ti] = r;
          if (p.o.done) p.o.done[ti] = done ? 1 : 0;
          if (LOG && p.o.cash) p.o.cash[ti] = st.b;
          if (LOG && p.o.asset) p.o.asset[ti] = vn;
          if (LOG && p.o.hold) {
#pragma unroll
            for (int k = 0; k < KA; ++k) p.o.hold[ti * KA + k] = (int16_t)st.h[k];
          }
          MetricAcc m = m_get(st);
          metric_push(m, vn);
          FIN_TR(threadIdx.x == 128, t, 21);
          if (done) {
            double em[3];
            metric_finish(m, 252.0, 0.0, em);
            if (p.o.ep_metrics && st.cnt < p.o.ep_capacity) {
              double* dst = p.o.ep_metrics + ((size_t)st.cnt * e.N + env) * 3;
              dst[0] = em[0]; dst[1] = em[1]; dst[2] = em[2];
            }
            ++st.cnt;
            agg_episode_g(e.agg_env + env, (size_t)e.N, em);
            if (e.autoreset) {
              st.b = e.cash0;
#pragma unroll
              for (int k = 0; k < KA; ++k) st.h[k] = 0;
#pragma unroll
              for (int k = 0; k < KOU; ++k) st.ou[k] = 0.f;
              if (ENS && p.n_ddpg > 1)
                for (int q = 0; q < p.n_ddpg; ++q)
                  for (int k = 0; k < KA; ++k) e.ou[((size_t)q * e.K + k) * e.N + env] = 0.f;
              st.t_ep = 0;
              st.vc = e.cash0;
              if (e.wadv) st.w = (st.w + 1) % e.W;
              metric_start(m, e.cash0);
            }
          }
          m_put(st, m);
        },
        st.zsm ? st.d0 : -1);   // uniform tile: its day's rows were staged by stage()
  }

  __device__ __forceinline__ static void finalize(State& st, const TcParams& p, int env, int gtid, int bar_id,
                                                  int tile) {
    finalize_rows(st, p, env, gtid, bar_id, tile, blockIdx.x * p.tiles_per_cta + tile, true);
  }
  // end of a segment of the balanced schedule: the state goes back to the env; the tile's
  // aggregate row (indexed by the tile, as in the one-tile-per-CTA layout) only at its end
  __device__ __forceinline__ static void finalize_seg(State& st, const TcParams& p, int env, int gtid, int bar_id,
                                                      int tile, int t1) {
    const bool last = t1 == p.T;
    if (!last && st.live && !(LOG && p.act_only)) {
      p.e.seg_cnt[env] = st.cnt;
      p.e.seg_rsum[env] = st.rsum;
    }
    finalize_rows(st, p, env, gtid, bar_id, 0, tile, last);
  }
  __device__ __forceinline__ static void finalize_rows(State& st, const TcParams& p, int env, int gtid, int bar_id,
                                                       int group, int agg_row, bool last) {
    const EnvDev& e = p.e;
    if (LOG && p.act_only) {   // fin_ensemble_act: only the single-DDPG register state may be committed
      if (ENS && p.commit_ou && p.n_ddpg == 1 && st.live) {
#pragma unroll
        for (int k = 0; k < KOU; ++k) e.ou[(size_t)k * e.N + env] = st.ou[k];
      }
      return;
    }
    if (st.live) {
      e.cash[env] = st.b;
      e.vcur[env] = st.vc;
      store_hold<KA>(e, env, st.h);
      e.t_ep[env] = st.t_ep;
      e.window[env] = st.w;
      const MetricAcc m = m_get(st);
      e.m_v0[env] = m.v0; e.m_vprev[env] = m.vprev; e.m_peak[env] = m.peak; e.m_mdd[env] = m.mdd;
      e.m_mean[env] = m.mean; e.m_m2[env] = m.m2; e.m_n[env] = m.n;
      if (ENS && p.n_ddpg == 1) {
#pragma unroll
        for (int k = 0; k < KOU; ++k) e.ou[(size_t)k * e.N + env] = st.ou[k];
      }
      if (p.o.ep_count) p.o.ep_count[env] = st.cnt;
      if (st.oor) set_flag(e, FIN_FLAG_ACTION_RANGE);
      if (st.bad) set_flag(e, FIN_FLAG_BAD_INDEX);
      if (st.nonfinite) set_flag(e, FIN_FLAG_NONFINITE);
    }
    if (!last) return;
    AggAcc agg;
    agg_init(agg);
    if (st.live) {
#pragma unroll
      for (int j = 0; j < FIN_AGG_LEN; ++j) agg.s[j] = e.agg_env[(size_t)j * e.N + env];
    }
    agg.s[FIN_AGG_SUM_REWARD] = st.rsum;
    if (p.o.agg_partial)
      agg_group_write(agg, p.o.agg_partial + (size_t)agg_row * FIN_AGG_LEN, gtid, bar_id, group);
  }
};

// ---------------------------------------------------------------- K7 probe
// Obs = StockObs<..> for the factored stock nets (X = the private columns of x, the
// shared columns enter through z1s), void for the crypto Q-net (X = x).
template <class Plan, class Obs>
struct ProbeOps {
  static constexpr bool kStream = false;
  static constexpr int kStageBytes = 16;
  static constexpr bool kStageBias = true;
  static constexpr bool kSplitOK = false;
  static constexpr bool kSplitAddend = false;
  static constexpr bool kSegments = false;
  static constexpr bool kL1Init = false;
  static constexpr int kOffB = 0;
  static constexpr int kOffImgT = 0;
  static constexpr bool kL1Bcast = false;   // (crypto only: broadcast layer-1 A operand)
  static constexpr bool kEpiPipe = false;
  static constexpr bool kFactored = !std::is_void<Obs>::value;
  struct State {
    int b;
  };
  __device__ __forceinline__ static int col_of(int j) {
    if constexpr (kFactored) return j < Obs::kEnv ? Obs::env_col(j) : -1;
    else return j;
  }
  __device__ __forceinline__ static void init(State& st, const TcParams& p, int env, int row) { st.b = env; }
  __device__ __forceinline__ static void stage(State&, const TcParams&, int, int, int, uint8_t*, int) {}
  __device__ __forceinline__ static const float* l1_addend(State& st, const TcParams& p, int m, uint8_t*) {
    // never null for a factored net (the epilogue's addend branch must be warp-uniform):
    // rows past B read row 0 and their outputs are dropped
    if constexpr (kFactored) return p.z1s + (size_t)(st.b < p.B ? st.b : 0) * Plan::kH1;
    else return nullptr;
  }
  __device__ __forceinline__ static void build_obs(State& st, const TcParams& p, int env, int row, int t, int m,
                                                   uint32_t xa, uint8_t*) {
    constexpr int KT8 = Plan::kIn / 8;
    const bool live = st.b < p.B;
    const uint16_t* x = p.x_in + (size_t)st.b * p.in_dim;
#pragma unroll 1
    for (int c = 0; c < KT8; ++c) {
      uint32_t w4[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int c0 = col_of(8 * c + 2 * j), c1 = col_of(8 * c + 2 * j + 1);
        const uint32_t lo = (live && c0 >= 0 && c0 < p.in_dim) ? x[c0] : 0u;
        const uint32_t hi = (live && c1 >= 0 && c1 < p.in_dim) ? x[c1] : 0u;
        w4[j] = lo | (hi << 16);
      }
      tc::sts128(xa + tc::cm_off(row, c, KT8), w4[0], w4[1], w4[2], w4[3]);
    }
  }
  __device__ __forceinline__ static uint16_t* hidden_ptr(State& st, const TcParams& p, int env, int t, int m, int l,
                                                         int hid) {
    if (st.b >= p.B || !p.hid_out) return nullptr;
    return p.hid_out + ((size_t)st.b * Plan::kNH + l) * hid;
  }
  __device__ __forceinline__ static void prepare(State&, const TcParams&, int, int, int) {}
  __device__ __forceinline__ static void consume(State& st, const TcParams& p, int env, int t, int m,
                                                 const float* z) {
    if (st.b >= p.B) return;
    for (int k = 0; k < p.out_dim; ++k) p.z_out[(size_t)st.b * p.out_dim + k] = z[k];
  }
  __device__ __forceinline__ static void finish_step(State&, const TcParams&, int, int, uint8_t*, uint8_t*) {}
  __device__ __forceinline__ static void finalize(State&, const TcParams&, int, int, int, int) {}
};

}  // namespace

namespace fin {

int num_sms() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
  }
  return n;
}

// CTA layout for a launch when there are more tiles than SMs.  Default ("dual"): two
// CTAs per SM with one tile each -- each tile has its own weight stream (2-slot ring)
// and MMA issuer, so one tile's tensor-core phases overlap the other's env work (with
// two tiles sharing one stream they advance in lockstep and the tensor core idles
// during every env phase); the env warpgroup still gets 216 registers (setmaxnreg).
// "pair" (FIN_TC_MODE=pair): one CTA with two tiles sharing each streamed weight stage.
// With fewer tiles than SMs: one tile per CTA (latency-bound: spread over the SMs).
#ifndef FIN_DUAL_RING
#define FIN_DUAL_RING 2   // weight-ring slots per CTA in the dual layout
#endif
constexpr int kDualRing = FIN_DUAL_RING;
template <class Plan, bool RES, class Ops>
cudaError_t launch_auto(const TcParams& p, int n_envs, int* tiles, cudaStream_t s) {
  const int n_tiles = (n_envs + tc::kTileM - 1) / tc::kTileM;
  if constexpr (Ops::kStream) {   // streamed noise: small N, one tile per CTA only
    *tiles = 1;
    // streamed-weight plan: the hidden epilogues split over two warpgroups (FIN_SPLIT=0: not)
    const char* sp = getenv("FIN_SPLIT");
    if constexpr (!RES)
      if (!(sp && sp[0] == '0') && tc::Smem<Plan, RES, 1, Ops>::total(p.M) + 1024 <= tc::kSmemLimit)
        return tc::launch<Plan, RES, 1, Ops, tc::kRing, 1, 2>(p, n_envs, s);
    return tc::launch<Plan, RES, 1, Ops>(p, n_envs, s);
  }
  const char* mode = getenv("FIN_TC_MODE");   // read per launch (tests switch it)
  const bool pair = mode && mode[0] == 'p';
  if constexpr (!RES) {
    // two CTAs must fit one SM's shared memory (the bias of up to 4 members is staged)
    const bool fits = 2 * tc::Smem<Plan, RES, 1, Ops, kDualRing>::total(p.M) <= tc::kSmemLimit;
    if (!pair && fits && n_tiles > num_sms()) {
      *tiles = 1;
      return tc::launch<Plan, RES, 1, Ops, kDualRing, 2>(p, n_envs, s, p.q_ctr ? p.seg_grid : 0);
    }
  }
  if (n_tiles > num_sms() && p.M <= tc::Smem<Plan, RES, 2, Ops>::max_members()) {
    *tiles = 2;
    return tc::launch<Plan, RES, 2, Ops>(p, n_envs, s);
  }
  *tiles = 1;
  return tc::launch<Plan, RES, 1, Ops>(p, n_envs, s);
}

// The balanced persistent schedule of a dual-layout launch: the grid of
// resident CTAs (2 per SM) when there are more tiles than that, else 0 (one tile per CTA).
// FIN_SEG=0 disables it (A/B runs).
template <class Plan, bool RES, class Ops>
int seg_grid_auto(const TcParams& p, int n_envs) {
  if constexpr (RES || !Ops::kSegments) {
    return 0;
  } else {
    const char* mode = getenv("FIN_TC_MODE");
    const char* seg = getenv("FIN_SEG");
    if ((mode && mode[0] == 'p') || (seg && seg[0] == '0') || p.act_only) return 0;
    const int n_tiles = (n_envs + tc::kTileM - 1) / tc::kTileM;
    if (2 * tc::Smem<Plan, RES, 1, Ops, kDualRing>::total(p.M) > tc::kSmemLimit || n_tiles <= num_sms()) return 0;
    // two CTAs per SM (the dual layout's __launch_bounds__ minimum and shared-memory fit);
    // the cooperative launch verifies that all of them are resident (else: plain grid)
    const int grid = 2 * num_sms();
    return n_tiles > grid ? grid : 0;
  }
}

template <class Plan, bool RES, class Ops>
struct StockKernel {
  using P = Plan;
  static constexpr bool R = RES;
  using O = Ops;
};

// net: 0 = PlanStockC1 (K=30, I=8), 1 = PlanStockSmall (K=4, I=4), 3 = PlanStockPaper (K=30, I=8;
// the paper's 64-32 net, 10 KB of weights: resident in shared memory, env-issued MMAs)
template <class F>
auto dispatch_stock(int net, const tc::TcParams& p, F&& f) -> decltype(f(StockKernel<PlanStockC1, false,
                                                                            StockOps<30, 8, PlanStockC1, false>>{})) {
  const bool single = p.M == 1 && p.kinds[0] != FIN_DDPG_OU;
  const bool logs = p.act_only || p.o.mlp_out || p.o.mlp_hidden || p.o.cash || p.o.asset || p.o.hold || p.o.actions ||
                    p.o.obs_private || p.o.day;
  if (p.noise_ready) {   // streamed small-N noise (api.cu plan_noise): the STREAM instantiations
    if (FIN_STREAM_EARLY && net == 0 && single && !logs && p.noise_mode == FIN_NOISE_PHILOX)
      return f(StockKernel<PlanStockC1, false, StockOps<30, 8, PlanStockC1, false, false, true, true>>{});
    if (net == 0 && single && !logs)
      return f(StockKernel<PlanStockC1, false, StockOps<30, 8, PlanStockC1, false, false, true>>{});
    if (net == 0 && single) return f(StockKernel<PlanStockC1, false, StockOps<30, 8, PlanStockC1, false, true, true>>{});
    if (net == 0) return f(StockKernel<PlanStockC1, false, StockOps<30, 8, PlanStockC1, true, true, true>>{});
    if (net == 3 && single && !logs)
      return f(StockKernel<PlanStockPaper, true, StockOps<30, 8, PlanStockPaper, false, false, true>>{});
    if (net == 3 && single)
      return f(StockKernel<PlanStockPaper, true, StockOps<30, 8, PlanStockPaper, false, true, true>>{});
    if (net == 3) return f(StockKernel<PlanStockPaper, true, StockOps<30, 8, PlanStockPaper, true, true, true>>{});
    return f(StockKernel<PlanStockSmall, true, StockOps<4, 4, PlanStockSmall, true, true, true>>{});
  }
  if (net == 0 && single && !logs) return f(StockKernel<PlanStockC1, false, StockOps<30, 8, PlanStockC1, false, false>>{});
  if (net == 0 && single) return f(StockKernel<PlanStockC1, false, StockOps<30, 8, PlanStockC1, false>>{});
  if (net == 0) return f(StockKernel<PlanStockC1, false, StockOps<30, 8, PlanStockC1, true>>{});
  if (net == 3 && single && !logs)
    return f(StockKernel<PlanStockPaper, true, StockOps<30, 8, PlanStockPaper, false, false>>{});
  if (net == 3 && single) return f(StockKernel<PlanStockPaper, true, StockOps<30, 8, PlanStockPaper, false>>{});
  if (net == 3) return f(StockKernel<PlanStockPaper, true, StockOps<30, 8, PlanStockPaper, true>>{});
  return f(StockKernel<PlanStockSmall, true, StockOps<4, 4, PlanStockSmall, true>>{});
}

cudaError_t launch_stock_rollout(int net, const tc::TcParams& p, int n_envs, int* tiles, cudaStream_t s) {
  if (net != 0 && net != 1 && net != 3) return cudaErrorInvalidValue;
  return dispatch_stock(net, p, [&](auto k) {
    using K = decltype(k);
    return launch_auto<typename K::P, K::R, typename K::O>(p, n_envs, tiles, s);
  });
}

int stock_seg_grid(int net, const tc::TcParams& p, int n_envs) {
  if (net != 0 && net != 1 && net != 3) return 0;
  return dispatch_stock(net, p, [&](auto k) {
    using K = decltype(k);
    return seg_grid_auto<typename K::P, K::R, typename K::O>(p, n_envs);
  });
}

// net: 0 = PlanStockC1, 1 = PlanStockSmall, 2 = PlanCrypto, 3 = PlanStockPaper, 4 = PlanCryptoPaper
cudaError_t launch_mlp_probe(int net, const tc::TcParams& p, int n_rows, cudaStream_t s) {
  int tiles = 0;
  if (net == 0) return launch_auto<PlanStockC1, false, ProbeOps<PlanStockC1, ObsC1>>(p, n_rows, &tiles, s);
  if (net == 1) return launch_auto<PlanStockSmall, true, ProbeOps<PlanStockSmall, ObsSmall>>(p, n_rows, &tiles, s);
  if (net == 2) return launch_auto<PlanCrypto, true, ProbeOps<PlanCrypto, void>>(p, n_rows, &tiles, s);
  if (net == 3) return launch_auto<PlanStockPaper, true, ProbeOps<PlanStockPaper, ObsC1>>(p, n_rows, &tiles, s);
  if (net == 4) return launch_auto<PlanCryptoPaper, true, ProbeOps<PlanCryptoPaper, void>>(p, n_rows, &tiles, s);
  return cudaErrorInvalidValue;
}

}  // namespace fin
