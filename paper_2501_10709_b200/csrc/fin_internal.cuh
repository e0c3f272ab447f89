// fin_internal.cuh -- device-side handle layout and shared device helpers of
// libfinenv.so.  Nothing here is shared with oracle/ (which is independent
// Python); this is the CUDA product path only.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <cstdio>

#include "../../include/fin.h"

#define FIN_HOLD_MAX 32767   // holdings are int16 (reading R-HOLD)
#define FIN_MAX_ASSETS 32
#define FIN_MAX_MEMBERS 32   // ensemble members per rollout (Ensemble-3 = 30)
#define FIN_STAGE_MEMBERS 4  // members whose bias / z1s rows live in shared memory (the rest: L2)

// Device-side bounds checks (compute-sanitizer is closed on this pool): a build with
// FIN_NVCC_FLAGS=-DFIN_CHECKS=1 traps on any violated index assumption of the hot kernels
// (trajectory rows, market days, work items, shared-memory staging); production builds
// compile them out.
#ifndef FIN_CHECKS
#define FIN_CHECKS 0
#endif
#if FIN_CHECKS
#define FIN_CHECK(cond)                                                                          \
  do {                                                                                           \
    if (!(cond)) {                                                                               \
      printf("FIN_CHECK failed: %s (%s:%d) block %d thread %d\n", #cond, __FILE__, __LINE__,     \
             (int)blockIdx.x, (int)threadIdx.x);                                                 \
      asm volatile("trap;");                                                                     \
    }                                                                                            \
  } while (0)
#else
#define FIN_CHECK(cond) \
  do {                  \
  } while (0)
#endif

// Flat, by-value kernel parameter block describing one env handle on the device.
// Internal state is SoA: element [k][i] of a [K][N] array is at k*N + i.
struct EnvDev {
  // ---- configuration (fin_env_config, validated on the host)
  int32_t task, N, K, I, rows, L;
  int32_t wstride, woff, W, wblock, wbase, wadv;
  int32_t max_trade, max_hold, autoreset;
  int32_t kp;            // K padded to a multiple of 4 (market channel stride)
  int32_t row_floats;    // floats per market row: (2+I)*kp (stock) or 144 (crypto)
  double cash0, cost, scale;
  double rcash0;
  float rmax_trade;      // fl(1 / max_trade) (host division): the observation's h / max_trade
  float rmax_hold;       // crypto: fl(1 / max_hold) (host division): the observation's tau / max_hold         // fl(1 / cash0) (host division): the observation's b / b0 by Markstein's correction
  double up, dn;         // fl(1 + cost), fl(1 - cost)
  float noise_std, ou_theta, ou_sigma, eps;
  uint64_t seed;
  int64_t env_offset;
  int64_t t_global;      // global step counter (Philox counter word), advanced per step
  const float* market;   // [rows][row_floats]
  const double* px;      // stock: [rows][kPriceRows][kp] f64 price rows of each day (env_stock.cuh)
  // ---- state (library-owned device memory)
  double* cash;          // [N]
  double* vcur;          // [N] stock: total asset v = b + sum_k h_k p_k at the env's current day
                         //     (P:132), cached: a step's pre-trade v is the previous post-trade v
  int16_t* hold;         // stock: asset octets [ceil(K/8)][N][8] (hold_at); crypto: [N] position in {-1,0,1}
  int32_t* t_ep;         // [N]
  int32_t* window;       // [N]
  int32_t* tau;          // [N] crypto holding time
  float* ou;             // [ou_slots][K][N] DDPG OU noise state (slot i: the i-th DDPG member of a call)
  int32_t ou_slots;      // allocated slots (grown on demand by fin_rollout)
  // online episode-metric state (persisted across calls)
  double* m_v0;          // equity at episode start
  double* m_vprev;       // last equity
  double* m_peak;        // running peak
  double* m_mdd;         // running min drawdown (<= 0)
  double* m_mean;        // Welford mean of returns
  double* m_m2;          // Welford M2
  int32_t* m_n;          // number of returns
  double* agg_env;       // [FIN_AGG_LEN][N] per-env aggregate partials of the running rollout (fused
                         // stock rollout: touched once per episode, kept out of the registers)
  int32_t* seg_cnt;      // [N] balanced schedule: episodes completed so far in this call (head -> tail)
  double* seg_rsum;      // [N] balanced schedule: reward sum so far in this call (head -> tail)
  uint32_t* seg_flag;    // [ceil(N / 128)] balanced schedule: epoch of the last published head per tile
  uint32_t* flags;       // sticky device error word; flags[FIN_CTR_*] are event counters (fin_env_counters)
};
// counters after the flags word (same 64-B block)
#define FIN_CTR_EXACT_REDO 4
// streamed small-N noise: steps per published group (k_stream_noise / noise_wait)
#define FIN_NOISE_GROUP 8   // stock: steps whose buys took the exact out-of-line affordability path

struct TrajDev {
  float* reward;
  uint8_t* done;
  int16_t* actions;
  double* cash;
  int16_t* hold;
  double* asset;
  float* mlp_out;
  uint16_t* mlp_hidden;
  double* ep_metrics;
  int32_t* ep_count;
  int32_t ep_capacity;
  double* agg_partial;   // [gridDim][FIN_AGG_LEN] scratch, reduced by k_agg_finalize
  uint16_t* obs_private; // [T][N][P] bf16 bits of the env-private observation entries (stock)
  int32_t* day;          // [T][N] market day of the step (stock)
};

// ----------------------------------------------------------------- exact fp64
// Every env-side float64 operation uses explicit round-to-nearest intrinsics so
// the compiler can never contract a*b+c into an FMA: the op order and rounding
// equal DESIGN.md §4.2 (the oracle's order) by construction.
__device__ __forceinline__ double fadd64(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double fsub64(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double fmul64(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double fdiv64(double a, double b) { return __ddiv_rn(a, b); }
// a / b correctly rounded from y = fl(1 / b) without a call (the slow-path CALL of __ddiv_rn makes
// ptxas keep the env state out of its caller-saved registers): q = fl(a y), r = a - b q exactly (fma),
// q' = fl(q + r y) -- Markstein's correction, the correctly rounded quotient whenever y is the
// correctly rounded reciprocal and nothing over- or underflows (b = b0 > 0 here, |a| < 2^1000)
__device__ __forceinline__ double fdiv64_rcp(double a, double b, double y) {
  const double q = __dmul_rn(a, y);
  const double r = __fma_rn(-q, b, a);
  return __fma_rn(r, y, q);
}

// Price rows of day d, precomputed on the host at create (px), staged per step:
//   P  = p_d   close of the execution day (exact widening of the fp32 market)
//   U  = u_d   = fl(p_d * (1 + c)), the buy price per share
//   MP = -2^52 p_d,  MU = -2^52 u_d   (exact scalings)
//   RU = fl(fl(1 / u_d) (1 + 2^-40))  (estimate of the affordable count only, biased up)
//   PN = p_d+1, MPN = -2^52 p_d+1     (marking day; 0 on the last row)
//   META[0] = min_k u_k               (cash below it buys nothing more this step)
enum { kRowP = 0, kRowU, kRowMP, kRowMU, kRowRU, kRowPN, kRowMPN, kRowMeta, kPriceRows };

// Exact int -> double for 0 <= n < 2^31 on the fp64 pipe: the bit pattern
// 0x43300000:n is 2^52 + n exactly and subtracting 2^52 is exact.  Replaces the
// I2F.F64 conversion, which runs on the narrow XU pipe (ncu round 1: XU was the
// busiest pipe of the step kernels).
__device__ __forceinline__ double nn2d(int n) {
  return __dsub_rn(__hiloint2double(0x43300000, n), 4503599627370496.0);
}

// Stock holdings layout: asset octets, element (k, i) at ((k / 8) * N + i) * 8 + k % 8,
// so one env's 8 assets are one 16-byte vector and a warp's octet row is 512
// contiguous bytes.  Padding assets (k >= K) are kept at 0.
__device__ __forceinline__ size_t hold_at(int N, int k, int i) {
  return (((size_t)(k >> 3) * N + i) << 3) + (k & 7);
}
template <int KA>
__device__ __forceinline__ void load_hold(const EnvDev& e, int i, int (&h)[KA]) {
  const uint4* q = reinterpret_cast<const uint4*>(e.hold);
#pragma unroll
  for (int o = 0; o < (KA + 7) / 8; ++o) {
    const uint4 v = q[(size_t)o * e.N + i];
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int j = 0; j < 8; ++j)
      if (8 * o + j < KA) h[8 * o + j] = (int)((j & 1) ? (w[j >> 1] >> 16) : (w[j >> 1] & 0xffffu));
  }
}
template <int KA>
__device__ __forceinline__ void store_hold(const EnvDev& e, int i, const int (&h)[KA]) {
  uint4* q = reinterpret_cast<uint4*>(e.hold);
#pragma unroll
  for (int o = 0; o < (KA + 7) / 8; ++o) {
    uint32_t w[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int k0 = 8 * o + 2 * j, k1 = k0 + 1;
      const uint32_t lo = k0 < KA ? (uint32_t)h[k0] : 0u, hi = k1 < KA ? (uint32_t)h[k1] : 0u;
      w[j] = __byte_perm(lo, hi, 0x5410);
    }
    q[(size_t)o * e.N + i] = make_uint4(w[0], w[1], w[2], w[3]);
  }
}

__device__ __forceinline__ void set_flag(const EnvDev& e, uint32_t bit) { atomicOr(e.flags, bit); }

// ----------------------------------------------------------------- windows (R10)
__device__ __forceinline__ int32_t window_of(const EnvDev& e, int64_t g) {
  int64_t w = ((int64_t)e.wbase + g / e.wblock) % e.W;
  return (int32_t)w;
}
__device__ __forceinline__ int32_t day_of(const EnvDev& e, int32_t w, int32_t t) {
  return e.woff + w * e.wstride + t;
}

// h / d correctly rounded in fp32 for integer |h| < 2^24 and d >= 1, without the IEEE
// division subroutine: q = h * (1/d) then one FMA residual correction (exhaustively
// checked for |h| < 2^15 and the divisors used here); the bf16 of the
// result therefore equals q(h / d) of the oracle.
__device__ __forceinline__ float div_int_f32(int h, float d, float inv_d) {
  const float hf = (float)h;
  const float q = __fmul_rn(hf, inv_d);
  const float r = __fmaf_rn(-q, d, hf);
  return __fmaf_rn(r, inv_d, q);
}
// ----------------------------------------------------------------- online metrics
// Per-episode accumulators: equity v_0 .. v_L, returns
// r_t = v_t / v_{t-1} - 1 (Welford mean / M2), running peak and min drawdown.
struct MetricAcc {
  double v0, vprev, peak, mdd, mean, m2;
  int32_t n;
};

__device__ __forceinline__ void metric_start(MetricAcc& m, double v) {
  m.v0 = v; m.vprev = v; m.peak = v; m.mdd = 0.0; m.mean = 0.0; m.m2 = 0.0; m.n = 0;
}

// 1 / x from the MUFU seed and two Newton steps (<= 1 ulp): a fraction of the cost of a
// correctly rounded division or __drcp_rn
__device__ __forceinline__ double rcp_nr(double x) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  double e = __fma_rn(-x, y, 1.0);
  y = __fma_rn(y, e, y);
  e = __fma_rn(-x, y, 1.0);
  return __fma_rn(y, e, y);
}

// 1 / sqrt(x) for normal x > 0 from the MUFU seed and two Newton steps (~1 ulp), inline: the
// library rsqrt carries a slow-path CALL, which makes ptxas keep the rollout's env state out of
// caller-saved registers (spills around every step)
__device__ __forceinline__ double rsqrt_nr(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  double h = __dmul_rn(0.5, x);
  double e = __fma_rn(-h, __dmul_rn(y, y), 0.5);
  y = __fma_rn(y, e, y);
  e = __fma_rn(-h, __dmul_rn(y, y), 0.5);
  return __fma_rn(y, e, y);
}

// Branch-free, no division: r = (v - v_prev) * rcp(v_prev) (v - v_prev exact, within
// ~2 ulp of v / v_prev - 1), Welford with rcp(n), drawdown (v - peak) * rcp(peak) with
// the running peak (exactly 0 at a peak).  The earlier form divided, and its "new
// maximum drawdown" branch was taken by some env of nearly every warp.
__device__ __forceinline__ void metric_push(MetricAcc& m, double v) {
  const double r = fmul64(fsub64(v, m.vprev), rcp_nr(m.vprev));
  m.n += 1;
  const double delta = fsub64(r, m.mean);
  m.mean = fadd64(m.mean, fmul64(delta, rcp_nr(nn2d(m.n))));
  m.m2 = fadd64(m.m2, fmul64(delta, fsub64(r, m.mean)));
  m.peak = fmax(m.peak, v);
  m.mdd = fmin(m.mdd, fmul64(fsub64(v, m.peak), rcp_nr(m.peak)));
  m.vprev = v;
}

// The same push with its three reciprocals formed from the pre-step state (metric_rcps: before
// the trade, off the serial cash chain): rv = rcp(v_prev), rn = rcp(n + 1), rp = rcp(peak).  The
// drawdown uses the old peak: when v exceeds it the new peak is v and the term is 0 either way.
struct MetricRcp {
  double rv, rn, rp;
};
__device__ __forceinline__ MetricRcp metric_rcps(double vprev, double peak, int n) {
  return MetricRcp{rcp_nr(vprev), rcp_nr(nn2d(n + 1)), rcp_nr(peak)};
}
__device__ __forceinline__ void metric_push_pre(MetricAcc& m, double v, const MetricRcp& q) {
  const double r = fmul64(fsub64(v, m.vprev), q.rv);
  m.n += 1;
  const double delta = fsub64(r, m.mean);
  m.mean = fadd64(m.mean, fmul64(delta, q.rn));
  m.m2 = fadd64(m.m2, fmul64(delta, fsub64(r, m.mean)));
  const double dd = v > m.peak ? 0.0 : fmul64(fsub64(v, m.peak), q.rp);
  m.peak = fmax(m.peak, v);
  m.mdd = fmin(m.mdd, dd);
  m.vprev = v;
}

// (cum, sharpe, mdd) of a finished episode; Sharpe = sqrt(ppy) mean / std(ddof 1),
// NaN when n < 2 or std == 0 (reading R21).  Reciprocals instead of divisions (each
// within an ulp): when episodes end at different steps across a warp this runs
// divergently on most steps, so its cost matters.
__device__ __forceinline__ void metric_finish(const MetricAcc& m, double ppy, double rf, double out[3]) {
  out[0] = fmul64(fsub64(m.vprev, m.v0), rcp_nr(m.v0));   // exactly 0 for a flat curve
  double sh = __longlong_as_double(0x7ff8000000000000ULL);
  if (m.n >= 2) {
    const double var = fmul64(m.m2, rcp_nr(nn2d(m.n - 1)));
    if (var > 0.0) sh = fmul64(fmul64(sqrt(ppy), fsub64(m.mean, rf)), rsqrt_nr(var));
  }
  out[1] = sh;
  out[2] = m.mdd;
}

// ----------------------------------------------------------------- block aggregate
// Per-block partial of the FIN_AGG_* vector, reduced across the block in smem in a
// fixed order (deterministic), written to agg_partial[blockIdx.x][.].
struct AggAcc {
  double s[FIN_AGG_LEN];
};
__device__ __forceinline__ void agg_init(AggAcc& a) {
#pragma unroll
  for (int j = 0; j < FIN_AGG_NSUM; ++j) a.s[j] = 0.0;
  a.s[FIN_AGG_MIN_MDD] = __longlong_as_double(0x7ff0000000000000ULL);  // +inf
  a.s[7] = __longlong_as_double(0x7ff0000000000000ULL);
}
__device__ __forceinline__ void agg_episode(AggAcc& a, const double m[3]) {
  a.s[FIN_AGG_EPISODES] += 1.0;
  a.s[FIN_AGG_SUM_CUM] += m[0];
  if (isfinite(m[1])) { a.s[FIN_AGG_SUM_SHARPE] += m[1]; a.s[FIN_AGG_N_SHARPE] += 1.0; }
  a.s[FIN_AGG_SUM_MDD] += m[2];
  a.s[FIN_AGG_MIN_MDD] = fmin(a.s[FIN_AGG_MIN_MDD], m[2]);
  a.s[7] = fmin(a.s[7], m[0]);
}

// the same accumulator kept in global memory, element j of env i at base[j * stride]
__device__ __forceinline__ void agg_init_g(double* base, size_t stride) {
  AggAcc a;
  agg_init(a);
#pragma unroll
  for (int j = 0; j < FIN_AGG_LEN; ++j) base[j * stride] = a.s[j];
}
__device__ __forceinline__ void agg_episode_g(double* base, size_t stride, const double m[3]) {
  AggAcc a;
#pragma unroll
  for (int j = 0; j < FIN_AGG_LEN; ++j) a.s[j] = base[j * stride];
  agg_episode(a, m);
#pragma unroll
  for (int j = 0; j < FIN_AGG_LEN; ++j) base[j * stride] = a.s[j];
}

// Block-wide deterministic reduction (blockDim.x a multiple of 32, <= 1024).
__device__ inline void agg_block_write(const AggAcc& a, double* partial_row) {
  __shared__ double red[32][FIN_AGG_LEN];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  double v[FIN_AGG_LEN];
#pragma unroll
  for (int j = 0; j < FIN_AGG_LEN; ++j) v[j] = a.s[j];
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
#pragma unroll
    for (int j = 0; j < FIN_AGG_LEN; ++j) {
      double o = __shfl_down_sync(0xffffffffu, v[j], off);
      v[j] = (j < FIN_AGG_NSUM) ? v[j] + o : fmin(v[j], o);
    }
  }
  if (lane == 0) {
#pragma unroll
    for (int j = 0; j < FIN_AGG_LEN; ++j) red[wid][j] = v[j];
  }
  __syncthreads();
  if (threadIdx.x < FIN_AGG_LEN) {
    const int j = threadIdx.x;
    double s = red[0][j];
    for (int w = 1; w < nw; ++w) s = (j < FIN_AGG_NSUM) ? s + red[w][j] : fmin(s, red[w][j]);
    partial_row[j] = s;
  }
}

// Same reduction for a 128-thread warpgroup that synchronises on named barrier
// ``bar_id`` (used inside warp-specialised kernels where other warps are busy).
__device__ inline void agg_group_write(const AggAcc& a, double* partial_row, int group_tid, int bar_id,
                                       int group = 0) {
  __shared__ double red_all[2][4][FIN_AGG_LEN];   // one scratch per warpgroup (<= 2 per CTA)
  double (*red_g)[FIN_AGG_LEN] = red_all[group & 1];
  const int lane = group_tid & 31, wid = group_tid >> 5;
  double v[FIN_AGG_LEN];
#pragma unroll
  for (int j = 0; j < FIN_AGG_LEN; ++j) v[j] = a.s[j];
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
#pragma unroll
    for (int j = 0; j < FIN_AGG_LEN; ++j) {
      double o = __shfl_down_sync(0xffffffffu, v[j], off);
      v[j] = (j < FIN_AGG_NSUM) ? v[j] + o : fmin(v[j], o);
    }
  }
  if (lane == 0) {
#pragma unroll
    for (int j = 0; j < FIN_AGG_LEN; ++j) red_g[wid][j] = v[j];
  }
  asm volatile("bar.sync %0, %1;" ::"r"(bar_id), "r"(128) : "memory");
  if (group_tid < FIN_AGG_LEN) {
    const int j = group_tid;
    double s = red_g[0][j];
    for (int w = 1; w < 4; ++w) s = (j < FIN_AGG_NSUM) ? s + red_g[w][j] : fmin(s, red_g[w][j]);
    partial_row[j] = s;
  }
}

// round half away from zero of an fp32 value (R18), exact: y - trunc(y) is exact
__device__ __forceinline__ int rha_f32(float y) {
  const float n = truncf(y);
  const float f = fabsf(__fsub_rn(y, n));
  int r = (int)n;
  if (f >= 0.5f) r += (y >= 0.f) ? 1 : -1;
  return r;
}

// ----------------------------------------------------------------- host launchers
namespace fin {
cudaError_t launch_stock_reset(const EnvDev& e, const uint8_t* mask, cudaStream_t s);
cudaError_t launch_stock_step(const EnvDev& e, const int16_t* actions, const TrajDev& o, cudaStream_t s);
cudaError_t launch_stock_replay(const EnvDev& e, const int16_t* actions, int T, const TrajDev& o,
                                int* n_blocks, cudaStream_t s);
cudaError_t launch_stock_get_state(const EnvDev& e, double* cash, int16_t* hold, double* asset,
                                   int32_t* t_ep, int32_t* window, cudaStream_t s);
cudaError_t launch_stock_set_state(const EnvDev& e, const double* cash, const int16_t* hold,
                                   const int32_t* t_ep, const int32_t* window, cudaStream_t s);
cudaError_t launch_crypto_reset(const EnvDev& e, const uint8_t* mask, cudaStream_t s);
cudaError_t launch_crypto_step(const EnvDev& e, const int16_t* actions, const TrajDev& o, cudaStream_t s);
cudaError_t launch_crypto_get_state(const EnvDev& e, double* cash, int16_t* hold, double* asset,
                                    int32_t* t_ep, cudaStream_t s);
cudaError_t launch_crypto_set_state(const EnvDev& e, const double* cash, const int16_t* hold,
                                    const int32_t* t_ep, const int32_t* tau, cudaStream_t s);
cudaError_t launch_agg_finalize(const double* partial, int n_blocks, double* agg, cudaStream_t s);
cudaError_t launch_episode_metrics(const double* equity, const uint8_t* done, int T, int N, double reset_eq,
                                   double ppy, double rf, double* ep, int cap, int32_t* cnt,
                                   double* partial, int* n_blocks, cudaStream_t s);
cudaError_t launch_market_prepare(const float* ohlcv, int D, int K, int warmup, const int32_t* ind, int I,
                                  double magnitude, uint64_t seed, float* market, double* raw, cudaStream_t s);
cudaError_t launch_member_weights(const double* stats, int M, double thr, double tau, float* w, double* sharpe,
                                  cudaStream_t s);
cudaError_t launch_philox_normals(uint64_t seed, int64_t off, int N, int K, int member, int64_t t,
                                  float* out, cudaStream_t s);
}  // namespace fin
