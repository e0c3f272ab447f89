// metrics.cu -- K6 episode metrics from a stored equity log, and the Philox probe.
//
// PAPER.md §6.1 cumulative return and max drawdown, Eq. 6
// Sharpe with r_f, annualised by sqrt(periods_per_year) (252 for
// daily bars, BASELINE configs[2]); reading R21-R23.  Equity log [T+1][N]:
// row 0 = equity at the start, row t = v' of transition t; an episode ends at a
// done transition and the next starts at ``reset_equity``.
//
// Decomposition: time is cut into chunks; pass A summarises each (chunk, env)
// (number of dones and the open-episode segment after the last done) as a
// monoid element; pass B scans the chunk summaries of each env in order
// (exclusive episode count + the accumulator entering each chunk); pass C
// re-walks each chunk from its carried-in accumulator and writes the episodes
// that end inside it.  Threads of a warp own consecutive envs, so every read of
// row t is coalesced.  Monoids: Welford (n, mean, M2) with Chan's combine;
// drawdown (max, min, mdd) with mdd(A.B) = min(A.mdd, B.mdd, B.min/A.max - 1).
#include "fin_internal.cuh"
#include "philox.cuh"
#include "sm100.cuh"

namespace {

constexpr int kThreads = 128;

struct Seg {       // summary of a run of equity points v_a..v_b following v_{a-1}
  double vlast, vmax, vmin, mdd, mean, m2;
  int32_t n;       // number of returns (= points)
  int32_t dones;   // number of done transitions in the chunk (pass A only)
};

__device__ __forceinline__ void seg_empty(Seg& s) {
  s.vlast = 0; s.vmax = -1.0; s.vmin = __longlong_as_double(0x7ff0000000000000ULL); s.mdd = 0; s.mean = 0; s.m2 = 0;
  s.n = 0; s.dones = 0;
}

// push equity point v (with previous point vp) onto a segment
__device__ __forceinline__ void seg_push(Seg& s, double vp, double v) {
  double r = fsub64(fdiv64(v, vp), 1.0);
  s.n += 1;
  double delta = fsub64(r, s.mean);
  s.mean = fadd64(s.mean, fmul64(delta, __drcp_rn(nn2d(s.n))));
  s.m2 = fadd64(s.m2, fmul64(delta, fsub64(r, s.mean)));
  if (s.n == 1) { s.vmax = v; s.vmin = v; s.mdd = 0.0; }
  else {
    if (v > s.vmax) s.vmax = v;
    if (v < fmul64(fadd64(s.mdd, 1.0 + 1e-12), s.vmax)) {   // see metric_push
      const double dd = fsub64(fdiv64(v, s.vmax), 1.0);
      if (dd < s.mdd) s.mdd = dd;
    }
    if (v < s.vmin) s.vmin = v;
  }
  s.vlast = v;
}

// accumulator (episode so far, MetricAcc) followed by a segment
__device__ __forceinline__ void acc_combine(MetricAcc& m, const Seg& s) {
  if (s.n == 0) return;
  // Welford / Chan combine of the return statistics
  const double na = (double)m.n, nb = (double)s.n, nn = na + nb;
  const double delta = fsub64(s.mean, m.mean);
  const double mean = fadd64(m.mean, fmul64(delta, fdiv64(nb, nn)));
  const double m2 = fadd64(fadd64(m.m2, s.m2), fmul64(fmul64(delta, delta), fdiv64(fmul64(na, nb), nn)));
  m.mean = mean; m.m2 = m2; m.n += s.n;
  // drawdown monoid, the accumulator's peak already includes v_0
  double cand = fsub64(fdiv64(s.vmin, m.peak), 1.0);
  double mdd = m.mdd;
  if (s.mdd < mdd) mdd = s.mdd;
  if (cand < mdd) mdd = cand;
  m.mdd = mdd > 0.0 ? 0.0 : mdd;
  if (s.vmax > m.peak) m.peak = s.vmax;
  m.vprev = s.vlast;
}

__global__ void k_pass_a(const double* __restrict__ eq, const uint8_t* __restrict__ done, int T, int N, int chunk,
                         double reset_eq,
                         Seg* __restrict__ seg) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int c = blockIdx.y;
  if (i >= N) return;
  const int t0 = c * chunk, t1 = min(T, t0 + chunk);
  Seg s;
  seg_empty(s);
  // the transition before the chunk ended an episode: the next one starts at reset_eq
  double vp = (t0 > 0 && done[(size_t)(t0 - 1) * N + i]) ? reset_eq : eq[(size_t)t0 * N + i];
  int dones = 0;
  for (int t = t0; t < t1; ++t) {
    const double v = eq[(size_t)(t + 1) * N + i];
    seg_push(s, vp, v);
    vp = v;
    if (done[(size_t)t * N + i]) { ++dones; seg_empty(s); vp = reset_eq; }
  }
  s.dones = dones;
  seg[(size_t)c * N + i] = s;
}

__global__ void k_pass_b(const double* __restrict__ eq, int N, int nchunks, double reset_eq,
                         const Seg* __restrict__ seg, MetricAcc* __restrict__ carry, int32_t* __restrict__ base) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N) return;
  MetricAcc m;
  metric_start(m, eq[i]);
  int cnt = 0;
  for (int c = 0; c < nchunks; ++c) {
    carry[(size_t)c * N + i] = m;
    base[(size_t)c * N + i] = cnt;
    const Seg s = seg[(size_t)c * N + i];
    if (s.dones > 0) { metric_start(m, reset_eq); cnt += s.dones; }
    acc_combine(m, s);
  }
}

// Pass C walks a chunk from its carried-in accumulator (carry == null: one chunk,
// the single fused pass, starting at row 0).  The equity / done rows of the next U
// steps are loaded ahead of the arithmetic of the current U (registers), so each
// thread keeps 9 U bytes in flight.
__global__ void k_pass_c(const double* __restrict__ eq, const uint8_t* __restrict__ done, int T, int N, int chunk,
                         double reset_eq, double ppy, double rf, const MetricAcc* __restrict__ carry,
                         const int32_t* __restrict__ base, double* __restrict__ ep, int cap,
                         int32_t* __restrict__ cnt_out, double* __restrict__ partial) {
  constexpr int U = 8;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int c = blockIdx.y;
  AggAcc agg;
  agg_init(agg);
  if (i < N) {
    const int t0 = c * chunk, t1 = min(T, t0 + chunk);
    MetricAcc m;
    int k = 0;
    if (carry) {
      m = carry[(size_t)c * N + i];
      k = base[(size_t)c * N + i];
    } else {
      metric_start(m, __ldg(eq + i));
    }
    double vb[U];
    uint8_t db[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      vb[u] = t0 + u < t1 ? __ldg(eq + (size_t)(t0 + u + 1) * N + i) : 0.0;
      db[u] = t0 + u < t1 ? __ldg(done + (size_t)(t0 + u) * N + i) : 0;
    }
    for (int t = t0; t < t1; t += U) {
      double vn[U];
      uint8_t dn[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int tn = t + U + u;
        vn[u] = tn < t1 ? __ldg(eq + (size_t)(tn + 1) * N + i) : 0.0;
        dn[u] = tn < t1 ? __ldg(done + (size_t)tn * N + i) : 0;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (t + u < t1) {
          metric_push(m, vb[u]);
          if (db[u]) {
            double em[3];
            metric_finish(m, ppy, rf, em);
            if (ep && k < cap) {
              double* d = ep + ((size_t)k * N + i) * 3;
              d[0] = em[0]; d[1] = em[1]; d[2] = em[2];
            }
            agg_episode(agg, em);
            ++k;
            metric_start(m, reset_eq);
          }
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        vb[u] = vn[u];
        db[u] = dn[u];
      }
    }
    if (c == gridDim.y - 1 && cnt_out) cnt_out[i] = k;
  }
  if (partial) agg_block_write(agg, partial + ((size_t)c * gridDim.x + blockIdx.x) * FIN_AGG_LEN);
}

// ------------------------------------------------------------ single fused pass
// When the envs alone fill the GPU (one chunk), every thread walks its env's whole
// log once.  The accumulator is cheaper than MetricAcc's Welford form (K6 was bound
// by fp64 issue, not HBM: a correctly rounded division and reciprocal per point):
//   r_t  = (v_t - v_{t-1}) * rcp(v_{t-1})   -- v_t - v_{t-1} is exact (Sterbenz) and
//          rcp(v) (MUFU seed + 2 Newton steps, <= 1 ulp) is computed once per point,
//          when v becomes the previous point: r within ~2 ulp of v_t / v_{t-1} - 1
//   shifted sums S1 = sum (r - r_1), S2 = sum (r - r_1)^2 with the episode's first
//          return r_1 as the shift: var = (S2 - S1^2 / n) / (n - 1), relative error
//          O(n eps (1 + (mean - r_1)^2 / var)); identical returns give S1 = S2 = 0, so
//          a flat equity curve still yields std = 0 -> NaN (reading R21)
//   drawdown (v - peak) * rcp(peak), rcp(peak) = rcp(v) of the point that set the peak
//          (~2 ulp relative, exactly 0 at a peak).
// Tolerances of the parity tests (rel 1e-9 cum / MDD, 1e-7 Sharpe) hold with room.
struct FastAcc {
  double v0, vprev, rinv, peak, rpeak, mdd, k, s1, s2;
  int32_t n;
};

__device__ __forceinline__ void fast_start(FastAcc& a, double v) {
  a.v0 = v; a.vprev = v; a.rinv = rcp_nr(v); a.peak = v; a.rpeak = a.rinv; a.mdd = 0.0;
  a.k = 0.0; a.s1 = 0.0; a.s2 = 0.0; a.n = 0;
}

// branch-free: the drawdown (v - peak) * rcp(peak) reuses rcp(v) of the new peak (a
// data-dependent division branch was taken by some env of nearly every warp)
__device__ __forceinline__ void fast_push(FastAcc& a, double v) {
  const double r = fmul64(fsub64(v, a.vprev), a.rinv);
  const double rv = rcp_nr(v);
  a.rinv = rv;
  a.vprev = v;
  a.k = a.n == 0 ? r : a.k;
  const double x = fsub64(r, a.k);
  a.s1 = fadd64(a.s1, x);
  a.s2 = __fma_rn(x, x, a.s2);
  a.n += 1;
  const bool up = v > a.peak;
  a.peak = up ? v : a.peak;
  a.rpeak = up ? rv : a.rpeak;
  a.mdd = fmin(a.mdd, fmul64(fsub64(v, a.peak), a.rpeak));
}

__device__ __forceinline__ void fast_finish(const FastAcc& a, double ppy, double rf, double out[3]) {
  out[0] = fmul64(fsub64(a.vprev, a.v0), rcp_nr(a.v0));   // exact 0 for a flat curve
  double sh = __longlong_as_double(0x7ff8000000000000ULL);
  if (a.n >= 2) {
    const double rn = rcp_nr(nn2d(a.n));
    const double mean = fadd64(a.k, fmul64(a.s1, rn));
    const double var = fmul64(fsub64(a.s2, fmul64(fmul64(a.s1, a.s1), rn)), rcp_nr(nn2d(a.n - 1)));
    if (var > 0.0) sh = fmul64(fmul64(sqrt(ppy), fsub64(mean, rf)), rsqrt_nr(var));
  }
  out[1] = sh;
  out[2] = a.mdd;
}

// Episode end: metrics row, per-thread aggregate (shared memory, touched only here).
#ifndef FIN_K6_MINB
#define FIN_K6_MINB 6
#endif
#ifndef FIN_K6_NOINLINE
#define FIN_K6_NOINLINE 0
#endif
#if FIN_K6_NOINLINE
#define FIN_K6_EP_ATTR __noinline__
#else
#define FIN_K6_EP_ATTR __forceinline__
#endif
__device__ FIN_K6_EP_ATTR void fast_episode(FastAcc& a, double ppy, double rf, double* ep, int cap, int N, int i,
                                            int k, double* sagg, double reset_eq) {
  double em[3];
  fast_finish(a, ppy, rf, em);
  if (ep && k < cap) {
    double* d = ep + ((size_t)k * N + i) * 3;
    d[0] = em[0]; d[1] = em[1]; d[2] = em[2];
  }
  AggAcc g;   // the thread's aggregate partial lives in shared memory (touched once per episode)
#pragma unroll
  for (int j = 0; j < FIN_AGG_LEN; ++j) g.s[j] = sagg[j * kThreads];
  agg_episode(g, em);
#pragma unroll
  for (int j = 0; j < FIN_AGG_LEN; ++j) sagg[j * kThreads] = g.s[j];
  fast_start(a, reset_eq);
}

__device__ __forceinline__ void sagg_init(double* sagg) {
  AggAcc g;
  agg_init(g);
#pragma unroll
  for (int j = 0; j < FIN_AGG_LEN; ++j) sagg[j * kThreads] = g.s[j];
}

// one thread per env, the whole log; the next U rows are loaded under the arithmetic
// of the current U.  Up to 8 blocks of 128 per SM (<= 64 registers): 32 warps in
// flight; the aggregate lives in shared memory.
__global__ void __launch_bounds__(kThreads, FIN_K6_MINB)
    k_metrics_fused(const double* __restrict__ eq, const uint8_t* __restrict__ done, int T, int N, double reset_eq,
                    double ppy, double rf, double* __restrict__ ep, int cap, int32_t* __restrict__ cnt_out,
                    double* __restrict__ partial) {
  constexpr int U = 8;
  __shared__ double s_agg[FIN_AGG_LEN * kThreads];
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  sagg_init(s_agg + threadIdx.x);
  if (i < N) {
    FastAcc a;
    fast_start(a, __ldg(eq + i));
    int k = 0;
    double vb[U];
    uint32_t db = 0;   // done bits of the current U rows
#pragma unroll
    for (int u = 0; u < U; ++u) {
      vb[u] = u < T ? __ldg(eq + (size_t)(u + 1) * N + i) : 0.0;
      db |= (u < T ? (uint32_t)__ldg(done + (size_t)u * N + i) : 0u) << u;
    }
    for (int t = 0; t < T; t += U) {
      double vn[U];
      uint32_t dn = 0;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int tn = t + U + u;
        vn[u] = tn < T ? __ldg(eq + (size_t)(tn + 1) * N + i) : 0.0;
        dn |= (tn < T ? (uint32_t)__ldg(done + (size_t)tn * N + i) : 0u) << u;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (t + u < T) {
          fast_push(a, vb[u]);
          if ((db >> u) & 1u) {
            fast_episode(a, ppy, rf, ep, cap, N, i, k, s_agg + threadIdx.x, reset_eq);
            ++k;
          }
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) vb[u] = vn[u];
      db = dn;
    }
    if (cnt_out) cnt_out[i] = k;
  }
  if (partial) {
    AggAcc g;
#pragma unroll
    for (int j = 0; j < FIN_AGG_LEN; ++j) g.s[j] = s_agg[j * kThreads + threadIdx.x];
    agg_block_write(g, partial + (size_t)blockIdx.x * FIN_AGG_LEN);
  }
}

// TMA-staged variant of the fused pass (N % 16 == 0, 16-B aligned logs): a producer
// warp streams, per 128-env block, chunks of R rows of the equity log (1 KB per row)
// and of the done log (128 B per row) into an S-slot shared-memory ring with 1-D bulk
// copies (cp.async.bulk, complete_tx on the slot's mbarrier), so S - 1 chunks are in
// flight per block without holding them in registers; the 4 consumer warps walk the
// rows out of shared memory (conflict-free 8-B / 1-B loads).
#ifndef FIN_K6_S
#define FIN_K6_S 3
#endif
#ifndef FIN_K6_R
#define FIN_K6_R 8
#endif
#ifndef FIN_K6_TMINB
#define FIN_K6_TMINB 5
#endif
constexpr int kK6S = FIN_K6_S, kK6R = FIN_K6_R;
struct K6Smem {
  double eq[kK6S][kK6R][kThreads];
  uint8_t dn[kK6S][kK6R][kThreads];
  double agg[FIN_AGG_LEN * kThreads];
  uint64_t full[kK6S], empty[kK6S];
};

__global__ void __launch_bounds__(kThreads + 32, FIN_K6_TMINB)
    k_metrics_tma(const double* __restrict__ eq, const uint8_t* __restrict__ done, int T, int N, double reset_eq,
                  double ppy, double rf, double* __restrict__ ep, int cap, int32_t* __restrict__ cnt_out,
                  double* __restrict__ partial) {
  extern __shared__ __align__(128) uint8_t k6_smem[];
  K6Smem& sm = *reinterpret_cast<K6Smem*>(k6_smem);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int i0 = blockIdx.x * kThreads;
  const int nb = min(kThreads, N - i0);           // envs of this block (multiple of 16)
  const int nchunks = (T + kK6R - 1) / kK6R;
  if (tid == 0) {
    for (int q = 0; q < kK6S; ++q) {
      sm100::mbar_init(&sm.full[q], 1);
      sm100::mbar_init(&sm.empty[q], kThreads / 32);
    }
    sm100::fence_mbar_init();
  }
  if (tid < kThreads) sagg_init(sm.agg + tid);
  __syncthreads();
  if (warp == kThreads / 32) {
    // ---- producer
    if (lane == 0) {
      for (int c = 0; c < nchunks; ++c) {
        const int slot = c % kK6S;
        if (c >= kK6S) sm100::mbar_wait(&sm.empty[slot], (uint32_t)(c / kK6S - 1) & 1u);
        const int rows = min(kK6R, T - c * kK6R);
        sm100::mbar_arrive_expect_tx(&sm.full[slot], (uint32_t)(rows * nb * 9));
        for (int r = 0; r < rows; ++r) {
          const size_t t = (size_t)c * kK6R + r;
          sm100::bulk_g2s(sm.eq[slot][r], eq + (t + 1) * N + i0, (uint32_t)nb * 8, &sm.full[slot]);
          sm100::bulk_g2s(sm.dn[slot][r], done + t * N + i0, (uint32_t)nb, &sm.full[slot]);
        }
      }
    }
  } else {
    // ---- consumers: thread tid owns env i0 + tid
    const bool live = tid < nb;
    const int i = i0 + tid;
    FastAcc a;
    fast_start(a, live ? __ldg(eq + i) : 1.0);
    int k = 0;
    for (int c = 0; c < nchunks; ++c) {
      const int slot = c % kK6S;
      sm100::mbar_wait(&sm.full[slot], (uint32_t)(c / kK6S) & 1u);
      const int rows = min(kK6R, T - c * kK6R);
      if (live) {
        if (rows == kK6R) {
          double v[kK6R];
          uint8_t d[kK6R];
#pragma unroll
          for (int r = 0; r < kK6R; ++r) { v[r] = sm.eq[slot][r][tid]; d[r] = sm.dn[slot][r][tid]; }
#pragma unroll
          for (int r = 0; r < kK6R; ++r) {
            fast_push(a, v[r]);
            if (d[r]) {
              fast_episode(a, ppy, rf, ep, cap, N, i, k, sm.agg + tid, reset_eq);
              ++k;
            }
          }
        } else {
          for (int r = 0; r < rows; ++r) {
            fast_push(a, sm.eq[slot][r][tid]);
            if (sm.dn[slot][r][tid]) {
              fast_episode(a, ppy, rf, ep, cap, N, i, k, sm.agg + tid, reset_eq);
              ++k;
            }
          }
        }
      }
      __syncwarp();
      if (lane == 0) sm100::mbar_arrive(&sm.empty[slot]);
    }
    if (live && cnt_out) cnt_out[i] = k;
  }
  __syncthreads();
  if (partial) {   // every thread takes part (agg_block_write synchronises the block); the
    AggAcc g;      // producer warp contributes the neutral element
    agg_init(g);
    if (tid < kThreads) {
#pragma unroll
      for (int j = 0; j < FIN_AGG_LEN; ++j) g.s[j] = sm.agg[j * kThreads + tid];
    }
    agg_block_write(g, partial + (size_t)blockIdx.x * FIN_AGG_LEN);
  }
}

__global__ void k_philox_normals(uint64_t seed, int64_t off, int N, int K, int member, int64_t t, float* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N) return;
  for (int blk = 0; blk * 4 < K; ++blk) {
    float z[4];
    philox_normals4((uint64_t)(off + i), (uint32_t)t, ((uint32_t)member << 16) | (uint32_t)blk, seed, z);
    for (int j = 0; j < 4 && blk * 4 + j < K; ++j) out[(size_t)i * K + blk * 4 + j] = z[j];
  }
}

// Pre-drawn exploration noise of a latency-bound (small-N) fused stock rollout
// (DESIGN.md §4.3 "small N"): the normals consume() / prepare() would draw in-kernel --
// the same Philox4x32-10 counters {global env id, t_global + t, m << 16 | counter, 0}
// and Box-Muller (reading R-NOISE, PAPER.md P:130 eps) through the same
// philox_normals8_v -- written in the supplied-noise layout [T][M][N][K]. One thread per
// (t, m, env, 8-asset block); grid-stride; total < 2^31 (the caller caps the buffer).
__global__ void k_pregen_noise(uint64_t seed, int64_t off, int N, int K, int M, int64_t t0, int T, float* out) {
  const uint32_t nb = (uint32_t)(K + 7) / 8;
  const uint32_t total = (uint32_t)T * (uint32_t)M * (uint32_t)N * nb;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const uint32_t pb = i % nb;
    const uint32_t r = i / nb;
    const uint32_t env = r % (uint32_t)N, tm = r / (uint32_t)N;
    const uint32_t m = tm % (uint32_t)M, t = tm / (uint32_t)M;
    const Normals8 v = philox_normals8_v((uint64_t)(off + env), (uint32_t)(t0 + t), (m << 16) | (2 * pb),
                                         (m << 16) | (2 * pb + 1), seed);
    const float z[8] = {v.a.x, v.a.y, v.a.z, v.a.w, v.b.x, v.b.y, v.b.z, v.b.w};
    float* dst = out + (size_t)r * K + 8 * pb;
#pragma unroll
    for (int j = 0; j < 8; ++j)
      if (8 * (int)pb + j < K) dst[j] = z[j];
  }
}

// The same normals streamed step by step while the rollout runs (small N: the rollout's
// tiles occupy few SMs; this kernel runs on the idle ones).  Every block takes its share of
// step t's (m, env, 8-asset block) items; after every FIN_NOISE_GROUP steps it counts the group
// finished in ready[t / FIN_NOISE_GROUP] (each thread's stores fenced, block barrier, one release
// add -- per group, so the consumers' acquire round trips are 1/8 of the steps); blocks never wait on the
// rollout, so the pair cannot deadlock whatever the order the blocks become resident in.
__global__ void k_stream_noise(uint64_t seed, int64_t off, int N, int K, int M, int64_t t0, int T, float* out,
                               uint32_t* ready) {
  const uint32_t nb = (uint32_t)(K + 7) / 8;
  const uint32_t per_t = (uint32_t)M * (uint32_t)N * nb;
  for (int t = 0; t < T; ++t) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < per_t; i += gridDim.x * blockDim.x) {
      const uint32_t pb = i % nb;
      const uint32_t r = i / nb;
      const uint32_t env = r % (uint32_t)N, m = r / (uint32_t)N;
      const Normals8 v = philox_normals8_v((uint64_t)(off + env), (uint32_t)(t0 + t), (m << 16) | (2 * pb),
                                           (m << 16) | (2 * pb + 1), seed);
      const float z[8] = {v.a.x, v.a.y, v.a.z, v.a.w, v.b.x, v.b.y, v.b.z, v.b.w};
      float* dst = out + ((size_t)t * M * N + r) * K + 8 * pb;
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (8 * (int)pb + j < K) dst[j] = z[j];
    }
    if ((t + 1) % FIN_NOISE_GROUP == 0 || t == T - 1) {   // publish a group of steps
      __threadfence();
      __syncthreads();
      if (threadIdx.x == 0)
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(ready + t / FIN_NOISE_GROUP) : "memory");
    }
  }
}

// Ensemble member weights from validation statistics (reading
// R-GATE): Sharpe_m = sum_m / count_m; discard Sharpe < threshold or NaN; softmax at
// temperature tau over the rest (shifted by the largest kept Sharpe); none kept -> the
// best finite Sharpe (lowest index on ties; member 0 if none is finite) gets 1.
__global__ void k_member_weights(const double* __restrict__ stats, int M, double thr, double tau, float* w,
                                 double* sharpe) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double sh[FIN_MAX_MEMBERS];
  bool keep[FIN_MAX_MEMBERS];
  bool any = false;
  double top = -__longlong_as_double(0x7ff0000000000000ULL);
  int best = -1;
  for (int m = 0; m < M; ++m) {
    const double c = stats[m * FIN_AGG_LEN + FIN_AGG_N_SHARPE];
    sh[m] = c > 0.0 ? stats[m * FIN_AGG_LEN + FIN_AGG_SUM_SHARPE] / c : __longlong_as_double(0x7ff8000000000000ULL);
    if (sharpe) sharpe[m] = sh[m];
    keep[m] = sh[m] == sh[m] && sh[m] >= thr;
    if (keep[m]) { any = true; top = fmax(top, sh[m]); }
    if (sh[m] == sh[m] && (best < 0 || sh[m] > sh[best])) best = m;
  }
  if (!any) {
    for (int m = 0; m < M; ++m) w[m] = m == (best < 0 ? 0 : best) ? 1.f : 0.f;
    return;
  }
  double ex[FIN_MAX_MEMBERS], tot = 0.0;
  for (int m = 0; m < M; ++m) {
    ex[m] = keep[m] ? exp((sh[m] - top) / tau) : 0.0;
    tot += ex[m];
  }
  for (int m = 0; m < M; ++m) w[m] = (float)(ex[m] / tot);
}

}  // namespace

namespace fin {

cudaError_t launch_member_weights(const double* stats, int M, double thr, double tau, float* w, double* sharpe,
                                  cudaStream_t s) {
  k_member_weights<<<1, 32, 0, s>>>(stats, M, thr, tau, w, sharpe);
  return cudaGetLastError();
}

cudaError_t launch_episode_metrics(const double* equity, const uint8_t* done, int T, int N, double reset_eq,
                                   double ppy, double rf, double* ep, int cap, int32_t* cnt, double* partial,
                                   int* n_blocks, cudaStream_t s) {
  // chunk length: enough (chunk, env) pairs to fill the GPU several times over
  const int env_blocks = (N + kThreads - 1) / kThreads;
  int nchunks = (2048 + env_blocks - 1) / env_blocks;
  if (nchunks > T) nchunks = T > 0 ? T : 1;
  if (nchunks > 4096) nchunks = 4096;
  const int chunk = (T + nchunks - 1) / nchunks > 0 ? (T + nchunks - 1) / nchunks : 1;
  nchunks = T > 0 ? (T + chunk - 1) / chunk : 1;
  dim3 grid(env_blocks, nchunks);
  *n_blocks = env_blocks * nchunks;
  if (nchunks == 1) {   // enough envs to fill the GPU: one fused pass, each row read once
#ifdef FIN_K6_OLD
    k_pass_c<<<grid, kThreads, 0, s>>>(equity, done, T, N, chunk, reset_eq, ppy, rf, nullptr, nullptr, ep, cap,
                                        cnt, partial);
#else
    const bool tma = N % 16 == 0 && ((uintptr_t)equity & 15) == 0 && ((uintptr_t)done & 15) == 0 && !getenv("FIN_K6_NOTMA");
    if (tma) {
      static bool attr = false;
      if (!attr) {
        cudaFuncSetAttribute(k_metrics_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(K6Smem));
        attr = true;
      }
      k_metrics_tma<<<env_blocks, kThreads + 32, sizeof(K6Smem), s>>>(equity, done, T, N, reset_eq, ppy, rf, ep, cap,
                                                                      cnt, partial);
    } else {
      k_metrics_fused<<<env_blocks, kThreads, 0, s>>>(equity, done, T, N, reset_eq, ppy, rf, ep, cap, cnt, partial);
    }
#endif
    return cudaGetLastError();
  }
  Seg* seg = nullptr;
  MetricAcc* carry = nullptr;
  int32_t* base = nullptr;
  cudaError_t err;
  if ((err = cudaMallocAsync(&seg, sizeof(Seg) * (size_t)nchunks * N, s)) != cudaSuccess) return err;
  if ((err = cudaMallocAsync(&carry, sizeof(MetricAcc) * (size_t)nchunks * N, s)) != cudaSuccess) return err;
  if ((err = cudaMallocAsync(&base, sizeof(int32_t) * (size_t)nchunks * N, s)) != cudaSuccess) return err;
  k_pass_a<<<grid, kThreads, 0, s>>>(equity, done, T, N, chunk, reset_eq, seg);
  k_pass_b<<<env_blocks, kThreads, 0, s>>>(equity, N, nchunks, reset_eq, seg, carry, base);
  k_pass_c<<<grid, kThreads, 0, s>>>(equity, done, T, N, chunk, reset_eq, ppy, rf, carry, base, ep, cap, cnt,
                                      partial);
  cudaFreeAsync(seg, s);
  cudaFreeAsync(carry, s);
  cudaFreeAsync(base, s);
  return cudaGetLastError();
}

cudaError_t launch_philox_normals(uint64_t seed, int64_t off, int N, int K, int member, int64_t t, float* out,
                                  cudaStream_t s) {
  k_philox_normals<<<(N + 127) / 128, 128, 0, s>>>(seed, off, N, K, member, t, out);
  return cudaGetLastError();
}

int num_sms();

// Load the producer's module and set its attributes before the rollout that waits on it is
// launched: with lazy module loading a first launch of k_stream_noise behind a running
// (spinning) rollout waits for the device to idle -- the pair would deadlock.
constexpr int kStreamSmem = 117 * 1024;   // > half an SM: a producer block never shares an SM with another
                                          // one or with a rollout CTA (> 100 KB), so it cannot steal issue
                                          // slots from a tile's step chain
cudaError_t load_stream_noise() {
  static cudaError_t st = cudaErrorNotReady;
  if (st == cudaErrorNotReady) {
    cudaFuncAttributes fa;
    st = cudaFuncGetAttributes(&fa, k_stream_noise);
    if (st == cudaSuccess)
      st = cudaFuncSetAttribute(k_stream_noise, cudaFuncAttributeMaxDynamicSharedMemorySize, kStreamSmem);
  }
  return st;
}

cudaError_t launch_stream_noise(uint64_t seed, int64_t off, int N, int K, int M, int64_t t0, int T, float* out,
                                uint32_t* ready, int blocks, cudaStream_t s) {
  if ((size_t)M * N * ((K + 7) / 8) >= (1ull << 31) || blocks <= 0) return cudaErrorInvalidValue;
  cudaError_t e = load_stream_noise();
  if (e != cudaSuccess) return e;
  k_stream_noise<<<blocks, 512, kStreamSmem, s>>>(seed, off, N, K, M, t0, T, out, ready);
  return cudaGetLastError();
}

cudaError_t launch_pregen_noise(uint64_t seed, int64_t off, int N, int K, int M, int64_t t0, int T, float* out,
                                cudaStream_t s) {
  const size_t total = (size_t)T * M * N * ((K + 7) / 8);
  if (total == 0) return cudaSuccess;
  if (total >= (1ull << 31)) return cudaErrorInvalidValue;
  const size_t blocks = (total + 255) / 256, cap = (size_t)num_sms() * 8;
  k_pregen_noise<<<(unsigned)(blocks < cap ? blocks : cap), 256, 0, s>>>(seed, off, N, K, M, t0, T, out);
  return cudaGetLastError();
}

}  // namespace fin
