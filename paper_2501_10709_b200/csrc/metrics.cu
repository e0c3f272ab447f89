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

__global__ void k_philox_normals(uint64_t seed, int64_t off, int N, int K, int member, int64_t t, float* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N) return;
  for (int blk = 0; blk * 4 < K; ++blk) {
    float z[4];
    philox_normals4((uint64_t)(off + i), (uint32_t)t, ((uint32_t)member << 16) | (uint32_t)blk, seed, z);
    for (int j = 0; j < 4 && blk * 4 + j < K; ++j) out[(size_t)i * K + blk * 4 + j] = z[j];
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
    k_pass_c<<<grid, kThreads, 0, s>>>(equity, done, T, N, chunk, reset_eq, ppy, rf, nullptr, nullptr, ep, cap,
                                        cnt, partial);
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

}  // namespace fin
