// crypto_gen.cu -- crypto market generation on the device: the
// synthetic stand-in for the paper's BTC LOB series (BASELINE configs[3]) as the
// [steps + 1][144] f32 tensor fin_env_create takes, drawn from counter-based
// Philox4x32-10 (reading R-CGEN; oracle/crypto_market.py states every formula):
//   N(t, s, j) = component j % 4 of the float64 Box-Muller normals of counter
//                (t, s, j / 4, 0);  U(t, s, j) = uniform of word j % 4 of that counter
//   log m_t = log m_{t-1} + ((-0.5 sigma) sigma + sigma N(t, 1, 0)),  m_0 = m0
//   book: half-spread m 1e-4 exp(0.5 N(t, 2, 0)), level gaps m 0.5e-4 exp(0.5 N(t, 3|4, l)),
//         sizes -ln U(t, 5|6, l)
//   factors f_{0,k} = N(0, 7, k), f_t = phi f_{t-1} + sqrt(1 - phi^2) N(t, 7, k)
// The two serial recurrences (the log-mid running sum and the 101 AR(1) factors, 480,000
// steps for C3) are cut into chunks of kChunk steps: pass A runs each chunk from a zero
// state (one thread per chunk and stream), pass B carries the chunk boundary values
// serially over the chunks (one thread per stream), pass C re-runs each chunk from its
// true carry-in and writes the rows.  The book columns of a step depend only on its mid:
// one thread per step.  Float64 throughout, one f32 rounding per stored value.
//
// Stock OHLCV generation (fin_stock_market, reading R-SGEN, oracle/stock_market.py): the
// synthetic stand-in for the paper's daily bars with BASELINE configs[0]'s GBM
// (S0 ~ U(lo, hi), mu, sigma per day) and OHLV around the close, as the [D][5][K] f32
// tensor fin_market_prepare takes.  Streams 11..15 of the same counter scheme (d, s, k / 4):
//   l_{-1} = ln(lo + (hi - lo) U(0, 11, k));  l_d = l_{d-1} + ((mu - (0.5 sigma) sigma) + sigma N(d, 12, k))
//   open = exp(l_{d-1}), close = exp(l_d), high = max (1 + (0.5 sigma)|N(d, 13, k)|),
//   low = min (1 - (0.5 sigma)|N(d, 14, k)|), volume = exp(ln 1e6 + 0.5 N(d, 15, k)).
// Pass 1 draws the increments (one thread per day and block of 4 assets), pass 2 runs the
// running sum left to right (one thread per asset), pass 3 writes the bars.
#include "fin_internal.cuh"
#include "philox.cuh"

namespace {

constexpr int kChunk = 256;
constexpr int kRow = 144, kLevels = 10, kFactors = 101, kGroups = (kFactors + 3) / 4;
enum { kSMid = 1, kSHalf = 2, kSAskGap = 3, kSBidGap = 4, kSAskSz = 5, kSBidSz = 6, kSFactor = 7 };

struct Words {
  uint32_t w[4];
};
__device__ __forceinline__ Words draw(uint64_t seed, int64_t t, uint32_t s, uint32_t blk) {
  Words r;
  r.w[0] = (uint32_t)t; r.w[1] = s; r.w[2] = blk; r.w[3] = 0u;
  philox4x32_10(r.w, (uint32_t)seed, (uint32_t)(seed >> 32));
  return r;
}
__device__ __forceinline__ double u01_f64(uint32_t x) {   // exact: 25 significant bits
  return ((double)(x >> 8) + 0.5) * 5.9604644775390625e-08;
}
// the four float64 Box-Muller normals of one counter (oracle.philox.normals4)
__device__ __forceinline__ void normals4_f64(const Words& x, double z[4]) {
  const double u0 = u01_f64(x.w[0]), u1 = u01_f64(x.w[1]), u2 = u01_f64(x.w[2]), u3 = u01_f64(x.w[3]);
  const double r0 = sqrt(fmul64(-2.0, log(u0))), r1 = sqrt(fmul64(-2.0, log(u2)));
  const double twopi = 6.283185307179586;
  double s0, c0, s1, c1;
  sincos(fmul64(twopi, u1), &s0, &c0);
  sincos(fmul64(twopi, u3), &s1, &c1);
  z[0] = fmul64(r0, c0); z[1] = fmul64(r0, s0); z[2] = fmul64(r1, c1); z[3] = fmul64(r1, s1);
}
__device__ __forceinline__ double normal_f64(uint64_t seed, int64_t t, uint32_t s, int j) {
  double z[4];
  normals4_f64(draw(seed, t, s, (uint32_t)(j >> 2)), z);
  return z[j & 3];
}

struct GenParams {
  int64_t steps;
  uint64_t seed;
  double sigma, logm0, phi, gain, drift, phiC;   // phiC = phi^kChunk
};

// log-mid increment of step t >= 1
__device__ __forceinline__ double mid_inc(const GenParams& g, int64_t t) {
  return fadd64(g.drift, fmul64(g.sigma, normal_f64(g.seed, t, kSMid, 0)));
}

// ---- pass A: per-chunk sums (mid) and zero-start chunk ends (factors)
__global__ void k_mid_chunks(GenParams g, int nch, double* __restrict__ csum) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= nch) return;
  const int64_t t0 = 1 + (int64_t)c * kChunk, t1 = min(g.steps + 1, t0 + kChunk);
  double s = 0.0;
  for (int64_t t = t0; t < t1; ++t) s = fadd64(s, mid_inc(g, t));
  csum[c] = s;
}
__global__ void k_fac_chunks(GenParams g, int nch, double* __restrict__ cend /*[nch][kGroups*4]*/) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nch * kGroups) return;
  const int c = i / kGroups, grp = i % kGroups;
  const int64_t t0 = 1 + (int64_t)c * kChunk, t1 = min(g.steps + 1, t0 + kChunk);
  double f[4] = {0.0, 0.0, 0.0, 0.0};
  for (int64_t t = t0; t < t1; ++t) {
    double z[4];
    normals4_f64(draw(g.seed, t, kSFactor, (uint32_t)grp), z);
#pragma unroll
    for (int q = 0; q < 4; ++q) f[q] = fadd64(fmul64(g.phi, f[q]), fmul64(g.gain, z[q]));
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) cend[(size_t)c * kGroups * 4 + grp * 4 + q] = f[q];
}

// ---- pass B: carry-in of every chunk (serial over chunks, one thread per stream)
__global__ void k_carry(GenParams g, int nch, const double* __restrict__ csum, double* __restrict__ cin_mid,
                        const double* __restrict__ cend, double* __restrict__ cin_fac) {
  const int i = threadIdx.x;   // 0: mid, 1 + k: factor k
  if (i == 0) {
    double acc = g.logm0;
    for (int c = 0; c < nch; ++c) {
      cin_mid[c] = acc;
      acc = fadd64(acc, csum[c]);
    }
  } else if (i <= kGroups * 4) {
    const int k = i - 1;
    double f = k < kFactors ? normal_f64(g.seed, 0, kSFactor, k) : 0.0;   // f_0
    for (int c = 0; c < nch; ++c) {
      cin_fac[(size_t)c * kGroups * 4 + k] = f;
      f = fadd64(fmul64(g.phiC, f), cend[(size_t)c * kGroups * 4 + k]);
    }
  }
}

// ---- pass C: rows.  Mid: each chunk from its carry-in (also row 0); factors likewise.
__global__ void k_mid_fill(GenParams g, int nch, const double* __restrict__ cin_mid, double* __restrict__ mid) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c == 0) mid[0] = exp(g.logm0);
  if (c >= nch) return;
  const int64_t t0 = 1 + (int64_t)c * kChunk, t1 = min(g.steps + 1, t0 + kChunk);
  double acc = cin_mid[c];
  for (int64_t t = t0; t < t1; ++t) {
    acc = fadd64(acc, mid_inc(g, t));
    mid[t] = exp(acc);
  }
}
__global__ void k_fac_fill(GenParams g, int nch, const double* __restrict__ cin_fac, float* __restrict__ rows) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nch * kGroups) return;
  const int c = i / kGroups, grp = i % kGroups;
  const int64_t t0 = 1 + (int64_t)c * kChunk, t1 = min(g.steps + 1, t0 + kChunk);
  double f[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) f[q] = cin_fac[(size_t)c * kGroups * 4 + grp * 4 + q];
  if (c == 0) {   // row 0: f_0
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if (grp * 4 + q < kFactors) rows[41 + grp * 4 + q] = (float)f[q];
  }
  for (int64_t t = t0; t < t1; ++t) {
    double z[4];
    normals4_f64(draw(g.seed, t, kSFactor, (uint32_t)grp), z);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      f[q] = fadd64(fmul64(g.phi, f[q]), fmul64(g.gain, z[q]));
      if (grp * 4 + q < kFactors) rows[(size_t)t * kRow + 41 + grp * 4 + q] = (float)f[q];
    }
  }
}
// the book of step t from its mid (one thread per step)
__global__ void k_book(GenParams g, const double* __restrict__ mid, float* __restrict__ rows) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t > g.steps) return;
  float* r = rows + (size_t)t * kRow;
  const double m = mid[t];
  const double h = fmul64(fmul64(m, 1e-4), exp(fmul64(0.5, normal_f64(g.seed, t, kSHalf, 0))));
  double za[12], zb[12];
#pragma unroll
  for (int b = 0; b < 3; ++b) {
    normals4_f64(draw(g.seed, t, kSAskGap, (uint32_t)b), za + 4 * b);
    normals4_f64(draw(g.seed, t, kSBidGap, (uint32_t)b), zb + 4 * b);
  }
  double ask = fadd64(m, h), bid = fsub64(m, h);
  r[0] = (float)m;
  r[1] = (float)ask;
  r[21] = (float)bid;
#pragma unroll
  for (int l = 1; l < kLevels; ++l) {
    ask = fadd64(ask, fmul64(fmul64(m, 0.5e-4), exp(fmul64(0.5, za[l - 1]))));
    bid = fsub64(bid, fmul64(fmul64(m, 0.5e-4), exp(fmul64(0.5, zb[l - 1]))));
    r[1 + l] = (float)ask;
    r[21 + l] = (float)bid;
  }
#pragma unroll
  for (int b = 0; b < 3; ++b) {
    const Words wa = draw(g.seed, t, kSAskSz, (uint32_t)b), wb = draw(g.seed, t, kSBidSz, (uint32_t)b);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int l = 4 * b + q;
      if (l < kLevels) {
        r[11 + l] = (float)(-log(u01_f64(wa.w[q])));
        r[31 + l] = (float)(-log(u01_f64(wb.w[q])));
      }
    }
  }
  r[142] = 0.f;
  r[143] = 0.f;
}

// ---- stock OHLCV (R-SGEN)
enum { kSInit = 11, kSClose = 12, kSHigh = 13, kSLow = 14, kSVol = 15 };
struct SGen {
  int D, K;
  uint64_t seed;
  double drift, sigma, hs, lo, span, lv0;
};
__global__ void k_sgen_inc(SGen g, double* __restrict__ inc /*[D][K]*/) {
  const int nb = (g.K + 3) >> 2;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= g.D * nb) return;
  const int d = i / nb, b = i % nb;
  double z[4];
  normals4_f64(draw(g.seed, d, kSClose, (uint32_t)b), z);
#pragma unroll
  for (int j = 0; j < 4; ++j)
    if (4 * b + j < g.K) inc[(size_t)d * g.K + 4 * b + j] = fadd64(g.drift, fmul64(g.sigma, z[j]));
}
__global__ void k_sgen_scan(SGen g, const double* __restrict__ inc, double* __restrict__ lp /*[D + 1][K]*/) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= g.K) return;
  const Words w = draw(g.seed, 0, kSInit, (uint32_t)(k >> 2));
  double l = log(fadd64(g.lo, fmul64(g.span, u01_f64(w.w[k & 3]))));
  lp[k] = l;
  for (int d = 0; d < g.D; ++d) {   // left to right, as the definition
    l = fadd64(l, inc[(size_t)d * g.K + k]);
    lp[(size_t)(d + 1) * g.K + k] = l;
  }
}
__global__ void k_sgen_bars(SGen g, const double* __restrict__ lp, float* __restrict__ out /*[D][5][K]*/) {
  const int nb = (g.K + 3) >> 2;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= g.D * nb) return;
  const int d = i / nb, b = i % nb;
  double zh[4], zl[4], zv[4];
  normals4_f64(draw(g.seed, d, kSHigh, (uint32_t)b), zh);
  normals4_f64(draw(g.seed, d, kSLow, (uint32_t)b), zl);
  normals4_f64(draw(g.seed, d, kSVol, (uint32_t)b), zv);
  float* row = out + (size_t)d * 5 * g.K;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int k = 4 * b + j;
    if (k >= g.K) break;
    const double o = exp(lp[(size_t)d * g.K + k]), c = exp(lp[(size_t)(d + 1) * g.K + k]);
    row[k] = (float)o;
    row[g.K + k] = (float)fmul64(fmax(o, c), fadd64(1.0, fmul64(g.hs, fabs(zh[j]))));
    row[2 * g.K + k] = (float)fmul64(fmin(o, c), fsub64(1.0, fmul64(g.hs, fabs(zl[j]))));
    row[3 * g.K + k] = (float)c;
    row[4 * g.K + k] = (float)exp(fadd64(g.lv0, fmul64(0.5, zv[j])));
  }
}

}  // namespace

namespace fin {

cudaError_t launch_stock_market(int D, int K, uint64_t seed, double mu, double sigma, double s0_lo, double s0_hi,
                                float* ohlcv, cudaStream_t s) {
  SGen g;
  g.D = D;
  g.K = K;
  g.seed = seed;
  g.sigma = sigma;
  g.drift = mu - (0.5 * sigma) * sigma;
  g.hs = 0.5 * sigma;
  g.lo = s0_lo;
  g.span = s0_hi - s0_lo;
  g.lv0 = log(1e6);
  double *inc = nullptr, *lp = nullptr;
  cudaError_t e = cudaMallocAsync(&inc, sizeof(double) * (size_t)D * K, s);
  if (e == cudaSuccess) e = cudaMallocAsync(&lp, sizeof(double) * (size_t)(D + 1) * K, s);
  if (e != cudaSuccess) return e;
  const int n = D * ((K + 3) / 4);
  k_sgen_inc<<<(n + 127) / 128, 128, 0, s>>>(g, inc);
  k_sgen_scan<<<(K + 31) / 32, 32, 0, s>>>(g, inc, lp);
  k_sgen_bars<<<(n + 127) / 128, 128, 0, s>>>(g, lp, ohlcv);
  e = cudaGetLastError();
  cudaFreeAsync(inc, s);
  cudaFreeAsync(lp, s);
  return e;
}


cudaError_t launch_crypto_market(int64_t steps, uint64_t seed, double sigma, double m0, double phi, float* rows,
                                 cudaStream_t s) {
  GenParams g;
  g.steps = steps;
  g.seed = seed;
  g.sigma = sigma;
  g.logm0 = log(m0);
  g.phi = phi;
  g.gain = sqrt(1.0 - phi * phi);
  g.drift = (-0.5 * sigma) * sigma;
  double pc = 1.0;
  for (int i = 0; i < kChunk; ++i) pc *= phi;
  g.phiC = pc;
  const int nch = (int)((steps + kChunk - 1) / kChunk);
  const size_t nf = (size_t)(nch > 0 ? nch : 1) * kGroups * 4;
  double *mid = nullptr, *csum = nullptr, *cin_mid = nullptr, *cend = nullptr, *cin_fac = nullptr;
  cudaError_t e = cudaMallocAsync(&mid, sizeof(double) * (size_t)(steps + 1), s);
  if (e == cudaSuccess) e = cudaMallocAsync(&csum, sizeof(double) * (nch + 1), s);
  if (e == cudaSuccess) e = cudaMallocAsync(&cin_mid, sizeof(double) * (nch + 1), s);
  if (e == cudaSuccess) e = cudaMallocAsync(&cend, sizeof(double) * nf, s);
  if (e == cudaSuccess) e = cudaMallocAsync(&cin_fac, sizeof(double) * nf, s);
  if (e != cudaSuccess) return e;
  if (nch > 0) {
    k_mid_chunks<<<(nch + 127) / 128, 128, 0, s>>>(g, nch, csum);
    k_fac_chunks<<<(nch * kGroups + 127) / 128, 128, 0, s>>>(g, nch, cend);
  }
  k_carry<<<1, 128, 0, s>>>(g, nch, csum, cin_mid, cend, cin_fac);
  k_mid_fill<<<(nch + 128) / 128, 128, 0, s>>>(g, nch, cin_mid, mid);
  if (nch > 0) {
    k_fac_fill<<<(nch * kGroups + 127) / 128, 128, 0, s>>>(g, nch, cin_fac, rows);
  } else {   // steps == 0: row 0 only
    k_fac_fill<<<1, 128, 0, s>>>(g, 1, cin_fac, rows);
  }
  k_book<<<(unsigned)((steps + 1 + 127) / 128), 128, 0, s>>>(g, mid, rows);
  e = cudaGetLastError();
  cudaFreeAsync(mid, s);
  cudaFreeAsync(csum, s);
  cudaFreeAsync(cin_mid, s);
  cudaFreeAsync(cend, s);
  cudaFreeAsync(cin_fac, s);
  return e;
}

}  // namespace fin
