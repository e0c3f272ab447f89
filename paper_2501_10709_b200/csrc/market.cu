// market.cu -- market preparation on the device: the step before
// the rollout.  From raw f32 OHLCV [D][5][K] (D = hidden warm-up days + stored rows):
//   * per-asset price-scale perturbation (§5.1; reading R-PERTURB):
//     c_k = 1 + m (2 u_k - 1), u_k from Philox4x32-10 (counter (k, 0, "MKTP", 0), key =
//     seed), applied to open / high / low / close;
//   * the paper's indicator families with the parameters of reading R11, in
//     float64 with the definitions' operation order (explicit _rn intrinsics);
//   * the stored tensor market[d][c][k] f32 the env consumes: close, close / close[0],
//     indicators z-scored per (asset, indicator) over the stored rows.
// One block per (asset, indicator): the window families one thread per day, the
// recurrences serially (bit-identical either way: every value is computed in the
// definition's own order).
#include "fin_internal.cuh"
#include "philox.cuh"

namespace {

constexpr int kMaxInd = 16;
constexpr uint32_t kPerturbWord = 0x4D4B5450u;   // "MKTP"

struct IndList {
  int32_t id[kMaxInd];
};

// one price channel (1 = high, 2 = low, 3 = close) of asset k on day d, scaled by c_k
__device__ __forceinline__ double px(const float* __restrict__ x, int K, int k, int d, int ch, double ck) {
  return fmul64((double)__ldg(x + ((size_t)d * 5 + ch) * K + k), ck);
}

// mean of channel ch over days [lo, d] (sum in day order, then one division)
__device__ double wmean(const float* x, int K, int k, int d, int n, int ch, double ck) {
  const int lo = d - n + 1 > 0 ? d - n + 1 : 0;
  double s = 0.0;
  for (int j = lo; j <= d; ++j) s = fadd64(s, px(x, K, k, j, ch, ck));
  return fdiv64(s, (double)(d + 1 - lo));
}

__device__ double typical(const float* x, int K, int k, int d, double ck) {
  return fdiv64(fadd64(fadd64(px(x, K, k, d, 1, ck), px(x, K, k, d, 2, ck)), px(x, K, k, d, 3, ck)), 3.0);
}

// indicator series value of day d for the running recurrences, window values directly
struct Ema {
  double e;
  double a;
  __device__ double step(double v, int d) {
    e = d == 0 ? v : fadd64(e, fmul64(a, fsub64(v, e)));
    return e;
  }
};

// value of indicator ``id`` on day d for the window families (each day independent: the
// window is summed in day order exactly as the sequential definition does)
__device__ double window_value(const float* x, int K, int k, int d, int id, double ck) {
  if (id == FIN_IND_BOLL_UB || id == FIN_IND_BOLL_LB) {
    const int lo = d - 19 > 0 ? d - 19 : 0;
    const double m = wmean(x, K, k, d, 20, 3, ck);
    double s = 0.0;
    for (int j = lo; j <= d; ++j) {
      const double dv = fsub64(px(x, K, k, j, 3, ck), m);
      s = fadd64(s, fmul64(dv, dv));
    }
    const double sd = sqrt(fdiv64(s, (double)(d + 1 - lo)));
    return id == FIN_IND_BOLL_UB ? fadd64(m, fmul64(2.0, sd)) : fsub64(m, fmul64(2.0, sd));
  }
  if (id == FIN_IND_CCI30) {
    const int lo = d - 29 > 0 ? d - 29 : 0;
    double s = 0.0;
    for (int j = lo; j <= d; ++j) s = fadd64(s, typical(x, K, k, j, ck));
    const double m = fdiv64(s, (double)(d + 1 - lo));
    double q = 0.0;
    for (int j = lo; j <= d; ++j) q = fadd64(q, fabs(fsub64(typical(x, K, k, j, ck), m)));
    const double mad = fdiv64(q, (double)(d + 1 - lo));
    return mad == 0.0 ? 0.0 : fdiv64(fsub64(typical(x, K, k, d, ck), m), fmul64(0.015, mad));
  }
  if (id == FIN_IND_SMA30) return wmean(x, K, k, d, 30, 3, ck);
  return wmean(x, K, k, d, 60, 3, ck);   // FIN_IND_SMA60
}

// One block per (asset k, slot i): slot i < I is indicator ind.id[i], slot I the two price
// channels.  Window families: one thread per day; the recurrences (MACD's EMAs, Wilder's
// RSI and DX) run serially in thread 0; the z-score's two sums run serially (the
// definition's order) and its elementwise division in parallel.
__global__ void k_market_prepare(const float* __restrict__ x, int D, int K, int warmup, IndList ind, int I,
                                 double magnitude, uint64_t seed, float* __restrict__ market,
                                 double* __restrict__ raw) {
  const int k = blockIdx.x;
  const int i = blockIdx.y;
  const int rows = D - warmup;
  uint32_t c4[4] = {(uint32_t)k, 0u, kPerturbWord, 0u};
  philox4x32_10(c4, (uint32_t)seed, (uint32_t)(seed >> 32));
  const double u = ((double)(c4[0] >> 8) + 0.5) * 5.9604644775390625e-08;   // exact in f64 (25 bits)
  const double ck = fadd64(1.0, fmul64(magnitude, fsub64(fmul64(2.0, u), 1.0)));
  const int C = 2 + I;
  if (i == I) {   // the two price channels
    const double c0 = px(x, K, k, warmup, 3, ck);
    for (int d = threadIdx.x; d < rows; d += blockDim.x) {
      const double c = px(x, K, k, warmup + d, 3, ck);
      market[((size_t)d * C + 0) * K + k] = (float)c;
      market[((size_t)d * C + 1) * K + k] = (float)fdiv64(c, c0);
    }
    return;
  }
  const int id = ind.id[i];
  double* out = raw + ((size_t)i * K + k) * rows;   // scratch [I][K][rows]
  const bool windowed = id == FIN_IND_BOLL_UB || id == FIN_IND_BOLL_LB || id == FIN_IND_CCI30 ||
                        id == FIN_IND_SMA30 || id == FIN_IND_SMA60;
  if (windowed) {
    for (int d = warmup + threadIdx.x; d < D; d += blockDim.x) out[d - warmup] = window_value(x, K, k, d, id, ck);
  } else if (threadIdx.x == 0) {
    // ---- the recurrences over all D days; stored days go to the scratch
    Ema e12{0.0, 2.0 / 13.0}, e26{0.0, 2.0 / 27.0};
    double gain = 0.0, loss = 0.0, sp = 0.0, sm = 0.0, st = 0.0;
    const double a30 = 1.0 / 30.0;
    for (int d = 0; d < D; ++d) {
      double v = 0.0;
      if (id == FIN_IND_MACD) {
        const double c = px(x, K, k, d, 3, ck);
        v = fsub64(e12.step(c, d), e26.step(c, d));
      } else if (id == FIN_IND_RSI30) {
        if (d == 0) {
          v = 50.0;
        } else {
          const double delta = fsub64(px(x, K, k, d, 3, ck), px(x, K, k, d - 1, 3, ck));
          const double g = delta > 0.0 ? delta : 0.0;
          const double l = delta < 0.0 ? -delta : 0.0;
          if (d == 1) { gain = g; loss = l; }
          else {
            gain = fadd64(gain, fmul64(a30, fsub64(g, gain)));
            loss = fadd64(loss, fmul64(a30, fsub64(l, loss)));
          }
          v = loss == 0.0 ? 100.0 : fsub64(100.0, fdiv64(100.0, fadd64(1.0, fdiv64(gain, loss))));
        }
      } else if (id == FIN_IND_DX30) {
        if (d > 0) {
          const double hd = px(x, K, k, d, 1, ck), hp = px(x, K, k, d - 1, 1, ck);
          const double ld = px(x, K, k, d, 2, ck), lp = px(x, K, k, d - 1, 2, ck);
          const double cp = px(x, K, k, d - 1, 3, ck);
          const double up = fsub64(hd, hp), dn = fsub64(lp, ld);
          const double pdm = (up > dn && up > 0.0) ? up : 0.0;
          const double mdm = (dn > up && dn > 0.0) ? dn : 0.0;
          const double tr = fmax(fsub64(hd, ld), fmax(fabs(fsub64(hd, cp)), fabs(fsub64(ld, cp))));
          if (d == 1) { sp = pdm; sm = mdm; st = tr; }
          else {
            sp = fadd64(sp, fmul64(a30, fsub64(pdm, sp)));
            sm = fadd64(sm, fmul64(a30, fsub64(mdm, sm)));
            st = fadd64(st, fmul64(a30, fsub64(tr, st)));
          }
          const double pdi = st > 0.0 ? fdiv64(fmul64(100.0, sp), st) : 0.0;
          const double mdi = st > 0.0 ? fdiv64(fmul64(100.0, sm), st) : 0.0;
          const double s = fadd64(pdi, mdi);
          v = s > 0.0 ? fdiv64(fmul64(100.0, fabs(fsub64(pdi, mdi))), s) : 0.0;
        }
      }
      if (d >= warmup) out[d - warmup] = v;
    }
  }
  __syncthreads();
  // ---- z-score over the stored rows (two-pass population mean / std, sums in day order)
  __shared__ double sh_m, sh_sd;
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int d = 0; d < rows; ++d) s = fadd64(s, out[d]);
    const double m = fdiv64(s, (double)rows);
    double q = 0.0;
    for (int d = 0; d < rows; ++d) {
      const double dv = fsub64(out[d], m);
      q = fadd64(q, fmul64(dv, dv));
    }
    sh_m = m;
    sh_sd = sqrt(fdiv64(q, (double)rows));
  }
  __syncthreads();
  const double m = sh_m, sd = sh_sd;
  for (int d = threadIdx.x; d < rows; d += blockDim.x)
    market[((size_t)d * C + 2 + i) * K + k] = sd == 0.0 ? 0.f : (float)fdiv64(fsub64(out[d], m), sd);
}

}  // namespace

namespace fin {

cudaError_t launch_market_prepare(const float* ohlcv, int D, int K, int warmup, const int32_t* ind, int I,
                                  double magnitude, uint64_t seed, float* market, double* raw, cudaStream_t s) {
  IndList l;
  for (int j = 0; j < kMaxInd; ++j) l.id[j] = j < I ? ind[j] : -1;
  k_market_prepare<<<dim3(K, I + 1), 128, 0, s>>>(ohlcv, D, K, warmup, l, I, magnitude, seed, market, raw);
  return cudaGetLastError();
}

}  // namespace fin
