// ppo.cu -- the learner's policy-gradient step (Eq. 3-4, P:176-195;
// PPO's clipped surrogate; reading R-PPO; oracle/learn.py states every formula):
//   head:     per sample s, float64: mu = tanh(z3), log pi = -sum (a - mu)^2 / (2 sigma^2) - K ln(sigma
//             sqrt(2 pi)), rho = exp(log pi - log pi_old), c = rho A unless the clipped term is the
//             minimum (then 0), g3 = d(-L)/dz3 = -(c / B) ((a - mu) / sigma^2) (1 - mu^2)  -> f32
//   backward: g2 = (g3 W3) * [h2 > 0],  g1 = (g2 W2) * [h1 > 0]   (rows = samples)
//             dW3 = g3^T h2, dW2 = g2^T h1, dW1 = g1^T x, db_l = column sums of g_l
//   Adam:     m, v, theta updates of the flat parameter vector (fin_adam_step)
// The contractions run as fp32 CUDA-core GEMMs (64 x 64 tiles, 4 x 4 per thread, split-K over the
// samples with partial sums reduced in a fixed order: deterministic); the hidden activations and
// inputs are the bf16 values the device forward (fin_mlp_forward) produced and consumed.
#include <cuda_bf16.h>

#include "fin_internal.cuh"
#include "gemm_f32.cuh"
#include "philox.cuh"

namespace {

using gemmf::bf16_at;
constexpr int kThr = gemmf::kThr;

// ---- head: one thread per sample; stats partials per block [4]: sum L, sum rho, clipped, n
__global__ void k_ppo_head(int B, int K, const float* __restrict__ z, const float* __restrict__ a,
                           const float* __restrict__ logp_old, const float* __restrict__ adv, double sigma,
                           double eps, float* __restrict__ g3, double* __restrict__ part) {
  __shared__ double red[4][kThr / 32];
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  double st[4] = {0.0, 0.0, 0.0, 0.0};
  if (s < B) {
    const double inv_s2 = 1.0 / (sigma * sigma);
    const double cst = (double)K * log(sigma * sqrt(2.0 * 3.141592653589793));
    double q = 0.0;
    for (int k = 0; k < K; ++k) {
      const double mu = tanh((double)z[(size_t)s * K + k]);
      const double d = (double)a[(size_t)s * K + k] - mu;
      q += d * d;
    }
    const double logp = -q * 0.5 * inv_s2 - cst;
    const double rho = exp(logp - (double)logp_old[s]);
    const double A = (double)adv[s];
    const double clipped = fmin(fmax(rho, 1.0 - eps), 1.0 + eps);
    const bool active = !((A > 0.0 && rho > 1.0 + eps) || (A < 0.0 && rho < 1.0 - eps));
    const double c = active ? rho * A : 0.0;
    const double scale = -c / (double)B * inv_s2;
    for (int k = 0; k < K; ++k) {
      const double mu = tanh((double)z[(size_t)s * K + k]);
      g3[(size_t)s * K + k] = (float)(scale * ((double)a[(size_t)s * K + k] - mu) * (1.0 - mu * mu));
    }
    st[0] = fmin(rho * A, clipped * A);
    st[1] = rho;
    st[2] = active ? 0.0 : 1.0;
    st[3] = 1.0;
  }
  for (int j = 0; j < 4; ++j) {
    double v = st[j];
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0) red[j][threadIdx.x >> 5] = v;
  }
  __syncthreads();
  if (threadIdx.x < 4) {
    double v = 0.0;
    for (int w = 0; w < kThr / 32; ++w) v += red[threadIdx.x][w];
    part[(size_t)blockIdx.x * 4 + threadIdx.x] = v;
  }
}

// ---- DQN family head (reading R-DQN): one thread per transition, float64; g_out = dL/d out
__device__ __forceinline__ void qvals(const float* o, int O, bool dueling, double* q) {
  if (!dueling) {
    for (int j = 0; j < O; ++j) q[j] = (double)o[j];
    return;
  }
  const int n = O - 1;
  double m = 0.0;
  for (int j = 0; j < n; ++j) m += (double)o[j];
  m /= n;
  for (int j = 0; j < n; ++j) q[j] = (double)o[n] + (double)o[j] - m;
}
__global__ void k_dqn_head(int B, int O, const float* __restrict__ out, const uint8_t* __restrict__ act,
                           const float* __restrict__ rew, const uint8_t* __restrict__ done,
                           const float* __restrict__ qt, const float* __restrict__ qo, double gamma, int dueling,
                           float* __restrict__ g, double* __restrict__ part) {
  __shared__ double red[4][kThr / 32];
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  double st[4] = {0.0, 0.0, 0.0, 0.0};
  if (s < B) {
    const bool du = dueling != 0;
    const int n = du ? O - 1 : O;
    double q[8], t[8];
    qvals(qt + (size_t)s * O, O, du, t);
    double boot;
    if (qo) {   // Double DQN: the online net picks, the target net evaluates (lowest index on ties)
      double w[8];
      qvals(qo + (size_t)s * O, O, du, w);
      int best = 0;
      for (int j = 1; j < n; ++j)
        if (w[j] > w[best]) best = j;
      boot = t[best];
    } else {
      boot = t[0];
      for (int j = 1; j < n; ++j) boot = fmax(boot, t[j]);
    }
    const double y = (double)rew[s] + gamma * (done[s] ? 0.0 : 1.0) * boot;
    qvals(out + (size_t)s * O, O, du, q);
    const int a = act[s];
    const double d = q[a] - y;
    const double c = 2.0 * d / (double)B;
    for (int j = 0; j < O; ++j) {
      double v;
      if (du) v = j < n ? c * ((j == a ? 1.0 : 0.0) - 1.0 / n) : c;
      else v = j == a ? c : 0.0;
      g[(size_t)s * O + j] = (float)v;
    }
    st[0] = d * d;
    st[1] = q[a];
    st[2] = y;
    st[3] = 1.0;
  }
  for (int j = 0; j < 4; ++j) {
    double v = st[j];
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0) red[j][threadIdx.x >> 5] = v;
  }
  __syncthreads();
  if (threadIdx.x < 4) {
    double v = 0.0;
    for (int w = 0; w < kThr / 32; ++w) v += red[threadIdx.x][w];
    part[(size_t)blockIdx.x * 4 + threadIdx.x] = v;
  }
}

__global__ void k_stats_final(const double* __restrict__ part, int nb, double* __restrict__ stats) {
  if (threadIdx.x < 4) {
    double v = 0.0;
    for (int b = 0; b < nb; ++b) v += part[(size_t)b * 4 + threadIdx.x];
    stats[threadIdx.x] = v;
  }
  __syncthreads();
  if (threadIdx.x == 0) {   // -> L (mean surrogate), mean rho, clipped fraction, B
    const double n = stats[3];
    stats[0] /= n;
    stats[1] /= n;
    stats[2] /= n;
  }
}

__global__ void k_adam(int64_t n, float* __restrict__ th, float* __restrict__ m, float* __restrict__ v,
                       const float* __restrict__ g, float b1, float b2, float lr_c, float inv_c2, float eps) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const float gi = g[i];
  const float mi = fmaf(b1, m[i], (1.f - b1) * gi);
  const float vi = fmaf(b2, v[i], (1.f - b2) * gi * gi);
  m[i] = mi;
  v[i] = vi;
  th[i] -= lr_c * mi / (sqrtf(vi * inv_c2) + eps);
}

// ---- the learner's view of the rollout's samples (sample s = idx[s] = t N + env)
// the full observation (PAPER.md P:129 order: b / b0, close_norm (K), h / max_trade (K), features
// indicator-major (I K)) from the logged env-private entries and the step's market day; the shared
// entries are bf16 of the f32 market value, as the z1s precompute (zshared.cu) quantises them
__global__ void k_gather_obs(EnvDev e, const uint16_t* __restrict__ priv, int P, const int32_t* __restrict__ day,
                             const int64_t* __restrict__ idx, int B, uint16_t* __restrict__ x) {
  const int in_dim = 1 + 2 * e.K + e.I * e.K;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (int64_t)B * in_dim) return;
  const int s = (int)(i / in_dim), c = (int)(i % in_dim);
  const int64_t r = idx[s];
  const uint16_t* pv = priv + (size_t)r * P;
  const float* mrow = e.market + (size_t)day[r] * e.row_floats;
  uint16_t v;
  if (c == 0) {
    v = pv[0];
  } else if (c <= e.K) {
    v = __bfloat16_as_ushort(__float2bfloat16_rn(mrow[e.kp + (c - 1)]));
  } else if (c <= 2 * e.K) {
    v = pv[c - e.K];
  } else {
    const int j = c - 1 - 2 * e.K;
    v = __bfloat16_as_ushort(__float2bfloat16_rn(mrow[(2 + j / e.K) * e.kp + (j % e.K)]));
  }
  x[i] = v;
}

// the rollout's Philox noise of member m at the samples' (global env id, global step)
__global__ void k_noise_at(uint64_t seed, int64_t off, int N, int64_t t_base, const int64_t* __restrict__ idx, int B,
                           int K, int member, float* __restrict__ out) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= B) return;
  const int64_t r = idx[s];
  const int64_t t = r / N, env = r % N;
  for (int blk = 0; blk * 4 < K; ++blk) {
    float z[4];
    philox_normals4((uint64_t)(off + env), (uint32_t)(t_base + t), ((uint32_t)member << 16) | (uint32_t)blk, seed, z);
    for (int j = 0; j < 4 && blk * 4 + j < K; ++j) out[(size_t)s * K + blk * 4 + j] = z[j];
  }
}

// the rollout policy's Gaussian sample and its log-density: a = tanh(z_old) + sigma eps (stored
// f32), log pi_old(a) = -sum (a - tanh(z_old))^2 / (2 sigma^2) - K ln(sigma sqrt(2 pi)), float64
__global__ void k_ppo_prepare(int B, int K, const float* __restrict__ z, const float* __restrict__ eps, double sigma,
                              float* __restrict__ a, float* __restrict__ logp) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= B) return;
  double q = 0.0;
  for (int k = 0; k < K; ++k) {
    const double mu = tanh((double)z[(size_t)s * K + k]);
    const float ak = (float)(mu + sigma * (double)eps[(size_t)s * K + k]);
    a[(size_t)s * K + k] = ak;
    const double d = (double)ak - mu;
    q += d * d;
  }
  logp[s] = (float)(-q / (2.0 * sigma * sigma) - (double)K * log(sigma * sqrt(2.0 * 3.141592653589793)));
}

// fin_policy_load: the tcgen05 image and the factored net's shared W1 columns gathered from the f32
// master weights through the handle's tables, bf16 round to nearest even on the way
__global__ void k_policy_gather(int64_t n, const int32_t* __restrict__ src, const float* w0, const float* w1,
                                const float* w2, const float* w3, uint16_t* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int32_t t = src[i];
  uint16_t v = 0;
  if (t >= 0) {
    const int l = t >> 24, idx = t & 0xffffff;
    const float* w = l == 0 ? w0 : l == 1 ? w1 : l == 2 ? w2 : w3;
    v = __bfloat16_as_ushort(__float2bfloat16_rn(w[idx]));
  }
  out[i] = v;
}
__global__ void k_w1s_gather(int64_t n, const int32_t* __restrict__ src, const float* __restrict__ w0,
                             float* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  out[i] = __bfloat162float(__float2bfloat16_rn(w0[src[i]]));
}

__global__ void k_to_bf16(int64_t n, const float* __restrict__ x, uint16_t* __restrict__ y) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) y[i] = __bfloat16_as_ushort(__float2bfloat16_rn(x[i]));
}

}  // namespace

#ifndef FIN_TC_WGRAD
#define FIN_TC_WGRAD 1   // weight gradients on the tensor cores (tc_gemm.cu); 0: fp32 CUDA-core GEMMs
#endif

namespace fin {

cudaError_t launch_wgrad_tc(int M, int N, int K, const float* g, int ldg, const uint16_t* xh, const float* xf,
                            int ldx, float* dw, cudaStream_t s);
cudaError_t launch_gemm_tc(int M, int N, int K, const float* g, int ldg, int arow, const uint16_t* xh, const float* xf,
                           int ldx, float* C, const void* mask, int ldm, int maskf, cudaStream_t s, int wt = 0,
                           const float* bias = nullptr, int relu = 0);

cudaError_t launch_gather_obs(const EnvDev& e, const uint16_t* priv, int P, const int32_t* day, const int64_t* idx,
                              int B, uint16_t* x, cudaStream_t s) {
  const int64_t n = (int64_t)B * (1 + 2 * e.K + e.I * e.K);
  k_gather_obs<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(e, priv, P, day, idx, B, x);
  return cudaGetLastError();
}
cudaError_t launch_noise_at(uint64_t seed, int64_t off, int N, int64_t t_base, const int64_t* idx, int B, int K,
                            int member, float* out, cudaStream_t s) {
  k_noise_at<<<(B + 127) / 128, 128, 0, s>>>(seed, off, N, t_base, idx, B, K, member, out);
  return cudaGetLastError();
}
cudaError_t launch_ppo_prepare(int B, int K, const float* z, const float* eps, double sigma, float* a, float* logp,
                               cudaStream_t s) {
  k_ppo_prepare<<<(B + 127) / 128, 128, 0, s>>>(B, K, z, eps, sigma, a, logp);
  return cudaGetLastError();
}
cudaError_t launch_policy_gather(int64_t n_pack, const int32_t* pack_src, const float* const (&w)[4], uint16_t* wpack,
                                 int64_t n_w1s, const int32_t* w1s_src, float* w1s, cudaStream_t s) {
  k_policy_gather<<<(unsigned)((n_pack + 255) / 256), 256, 0, s>>>(n_pack, pack_src, w[0], w[1], w[2], w[3], wpack);
  if (n_w1s > 0) k_w1s_gather<<<(unsigned)((n_w1s + 255) / 256), 256, 0, s>>>(n_w1s, w1s_src, w[0], w1s);
  return cudaGetLastError();
}
cudaError_t launch_to_bf16(int64_t n, const float* x, uint16_t* y, cudaStream_t s) {
  k_to_bf16<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(n, x, y);
  return cudaGetLastError();
}

// the backward pass from g3 = dL/d z_out [B][K] (device, f32): g2, g1, weight and bias gradients
cudaError_t backward(int B, int in, int H1, int H2, int K, const uint16_t* x, const uint16_t* hid, const float* g3,
                     const float* w2, const float* w3, float* dw1, float* db1, float* dw2, float* db2, float* dw3,
                     float* db3, cudaStream_t s) {
  using namespace gemmf;
  const int Hs = H1 > H2 ? H1 : H2;   // hidden log row width ([B][2][Hs], fin_mlp_forward)
  size_t scr_n = colsum_floats(B, H1 > H2 ? (H1 > K ? H1 : K) : (H2 > K ? H2 : K));
  for (size_t q : {split_floats(K, H2, B), split_floats(H2, H1, B), split_floats(H1, in, B)}) scr_n = q > scr_n ? q : scr_n;
  float *g2 = nullptr, *g1 = nullptr, *scr = nullptr;
  cudaError_t e = cudaMallocAsync(&g2, sizeof(float) * (size_t)B * H2, s);
  if (e == cudaSuccess) e = cudaMallocAsync(&g1, sizeof(float) * (size_t)B * H1, s);
  if (e == cudaSuccess) e = cudaMallocAsync(&scr, sizeof(float) * scr_n, s);
  if (e != cudaSuccess) return e;
#if FIN_TC_WGRAD
  // g2 = (g3 W3) * [h2 > 0], g1 = (g2 W2) * [h1 > 0] (rows = samples; masks = the hidden log, row
  // stride 2 Hs) on the tensor cores
  // (the short K = k_out contraction stays on the CUDA cores: 77 vs 170 us at B = 65,536)
  e = gemm<false, kBF32, kMaskBF16>(B, H2, K, g3, K, w3, nullptr, H2, g2, hid + Hs, 2 * Hs, nullptr, 0, scr, s);
  if (e == cudaSuccess) e = launch_gemm_tc(B, H1, H2, g2, H2, 1, nullptr, w2, H1, g1, hid, 2 * Hs, 0, s);
#else
  // g2 = (g3 W3) * [h2 > 0]: A = g3 [B][K] row-major, B = W3 [K][H2], mask = h2 (row stride 2 Hs)
  e = gemm<false, kBF32, kMaskBF16>(B, H2, K, g3, K, w3, nullptr, H2, g2, hid + Hs, 2 * Hs, nullptr, 0, scr, s);
  // g1 = (g2 W2) * [h1 > 0]: A = g2 [B][H2] row-major, B = W2 [H2][H1], mask = h1 (row stride 2 Hs)
  if (e == cudaSuccess)
    e = gemm<false, kBF32, kMaskBF16>(B, H1, H2, g2, H2, w2, nullptr, H1, g1, hid, 2 * Hs, nullptr, 0, scr, s);
#endif
  // weight gradients dW_l = g_l^T a_l over the batch (a_l the bf16 activations): tensor cores
#if FIN_TC_WGRAD
  if (e == cudaSuccess) e = launch_wgrad_tc(K, H2, B, g3, K, hid + Hs, nullptr, 2 * Hs, dw3, s);
  if (e == cudaSuccess) e = launch_wgrad_tc(H2, H1, B, g2, H2, hid, nullptr, 2 * Hs, dw2, s);
  if (e == cudaSuccess) e = launch_wgrad_tc(H1, in, B, g1, H1, x, nullptr, in, dw1, s);
#else
  // (CUDA-core form: A = g_l [B][M] (k = sample: AKM), B = activations [B][N])
  if (e == cudaSuccess)
    e = gemm<true, kBBF16, kMaskNone>(K, H2, B, g3, K, nullptr, hid + Hs, 2 * Hs, dw3, nullptr, 0, nullptr, 0, scr, s);
  if (e == cudaSuccess)
    e = gemm<true, kBBF16, kMaskNone>(H2, H1, B, g2, H2, nullptr, hid, 2 * Hs, dw2, nullptr, 0, nullptr, 0, scr, s);
  if (e == cudaSuccess)
    e = gemm<true, kBBF16, kMaskNone>(H1, in, B, g1, H1, nullptr, x, in, dw1, nullptr, 0, nullptr, 0, scr, s);
#endif
  // (scr is free again: the split partials were reduced above)
  colsum(B, K, g3, K, db3, scr, s);
  colsum(B, H2, g2, H2, db2, scr, s);
  colsum(B, H1, g1, H1, db1, scr, s);
  if (e == cudaSuccess) e = cudaGetLastError();
  cudaFreeAsync(g2, s);
  cudaFreeAsync(g1, s);
  cudaFreeAsync(scr, s);
  return e;
}

cudaError_t launch_ppo_grad(int B, int in, int H1, int H2, int K, const uint16_t* x, const uint16_t* hid,
                            const float* z, const float* a, const float* logp_old, const float* adv, double sigma,
                            double eps, const float* w2, const float* w3, float* dw1, float* db1, float* dw2,
                            float* db2, float* dw3, float* db3, double* stats, cudaStream_t s) {
  const int nb = (B + kThr - 1) / kThr;
  float* g3 = nullptr;
  double* part = nullptr;
  cudaError_t e = cudaMallocAsync(&g3, sizeof(float) * (size_t)B * K, s);
  if (e == cudaSuccess) e = cudaMallocAsync(&part, sizeof(double) * 4 * (size_t)nb, s);
  if (e != cudaSuccess) return e;
  k_ppo_head<<<nb, kThr, 0, s>>>(B, K, z, a, logp_old, adv, sigma, eps, g3, part);
  k_stats_final<<<1, 32, 0, s>>>(part, nb, stats);
  e = backward(B, in, H1, H2, K, x, hid, g3, w2, w3, dw1, db1, dw2, db2, dw3, db3, s);
  cudaFreeAsync(g3, s);
  cudaFreeAsync(part, s);
  return e;
}

cudaError_t launch_dqn_grad(int B, int in, int H1, int H2, int O, const uint16_t* x, const uint16_t* hid,
                            const float* out, const uint8_t* act, const float* rew, const uint8_t* done,
                            const float* qt, const float* qo, double gamma, int dueling, const float* w2,
                            const float* w3, float* dw1, float* db1, float* dw2, float* db2, float* dw3, float* db3,
                            double* stats, cudaStream_t s) {
  const int nb = (B + kThr - 1) / kThr;
  float* g3 = nullptr;
  double* part = nullptr;
  cudaError_t e = cudaMallocAsync(&g3, sizeof(float) * (size_t)B * O, s);
  if (e == cudaSuccess) e = cudaMallocAsync(&part, sizeof(double) * 4 * (size_t)nb, s);
  if (e != cudaSuccess) return e;
  k_dqn_head<<<nb, kThr, 0, s>>>(B, O, out, act, rew, done, qt, qo, gamma, dueling, g3, part);
  k_stats_final<<<1, 32, 0, s>>>(part, nb, stats);
  e = backward(B, in, H1, H2, O, x, hid, g3, w2, w3, dw1, db1, dw2, db2, dw3, db3, s);
  cudaFreeAsync(g3, s);
  cudaFreeAsync(part, s);
  return e;
}

cudaError_t launch_adam(int64_t n, float* th, float* m, float* v, const float* g, int step, double lr, double b1,
                        double b2, double eps, cudaStream_t s) {
  const double c1 = 1.0 - pow(b1, (double)step), c2 = 1.0 - pow(b2, (double)step);
  k_adam<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(n, th, m, v, g, (float)b1, (float)b2, (float)(lr / c1),
                                                     (float)(1.0 / c2), (float)eps);
  return cudaGetLastError();
}

}  // namespace fin
