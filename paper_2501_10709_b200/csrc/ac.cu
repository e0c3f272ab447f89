// ac.cu -- the DDPG / SAC updates' device pieces (the stock ensemble's other
// two members; reading R-AC, every formula stated in
// oracle/learn.py):
//   critics:   fin_dense_forward / fin_dense_backward -- a 3-layer ReLU MLP in fp32 on the
//              concatenated input [x(s); a] (fin_concat_obs_action), its parameter gradients and
//              its gradient with respect to the input (dQ/da for the actor)
//   heads:     fin_squash (a = tanh(z + sigma eps) and log pi, float64), fin_critic_head (target y and
//              the squared TD loss, float64), fin_actor_head (DDPG / SAC dL/dz, float64)
//   the actor's backward is the policy MLP's (fin_policy_backward, ppo.cu); fin_soft_update blends
//   target networks (float64, one f32 rounding: bit-identical to the oracle).
#include <cuda_bf16.h>

#include "fin_internal.cuh"
#include "gemm_f32.cuh"

namespace {

constexpr int kThr = 256;

// [x bf16 (S) ; a f32 (K)] -> f32 [B][S + K]
__global__ void k_concat(int B, int S, const uint16_t* __restrict__ x, int K, const float* __restrict__ a,
                         float* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int D = S + K;
  if (i >= (int64_t)B * D) return;
  const int64_t s = i / D;
  const int c = (int)(i % D);
  out[i] = c < S ? gemmf::bf16_at(x, (size_t)s * S + c) : a[(size_t)s * K + (c - S)];
}

// ln(1 - tanh(u)^2) = 2 (ln 2 - u - softplus(-2 u))
__device__ __forceinline__ double log1m_tanh2(double u) {
  const double x = -2.0 * u;
  const double sp = fmax(x, 0.0) + log1p(exp(-fabs(x)));
  return 2.0 * (0.6931471805599453 - u - sp);
}

// a = tanh(z + sigma eps) (eps NULL: tanh z); logp (optional) = sum_k [-eps^2 / 2 - ln(sigma sqrt(2 pi))
// - ln(1 - tanh(u)^2)]
__global__ void k_squash(int B, int K, const float* __restrict__ z, const float* __restrict__ eps, double sigma,
                         float* __restrict__ a, float* __restrict__ logp) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= B) return;
  const double c = log(sigma * sqrt(2.0 * 3.141592653589793));
  double acc = 0.0;
  for (int k = 0; k < K; ++k) {
    const double e = eps ? (double)eps[(size_t)s * K + k] : 0.0;
    const double u = (double)z[(size_t)s * K + k] + sigma * e;
    a[(size_t)s * K + k] = (float)tanh(u);
    if (eps) acc += -0.5 * e * e - c - log1m_tanh2(u);
  }
  if (logp) logp[s] = (float)acc;
}

// stats partials per block [4] (sum over the block's samples), reduced in a fixed order
__device__ __forceinline__ void block_stats(const double (&st)[4], double* part) {
  __shared__ double red[4][kThr / 32];
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

// y = r + gamma (1 - d) (min(q1', q2') - alpha logp'); L = (q - y)^2, g = 2 (q - y) / B
__global__ void k_critic_head(int B, const float* __restrict__ q, const float* __restrict__ r,
                              const uint8_t* __restrict__ done, const float* __restrict__ q1n,
                              const float* __restrict__ q2n, const float* __restrict__ lpn, double gamma, double alpha,
                              float* __restrict__ g, double* __restrict__ part) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  double st[4] = {0.0, 0.0, 0.0, 0.0};
  if (s < B) {
    double boot = (double)q1n[s];
    if (q2n && (double)q2n[s] < boot) boot = (double)q2n[s];
    if (lpn) boot = boot - alpha * (double)lpn[s];
    const double y = (double)r[s] + gamma * (done[s] ? 0.0 : 1.0) * boot;
    const double d = (double)q[s] - y;
    g[s] = (float)(2.0 * d / (double)B);
    st[0] = d * d;
    st[1] = (double)q[s];
    st[2] = y;
    st[3] = 1.0;
  }
  block_stats(st, part);
}

// DDPG (lp == NULL): g_z = -(1/B) dq1 (1 - a^2), L = -q1.  SAC: the smaller critic m (Q1 on ties),
// g_z = (1/B) (2 alpha a - dq_m (1 - a^2)), L = alpha logp - q_m.  dq rows have stride ldq.
__global__ void k_actor_head(int B, int K, const float* __restrict__ a, const float* __restrict__ lp,
                             const float* __restrict__ q1, const float* __restrict__ dq1, const float* __restrict__ q2,
                             const float* __restrict__ dq2, int ldq, double alpha, float* __restrict__ gz,
                             double* __restrict__ part) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  double st[4] = {0.0, 0.0, 0.0, 0.0};
  if (s < B) {
    const bool two = q2 && (double)q2[s] < (double)q1[s];
    const double qm = two ? (double)q2[s] : (double)q1[s];
    const float* dq = (two ? dq2 : dq1) + (size_t)s * ldq;
    const double inv = 1.0 / (double)B;
    for (int k = 0; k < K; ++k) {
      const double ak = (double)a[(size_t)s * K + k];
      const double t = (double)dq[k] * (1.0 - ak * ak);
      gz[(size_t)s * K + k] = (float)(lp ? (2.0 * alpha * ak - t) * inv : -t * inv);
    }
    st[0] = lp ? alpha * (double)lp[s] - qm : -qm;
    st[1] = qm;
    st[2] = lp ? (double)lp[s] : 0.0;
    st[3] = 1.0;
  }
  block_stats(st, part);
}

// [0] and [1], [2] divided by the count [3]
__global__ void k_stats_mean(const double* __restrict__ part, int nb, double* __restrict__ stats) {
  if (threadIdx.x < 4) {
    double v = 0.0;
    for (int b = 0; b < nb; ++b) v += part[(size_t)b * 4 + threadIdx.x];
    stats[threadIdx.x] = v;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const double n = stats[3];
    stats[0] /= n;
    stats[1] /= n;
    stats[2] /= n;
  }
}

// theta_t = f32(tau theta + (1 - tau) theta_t), float64 products and sum, no contraction
__global__ void k_soft_update(int64_t n, float* __restrict__ t, const float* __restrict__ o, double tau, double omt) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  t[i] = (float)__dadd_rn(__dmul_rn(tau, (double)o[i]), __dmul_rn(omt, (double)t[i]));
}

}  // namespace

#ifndef FIN_TC_WGRAD
#define FIN_TC_WGRAD 1
#endif

namespace fin {

cudaError_t launch_wgrad_tc(int M, int N, int K, const float* g, int ldg, const uint16_t* xh, const float* xf,
                            int ldx, float* dw, cudaStream_t s);
cudaError_t launch_gemm_tc(int M, int N, int K, const float* g, int ldg, int arow, const uint16_t* xh, const float* xf,
                           int ldx, float* C, const void* mask, int ldm, int maskf, cudaStream_t s, int wt = 0,
                           const float* bias = nullptr, int relu = 0);

cudaError_t launch_concat_sa(int B, int S, const uint16_t* x, int K, const float* a, float* out, cudaStream_t s) {
  const int64_t n = (int64_t)B * (S + K);
  k_concat<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(B, S, x, K, a, out);
  return cudaGetLastError();
}

cudaError_t launch_squash(int B, int K, const float* z, const float* eps, double sigma, float* a, float* logp,
                          cudaStream_t s) {
  k_squash<<<(B + 127) / 128, 128, 0, s>>>(B, K, z, eps, sigma, a, logp);
  return cudaGetLastError();
}

cudaError_t launch_critic_head(int B, const float* q, const float* r, const uint8_t* done, const float* q1n,
                               const float* q2n, const float* lpn, double gamma, double alpha, float* g, double* stats,
                               cudaStream_t s) {
  const int nb = (B + kThr - 1) / kThr;
  double* part = nullptr;
  cudaError_t e = cudaMallocAsync(&part, sizeof(double) * 4 * (size_t)nb, s);
  if (e != cudaSuccess) return e;
  k_critic_head<<<nb, kThr, 0, s>>>(B, q, r, done, q1n, q2n, lpn, gamma, alpha, g, part);
  k_stats_mean<<<1, 32, 0, s>>>(part, nb, stats);
  e = cudaGetLastError();
  cudaFreeAsync(part, s);
  return e;
}

cudaError_t launch_actor_head(int B, int K, const float* a, const float* lp, const float* q1, const float* dq1,
                              const float* q2, const float* dq2, int ldq, double alpha, float* gz, double* stats,
                              cudaStream_t s) {
  const int nb = (B + kThr - 1) / kThr;
  double* part = nullptr;
  cudaError_t e = cudaMallocAsync(&part, sizeof(double) * 4 * (size_t)nb, s);
  if (e != cudaSuccess) return e;
  k_actor_head<<<nb, kThr, 0, s>>>(B, K, a, lp, q1, dq1, q2, dq2, ldq, alpha, gz, part);
  k_stats_mean<<<1, 32, 0, s>>>(part, nb, stats);
  e = cudaGetLastError();
  cudaFreeAsync(part, s);
  return e;
}

cudaError_t launch_soft_update(int64_t n, float* t, const float* o, double tau, cudaStream_t s) {
  k_soft_update<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(n, t, o, tau, 1.0 - tau);
  return cudaGetLastError();
}

// critic forward: hidden f32 [B][H1 + H2] (h1 then h2 per row), out f32 [B][O]
cudaError_t dense_forward(int B, int in, int H1, int H2, int O, const float* x, const float* w1, const float* b1,
                          const float* w2, const float* b2, const float* w3, const float* b3, float* hid, float* out,
                          cudaStream_t s) {
  using namespace gemmf;
  const int Hs = H1 + H2;
  // z = x W^T + b: A = x row-major [B][in], B(k, n) = W[n][k] (transposed mode), bias + ReLU epilogue;
  // hidden rows are written with stride Hs through a [B][Hs] view (one GEMM per layer, N = H_l)
  float *h1 = nullptr, *h2 = nullptr;
  cudaError_t e = cudaMallocAsync(&h1, sizeof(float) * (size_t)B * H1, s);
  if (e == cudaSuccess) e = cudaMallocAsync(&h2, sizeof(float) * (size_t)B * H2, s);
  if (e != cudaSuccess) return e;
#if FIN_TC_WGRAD
  // the two wide layers on the tensor cores (weights pre-split once per call), the output layer (N = O,
  // a few columns) on the CUDA cores
  e = launch_gemm_tc(B, H1, in, x, in, 1, nullptr, w1, in, h1, nullptr, 0, 0, s, 1, b1, 1);
  if (e == cudaSuccess) e = launch_gemm_tc(B, H2, H1, h1, H1, 1, nullptr, w2, H1, h2, nullptr, 0, 0, s, 1, b2, 1);
#else
  e = gemm<false, kBF32T, kMaskNone>(B, H1, in, x, in, w1, nullptr, in, h1, nullptr, 0, b1, 1, nullptr, s);
  if (e == cudaSuccess)
    e = gemm<false, kBF32T, kMaskNone>(B, H2, H1, h1, H1, w2, nullptr, H1, h2, nullptr, 0, b2, 1, nullptr, s);
#endif
  if (e == cudaSuccess)
    e = gemm<false, kBF32T, kMaskNone>(B, O, H2, h2, H2, w3, nullptr, H2, out, nullptr, 0, b3, 0, nullptr, s);
  if (e == cudaSuccess && hid) {
    e = cudaMemcpy2DAsync(hid, sizeof(float) * Hs, h1, sizeof(float) * H1, sizeof(float) * H1, B,
                          cudaMemcpyDeviceToDevice, s);
    if (e == cudaSuccess)
      e = cudaMemcpy2DAsync(hid + H1, sizeof(float) * Hs, h2, sizeof(float) * H2, sizeof(float) * H2, B,
                            cudaMemcpyDeviceToDevice, s);
  }
  cudaFreeAsync(h1, s);
  cudaFreeAsync(h2, s);
  return e;
}

// critic backward from g3 = dL/d out [B][O]: parameter gradients (dw1 == NULL: skipped) and g_x [B][in]
// (NULL: skipped)
cudaError_t dense_backward(int B, int in, int H1, int H2, int O, const float* x, const float* hid, const float* g3,
                           const float* w1, const float* w2, const float* w3, float* dw1, float* db1, float* dw2,
                           float* db2, float* dw3, float* db3, float* gx, cudaStream_t s) {
  using namespace gemmf;
  const int Hs = H1 + H2;
  const bool params = dw1 != nullptr;
  size_t scr_n = gx ? split_floats(B, in, H1) : 1;   // the g_x GEMM may split over H1
  if (params) {
    const size_t c = colsum_floats(B, H1 > H2 ? (H1 > O ? H1 : O) : (H2 > O ? H2 : O));
    for (size_t q : {c, split_floats(O, H2, B), split_floats(H2, H1, B), split_floats(H1, in, B)})
      scr_n = q > scr_n ? q : scr_n;
  }
  float *g2 = nullptr, *g1 = nullptr, *scr = nullptr;
  cudaError_t e = cudaMallocAsync(&g2, sizeof(float) * (size_t)B * H2, s);
  if (e == cudaSuccess) e = cudaMallocAsync(&g1, sizeof(float) * (size_t)B * H1, s);
  if (e == cudaSuccess) e = cudaMallocAsync(&scr, sizeof(float) * scr_n, s);
  if (e != cudaSuccess) return e;
#if FIN_TC_WGRAD
  // g2 = (g3 W3) * [h2 > 0], g1 = (g2 W2) * [h1 > 0], g_x = g1 W1 (rows = samples) on the tensor cores
  e = gemm<false, kBF32, kMaskF32>(B, H2, O, g3, O, w3, nullptr, H2, g2, hid + H1, Hs, nullptr, 0, nullptr, s);
  if (e == cudaSuccess) e = launch_gemm_tc(B, H1, H2, g2, H2, 1, nullptr, w2, H1, g1, hid, Hs, 1, s);
  if (e == cudaSuccess && gx) e = launch_gemm_tc(B, in, H1, g1, H1, 1, nullptr, w1, in, gx, nullptr, 0, 0, s);
#else
  // g2 = (g3 W3) * [h2 > 0]: A = g3 [B][O], B = W3 [O][H2]; g1 = (g2 W2) * [h1 > 0]
  e = gemm<false, kBF32, kMaskF32>(B, H2, O, g3, O, w3, nullptr, H2, g2, hid + H1, Hs, nullptr, 0, nullptr, s);
  if (e == cudaSuccess)
    e = gemm<false, kBF32, kMaskF32>(B, H1, H2, g2, H2, w2, nullptr, H1, g1, hid, Hs, nullptr, 0, nullptr, s);
  // g_x = g1 W1: A = g1 [B][H1], B = W1 [H1][in]
  if (e == cudaSuccess && gx)
    e = gemm<false, kBF32, kMaskNone>(B, in, H1, g1, H1, w1, nullptr, in, gx, nullptr, 0, nullptr, 0, scr, s);
#endif
  if (e == cudaSuccess && params) {
#if FIN_TC_WGRAD
    e = launch_wgrad_tc(O, H2, B, g3, O, nullptr, hid + H1, Hs, dw3, s);
    if (e == cudaSuccess) e = launch_wgrad_tc(H2, H1, B, g2, H2, nullptr, hid, Hs, dw2, s);
    if (e == cudaSuccess) e = launch_wgrad_tc(H1, in, B, g1, H1, nullptr, x, in, dw1, s);
#else
    e = gemm<true, kBF32, kMaskNone>(O, H2, B, g3, O, hid + H1, nullptr, Hs, dw3, nullptr, 0, nullptr, 0, scr, s);
    if (e == cudaSuccess)
      e = gemm<true, kBF32, kMaskNone>(H2, H1, B, g2, H2, hid, nullptr, Hs, dw2, nullptr, 0, nullptr, 0, scr, s);
    if (e == cudaSuccess)
      e = gemm<true, kBF32, kMaskNone>(H1, in, B, g1, H1, x, nullptr, in, dw1, nullptr, 0, nullptr, 0, scr, s);
#endif
    colsum(B, O, g3, O, db3, scr, s);
    colsum(B, H2, g2, H2, db2, scr, s);
    colsum(B, H1, g1, H1, db1, scr, s);
  }
  if (e == cudaSuccess) e = cudaGetLastError();
  cudaFreeAsync(g2, s);
  cudaFreeAsync(g1, s);
  cudaFreeAsync(scr, s);
  return e;
}

}  // namespace fin
