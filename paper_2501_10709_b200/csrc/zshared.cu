// zshared.cu -- the shared part of layer 1 for the factored stock policy:
//     z1s[r][n] = sum_s W1_shared[n][s] * q(x_shared(r))[s]  (+ b1[n])
// (the layer-1 bias is folded in here, in float64, when it is non-zero: the rollout and
// the probe then never add it in their epilogues)
// for every market day r (rollouts) or every probe row r (fin_mlp_forward), in
// float64 (bf16 x bf16 products are exact in float64), rounded once to fp32.
// One CTA per row: the row's shared inputs are converted to bf16 once into shared
// memory, then thread n accumulates output n over the transposed weights (coalesced).
#include <cuda_bf16.h>

#include "fin_internal.cuh"
#include "tc_plan.cuh"

namespace {

template <class Obs>
__device__ __forceinline__ float market_shared_value(const float* mrow, int kp, int s) {
  constexpr int KA = (Obs::kEnv - 1);
  // close_norm (channel 1) for s < K, then indicator-major features (channel 2 + j / K)
  if (s < KA) return mrow[kp + s];
  const int j = s - KA;
  return mrow[(2 + j / KA) * kp + (j % KA)];
}

template <class Obs>
__global__ void k_z1s_market(const float* __restrict__ w1s_t /*[S][H]*/, const float* __restrict__ b1, int H,
                             const float* __restrict__ market, int row_floats, int kp, float* __restrict__ z1s /*[rows][H]*/) {
  __shared__ double xs[Obs::kShared];
  const int r = blockIdx.x;
  const float* mrow = market + (size_t)r * row_floats;
  for (int s = threadIdx.x; s < Obs::kShared; s += blockDim.x)
    xs[s] = (double)__bfloat162float(__float2bfloat16_rn(market_shared_value<Obs>(mrow, kp, s)));
  __syncthreads();
  for (int n = threadIdx.x; n < H; n += blockDim.x) {
    double acc = 0.0;
    for (int s = 0; s < Obs::kShared; ++s) acc = fma((double)w1s_t[(size_t)s * H + n], xs[s], acc);
    if (b1) acc += (double)b1[n];
    z1s[(size_t)r * H + n] = (float)acc;
  }
}

// probe rows: kRows rows per CTA, so each weight read from L2 feeds kRows independent float64
// chains (the one-row form re-read all of W1_shared per row: 18 GB of L2 traffic at B = 65,536);
// the same fma order per output as k_z1s_market (s ascending, then + b1), so the same bits
constexpr int kRows = 16;
template <class Obs>
__global__ void k_z1s_probe(const float* __restrict__ w1s_t, const float* __restrict__ b1, int H,
                            const uint16_t* __restrict__ x, int in_dim, int B, float* __restrict__ z1s) {
  __shared__ __align__(16) double xs[Obs::kShared][kRows];   // [s][row]: a thread reads its rows' values
  const int r0 = blockIdx.x * kRows;                          // of one s as 8 x 16 B
  for (int i = threadIdx.x; i < Obs::kShared * kRows; i += blockDim.x) {
    const int rr = i / Obs::kShared, sidx = i % Obs::kShared;
    const int col = Obs::shared_col(sidx);
    const uint16_t bits = (r0 + rr < B && col < in_dim) ? x[(size_t)(r0 + rr) * in_dim + col] : (uint16_t)0;
    xs[sidx][rr] = (double)__uint_as_float((uint32_t)bits << 16);
  }
  __syncthreads();
  for (int n = threadIdx.x; n < H; n += blockDim.x) {
    double acc[kRows];
#pragma unroll
    for (int rr = 0; rr < kRows; ++rr) acc[rr] = 0.0;
    for (int sidx = 0; sidx < Obs::kShared; ++sidx) {
      const double w = (double)w1s_t[(size_t)sidx * H + n];
      const double2* xv = reinterpret_cast<const double2*>(xs[sidx]);
#pragma unroll
      for (int q = 0; q < kRows / 2; ++q) {
        const double2 v = xv[q];
        acc[2 * q] = fma(w, v.x, acc[2 * q]);
        acc[2 * q + 1] = fma(w, v.y, acc[2 * q + 1]);
      }
    }
    const double bn = b1 ? (double)b1[n] : 0.0;
#pragma unroll
    for (int rr = 0; rr < kRows; ++rr) {
      if (r0 + rr >= B) break;
      double a = acc[rr];
      if (b1) a += bn;
      z1s[(size_t)(r0 + rr) * H + n] = (float)a;
    }
  }
}

}  // namespace

namespace fin {

// net 0 = C1 (K=30, I=8), 3 = the paper's 301-64-32-30 on the C1 env, net 1 = small (K=4, I=4)
cudaError_t launch_z1s_market(int net, const float* w1s_t, const float* b1, int H, const EnvDev& e, float* z1s,
                              cudaStream_t s) {
  if (net == 0 || net == 3) k_z1s_market<ObsC1><<<e.rows, 256, 0, s>>>(w1s_t, b1, H, e.market, e.row_floats, e.kp, z1s);
  else if (net == 1) k_z1s_market<ObsSmall><<<e.rows, 128, 0, s>>>(w1s_t, b1, H, e.market, e.row_floats, e.kp, z1s);
  else return cudaErrorInvalidValue;
  return cudaGetLastError();
}

cudaError_t launch_z1s_probe(int net, const float* w1s_t, const float* b1, int H, const uint16_t* x, int B, int in_dim,
                             float* z1s, cudaStream_t s) {
  const unsigned blocks = (unsigned)((B + kRows - 1) / kRows);
  if (net == 0 || net == 3) k_z1s_probe<ObsC1><<<blocks, 256, 0, s>>>(w1s_t, b1, H, x, in_dim, B, z1s);
  else if (net == 1) k_z1s_probe<ObsSmall><<<blocks, 128, 0, s>>>(w1s_t, b1, H, x, in_dim, B, z1s);
  else return cudaErrorInvalidValue;
  return cudaGetLastError();
}

}  // namespace fin
