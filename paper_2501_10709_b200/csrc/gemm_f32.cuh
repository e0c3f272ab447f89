// gemm_f32.cuh -- the learner's fp32 CUDA-core contractions: the
// backward passes of fin_ppo_grad / fin_dqn_grad / fin_policy_backward and the critics'
// forward and backward (fin_dense_forward / fin_dense_backward).  Deterministic: 64 x 64 output
// tiles, 4 x 4 per thread, split-K over long reductions with the partials summed in a fixed order.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace gemmf {
namespace {   // internal linkage: each including translation unit keeps its own kernels

constexpr int kTile = 64, kBK = 16, kThr = 256;

__device__ __forceinline__ float bf16_at(const uint16_t* p, size_t i) {
  return __uint_as_float((uint32_t)p[i] << 16);
}

// B operand modes: B(k, n) = Bf[k ldb + n] (f32), bf16 Bh[k ldb + n], or Bf[n ldb + k] (f32, the
// transposed [out][in] weight of a forward layer)
enum { kBF32 = 0, kBBF16 = 1, kBF32T = 2 };
// output mask modes (applied when the GEMM is not split): none, bf16 > 0, f32 > 0 at mask[m ldm + n]
enum { kMaskNone = 0, kMaskBF16 = 1, kMaskF32 = 2 };

// C[m][n] = sum_k A(m, k) B(k, n) over k in this split's range, A(m, k) = AKM ? A[k lda + m] :
// A[m lda + k]; out: part[split][M][N] (or C when not split); epilogue (not split): + bias[n],
// ReLU, mask
template <bool AKM, int BM, int MM>
__global__ void __launch_bounds__(kThr) k_gemm(int M, int N, int Ktot, int kchunk, const float* __restrict__ A,
                                               int lda, const float* __restrict__ Bf, const uint16_t* __restrict__ Bh,
                                               int ldb, float* __restrict__ out, const void* __restrict__ mask, int ldm,
                                               const float* __restrict__ bias, int relu) {
  __shared__ float As[kBK][kTile + 4];
  __shared__ float Bs[kBK][kTile + 4];
  const int m0 = blockIdx.y * kTile, n0 = blockIdx.x * kTile;
  const int k0 = blockIdx.z * kchunk, k1 = min(Ktot, k0 + kchunk);
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  float acc[4][4] = {};
  for (int kb = k0; kb < k1; kb += kBK) {
    for (int e = threadIdx.x; e < kBK * kTile; e += kThr) {
      const int kk = e / kTile, mm = e % kTile;   // consecutive threads: consecutive m (AKM) / n
      const int k = kb + kk;
      if (AKM) As[kk][mm] = (k < k1 && m0 + mm < M) ? A[(size_t)k * lda + m0 + mm] : 0.f;
      if (BM != kBF32T) {
        float bv = 0.f;
        if (k < k1 && n0 + mm < N) bv = BM == kBBF16 ? bf16_at(Bh, (size_t)k * ldb + n0 + mm) : Bf[(size_t)k * ldb + n0 + mm];
        Bs[kk][mm] = bv;
      }
    }
    for (int e = threadIdx.x; e < kBK * kTile; e += kThr) {   // row-major operands: consecutive k
      const int mm = e / kBK, kk = e % kBK;
      const int k = kb + kk;
      if (!AKM) As[kk][mm] = (k < k1 && m0 + mm < M) ? A[(size_t)(m0 + mm) * lda + k] : 0.f;
      if (BM == kBF32T) Bs[kk][mm] = (k < k1 && n0 + mm < N) ? Bf[(size_t)(n0 + mm) * ldb + k] : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < kBK; ++kk) {
      float av[4], bv[4];
#pragma unroll
      for (int r = 0; r < 4; ++r) av[r] = As[kk][ty * 4 + r];
#pragma unroll
      for (int c = 0; c < 4; ++c) bv[c] = Bs[kk][tx * 4 + c];
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c) acc[r][c] = fmaf(av[r], bv[c], acc[r][c]);
    }
    __syncthreads();
  }
  float* dst = out + (size_t)blockIdx.z * M * N;
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const int m = m0 + ty * 4 + r;
    if (m >= M) continue;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int n = n0 + tx * 4 + c;
      if (n >= N) continue;
      float v = acc[r][c];
      if (bias) v += bias[n];
      if (relu) v = fmaxf(v, 0.f);
      if (MM == kMaskBF16 && !(bf16_at(static_cast<const uint16_t*>(mask), (size_t)m * ldm + n) > 0.f)) v = 0.f;
      if (MM == kMaskF32 && !(static_cast<const float*>(mask)[(size_t)m * ldm + n] > 0.f)) v = 0.f;
      dst[(size_t)m * N + n] = v;
    }
  }
}

// The same contraction with 128 x 128 output tiles, 8 x 8 per thread, K in blocks of 8 prefetched
// into registers one block ahead (double-buffered shared memory, one barrier per block): the large
// GEMMs (M, N >= 128) of the learner.  Same operand modes, epilogue and split-K contract as k_gemm.
template <bool AKM, int BM, int MM>
__global__ void __launch_bounds__(kThr) k_gemm128(int M, int N, int Ktot, int kchunk, const float* __restrict__ A,
                                                  int lda, const float* __restrict__ Bf,
                                                  const uint16_t* __restrict__ Bh, int ldb, float* __restrict__ out,
                                                  const void* __restrict__ mask, int ldm,
                                                  const float* __restrict__ bias, int relu) {
  constexpr int T = 128, BK = 8;
  __shared__ __align__(16) float As[2][BK][T + 4];
  __shared__ __align__(16) float Bs[2][BK][T + 4];
  const int tid = threadIdx.x;
  const int m0 = blockIdx.y * T, n0 = blockIdx.x * T;
  const int k0 = blockIdx.z * kchunk, k1 = min(Ktot, k0 + kchunk);
  const int tx = tid % 16, ty = tid / 16;
  float acc[8][8];
#pragma unroll
  for (int r = 0; r < 8; ++r)
#pragma unroll
    for (int c = 0; c < 8; ++c) acc[r][c] = 0.f;
  float ra[4], rb[4];
  // operands contiguous along M / N: element (kk = tid / 32, col (tid % 32) + 32 j); contiguous
  // along K: element (row tid / 2, kk = (tid % 2) 4 + j)
  auto load = [&](int kb) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      if (AKM) {
        const int k = kb + tid / 32, m = m0 + (tid % 32) + 32 * j;
        ra[j] = (k < k1 && m < M) ? A[(size_t)k * lda + m] : 0.f;
      } else {
        const int k = kb + (tid % 2) * 4 + j, m = m0 + tid / 2;
        ra[j] = (k < k1 && m < M) ? A[(size_t)m * lda + k] : 0.f;
      }
      if (BM == kBF32T) {
        const int k = kb + (tid % 2) * 4 + j, n = n0 + tid / 2;
        rb[j] = (k < k1 && n < N) ? Bf[(size_t)n * ldb + k] : 0.f;
      } else {
        const int k = kb + tid / 32, n = n0 + (tid % 32) + 32 * j;
        rb[j] = (k < k1 && n < N) ? (BM == kBBF16 ? bf16_at(Bh, (size_t)k * ldb + n) : Bf[(size_t)k * ldb + n]) : 0.f;
      }
    }
  };
  auto store = [&](int buf) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      if (AKM) As[buf][tid / 32][(tid % 32) + 32 * j] = ra[j];
      else As[buf][(tid % 2) * 4 + j][tid / 2] = ra[j];
      if (BM == kBF32T) Bs[buf][(tid % 2) * 4 + j][tid / 2] = rb[j];
      else Bs[buf][tid / 32][(tid % 32) + 32 * j] = rb[j];
    }
  };
  load(k0);
  store(0);
  __syncthreads();
  int buf = 0;
  for (int kb = k0; kb < k1; kb += BK) {
    const bool more = kb + BK < k1;
    if (more) load(kb + BK);
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      const float4 a0 = *reinterpret_cast<const float4*>(&As[buf][kk][ty * 8]);
      const float4 a1 = *reinterpret_cast<const float4*>(&As[buf][kk][ty * 8 + 4]);
      const float4 b0 = *reinterpret_cast<const float4*>(&Bs[buf][kk][tx * 8]);
      const float4 b1 = *reinterpret_cast<const float4*>(&Bs[buf][kk][tx * 8 + 4]);
      const float a[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
      const float b[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
      for (int r = 0; r < 8; ++r)
#pragma unroll
        for (int c = 0; c < 8; ++c) acc[r][c] = fmaf(a[r], b[c], acc[r][c]);
    }
    if (more) store(buf ^ 1);
    __syncthreads();
    buf ^= 1;
  }
  float* dst = out + (size_t)blockIdx.z * M * N;
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    const int m = m0 + ty * 8 + r;
    if (m >= M) continue;
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const int n = n0 + tx * 8 + c;
      if (n >= N) continue;
      float v = acc[r][c];
      if (bias) v += bias[n];
      if (relu) v = fmaxf(v, 0.f);
      if (MM == kMaskBF16 && !(bf16_at(static_cast<const uint16_t*>(mask), (size_t)m * ldm + n) > 0.f)) v = 0.f;
      if (MM == kMaskF32 && !(static_cast<const float*>(mask)[(size_t)m * ldm + n] > 0.f)) v = 0.f;
      dst[(size_t)m * N + n] = v;
    }
  }
}

// fixed-order sum of the split partials: C[i] = sum_z part[z][i]
__global__ void k_sum_splits(const float* __restrict__ part, int splits, size_t n, float* __restrict__ C) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  float v = 0.f;
  for (int z = 0; z < splits; ++z) v += part[(size_t)z * n + i];
  C[i] = v;
}

// column sums of g [B][H] (row stride ldg; bias gradients), deterministic: block (column group of
// 32, row chunk) -> 8 row-strided partials per column reduced in a fixed order -> part[chunk][H];
// then the chunks summed in order
constexpr int kColRows = 2048;
__global__ void k_colsum_part(int B, int H, const float* __restrict__ g, int ldg, float* __restrict__ part) {
  __shared__ float red[8][33];
  const int j = blockIdx.x * 32 + (threadIdx.x & 31), r = threadIdx.x >> 5;
  const int s0 = blockIdx.y * kColRows, s1 = min(B, s0 + kColRows);
  float v = 0.f;
  if (j < H)
    for (int s = s0 + r; s < s1; s += 8) v += g[(size_t)s * ldg + j];
  red[r][threadIdx.x & 31] = v;
  __syncthreads();
  if (r == 0 && j < H) {
    float t = 0.f;
    for (int q = 0; q < 8; ++q) t += red[q][threadIdx.x & 31];
    part[(size_t)blockIdx.y * H + j] = t;
  }
}
__global__ void k_colsum_final(int chunks, int H, const float* __restrict__ part, float* __restrict__ out) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= H) return;
  float v = 0.f;
  for (int c = 0; c < chunks; ++c) v += part[(size_t)c * H + j];
  out[j] = v;
}

// launch plan of one GEMM: tile size (128 for M, N >= 128), K split (~2 waves of blocks, >= 64 rows of K
// per split; none with an epilogue), K chunk (a multiple of 16) and the splits used
struct GemmPlan {
  int big, kchunk, used;
};
inline GemmPlan plan_for(int M, int N, int K, bool epi) {
  GemmPlan g;
  g.big = (M >= 128 && N >= 128) ? 1 : 0;
  const int T = g.big ? 128 : kTile;
  const int tiles = ((M + T - 1) / T) * ((N + T - 1) / T);
  int s = (2 * 148 + tiles - 1) / tiles;
  const int maxs = (K + 4 * kBK - 1) / (4 * kBK);
  if (s > maxs) s = maxs;
  if (s < 1 || epi) s = 1;
  g.kchunk = ((K + s - 1) / s + kBK - 1) / kBK * kBK;
  g.used = (K + g.kchunk - 1) / g.kchunk;
  if (g.used < 1) g.used = 1;
  return g;
}
// floats of split partials one split GEMM needs (1 when it is not split)
inline size_t split_floats(int M, int N, int K) {
  const GemmPlan g = plan_for(M, N, K, false);
  return g.used > 1 ? (size_t)g.used * M * N : (size_t)1;
}
inline size_t colsum_floats(int B, int H) { return (size_t)((B + kColRows - 1) / kColRows) * H; }

// C[M][N] with split-K (no epilogue) or one pass with the bias / ReLU / mask epilogue
template <bool AKM, int BM, int MM>
cudaError_t gemm(int M, int N, int K, const float* A, int lda, const float* Bf, const uint16_t* Bh, int ldb, float* C,
                 const void* mask, int ldm, const float* bias, int relu, float* scratch, cudaStream_t s) {
  const GemmPlan g = plan_for(M, N, K, MM != kMaskNone || bias || relu);
  float* out = g.used <= 1 ? C : scratch;
  if (g.big) {
    dim3 grid((N + 127) / 128, (M + 127) / 128, g.used);
    k_gemm128<AKM, BM, MM><<<grid, kThr, 0, s>>>(M, N, K, g.kchunk, A, lda, Bf, Bh, ldb, out, mask, ldm, bias, relu);
  } else {
    dim3 grid((N + kTile - 1) / kTile, (M + kTile - 1) / kTile, g.used);
    k_gemm<AKM, BM, MM><<<grid, kThr, 0, s>>>(M, N, K, g.kchunk, A, lda, Bf, Bh, ldb, out, mask, ldm, bias, relu);
  }
  if (g.used > 1) {
    const size_t n = (size_t)M * N;
    k_sum_splits<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(scratch, g.used, n, C);
  }
  return cudaGetLastError();
}

// out[j] = sum_s g[s ldg + j] for j < H (scratch: colsum_floats(B, H))
inline void colsum(int B, int H, const float* g, int ldg, float* out, float* scratch, cudaStream_t s) {
  const int chunks = (B + kColRows - 1) / kColRows;
  k_colsum_part<<<dim3((H + 31) / 32, chunks), 256, 0, s>>>(B, H, g, ldg, scratch);
  k_colsum_final<<<(H + 127) / 128, 128, 0, s>>>(chunks, H, scratch, out);
}

}  // namespace
}  // namespace gemmf
