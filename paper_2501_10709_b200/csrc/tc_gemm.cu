// tc_gemm.cu -- the learner's contractions on the tensor cores: weight gradients dW = G^T X, the
// backpropagated products g W and the critics' forward layers x W^T + b
// (the backward passes of fin_ppo_grad / fin_dqn_grad / fin_policy_backward and
// fin_dense_backward, readings R-PPO / R-DQN / R-AC).
//
// dW[m][n] = sum_k G[k][m] X[k][n] over the batch k (G = dL/dz of a layer, fp32; X = the layer's input:
// bf16 activations of the policy forward, or fp32 for the critics).  One CTA owns a 128 x N_t output
// tile (N_t <= 256) and a K chunk of the batch; the chunks are summed afterwards in a fixed order
// (deterministic).  Per block of 32 batch rows, all 256 threads stage the operands into shared memory in
// the UMMA K-major canonical layout (a transpose: the batch is the contraction dimension), one thread
// issues tcgen05.mma kind::f16 into a TMEM accumulator, and the next block is staged while the MMAs run
// (two buffers, completion by tcgen05.commit on an mbarrier per buffer).
//
// Precision: fp32 operands are split into bf16 pairs, v = hi + lo with hi = bf16(v), lo = bf16(v - hi)
// (|v - hi - lo| <= 2^-16 |v|), and the product expanded to hi*hi + lo*hi (+ hi*lo for fp32 X); bf16 X is
// exact.  Products are exact in the fp32 accumulator, so the result is the fp32-accumulated sum of terms
// within ~2^-16 relative of the exact products -- the accuracy of the fp32 CUDA-core contraction it
// replaces, at tensor-core rate.
#include <cuda_bf16.h>

#include "fin_internal.cuh"
#include "gemm_f32.cuh"
#include "sm100.cuh"

namespace {

constexpr int kKB = 32;         // batch rows per block: two UMMA k-steps of 16
constexpr int kThreads = 256;
constexpr int kTileA = 128 * kKB * 2;   // 8 KB: 128 rows x 32 k bf16
constexpr int kTileB = 256 * kKB * 2;   // 16 KB: 256 rows x 32 k bf16

// byte offset of row r, k-group kc (8 consecutive k) in a [rows][32 k] K-major canonical tile:
// 8-row x 16-byte core matrices, LBO = 128 B (along K), SBO = 4 x 128 B (along the rows)
__device__ __forceinline__ uint32_t cm_off(int r, int kc) {
  return (uint32_t)(((r >> 3) * 4 + kc) * 128 + (r & 7) * 16);
}

__device__ __forceinline__ uint32_t bf16_pair(float a, float b) {
  return (uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(a)) |
         ((uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(b)) << 16);
}
// (hi, lo) bf16 pairs of two fp32 values: v = hi + lo + O(2^-16 v)
__device__ __forceinline__ void split_pair(float a, float b, uint32_t& hi, uint32_t& lo) {
  const float ha = __bfloat162float(__float2bfloat16_rn(a)), hb = __bfloat162float(__float2bfloat16_rn(b));
  hi = bf16_pair(ha, hb);
  lo = bf16_pair(a - ha, b - hb);
}

// AROW: A(m, k) = g[m * ldg + k] (row-major, the backpropagated product g W); else g[k * ldg + m] (G^T,
// the weight gradient).  MASK (not split): C(m, n) = 0 unless mask(m, n) > 0 (bf16 bits, or fp32 with
// MASKF), the ReLU derivative of the layer below.
// BPACK (with XF32): X is a weight matrix already split and laid out by k_pack_b -- per 256-column
// tile and 32-row block, the hi then the lo tile image -- so its staging is 16-byte copies.
template <bool XF32, bool AROW, bool MASK, bool MASKF, bool BPACK = false>
__global__ void __launch_bounds__(kThreads) k_gemm_tc(int M, int N, int K, int kchunk, const float* __restrict__ g,
                                                      int ldg, const uint16_t* __restrict__ xh,
                                                      const float* __restrict__ xf, int ldx,
                                                      float* __restrict__ out, const void* __restrict__ mask,
                                                      int ldm, const uint4* __restrict__ bpk = nullptr,
                                                      const float* __restrict__ bias = nullptr, int relu = 0) {
  extern __shared__ __align__(1024) uint8_t smem[];
  constexpr int kStage = 2 * kTileA + (XF32 ? 2 : 1) * kTileB;
  __shared__ uint64_t done[2];
  __shared__ uint32_t tslot;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int m0 = blockIdx.y * 128, n0 = blockIdx.x * 256;
  const int nt = min(256, (N - n0 + 15) / 16 * 16);   // this tile's UMMA N (multiple of 16)
  const int k0 = blockIdx.z * kchunk, k1 = min(K, k0 + kchunk);
  if (tid == 0) {
    sm100::mbar_init(&done[0], 1);
    sm100::mbar_init(&done[1], 1);
    sm100::fence_mbar_init();
  }
  if (warp == 0) {
    sm100::tmem_alloc(&tslot, 256);
    sm100::tmem_relinquish();
  }
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tm = tslot;
  const uint32_t idesc = sm100::make_idesc_bf16(128, nt);
  const int nblk = k1 > k0 ? (k1 - k0 + kKB - 1) / kKB : 0;
  const int r = tid & 127, kh = tid >> 7;   // staging: row r, batch rows kh * 16 .. + 15 of the block
  // raw operand values of one block, loaded one block ahead (the global-load latency overlaps the
  // barrier, the MMA issue and the wait for the buffer): G column m0 + r, X columns n0 + r, + 128
  float ga[16];
  float xa[2][16];
  uint16_t xb[2][16];
  uint4 xp[8];   // BPACK: this thread's 8 of the block's 2 x 256 x 64 B (hi, lo) image
  const int nbt = (K + kKB - 1) / kKB;   // BPACK: blocks per column tile in the packed image
  auto load = [&](int b) {
    const int kb = k0 + b * kKB + kh * 16;
    const bool mv = m0 + r < M;
    if constexpr (AROW) {   // 16 consecutive k of row m0 + r: four 16-byte loads when aligned
      const float* src = g + (size_t)(m0 + r) * ldg + kb;
      if (mv && kb + 16 <= k1 && ((ldg | kb) & 3) == 0) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float4 v = __ldg(reinterpret_cast<const float4*>(src) + j);
          ga[4 * j] = v.x; ga[4 * j + 1] = v.y; ga[4 * j + 2] = v.z; ga[4 * j + 3] = v.w;
        }
      } else {
#pragma unroll
        for (int j = 0; j < 16; ++j) ga[j] = (mv && kb + j < k1) ? src[j] : 0.f;
      }
    } else {
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const int k = kb + j;
        ga[j] = (mv && k < k1) ? g[(size_t)k * ldg + m0 + r] : 0.f;
      }
    }
    if constexpr (BPACK) {
      const uint4* src = bpk + ((size_t)blockIdx.x * nbt + (size_t)(k0 / kKB + b)) * (2 * 256 * 4);
#pragma unroll
      for (int j = 0; j < 8; ++j) xp[j] = __ldg(src + tid + 256 * j);
    }
#pragma unroll
    for (int h = 0; h < (BPACK ? 0 : 2); ++h) {
      const int n = r + 128 * h;
      const bool nv = n < nt && n0 + n < N;
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const int k = kb + j;
        if constexpr (XF32) xa[h][j] = (nv && k < k1) ? xf[(size_t)k * ldx + n0 + n] : 0.f;
        else xb[h][j] = (nv && k < k1) ? xh[(size_t)k * ldx + n0 + n] : (uint16_t)0;
      }
    }
  };
  if (nblk > 0) load(0);
  for (int b = 0; b < nblk; ++b) {
    const int buf = b & 1;
    uint8_t* st = smem + buf * kStage;
    const uint32_t sa = sm100::smem_u32(st);
    if (b >= 2) sm100::mbar_wait(&done[buf], (uint32_t)((b - 2) >> 1) & 1u);   // block b - 2's MMAs read it
    {   // A = G^T: row m0 + r, 16 consecutive batch rows -> (hi, lo) bf16
      uint32_t hi[8], lo[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) split_pair(ga[2 * j], ga[2 * j + 1], hi[j], lo[j]);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        sm100::st_shared_v4(sa + cm_off(r, kh * 2 + h), hi[4 * h], hi[4 * h + 1], hi[4 * h + 2], hi[4 * h + 3]);
        sm100::st_shared_v4(sa + kTileA + cm_off(r, kh * 2 + h), lo[4 * h], lo[4 * h + 1], lo[4 * h + 2],
                            lo[4 * h + 3]);
      }
    }
    if constexpr (BPACK) {   // the (hi, lo) tile images, 16 bytes per thread and copy
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const uint32_t off = (uint32_t)(tid + 256 * j) * 16u;   // hi image [0, 16 KB), lo [16 KB, 32 KB)
        sm100::st_shared_v4(sa + 2 * kTileA + off, xp[j].x, xp[j].y, xp[j].z, xp[j].w);
      }
    }
#pragma unroll
    for (int h = 0; h < (BPACK ? 0 : 2); ++h) {   // B = X: rows r, r + 128 of the tile, k-major
      const int n = r + 128 * h;
      if (n >= nt) continue;
      uint32_t hi[8], lo[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        if constexpr (XF32) split_pair(xa[h][2 * j], xa[h][2 * j + 1], hi[j], lo[j]);
        else hi[j] = (uint32_t)xb[h][2 * j] | ((uint32_t)xb[h][2 * j + 1] << 16);
      }
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        sm100::st_shared_v4(sa + 2 * kTileA + cm_off(n, kh * 2 + q), hi[4 * q], hi[4 * q + 1], hi[4 * q + 2],
                            hi[4 * q + 3]);
        if constexpr (XF32)
          sm100::st_shared_v4(sa + 2 * kTileA + kTileB + cm_off(n, kh * 2 + q), lo[4 * q], lo[4 * q + 1],
                              lo[4 * q + 2], lo[4 * q + 3]);
      }
    }
    if (b + 1 < nblk) load(b + 1);
    sm100::fence_proxy_async_smem();   // generic-proxy stores -> the tensor core's reads
    sm100::tc_fence_before();
    __syncthreads();
    if (tid == 0) {
      sm100::tc_fence_after();
#pragma unroll
      for (int s = 0; s < 2; ++s) {
        const uint64_t ahi = sm100::make_sdesc(sa + s * 256, 128, 512);
        const uint64_t alo = sm100::make_sdesc(sa + kTileA + s * 256, 128, 512);
        const uint64_t bhi = sm100::make_sdesc(sa + 2 * kTileA + s * 256, 128, 512);
        sm100::mma_bf16(tm, ahi, bhi, idesc, (b | s) ? 1u : 0u);
        sm100::mma_bf16(tm, alo, bhi, idesc, 1u);
        if constexpr (XF32) {
          const uint64_t blo = sm100::make_sdesc(sa + 2 * kTileA + kTileB + s * 256, 128, 512);
          sm100::mma_bf16(tm, ahi, blo, idesc, 1u);
        }
      }
      sm100::mma_commit(&done[buf]);
    }
  }
  if (nblk > 0) sm100::mbar_wait(&done[(nblk - 1) & 1], (uint32_t)((nblk - 1) >> 1) & 1u);
  sm100::tc_fence_after();
  // epilogue: warp w reads TMEM lanes 32 (w % 4) .. (rows m), 16-column chunks c = w / 4 (mod 2)
  float* dst = out + (size_t)blockIdx.z * M * N;
  const int q = warp & 3, m = m0 + 32 * q + lane;
  for (int c = warp >> 2; c * 16 < nt; c += 2) {
    uint32_t v[16];
    if (nblk > 0) {
      sm100::tmem_ld16(tm + ((uint32_t)(32 * q) << 16) + (uint32_t)(c * 16), v);
      sm100::tmem_wait_ld();
    } else {
#pragma unroll
      for (int j = 0; j < 16; ++j) v[j] = 0u;
    }
    const int nb = n0 + c * 16;
    // full 16-column chunk of an aligned row: 16-byte mask loads and stores
    const bool vec = m < M && nb + 16 <= N && (N & 3) == 0 && (!MASK || MASKF || (ldm & 7) == 0) &&
                     (!MASK || !MASKF || (ldm & 3) == 0);
    if (vec) {
      float y[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        y[j] = __uint_as_float(v[j]);
        if (bias) y[j] += bias[nb + j];
        if (relu) y[j] = fmaxf(y[j], 0.f);
      }
      if constexpr (MASK) {
        if constexpr (MASKF) {
          const float4* mk = reinterpret_cast<const float4*>(static_cast<const float*>(mask) + (size_t)m * ldm + nb);
#pragma unroll
          for (int q4 = 0; q4 < 4; ++q4) {
            const float4 mm = __ldg(mk + q4);
            if (!(mm.x > 0.f)) y[4 * q4] = 0.f;
            if (!(mm.y > 0.f)) y[4 * q4 + 1] = 0.f;
            if (!(mm.z > 0.f)) y[4 * q4 + 2] = 0.f;
            if (!(mm.w > 0.f)) y[4 * q4 + 3] = 0.f;
          }
        } else {
          const uint4* mk = reinterpret_cast<const uint4*>(static_cast<const uint16_t*>(mask) + (size_t)m * ldm + nb);
#pragma unroll
          for (int q8 = 0; q8 < 2; ++q8) {
            const uint4 mm = __ldg(mk + q8);
            const uint32_t w[4] = {mm.x, mm.y, mm.z, mm.w};
#pragma unroll
            for (int t = 0; t < 8; ++t) {
              const uint32_t bits = (t & 1) ? (w[t >> 1] & 0xffff0000u) : (w[t >> 1] << 16);
              if (!(__uint_as_float(bits) > 0.f)) y[8 * q8 + t] = 0.f;
            }
          }
        }
      }
      float4* o4 = reinterpret_cast<float4*>(dst + (size_t)m * N + nb);
#pragma unroll
      for (int q4 = 0; q4 < 4; ++q4) o4[q4] = make_float4(y[4 * q4], y[4 * q4 + 1], y[4 * q4 + 2], y[4 * q4 + 3]);
    } else if (m < M) {
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const int n = n0 + c * 16 + j;
        if (n < N) {
          float y = __uint_as_float(v[j]);
          if (bias) y += bias[n];   // (not split: the forward's epilogue, z = x W^T + b, then ReLU)
          if (relu) y = fmaxf(y, 0.f);
          if constexpr (MASK) {
            const bool on = MASKF ? static_cast<const float*>(mask)[(size_t)m * ldm + n] > 0.f
                                  : gemmf::bf16_at(static_cast<const uint16_t*>(mask), (size_t)m * ldm + n) > 0.f;
            if (!on) y = 0.f;
          }
          dst[(size_t)m * N + n] = y;
        }
      }
    }
  }
  sm100::tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    sm100::tc_fence_after();
    sm100::tmem_dealloc(tm, 256);
  }
}

// W [K][ldw] fp32 (K x N) -> per 256-column tile t and 32-row block b: the hi image then the lo image of
// the B operand tile (256 rows n x 32 k, K-major canonical), rows n >= N zero; one thread per 8 k of a row
// WT: W is stored [N][ldw] (the out-major weight of a forward layer: B(k, n) = W[n][k]), else [K][ldw]
template <bool WT>
__global__ void k_pack_b(int K, int N, const float* __restrict__ w, int ldw, uint4* __restrict__ out) {
  const int nbt = (K + kKB - 1) / kKB;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t total = (int64_t)((N + 255) / 256) * nbt * 256 * 4;
  if (i >= total) return;
  const int kc = (int)(i & 3), n = (int)((i >> 2) & 255);
  const int64_t tb = i >> 10;   // tile * nbt + block
  const int t = (int)(tb / nbt), b = (int)(tb % nbt);
  const int col = t * 256 + n;
  float v[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const int k = b * kKB + kc * 8 + j;
    v[j] = (col < N && k < K) ? (WT ? w[(size_t)col * ldw + k] : w[(size_t)k * ldw + col]) : 0.f;
  }
  uint32_t hi[4], lo[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) split_pair(v[2 * j], v[2 * j + 1], hi[j], lo[j]);
  uint4* base = out + tb * (2 * 256 * 4);
  const uint32_t off = cm_off(n, kc) / 16;
  base[off] = make_uint4(hi[0], hi[1], hi[2], hi[3]);
  base[256 * 4 + off] = make_uint4(lo[0], lo[1], lo[2], lo[3]);
}

}  // namespace

namespace fin {

template <bool XF32, bool AROW, bool MASK, bool MASKF, bool BPACK>
static cudaError_t run_tc_p(dim3 grid, int bytes, cudaStream_t s, int M, int N, int K, int kchunk, const float* g,
                            int ldg, const float* xf, int ldx, float* out, const void* mask, int ldm, const uint4* bp,
                            const float* bias, int relu) {
  auto kern = k_gemm_tc<XF32, AROW, MASK, MASKF, BPACK>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess)
    kern<<<grid, kThreads, bytes, s>>>(M, N, K, kchunk, g, ldg, nullptr, xf, ldx, out, mask, ldm, bp, bias, relu);
  return e;
}

template <bool XF32, bool AROW, bool MASK, bool MASKF>
static cudaError_t run_tc(dim3 grid, int bytes, cudaStream_t s, int M, int N, int K, int kchunk, const float* g,
                          int ldg, const uint16_t* xh, const float* xf, int ldx, float* out, const void* mask,
                          int ldm) {
  auto kern = k_gemm_tc<XF32, AROW, MASK, MASKF>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess)
    kern<<<grid, kThreads, bytes, s>>>(M, N, K, kchunk, g, ldg, xh, xf, ldx, out, mask, ldm, nullptr, nullptr, 0);
  return e;
}

// C [M][N] = sum_k A(m, k) X[k * ldx + n] over k < K with A(m, k) = G[k * ldg + m] (arow = 0: the weight
// gradient G^T X) or G[m * ldg + k] (arow = 1: the backpropagated product), X bf16 bits (xh) or fp32 (xf);
// mask (arow only; bf16 bits, or fp32 with maskf) zeroes C(m, n) where mask[m * ldm + n] <= 0.  Splits the
// batch-long contractions over CTAs (partials summed in a fixed order); allocates stream-ordered scratch
// for them and frees it on the stream.
cudaError_t launch_gemm_tc(int M, int N, int K, const float* g, int ldg, int arow, const uint16_t* xh, const float* xf,
                           int ldx, float* C, const void* mask, int ldm, int maskf, cudaStream_t s, int wt,
                           const float* bias, int relu) {
  const int gx = (N + 255) / 256, gy = (M + 127) / 128;
  const int tiles = gx * gy;
  int splits = (2 * 148 + tiles - 1) / tiles;
  const int maxs = (K + 8 * kKB - 1) / (8 * kKB);   // >= 256 batch rows per split
  if (splits > maxs) splits = maxs;
  if (splits < 1 || mask || bias || relu) splits = 1;
  const int kchunk = ((K + splits - 1) / splits + kKB - 1) / kKB * kKB;
  const int used = K > 0 ? (K + kchunk - 1) / kchunk : 1;
  float* part = C;
  cudaError_t e = cudaSuccess;
  if (used > 1) {
    e = cudaMallocAsync(&part, sizeof(float) * (size_t)used * M * N, s);
    if (e != cudaSuccess) return e;
  }
  const bool f32 = xf != nullptr;
  const int bytes = (2 * kTileA + (f32 ? 2 : 1) * kTileB) * 2;
  const dim3 grid(gx, gy, used);
  if (arow && f32 && used == 1) {   // a weight matrix read by every CTA: split and lay it out once
    const int nbt = (K + kKB - 1) / kKB;
    const size_t n16 = (size_t)gx * nbt * 2 * 256 * 4;
    uint4* bp = nullptr;
    e = cudaMallocAsync(&bp, n16 * 16, s);
    if (e != cudaSuccess) return e;
    const int64_t threads = (int64_t)gx * nbt * 256 * 4;
    if (wt) k_pack_b<true><<<(unsigned)((threads + 255) / 256), 256, 0, s>>>(K, N, xf, ldx, bp);
    else k_pack_b<false><<<(unsigned)((threads + 255) / 256), 256, 0, s>>>(K, N, xf, ldx, bp);
    if (!mask)
      e = run_tc_p<true, true, false, false, true>(grid, bytes, s, M, N, K, kchunk, g, ldg, xf, ldx, C, nullptr, 0, bp,
                                                   bias, relu);
    else if (maskf)
      e = run_tc_p<true, true, true, true, true>(grid, bytes, s, M, N, K, kchunk, g, ldg, xf, ldx, C, mask, ldm, bp,
                                                 bias, relu);
    else
      e = run_tc_p<true, true, true, false, true>(grid, bytes, s, M, N, K, kchunk, g, ldg, xf, ldx, C, mask, ldm, bp,
                                                  bias, relu);
    if (e == cudaSuccess) e = cudaGetLastError();
    cudaFreeAsync(bp, s);
    return e;
  }
  if (!arow) {
    e = f32 ? run_tc<true, false, false, false>(grid, bytes, s, M, N, K, kchunk, g, ldg, xh, xf, ldx, part, nullptr, 0)
            : run_tc<false, false, false, false>(grid, bytes, s, M, N, K, kchunk, g, ldg, xh, xf, ldx, part, nullptr, 0);
  } else if (!mask) {
    e = f32 ? run_tc<true, true, false, false>(grid, bytes, s, M, N, K, kchunk, g, ldg, xh, xf, ldx, part, nullptr, 0)
            : run_tc<false, true, false, false>(grid, bytes, s, M, N, K, kchunk, g, ldg, xh, xf, ldx, part, nullptr, 0);
  } else if (maskf) {
    e = f32 ? run_tc<true, true, true, true>(grid, bytes, s, M, N, K, kchunk, g, ldg, xh, xf, ldx, part, mask, ldm)
            : run_tc<false, true, true, true>(grid, bytes, s, M, N, K, kchunk, g, ldg, xh, xf, ldx, part, mask, ldm);
  } else {
    e = f32 ? run_tc<true, true, true, false>(grid, bytes, s, M, N, K, kchunk, g, ldg, xh, xf, ldx, part, mask, ldm)
            : run_tc<false, true, true, false>(grid, bytes, s, M, N, K, kchunk, g, ldg, xh, xf, ldx, part, mask, ldm);
  }
  if (e == cudaSuccess && used > 1) {
    const size_t n = (size_t)M * N;
    gemmf::k_sum_splits<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(part, used, n, C);
  }
  if (e == cudaSuccess) e = cudaGetLastError();
  if (used > 1) cudaFreeAsync(part, s);
  return e;
}

// dW [M][N] = sum_k G[k * ldg + m] X[k * ldx + n] over k < K (X bf16 bits xh or fp32 xf)
cudaError_t launch_wgrad_tc(int M, int N, int K, const float* g, int ldg, const uint16_t* xh, const float* xf,
                            int ldx, float* dw, cudaStream_t s) {
  return launch_gemm_tc(M, N, K, g, ldg, 0, xh, xf, ldx, dw, nullptr, 0, 0, s, 0, nullptr, 0);
}

}  // namespace fin
