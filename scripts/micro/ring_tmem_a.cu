// Micro-benchmark: does reading the A operand (activations) from TMEM instead of shared
// memory let the weight ring keep up with the tensor core?  One 128 KB layer (K = 256,
// N = 256 outputs) streamed in 16 KB stages through a 2-slot ring while the MMA lane issues:
//   V0  A in smem, N = 256 per MMA (2 k-steps per stage)           -- the fused rollout today
//   V1  A in TMEM, N = 256 per MMA                                   (TMEM: D 256 + A 128 cols)
//   V2  A in TMEM, two N = 128 halves (4 k-steps per stage)          (TMEM: D 128 + A 128 cols)
//   V3  A in smem, two N = 128 halves
// Grid 1 (one SM) and 296 (two CTAs per SM, as the dual layout) for the 256-column variants.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_2501_10709_b200/csrc ring_tmem_a.cu
#include <cstdint>
#include <cstdio>
#include <vector>
#include <algorithm>

#include "sm100.cuh"

constexpr int kStages = 8, kSB = 16384;

__device__ __forceinline__ void mma_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(acc)
      : "memory");
}

template <int V, int COLS>
__global__ void k(const uint8_t* __restrict__ w, int reps, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t full[2], empty[2], done;
  __shared__ uint32_t tslot;
  uint8_t* A = smem;            // 64 KB
  uint8_t* R = smem + 65536;    // 2 x 16 KB
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < 2; ++s) { sm100::mbar_init(&full[s], 1); sm100::mbar_init(&empty[s], 1); }
    sm100::mbar_init(&done, 1);
    sm100::fence_mbar_init();
  }
  if (warp == 1) { sm100::tmem_alloc(&tslot, COLS); sm100::tmem_relinquish(); }
  for (int i = threadIdx.x; i < (65536 + 2 * kSB) / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
  sm100::fence_proxy_async_smem();
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tm = tslot;
  const uint8_t* src = w + (size_t)(blockIdx.x % 148) * (kStages * kSB);
  uint32_t it_p = 0, it_m = 0;
  long long best = 1LL << 60;
  constexpr bool kTmemA = V == 1 || V == 2;
  constexpr int kN = (V == 0 || V == 1) ? 256 : 128;
  constexpr int kKs = kSB / (kN * 32);   // k-steps per stage (N x 16 bf16 each)
  const uint32_t a_tm = tm + (V == 1 ? 256 : 128);
  for (int r = 0; r < reps; ++r) {
    __syncthreads();
    const long long t0 = clock64();
    if (warp == 0 && lane == 0) {
      for (int s = 0; s < kStages; ++s, ++it_p) {
        const uint32_t slot = it_p & 1, ph = (it_p >> 1) & 1;
        sm100::mbar_wait(&empty[slot], ph ^ 1);
        sm100::mbar_arrive_expect_tx(&full[slot], kSB);
        sm100::bulk_g2s(R + slot * kSB, src + (size_t)s * kSB, kSB, &full[slot]);
      }
    } else if (warp == 1 && lane == 0) {
      const uint32_t idesc = sm100::make_idesc_bf16(128, kN);
      const uint32_t a = sm100::smem_u32(A), rb = sm100::smem_u32(R);
      for (int s = 0; s < kStages; ++s, ++it_m) {
        const uint32_t slot = it_m & 1, ph = (it_m >> 1) & 1;
        sm100::mbar_wait(&full[slot], ph);
        sm100::tc_fence_after();
        for (int j = 0; j < kKs; ++j) {
          const int ks = (s * kKs + j) % 16;   // K position (the halves reuse A)
          const uint64_t bd = sm100::make_sdesc(rb + slot * kSB + j * (kN * 32), 128, 256);
          if (kTmemA) mma_ts(tm, a_tm + ks * 8, bd, idesc, (s | j) ? 1u : 0u);
          else sm100::mma_bf16(tm, sm100::make_sdesc(a + ks * 256, 128, 4096), bd, idesc, (s | j) ? 1u : 0u);
        }
        sm100::mma_commit(&empty[slot]);
      }
      sm100::mma_commit(&done);
      sm100::mbar_wait(&done, (uint32_t)r & 1u);
      const long long dt = clock64() - t0;
      if (r > 0 && dt < best) best = dt;
      out[blockIdx.x] = best;
    }
  }
  sm100::tc_fence_before();
  __syncthreads();
  if (warp == 1) { sm100::tc_fence_after(); sm100::tmem_dealloc(tm, COLS); }
}

template <int V, int COLS>
void run(const uint8_t* w, long long* d, int grid) {
  const int smem = 65536 + 2 * kSB;
  cudaFuncSetAttribute(k<V, COLS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  k<V, COLS><<<grid, 128, smem>>>(w, 6, d);
  cudaError_t e = cudaDeviceSynchronize();
  std::vector<long long> h(grid);
  cudaMemcpy(h.data(), d, grid * 8, cudaMemcpyDeviceToHost);
  std::sort(h.begin(), h.end());
  printf("V%d grid %3d: 128 KB layer in %6lld cycles median (%4lld per 16 KB stage) %s\n", V, grid, h[grid / 2],
         h[grid / 2] / kStages, e == cudaSuccess ? "" : cudaGetErrorString(e));
}

int main() {
  uint8_t* w;
  cudaMalloc(&w, 148 * kStages * kSB);
  cudaMemset(w, 0, 148 * kStages * kSB);
  long long* d;
  cudaMalloc(&d, 296 * 8);
  for (int grid : {1, 296}) {
    run<0, 256>(w, d, grid);
    if (grid == 1) run<1, 512>(w, d, grid);
    run<2, 256>(w, d, grid);
    run<3, 256>(w, d, grid);
  }
  return 0;
}
