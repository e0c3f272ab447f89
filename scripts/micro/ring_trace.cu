// Micro-benchmark: timeline of the weight ring (producer -> MMA warp) for one 128 KB layer
// streamed in 16 KB stages through a ring of R slots, as the fused rollout does it.
// Records, per stage s: t_issue (producer issued the copy), t_full (the MMA lane saw the
// stage land), t_mma (the MMA lane issued its 2 k-steps and committed the slot back), and
// t_empty (the producer saw the slot free again).  Variants: the copy of a stage as 1 x 16 KB
// (one lane) or 4 x 4 KB (four lanes); grid 1 and 296 (two CTAs per SM).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_2501_10709_b200/csrc ring_trace.cu
#include <cstdint>
#include <cstdio>
#include <vector>
#include <algorithm>

#include "sm100.cuh"

constexpr int kStages = 8, kSB = 16384;

__global__ void k(const uint8_t* __restrict__ w, int ring, int split, int reps, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t full[8], empty[8], done;
  __shared__ uint32_t tslot;
  __shared__ long long t_issue[kStages], t_full[kStages], t_mma[kStages];
  uint8_t* A = smem;            // 64 KB
  uint8_t* R = smem + 65536;    // ring <= 4 x 16 KB
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < 8; ++s) { sm100::mbar_init(&full[s], 1); sm100::mbar_init(&empty[s], 1); }
    sm100::mbar_init(&done, 1);
    sm100::fence_mbar_init();
  }
  if (warp == 1) { sm100::tmem_alloc(&tslot, 256); sm100::tmem_relinquish(); }
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(A)[i] = 0x3c003c00u;
  sm100::fence_proxy_async_smem();
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tm = tslot;
  const uint8_t* src = w + (size_t)(blockIdx.x % 148) * (kStages * kSB);
  long long best = 1LL << 60;
  uint32_t it_p = 0, it_m = 0;
  for (int r = 0; r < reps; ++r) {
    __syncthreads();
    const long long t0 = clock64();
    if (warp == 0 && lane < split) {
      for (int s = 0; s < kStages; ++s, ++it_p) {
        const uint32_t slot = it_p % ring, ph = (it_p / ring) & 1;
        sm100::mbar_wait(&empty[slot], ph ^ 1);
        if (lane == 0) {
          sm100::mbar_arrive_expect_tx(&full[slot], kSB);
          if (r == reps - 1) t_issue[s] = clock64() - t0;
        }
        __syncwarp((1u << split) - 1);
        const int part = kSB / split;
        sm100::bulk_g2s(R + slot * kSB + lane * part, src + (size_t)s * kSB + lane * part, part, &full[slot]);
      }
    } else if (warp == 1 && lane == 0) {
      const uint32_t idesc = sm100::make_idesc_bf16(128, 256);
      const uint32_t a = sm100::smem_u32(A), rb = sm100::smem_u32(R);
      for (int s = 0; s < kStages; ++s, ++it_m) {
        const uint32_t slot = it_m % ring, ph = (it_m / ring) & 1;
        sm100::mbar_wait(&full[slot], ph);
        if (r == reps - 1) t_full[s] = clock64() - t0;
        sm100::tc_fence_after();
        for (int j = 0; j < 2; ++j)
          sm100::mma_bf16(tm, sm100::make_sdesc(a + (2 * s + j) * 256, 128, 4096),
                          sm100::make_sdesc(rb + slot * kSB + j * 256, 128, 512), idesc, (s | j) ? 1u : 0u);
        sm100::mma_commit(&empty[slot]);
        if (r == reps - 1) t_mma[s] = clock64() - t0;
      }
      sm100::mma_commit(&done);
      sm100::mbar_wait(&done, (uint32_t)r & 1u);
      const long long dt = clock64() - t0;
      if (r > 0 && dt < best) best = dt;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    long long* o = out + (size_t)blockIdx.x * (1 + 3 * kStages);
    o[0] = best;
    for (int s = 0; s < kStages; ++s) { o[1 + s] = t_issue[s]; o[1 + kStages + s] = t_full[s]; o[1 + 2 * kStages + s] = t_mma[s]; }
  }
  sm100::tc_fence_before();
  __syncthreads();
  if (warp == 1) { sm100::tc_fence_after(); sm100::tmem_dealloc(tm, 256); }
}

int main() {
  uint8_t* w;
  cudaMalloc(&w, 148 * kStages * kSB);
  cudaMemset(w, 0, 148 * kStages * kSB);
  long long* d;
  const int per = 1 + 3 * kStages;
  cudaMalloc(&d, 296 * per * 8);
  const int smem = 65536 + 4 * kSB;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int grid : {1, 296})
    for (int split : {1, 4})
      for (int ring : {2, 4}) {
        k<<<grid, 128, smem>>>(w, ring, split, 6, d);
        cudaError_t e = cudaDeviceSynchronize();
        std::vector<long long> h((size_t)grid * per);
        cudaMemcpy(h.data(), d, h.size() * 8, cudaMemcpyDeviceToHost);
        std::vector<long long> b(grid);
        for (int g = 0; g < grid; ++g) b[g] = h[(size_t)g * per];
        std::sort(b.begin(), b.end());
        printf("grid %3d ring %d, stage copied as %d x %2d KB: layer %6lld cycles (median CTA) %s\n", grid, ring, split,
               16 / split, b[grid / 2], e == cudaSuccess ? "" : cudaGetErrorString(e));
        printf("   CTA 0 stage: issue / landed / MMAs committed\n");
        for (int s = 0; s < kStages; ++s)
          printf("   %d: %6lld %6lld %6lld\n", s, h[1 + s], h[1 + kStages + s], h[1 + 2 * kStages + s]);
      }
  return 0;
}
