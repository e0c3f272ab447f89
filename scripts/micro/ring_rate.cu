// Micro-benchmark: weight streaming through a shared-memory ring, as the fused rollout's
// producer / MMA warps do it: lane 0 of warp 0 bulk-copies stages of ``sb`` bytes (L2-
// resident source, evict-last) into ``ring`` slots; lane 0 of warp 1 waits for each stage,
// issues its k-steps (N = 256, K = 16 each: sb / 8 KB of them) and commits the slot back.
// Cycles per 16 KB of weights for a 128 KB layer, and the same with all stages resident.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_2501_10709_b200/csrc ring_rate.cu
#include <cstdint>
#include <cstdio>

#include "sm100.cuh"

__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .b32 %%rx;\n\t.reg .pred %%px;\n\t"
      "elect.sync %%rx|%%px, %1;\n\t"
      "@%%px mov.s32 %0, 1;\n\t}"
      : "+r"(pred)
      : "r"(0xffffffffu));
  return pred != 0;
}

__device__ __forceinline__ bool try_wait_nohint(uint64_t* bar, uint32_t parity) {
  return sm100::mbar_try_wait_nh(bar, parity);
}

template <bool HINT>
__device__ __forceinline__ void wait(uint64_t* bar, uint32_t ph) {
  if (HINT) sm100::mbar_wait(bar, ph);
  else while (!try_wait_nohint(bar, ph)) {}
}

template <bool HINT, bool WARPWIDE>
__global__ void k(const uint8_t* __restrict__ w, int sb, int ring, int layer_bytes, int reps, long long* out, int cev, int lay) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t full[8], empty[8], done;
  __shared__ uint32_t tslot;
  uint8_t* A = smem;                 // 128 x 256 bf16 A operand (64 KB)
  uint8_t* R = smem + 65536;         // ring
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < ring; ++s) { sm100::mbar_init(&full[s], 1); sm100::mbar_init(&empty[s], 1); }
    sm100::mbar_init(&done, 1);
    sm100::fence_mbar_init();
  }
  if (warp == 1) { sm100::tmem_alloc(&tslot, 256); sm100::tmem_relinquish(); }
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(A)[i] = 0x3f803f80u;
  sm100::fence_proxy_async_smem();
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tm = tslot;
  const int stages = layer_bytes / sb;
  const int ks_per_stage = sb / 8192;   // N = 256 x K = 16 bf16 = 8 KB per k-step
  const uint64_t pol = sm100::l2_policy_evict_last();
  if (warp == 0 && lane == 0) {
    uint32_t it = 0;
    for (int r = 0; r < reps; ++r)
      for (int s = 0; s < stages; ++s, ++it) {
        const uint32_t slot = it % ring, ph = (it / ring) & 1;
        if (cev > 0) wait<HINT>(&empty[slot], ph ^ 1);
        else if (it >= (uint32_t)ring) break;   // resident modes: the ring holds the whole layer
        sm100::mbar_arrive_expect_tx(&full[slot], sb);
        sm100::bulk_g2s_hint(R + slot * sb, w + (size_t)s * sb, sb, &full[slot], pol);
      }
  } else if (warp == 1 && (WARPWIDE || lane == 0)) {
    uint32_t it = 0;
    const uint32_t idesc = sm100::make_idesc_bf16(128, 256);
    const uint32_t a = sm100::smem_u32(A), rb = sm100::smem_u32(R);
    long long best = 1LL << 60;
    for (int r = 0; r < reps; ++r) {
      const long long t0 = clock64();
      for (int s = 0; s < stages; ++s, ++it) {
        const uint32_t slot = it % ring, ph = (it / ring) & 1;
        if (cev > 0 || it < (uint32_t)ring) wait<HINT>(&full[slot], ph);   // (resident: first pass only)
        if (cev >= 0) sm100::tc_fence_after();
        for (int j = 0; j < ks_per_stage; ++j)
          if (!WARPWIDE || elect_one()) sm100::mma_bf16(tm, sm100::make_sdesc(a + (s * ks_per_stage + j) % 16 * 256, 128, 4096),
                          lay == 0 ? sm100::make_sdesc(rb + slot * sb + j * 256, 128, (uint32_t)ks_per_stage * 256)
                                   : sm100::make_sdesc(rb + slot * sb + j * 2 * 4096, 4096, 128),
                          idesc, (s | j) ? 1u : 0u);
        // release the slots every cev stages (one commit arrives on each of them)
        if (cev > 0 && ((s + 1) % cev == 0 || s + 1 == stages))
          for (int q = s - (s % cev); q <= s; ++q)
            if (!WARPWIDE || elect_one()) sm100::mma_commit(&empty[(it - (s - q)) % ring]);
      }
      if (!WARPWIDE || elect_one()) sm100::mma_commit(&done);
      wait<HINT>(&done, r & 1);
      const long long dt = clock64() - t0;
      if (r > 0 && dt < best) best = dt;
    }
    if (lane == 0) out[0] = best;
  }
  sm100::tc_fence_before();
  __syncthreads();
  if (warp == 1) { sm100::tc_fence_after(); sm100::tmem_dealloc(tm, 256); }
}

int main() {
  uint8_t* w;
  cudaMalloc(&w, 1 << 20);
  cudaMemset(w, 0, 1 << 20);
  long long* d;
  cudaMalloc(&d, 8);
  const int smem = 65536 + 131072;
  cudaFuncSetAttribute(k<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int hint = 1;
  for (int ww : {0, 1})
  for (int lay : {0})
  for (int sb : {8192, 16384, 32768})
    for (int ring : {2, 4, 8})
      for (int cev : {1, 2, 0}) {
        if (sb * ring > 131072 || (cev > 0 && 2 * cev > ring) || (cev <= 0 && sb * ring != 131072)) continue;
        if (cev > 0 && ring != 4 && !(sb == 32768 && ring == 2)) continue;
        if (ww) k<true, true><<<1, 128, smem>>>(w, sb, ring, 131072, 6, d, cev, lay);
        else k<true, false><<<1, 128, smem>>>(w, sb, ring, 131072, 6, d, cev, lay);
        printf("%s: ", ww ? "warp-wide loop, elect.sync MMA" : "lane-0 loop              ");
        long long h = 0;
        cudaError_t e = cudaDeviceSynchronize();
        cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
        printf("hint=%d stage=%2d KB ring=%d commit every %d stages%s: 128 KB layer in %6lld cycles (%.0f per 16 KB) %s\n",
               hint, sb / 1024, ring, cev, cev == 0 ? " (resident, no waits)" : cev < 0 ? " (resident, no waits, no fences)" : "", h, h / 8.0,
               e == cudaSuccess ? "" : cudaGetErrorString(e));
      }
  return 0;
}
