// Micro-benchmark: one 128 KB layer (K = 256, N = 256) streamed through the same 32 KB of ring memory
// as 2 x 16 KB slots or 4 x 8 KB slots, the copies issued by 1 or 2 producer lanes (alternating), while
// the MMA lane consumes each stage (N = 256, K = 16 per 8 KB).  Grid 1 and 296 (two CTAs per SM).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_2501_10709_b200/csrc ring_split.cu
#include <cstdint>
#include <cstdio>
#include <vector>
#include <algorithm>

#include "sm100.cuh"

__global__ void k(const uint8_t* __restrict__ w, int sb, int lanes, int reps, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t full[4], empty[4], done;
  __shared__ uint32_t tslot;
  uint8_t* A = smem;            // 64 KB
  uint8_t* R = smem + 65536;    // 32 KB ring
  const int ring = 32768 / sb, stages = 131072 / sb, ks = sb / 8192;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < 4; ++s) { sm100::mbar_init(&full[s], 1); sm100::mbar_init(&empty[s], 1); }
    sm100::mbar_init(&done, 1);
    sm100::fence_mbar_init();
  }
  if (warp == 1) { sm100::tmem_alloc(&tslot, 256); sm100::tmem_relinquish(); }
  for (int i = threadIdx.x; i < (65536 + 32768) / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
  sm100::fence_proxy_async_smem();
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tm = tslot;
  const uint8_t* src = w + (size_t)(blockIdx.x % 148) * 131072;
  uint32_t itp = 0, itm = 0;
  long long best = 1LL << 60;
  for (int r = 0; r < reps; ++r) {
    __syncthreads();
    const long long t0 = clock64();
    const int pw = warp == 0 ? 0 : (warp == 2 ? 1 : -1);   // producer index: lane 0 of warps 0 and 2
    if (pw >= 0 && pw < lanes && lane == 0) {
      for (int s = 0; s < stages; ++s, ++itp) {
        if ((s % lanes) != pw) continue;
        const uint32_t slot = itp % ring, ph = (itp / ring) & 1;
        sm100::mbar_wait(&empty[slot], ph ^ 1);
        sm100::mbar_arrive_expect_tx(&full[slot], sb);
        sm100::bulk_g2s(R + slot * sb, src + (size_t)s * sb, sb, &full[slot]);
      }
    } else if (warp == 1 && lane == 0) {
      const uint32_t idesc = sm100::make_idesc_bf16(128, 256);
      const uint32_t a = sm100::smem_u32(A), rb = sm100::smem_u32(R);
      for (int s = 0; s < stages; ++s, ++itm) {
        const uint32_t slot = itm % ring, ph = (itm / ring) & 1;
        sm100::mbar_wait(&full[slot], ph);
        sm100::tc_fence_after();
        for (int j = 0; j < ks; ++j) {
          const int kk = s * ks + j;
          sm100::mma_bf16(tm, sm100::make_sdesc(a + kk * 256, 128, 4096),
                          sm100::make_sdesc(rb + slot * sb + j * 256, 128, (uint32_t)ks * 256), idesc, kk ? 1u : 0u);
        }
        sm100::mma_commit(&empty[slot]);
      }
      sm100::mma_commit(&done);
      sm100::mbar_wait(&done, (uint32_t)r & 1u);
      const long long dt = clock64() - t0;
      if (r > 0 && dt < best) best = dt;
      out[blockIdx.x] = best;
    }
    if (warp == 0 && lanes > 1) itp += 0;   // (each lane counted every stage above)
  }
  sm100::tc_fence_before();
  __syncthreads();
  if (warp == 1) { sm100::tc_fence_after(); sm100::tmem_dealloc(tm, 256); }
}

int main() {
  uint8_t* w;
  cudaMalloc(&w, 148 * 131072);
  cudaMemset(w, 0, 148 * 131072);
  long long* d;
  cudaMalloc(&d, 296 * 8);
  const int smem = 65536 + 32768;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int grid : {1, 296})
    for (int sb : {16384, 8192})
      for (int lanes : {1, 2}) {
        k<<<grid, 128, smem>>>(w, sb, lanes, 8, d);
        cudaError_t e = cudaDeviceSynchronize();
        std::vector<long long> h(grid);
        cudaMemcpy(h.data(), d, grid * 8, cudaMemcpyDeviceToHost);
        std::sort(h.begin(), h.end());
        printf("grid %3d ring %d x %2d KB, %d issuing warp(s): 128 KB layer %6lld cycles (median CTA) %s\n", grid,
               32768 / sb, sb / 1024, lanes, h[grid / 2], e == cudaSuccess ? "" : cudaGetErrorString(e));
      }
  return 0;
}
