// Micro-benchmark: where the MMA warp's per-weight-stage overhead comes from.
// One CTA; A (128 x 256 bf16) and all of B (256 x 256 bf16, 16 k-steps of N = 256 x K = 16)
// resident in shared memory, so no copy is on the path unless a variant adds one.  Lane 0 of
// warp 1 issues the 16 k-steps of a 128 KB layer as 8 "stages" of 2 and does, per stage:
//   V0  nothing (16 MMAs back to back)
//   V1  tcgen05.fence::after_thread_sync
//   V2  tcgen05.commit to a per-stage mbarrier (no wait)
//   V3  try_wait on an mbarrier whose phase has already completed + fence
//   V4  V2 + V3 (the ring's sequence with the data already there)
//   V5  V0 while warp 0 bulk-copies 16 KB from L2 into a spare region per stage (smem writes)
//   V6  V4 + the copies of V5
//   V7  V4, descriptors from runtime values (the slot base read from shared memory)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_2501_10709_b200/csrc stage_cost.cu
#include <cstdint>
#include <cstdio>

#include "sm100.cuh"

template <int V>
__global__ void k(const uint8_t* __restrict__ w, int reps, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t st[8], ready, done, cpy;
  __shared__ uint32_t tslot, base_rt;
  uint8_t* A = smem;                  // 64 KB
  uint8_t* B = smem + 65536;          // 128 KB
  uint8_t* X = smem + 65536 + 131072; // 32 KB spare (copy target)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < 8; ++s) sm100::mbar_init(&st[s], 1);
    sm100::mbar_init(&ready, 1);
    sm100::mbar_init(&done, 1);
    sm100::mbar_init(&cpy, 1);
    sm100::fence_mbar_init();
    base_rt = sm100::smem_u32(B);
  }
  if (warp == 1) { sm100::tmem_alloc(&tslot, 256); sm100::tmem_relinquish(); }
  for (int i = threadIdx.x; i < (65536 + 131072) / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
  sm100::fence_proxy_async_smem();
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  if (threadIdx.x == 0) sm100::mbar_arrive(&ready);   // phase 0 of ``ready`` completes now
  __syncthreads();
  const uint32_t tm = tslot;
  const uint32_t idesc = sm100::make_idesc_bf16(128, 256);
  const uint32_t a = sm100::smem_u32(A);
  for (int r = 0; r < reps; ++r) {
    __syncthreads();
    if (warp == 0 && lane == 0 && (V == 5 || V == 6)) {
      for (int s = 0; s < 8; ++s) {
        sm100::mbar_arrive_expect_tx(&cpy, 16384);
        sm100::bulk_g2s(X + (s & 1) * 16384, w + (size_t)s * 16384, 16384, &cpy);
        sm100::mbar_wait(&cpy, (uint32_t)(r * 8 + s) & 1u);
      }
    }
    if (warp == 1 && lane == 0) {
      const uint32_t b = V == 7 ? *(volatile uint32_t*)&base_rt : sm100::smem_u32(B);
      const long long t0 = clock64();
#pragma unroll
      for (int s = 0; s < 8; ++s) {
        if (V == 3 || V == 4 || V == 6 || V == 7) sm100::mbar_wait(&ready, 0);
        if (V == 1 || V == 3 || V == 4 || V == 6 || V == 7) sm100::tc_fence_after();
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const int ks = 2 * s + j;
          sm100::mma_bf16(tm, sm100::make_sdesc(a + ks * 256, 128, 4096), sm100::make_sdesc(b + ks * 8192, 128, 256), idesc,
                          ks ? 1u : 0u);
        }
        if (V == 2 || V == 4 || V == 6 || V == 7) sm100::mma_commit(&st[s]);
      }
      sm100::mma_commit(&done);
      sm100::mbar_wait(&done, (uint32_t)r & 1u);
      const long long dt = clock64() - t0;
      if (r == reps - 1) out[V] = dt;
    }
  }
  sm100::tc_fence_before();
  __syncthreads();
  if (warp == 1) { sm100::tc_fence_after(); sm100::tmem_dealloc(tm, 256); }
}

template <int V>
void run(const uint8_t* w, long long* d) {
  const int smem = 65536 + 131072 + 32768;
  cudaFuncSetAttribute(k<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  long long best = 1LL << 60;
  for (int t = 0; t < 5; ++t) {
    k<V><<<1, 128, smem>>>(w, 4, d);
    long long h = 0;
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("V%d: %s\n", V, cudaGetErrorString(e)); return; }
    cudaMemcpy(&h, d + V, 8, cudaMemcpyDeviceToHost);
    if (h < best) best = h;
  }
  printf("V%d: 128 KB layer (16 k-steps, 8 stages of 2) %6lld cycles  (%.0f per stage)\n", V, best, best / 8.0);
}

int main() {
  uint8_t* w;
  cudaMalloc(&w, 1 << 20);
  cudaMemset(w, 0, 1 << 20);
  long long* d;
  cudaMalloc(&d, 8 * 8);
  run<0>(w, d); run<1>(w, d); run<2>(w, d); run<3>(w, d);
  run<4>(w, d); run<5>(w, d); run<6>(w, d); run<7>(w, d);
  return 0;
}
