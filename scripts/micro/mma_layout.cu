// Micro-benchmark: 16 back-to-back tcgen05.mma (M = 128, N = 256, K = 16, bf16) with the B operand
// (256 x 256, resident) in three shared-memory images: (0) one K-major image of all K (LBO 128,
// SBO 4096 -- K = 256 per 8-row group), (1) 8 stage images of K = 32 each (the fused rollout's
// packing: LBO 128, SBO 512, stages 16 KB apart), (2) 4 stage images of K = 64 (SBO 1024).
#include <cstdint>
#include <cstdio>

#include "sm100.cuh"

__global__ void k(int mode, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  uint8_t* A = smem;
  uint8_t* B = smem + 65536;
  for (int i = threadIdx.x; i < (65536 + 131072) / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3f803f80u;
  if (threadIdx.x == 0) { sm100::mbar_init(&bar, 1); sm100::fence_mbar_init(); }
  if (threadIdx.x < 32) { sm100::tmem_alloc(&tslot, 256); sm100::tmem_relinquish(); }
  sm100::fence_proxy_async_smem();
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tm = tslot;
  if (threadIdx.x == 0) {
    const uint32_t idesc = sm100::make_idesc_bf16(128, 256);
    const uint32_t a = sm100::smem_u32(A), b = sm100::smem_u32(B);
    long long best = 1LL << 60;
    for (int r = 0; r < 20; ++r) {
      const long long t0 = clock64();
      for (int j = 0; j < 16; ++j) {
        uint64_t bd;
        if (mode == 0) bd = sm100::make_sdesc(b + j * 256, 128, 4096);
        else if (mode == 1) bd = sm100::make_sdesc(b + (j / 2) * 16384 + (j % 2) * 256, 128, 512);
        else bd = sm100::make_sdesc(b + (j / 4) * 32768 + (j % 4) * 256, 128, 1024);
        sm100::mma_bf16(tm, sm100::make_sdesc(a + j * 256, 128, 4096), bd, idesc, j > 0 ? 1u : 0u);
      }
      sm100::mma_commit(&bar);
      sm100::mbar_wait(&bar, r & 1);
      const long long dt = clock64() - t0;
      if (dt < best) best = dt;
    }
    out[mode] = best;
  }
  sm100::tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) { sm100::tc_fence_after(); sm100::tmem_dealloc(tm, 256); }
}

int main() {
  long long* d;
  cudaMalloc(&d, 64);
  const int smem = 65536 + 131072;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const char* names[] = {"one K=256 image (SBO 4096)", "8 stages of K=32 (SBO 512)", "4 stages of K=64 (SBO 1024)"};
  for (int m = 0; m < 3; ++m) {
    k<<<1, 128, smem>>>(m, d);
    long long h;
    cudaDeviceSynchronize();
    cudaMemcpy(&h, d + m, 8, cudaMemcpyDeviceToHost);
    printf("%-32s: 16 MMAs in %5lld cycles (%s)\n", names[m], h, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
