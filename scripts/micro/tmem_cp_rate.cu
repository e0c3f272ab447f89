// Micro-benchmark: latency of n tcgen05.cp.128x256b (SBO = 0 broadcast source) issued by one
// thread, from issue to tcgen05.commit completion, vs n = 2 MMAs (M128 N256 K16).
#include <cstdint>
#include <cstdio>

#include "sm100.cuh"

__global__ void k(int n, int mode, long long* out) {
  extern __shared__ __align__(1024) uint8_t buf[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  for (int i = threadIdx.x; i < (65536 + 8192) / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(buf)[i] = 0x3f803f80u;
  if (threadIdx.x == 0) { sm100::mbar_init(&bar, 1); sm100::fence_mbar_init(); }
  if (threadIdx.x < 32) { sm100::tmem_alloc(&tslot, 256); sm100::tmem_relinquish(); }
  sm100::fence_proxy_async_smem();
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tm = tslot;
  if (threadIdx.x == 0) {
    const uint32_t img = sm100::smem_u32(buf + 65536);
    const uint32_t a = sm100::smem_u32(buf);
    uint32_t ph = 0;
    for (int rep = 0; rep < 4; ++rep) {
      long long t0 = clock64();
      if (mode == 0 || mode == 2)
        for (int g = 0; g < n; ++g) sm100::tmem_cp_128x256b(tm + 8 * g, sm100::make_sdesc(img + g * 256, 128, 0));
      if (mode >= 1) {
        const uint32_t idesc = sm100::make_idesc_bf16(128, 256);
        for (int j = 0; j < 2; ++j)
          sm100::mma_bf16(tm, sm100::make_sdesc(a + j * 256, 128, 512), sm100::make_sdesc(a + j * 256, 128, 512), idesc, 1);
      }
      sm100::mma_commit(&bar);
      sm100::mbar_wait(&bar, ph);
      ph ^= 1;
      long long t1 = clock64();
      out[rep] = t1 - t0;
    }
  }
  sm100::tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) sm100::tmem_dealloc(tm, 256);
}

int main() {
  long long* d;
  cudaMalloc(&d, 64);
  long long h[4];
  const char* names[] = {"cp only", "2 MMA only", "cp + 2 MMA"};
  for (int mode = 0; mode < 3; ++mode)
    for (int n : {1, 8, 16, 32}) {
      if (mode == 1 && n != 1) continue;
      cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 + 8192);
      k<<<1, 128, 65536 + 8192>>>(n, mode, d);
      cudaError_t e = cudaDeviceSynchronize();
      cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
      printf("%-12s n=%2d: cycles %lld %lld %lld %lld (%s)\n", names[mode], n, h[0], h[1], h[2], h[3], cudaGetErrorString(e));
    }
  return 0;
}
