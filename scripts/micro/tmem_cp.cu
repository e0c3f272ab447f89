// Micro-test: tcgen05.cp (shared -> TMEM) with a broadcast source (SBO = 0) and
// tcgen05.st (registers -> TMEM), read back with tcgen05.ld.  Prints the TMEM value seen
// by a few lanes / columns so the source layout can be checked.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_2501_10709_b200/csrc tmem_cp.cu
#include <cstdint>
#include <cstdio>

#include "sm100.cuh"

__device__ __forceinline__ void cp_128x256b(uint32_t taddr, uint64_t desc) {
  asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(taddr), "l"(desc) : "memory");
}
__device__ __forceinline__ void cp_32x128b_x4(uint32_t taddr, uint64_t desc) {
  asm volatile("tcgen05.cp.cta_group::1.32x128b.warpx4 [%0], %1;" ::"r"(taddr), "l"(desc) : "memory");
}
__device__ __forceinline__ void st_32x32b_x8(uint32_t taddr, const uint32_t (&r)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(r[0]),
               "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
               : "memory");
}

__global__ void k(int mode, uint32_t lbo, uint32_t sbo, float* out) {
  __shared__ __align__(1024) float src[4096];   // 16 KB
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) src[i] = (float)i;
  if (threadIdx.x == 0) {
    sm100::mbar_init(&bar, 1);
    sm100::fence_mbar_init();
  }
  if (threadIdx.x < 32) {
    sm100::tmem_alloc(&tslot, 64);
    sm100::tmem_relinquish();
  }
  sm100::fence_proxy_async_smem();
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tm = tslot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (mode == 2) {   // tcgen05.st: thread (lane r of quadrant q) writes row 32 q + r, 8 columns
    uint32_t r[8];
    for (int j = 0; j < 8; ++j) r[j] = __float_as_uint(1000.f * (32 * warp + lane) + j);
    st_32x32b_x8(tm + ((uint32_t)(32 * warp) << 16), r);
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    sm100::tc_fence_before();
    __syncthreads();
    sm100::tc_fence_after();
  } else {
    if (threadIdx.x == 0) {
      const uint64_t d = sm100::make_sdesc(sm100::smem_u32(src), lbo, sbo);
      if (mode == 0) cp_128x256b(tm, d);
      else cp_32x128b_x4(tm, d);
      sm100::mma_commit(&bar);
    }
    sm100::mbar_wait(&bar, 0);
    sm100::tc_fence_after();
  }
  uint32_t v[16];
  sm100::tmem_ld16(tm + ((uint32_t)(32 * warp) << 16), v);
  sm100::tmem_wait_ld();
  for (int j = 0; j < 16; ++j) out[threadIdx.x * 16 + j] = __uint_as_float(v[j]);
  sm100::tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) sm100::tmem_dealloc(tm, 64);
}

int main() {
  float* d;
  cudaMalloc(&d, 128 * 16 * 4);
  float h[128 * 16];
  const struct { int mode; uint32_t lbo, sbo; const char* name; } cases[] = {
      {0, 128, 256, "128x256b lbo128 sbo256"}, {0, 128, 0, "128x256b lbo128 sbo0"},
      {1, 128, 128, "32x128b.warpx4 sbo128"}, {1, 128, 0, "32x128b.warpx4 sbo0"}, {2, 0, 0, "tcgen05.st 32x32b.x8"}};
  for (auto& c : cases) {
    cudaMemset(d, 0, sizeof(h));
    k<<<1, 128>>>(c.mode, c.lbo, c.sbo, d);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    printf("== %s (%s)\n", c.name, cudaGetErrorString(e));
    for (int row : {0, 1, 7, 8, 9, 31, 32, 63, 64, 127}) {
      printf("row %3d:", row);
      for (int j = 0; j < 12; ++j) printf(" %6.0f", h[row * 16 + j]);
      printf("\n");
    }
  }
  return 0;
}
