// Microbenchmark: tcgen05.mma (kind::f16, M = 128, cta_group::1) issue-to-completion
// time for a run of k-steps with SWIZZLE_NONE vs SWIZZLE_128B K-major operands.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_2501_10709_b200/csrc mma_rate.cu
#include <cstdio>
#include <cstdint>
#include "sm100.cuh"

__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)layout << 61;
  return d;
}

__device__ __forceinline__ void mma_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(acc)
      : "memory");
}
__global__ void k(int N, int ksteps, int swz, int reps, long long* out, int M) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  uint8_t* A = smem;                 // 128 x 256 bf16 (64 KB)
  uint8_t* B = smem + 65536;         // N x 256 bf16 (<= 128 KB)
  for (int i = threadIdx.x; i < (65536 + N * 512) / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3f803f80u;
  if (threadIdx.x == 0) { sm100::mbar_init(&bar, 1); sm100::fence_mbar_init(); }
  if (threadIdx.x < 32) { sm100::tmem_alloc(&tslot, 512); sm100::tmem_relinquish(); }
  sm100::fence_proxy_async_smem();
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tm = tslot;
  if (threadIdx.x == 0) {
    const uint32_t idesc = sm100::make_idesc_bf16(M, N);
    const uint32_t a = sm100::smem_u32(A), b = sm100::smem_u32(B);
    long long best = 1LL << 60;
    for (int r = 0; r < reps; ++r) {
      const long long t0 = clock64();
      for (int j = 0; j < ksteps; ++j) {
        uint64_t ad, bd;
        if (swz == 0) {   // canonical no-swizzle K-major: core matrices 128 B, LBO 128 (K), SBO K/8*128 (M/N)
          ad = sdesc(a + j * 256, 128, 256 / 8 * 128, 0);
          bd = sdesc(b + j * 256, 128, 256 / 8 * 128, 0);
        } else {          // SWIZZLE_128B K-major: 8-row x 128-B atoms, SBO = 1024; K step of 16 = 32 B inside the atom
          const int kk = j * 16;  // element offset along K
          const int atom = kk / 64, in = (kk % 64) * 2;
          ad = sdesc(a + atom * (128 * 128) + in, 16, 1024, 2);
          bd = sdesc(b + atom * (N * 128) + in, 16, 1024, 2);
        }
        if (swz == 2) mma_ts(tm, tm + 256 + j * 8, bd, idesc, j > 0 ? 1u : 0u);
        else sm100::mma_bf16(tm, ad, bd, idesc, j > 0 ? 1u : 0u);
      }
      sm100::mma_commit(&bar);
      sm100::mbar_wait(&bar, r & 1);
      const long long dt = clock64() - t0;
      if (dt < best) best = dt;
    }
    out[0] = best;
  }
  sm100::tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) { sm100::tc_fence_after(); sm100::tmem_dealloc(tm, 512); }
}

int main() {
  long long* d; cudaMalloc(&d, 8);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 + 131072);
  for (int M : {64, 128})
  for (int swz = 0; swz < 1; swz += 2)
    for (int N : {32, 64, 128, 256})
      for (int ks : {1, 16}) {
        k<<<1, 128, 65536 + N * 512>>>(N, ks, swz, 20, d, M);
        long long h = 0; cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
        cudaError_t e = cudaGetLastError();
        const double flop = 2.0 * M * N * 16 * ks;
        printf("M=%d swz=%d N=%3d ksteps=%2d: %6lld cycles  %.0f FLOP/cycle %s\n", M, swz, N, ks, h, flop / h,
               e == cudaSuccess ? "" : cudaGetErrorString(e));
      }
  return 0;
}
