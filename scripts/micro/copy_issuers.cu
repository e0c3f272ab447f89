// Micro-benchmark: is the ~430-cycle cost of a 1-D bulk copy (copy_rate.cu) per issuing
// thread, per warp, or per SM?  A 128 KB L2-resident layer is copied into shared memory as n
// copies of sb bytes, all completing on one mbarrier (expect_tx of the total), issued by
//   mode 0: ``iss`` lanes of warp 0 (copy c by lane c % iss)
//   mode 1: lane 0 of ``iss`` warps (copy c by warp c % iss)
// Grid 1 and 296 (two CTAs per SM).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_2501_10709_b200/csrc copy_issuers.cu
#include <cstdint>
#include <cstdio>
#include <vector>
#include <algorithm>

#include "sm100.cuh"

__global__ void k(const uint8_t* __restrict__ w, int sb, int iss, int mode, int reps, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  const int n = 131072 / sb;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    sm100::mbar_init(&bar, 1);
    sm100::fence_mbar_init();
  }
  __syncthreads();
  const uint64_t pol = sm100::l2_policy_evict_last();
  const int me = mode == 0 ? (warp == 0 ? lane : -1) : (lane == 0 ? warp : -1);
  long long best = 1LL << 60;
  for (int r = 0; r < reps; ++r) {
    __syncthreads();
    const long long t0 = clock64();
    if (threadIdx.x == 0) sm100::mbar_arrive_expect_tx(&bar, 131072);
    __syncthreads();
    if (me >= 0 && me < iss)
      for (int c = me; c < n; c += iss)
        sm100::bulk_g2s_hint(smem + (size_t)(c % (65536 / sb)) * sb, w + (size_t)c * sb, sb, &bar, pol);
    sm100::mbar_wait(&bar, (uint32_t)r & 1u);
    const long long dt = clock64() - t0;
    if (r > 0 && dt < best) best = dt;
  }
  if (threadIdx.x == 0) out[blockIdx.x] = best;
}

int main() {
  uint8_t* w;
  cudaMalloc(&w, 1 << 20);
  cudaMemset(w, 1, 1 << 20);
  long long* d;
  cudaMalloc(&d, 296 * 8);
  const int smem = 65536;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int grid : {1, 296})
    for (int mode : {0, 1})
      for (int sb : {2048, 4096, 8192, 16384, 32768})
        for (int iss : {1, 2, 4, 8}) {
          if (131072 / sb < iss) continue;
          k<<<grid, 256, smem>>>(w, sb, iss, mode, 6, d);
          cudaError_t e = cudaDeviceSynchronize();
          std::vector<long long> h(grid);
          cudaMemcpy(h.data(), d, grid * 8, cudaMemcpyDeviceToHost);
          std::sort(h.begin(), h.end());
          const double med = (double)h[grid / 2];
          printf("grid %3d %s x%d, copy %2d KB: 128 KB in %6.0f cycles (%5.1f B/clk per CTA) %s\n", grid,
                 mode == 0 ? "lanes of one warp" : "lane 0 of warps  ", iss, sb / 1024, med, 131072.0 / med,
                 e == cudaSuccess ? "" : cudaGetErrorString(e));
        }
  return 0;
}
