// Micro-benchmark: 1-D bulk copies with and without the .L2::cache_hint (evict_last) operand.
// A 128 KB L2-resident layer as n copies of sb bytes, one mbarrier per copy, issued back to
// back by one thread and waited in order; grid 1 and 296 (two CTAs per SM, per-CTA layers).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_2501_10709_b200/csrc copy_hint.cu
#include <cstdint>
#include <cstdio>
#include <vector>
#include <algorithm>

#include "sm100.cuh"

template <int HINT>
__global__ void k(const uint8_t* __restrict__ w, int sb, int reps, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar[32];
  const int n = 131072 / sb;
  if (threadIdx.x == 0) {
    for (int s = 0; s < 32; ++s) sm100::mbar_init(&bar[s], 1);
    sm100::fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  const uint64_t pol = sm100::l2_policy_evict_last();
  const uint8_t* src = w + (size_t)(blockIdx.x % 148) * 131072;
  long long best = 1LL << 60;
  for (int r = 0; r < reps; ++r) {
    const long long t0 = clock64();
    for (int s = 0; s < n; ++s) {
      sm100::mbar_arrive_expect_tx(&bar[s], sb);
      if (HINT) sm100::bulk_g2s_hint(smem + (size_t)(s % (65536 / sb)) * sb, src + (size_t)s * sb, sb, &bar[s], pol);
      else sm100::bulk_g2s(smem + (size_t)(s % (65536 / sb)) * sb, src + (size_t)s * sb, sb, &bar[s]);
    }
    for (int s = 0; s < n; ++s) sm100::mbar_wait(&bar[s], (uint32_t)r & 1u);
    const long long dt = clock64() - t0;
    if (r > 0 && dt < best) best = dt;
  }
  out[blockIdx.x] = best;
}

int main() {
  uint8_t* w;
  cudaMalloc(&w, 148 * 131072);
  cudaMemset(w, 1, 148 * 131072);
  long long* d;
  cudaMalloc(&d, 296 * 8);
  cudaFuncSetAttribute(k<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  cudaFuncSetAttribute(k<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  for (int grid : {1, 296})
    for (int sb : {4096, 8192, 16384, 32768})
      for (int hint : {0, 1}) {
        if (hint) k<1><<<grid, 32, 65536>>>(w, sb, 6, d);
        else k<0><<<grid, 32, 65536>>>(w, sb, 6, d);
        cudaError_t e = cudaDeviceSynchronize();
        std::vector<long long> h(grid);
        cudaMemcpy(h.data(), d, grid * 8, cudaMemcpyDeviceToHost);
        std::sort(h.begin(), h.end());
        printf("grid %3d copy %2d KB %s: 128 KB in %6lld cycles median %s\n", grid, sb / 1024,
               hint ? "evict_last hint" : "no hint        ", h[grid / 2], e == cudaSuccess ? "" : cudaGetErrorString(e));
      }
  return 0;
}
