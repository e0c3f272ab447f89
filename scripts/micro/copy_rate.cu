// Micro-benchmark: L2 -> shared-memory weight streaming rate of 1-D bulk copies
// (cp.async.bulk, what the fused rollout's producer warp issues), per SM.
// Each CTA copies a 128 KB L2-resident layer into shared memory as n copies of sb bytes,
// all issued back to back by one thread (each on its own mbarrier), and times issue -> last
// completion.  Grid 1 (one SM alone), 2 CTAs on one SM, and 148 / 296 CTAs (every SM busy);
// plus the same with the copies issued in flight-limited fashion (at most ``depth``
// outstanding), which is what a ring of ``depth`` slots allows.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_2501_10709_b200/csrc copy_rate.cu
#include <cstdint>
#include <cstdio>
#include <vector>
#include <algorithm>

#include "sm100.cuh"

__global__ void k(const uint8_t* __restrict__ w, int sb, int depth, int reps, int span, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar[64];
  const int n = 131072 / sb;
  if (threadIdx.x == 0) {
    for (int s = 0; s < 64; ++s) sm100::mbar_init(&bar[s], 1);
    sm100::fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  const uint64_t pol = sm100::l2_policy_evict_last();
  const uint8_t* src = w + (size_t)(blockIdx.x % span) * 131072;
  long long best = 1LL << 60;
  uint32_t use[64] = {};
  for (int r = 0; r < reps; ++r) {
    const long long t0 = clock64();
    int issued = 0, waited = 0;
    while (waited < n) {
      while (issued < n && issued - waited < depth) {
        const int s = issued % 64;
        sm100::mbar_arrive_expect_tx(&bar[s], sb);
        sm100::bulk_g2s_hint(smem + (size_t)(issued % (65536 / sb)) * sb, src + (size_t)issued * sb, sb, &bar[s], pol);
        ++issued;
      }
      const int s = waited % 64;
      sm100::mbar_wait(&bar[s], use[s] & 1u);
      ++use[s];
      ++waited;
    }
    const long long dt = clock64() - t0;
    if (r > 0 && dt < best) best = dt;
  }
  out[blockIdx.x] = best;
}

int main() {
  uint8_t* w;
  const size_t wbytes = 148 * 131072;
  cudaMalloc(&w, wbytes);
  cudaMemset(w, 1, wbytes);
  long long* d;
  cudaMalloc(&d, 296 * 8);
  const int smem = 65536;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int grid : {1, 2, 148, 296})
    for (int span : {1, 148}) {
      if (grid == 1 && span > 1) continue;
      for (int sb : {4096, 8192, 16384, 32768})
        for (int depth : {1, 2, 4, 64}) {
          k<<<grid, 32, smem>>>(w, sb, depth, 6, span, d);
          cudaError_t e = cudaDeviceSynchronize();
          std::vector<long long> h(grid);
          cudaMemcpy(h.data(), d, grid * 8, cudaMemcpyDeviceToHost);
          std::sort(h.begin(), h.end());
          const double med = (double)h[grid / 2];
          printf("grid %3d (%s) copy %2d KB, <= %2d in flight: 128 KB in %6.0f cycles median (%5.1f B/clk per CTA) %s\n", grid,
                 span == 1 ? "same 128 KB" : "per-SM 128 KB", sb / 1024, depth, med, 131072.0 / med,
                 e == cudaSuccess ? "" : cudaGetErrorString(e));
        }
    }
  return 0;
}
