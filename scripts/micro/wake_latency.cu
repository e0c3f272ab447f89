// Micro-benchmark: mbarrier wake-up latency by wait flavour.  Warp 1 lane 0 waits on an
// mbarrier; warp 0 lane 0 spins ~``delay`` cycles, records clock64 and arrives; the waiter
// records clock64 when its wait returns.  Wake latency = t_wake - t_arrive (same SM clock).
//   kind 0: try_wait.parity with a 1e6 ns suspend-time hint (sm100::mbar_wait)
//   kind 1: try_wait.parity without a hint (hardware default time limit)
//   kind 2: test_wait.parity spin (never suspends)
// Then the 8 x 16 KB copy stream of copy_rate.cu (one mbarrier per copy, waited in order)
// with each flavour.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_2501_10709_b200/csrc wake_latency.cu
#include <cstdint>
#include <cstdio>

#include "sm100.cuh"

__device__ __forceinline__ bool test_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(sm100::smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
template <int KIND>
__device__ __forceinline__ void wait(uint64_t* bar, uint32_t ph) {
  if (KIND == 0) sm100::mbar_wait(bar, ph);
  else if (KIND == 1) while (!sm100::mbar_try_wait_nh(bar, ph)) {}
  else while (!test_wait(bar, ph)) {}
}

template <int KIND>
__global__ void k_wake(int delay, int reps, long long* out) {
  __shared__ uint64_t bar;
  __shared__ long long t_arr;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) { sm100::mbar_init(&bar, 1); sm100::fence_mbar_init(); }
  __syncthreads();
  long long sum = 0, mx = 0;
  for (int r = 0; r < reps; ++r) {
    __syncthreads();
    if (warp == 0 && lane == 0) {
      const long long t0 = clock64();
      while (clock64() - t0 < delay) {}
      *(volatile long long*)&t_arr = clock64();
      sm100::mbar_arrive(&bar);
    } else if (warp == 1 && lane == 0) {
      wait<KIND>(&bar, (uint32_t)r & 1u);
      const long long tw = clock64();
      __threadfence_block();
      const long long d = tw - *(volatile long long*)&t_arr;
      sum += d;
      mx = d > mx ? d : mx;
    }
  }
  if (warp == 1 && lane == 0) { out[0] = sum / reps; out[1] = mx; }
}

template <int KIND>
__global__ void k_copy(const uint8_t* __restrict__ w, int reps, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar[8];
  if (threadIdx.x == 0) {
    for (int s = 0; s < 8; ++s) sm100::mbar_init(&bar[s], 1);
    sm100::fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  long long best = 1LL << 60;
  for (int r = 0; r < reps; ++r) {
    const long long t0 = clock64();
    for (int s = 0; s < 8; ++s) {
      sm100::mbar_arrive_expect_tx(&bar[s], 16384);
      sm100::bulk_g2s(smem + (s & 3) * 16384, w + (size_t)s * 16384, 16384, &bar[s]);
    }
    for (int s = 0; s < 8; ++s) wait<KIND>(&bar[s], (uint32_t)r & 1u);
    const long long dt = clock64() - t0;
    if (r > 0 && dt < best) best = dt;
  }
  out[0] = best;
}

int main() {
  long long* d;
  cudaMalloc(&d, 16);
  uint8_t* w;
  cudaMalloc(&w, 1 << 20);
  cudaMemset(w, 1, 1 << 20);
  long long h[2];
  const char* names[3] = {"try_wait + 1 ms hint", "try_wait, no hint   ", "test_wait spin      "};
  for (int delay : {0, 200, 1000, 5000}) {
    k_wake<0><<<1, 64>>>(delay, 50, d); cudaDeviceSynchronize(); cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("%s delay %5d: wake latency mean %5lld max %5lld cycles\n", names[0], delay, h[0], h[1]);
    k_wake<1><<<1, 64>>>(delay, 50, d); cudaDeviceSynchronize(); cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("%s delay %5d: wake latency mean %5lld max %5lld cycles\n", names[1], delay, h[0], h[1]);
    k_wake<2><<<1, 64>>>(delay, 50, d); cudaDeviceSynchronize(); cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("%s delay %5d: wake latency mean %5lld max %5lld cycles\n", names[2], delay, h[0], h[1]);
  }
  cudaFuncSetAttribute(k_copy<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  cudaFuncSetAttribute(k_copy<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  cudaFuncSetAttribute(k_copy<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  k_copy<0><<<1, 32, 65536>>>(w, 6, d); cudaDeviceSynchronize(); cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost);
  printf("8 x 16 KB copies, waited in order, %s: %lld cycles\n", names[0], h[0]);
  k_copy<1><<<1, 32, 65536>>>(w, 6, d); cudaDeviceSynchronize(); cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost);
  printf("8 x 16 KB copies, waited in order, %s: %lld cycles\n", names[1], h[0]);
  k_copy<2><<<1, 32, 65536>>>(w, 6, d); cudaDeviceSynchronize(); cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost);
  printf("8 x 16 KB copies, waited in order, %s: %lld cycles\n", names[2], h[0]);
  return 0;
}
