// philox.cuh -- Philox4x32-10 (Salmon et al., SC'11) + Box-Muller on the device.
// Production-mode noise of the rollout: key = seed, counter =
// (global env id, global step, (member << 16) | block, 0), so the draws do not
// depend on how envs are partitioned over ranks.
//   u_i = ((x_i >> 8) + 0.5) * 2^-24 in (0, 1);  (z0, z1) = sqrt(-2 ln u0) (cos, sin)(2 pi u1)
#pragma once
#include <stdint.h>

__device__ __forceinline__ void philox4x32_10(uint32_t c[4], uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r > 0) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
    const uint32_t hi0 = __umulhi(0xD2511F53u, c[0]), lo0 = 0xD2511F53u * c[0];
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, c[2]), lo1 = 0xCD9E8D57u * c[2];
    const uint32_t n0 = hi1 ^ c[1] ^ k0, n2 = hi0 ^ c[3] ^ k1;
    c[0] = n0; c[1] = lo1; c[2] = n2; c[3] = lo0;
  }
}

__device__ __forceinline__ float philox_u01(uint32_t x) {
  return ((float)(x >> 8) + 0.5f) * 5.9604644775390625e-08f;  // 2^-24, exact
}

__device__ __forceinline__ void philox_normals4(uint64_t g, uint32_t t, uint32_t word2, uint64_t seed, float z[4]) {
  uint32_t c[4] = {(uint32_t)g, t, word2, 0u};
  philox4x32_10(c, (uint32_t)seed, (uint32_t)(seed >> 32));
  const float u0 = philox_u01(c[0]), u1 = philox_u01(c[1]), u2 = philox_u01(c[2]), u3 = philox_u01(c[3]);
  const float r0 = sqrtf(-2.0f * logf(u0)), r1 = sqrtf(-2.0f * logf(u2));
  float s0, c0, s1, c1;
  sincospif(2.0f * u1, &s0, &c0);
  sincospif(2.0f * u3, &s1, &c1);
  z[0] = r0 * c0; z[1] = r0 * s0; z[2] = r1 * c1; z[3] = r1 * s1;
}

__device__ __forceinline__ void philox_uniform2(uint64_t g, uint32_t t, uint64_t seed, float u[2]) {
  uint32_t c[4] = {(uint32_t)g, t, 0xFFFF0000u, 0u};
  philox4x32_10(c, (uint32_t)seed, (uint32_t)(seed >> 32));
  u[0] = philox_u01(c[0]);
  u[1] = philox_u01(c[1]);
}
