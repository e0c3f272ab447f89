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

// fp32 value of ((x >> 8) + 0.5) 2^-24: the +0.5 rounds away for x >> 8 >= 2^23 (the exact
// value needs 25 bits); the rollout's noise is compared with tolerances, and exact
// consumers (fin_market_prepare) form the value in f64
__device__ __forceinline__ float philox_u01(uint32_t x) {
  return ((float)(x >> 8) + 0.5f) * 5.9604644775390625e-08f;
}

// Box-Muller pair from (u_r, u_a): r = sqrt(-2 ln u_r) (accurate log: u_r can be
// 1 - 2^-25), angle 2 pi u_a evaluated as 2 pi (u_a - [u_a >= 1/2]) in [-pi, pi) with
// the fast sincos (absolute error ~4e-7 there).
__device__ __forceinline__ void box_muller(float ur, float ua, float& z0, float& z1) {
  float r;   // sqrt.approx (rel. error ~2^-23; no slow-path call in the env warps' code)
  asm("sqrt.approx.f32 %0, %1;" : "=f"(r) : "f"(-2.0f * logf(ur)));
  const float a = 6.283185307179586f * (ua >= 0.5f ? ua - 1.0f : ua);
  float s, c;
  __sincosf(a, &s, &c);
  z0 = r * c;
  z1 = r * s;
}

// Two counters (word2a, word2b) interleaved for instruction-level parallelism, out of
// line (one copy in the kernel), results returned in registers.
struct Normals8 {
  float4 a, b;
};
__device__ __forceinline__ Normals8 philox_normals8_v(uint64_t g, uint32_t t, uint32_t word2a, uint32_t word2b,
                                                           uint64_t seed) {
  uint32_t ca[4] = {(uint32_t)g, t, word2a, 0u};
  uint32_t cb[4] = {(uint32_t)g, t, word2b, 0u};
  uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r > 0) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
    const uint32_t ha0 = __umulhi(0xD2511F53u, ca[0]), la0 = 0xD2511F53u * ca[0];
    const uint32_t hb0 = __umulhi(0xD2511F53u, cb[0]), lb0 = 0xD2511F53u * cb[0];
    const uint32_t ha1 = __umulhi(0xCD9E8D57u, ca[2]), la1 = 0xCD9E8D57u * ca[2];
    const uint32_t hb1 = __umulhi(0xCD9E8D57u, cb[2]), lb1 = 0xCD9E8D57u * cb[2];
    const uint32_t na0 = ha1 ^ ca[1] ^ k0, na2 = ha0 ^ ca[3] ^ k1;
    const uint32_t nb0 = hb1 ^ cb[1] ^ k0, nb2 = hb0 ^ cb[3] ^ k1;
    ca[0] = na0; ca[1] = la1; ca[2] = na2; ca[3] = la0;
    cb[0] = nb0; cb[1] = lb1; cb[2] = nb2; cb[3] = lb0;
  }
  Normals8 o;
  box_muller(philox_u01(ca[0]), philox_u01(ca[1]), o.a.x, o.a.y);
  box_muller(philox_u01(ca[2]), philox_u01(ca[3]), o.a.z, o.a.w);
  box_muller(philox_u01(cb[0]), philox_u01(cb[1]), o.b.x, o.b.y);
  box_muller(philox_u01(cb[2]), philox_u01(cb[3]), o.b.z, o.b.w);
  return o;
}

// Four counters (word2 = w2[0..3]) interleaved: 16 normals (Box-Muller pairs of each counter's
// words 0-1 and 2-3, as philox_normals8_v per counter)
struct Normals16 {
  float v[16];
};
__device__ __forceinline__ Normals16 philox_normals16_v(uint64_t g, uint32_t t, const uint32_t (&w2)[4], uint64_t seed) {
  uint32_t c[4][4];
#pragma unroll
  for (int q = 0; q < 4; ++q) { c[q][0] = (uint32_t)g; c[q][1] = t; c[q][2] = w2[q]; c[q][3] = 0u; }
  uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r > 0) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint32_t h0 = __umulhi(0xD2511F53u, c[q][0]), l0 = 0xD2511F53u * c[q][0];
      const uint32_t h1 = __umulhi(0xCD9E8D57u, c[q][2]), l1 = 0xCD9E8D57u * c[q][2];
      const uint32_t n0 = h1 ^ c[q][1] ^ k0, n2 = h0 ^ c[q][3] ^ k1;
      c[q][0] = n0; c[q][1] = l1; c[q][2] = n2; c[q][3] = l0;
    }
  }
  Normals16 o;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    box_muller(philox_u01(c[q][0]), philox_u01(c[q][1]), o.v[4 * q], o.v[4 * q + 1]);
    box_muller(philox_u01(c[q][2]), philox_u01(c[q][3]), o.v[4 * q + 2], o.v[4 * q + 3]);
  }
  return o;
}

__device__ __forceinline__ void philox_normals4(uint64_t g, uint32_t t, uint32_t word2, uint64_t seed, float z[4]) {
  const Normals8 v = philox_normals8_v(g, t, word2, word2, seed);
  z[0] = v.a.x; z[1] = v.a.y; z[2] = v.a.z; z[3] = v.a.w;
}

__device__ __forceinline__ void philox_uniform2(uint64_t g, uint32_t t, uint64_t seed, float u[2]) {
  uint32_t c[4] = {(uint32_t)g, t, 0xFFFF0000u, 0u};
  philox4x32_10(c, (uint32_t)seed, (uint32_t)(seed >> 32));
  u[0] = philox_u01(c[0]);
  u[1] = philox_u01(c[1]);
}
