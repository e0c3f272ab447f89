// env_stock.cuh -- the stock SubEnv transition as a device function, shared by
// the single-step kernel (K1), the replay rollout (K4) and the fused policy
// rollout (K3).
//
// PAPER.md §3.1: state [b, p, h, f]; action = change in position
// h_{t+1} = h_t + a_t; reward R = v_{t+1} - v_t with v_t = b_t + p_t^T h_t;
// transaction costs (0.1% per side, BASELINE configs[0]).  Readings
// (DESIGN.md §3): R2 execute at p_t, mark at p_{t+1}; R3 sells first, then buys
// in ascending asset order; R4 proceeds n p (1-c), cost n p (1+c); R5 buy the
// largest affordable count; R6 clamp |a| <= max_trade; R8 reward * 2^-12;
// R-HOLD holdings <= 32767.
//
// Every float64 operation is an explicit _rn intrinsic in the order written, so
// cash / asset are bit-identical to the float64 definition (no FMA contraction).
#pragma once
#include "fin_internal.cuh"

// ``p`` / ``pn``: close prices of rows d and d+1 (fp32, widened exactly).
// h[] holds int holdings (updated in place), a[] the requested deltas.
// Returns via references: v (pre-trade asset at p), vn (post-trade asset at pn),
// act[] the action after the clamp (R6); oor set when an action was clamped.
template <int KP, typename PT>
__device__ __forceinline__ void stock_transition(const EnvDev& e, double& b, int (&h)[KP],
                                                 const PT* __restrict__ p, const PT* __restrict__ pn,
                                                 const int (&a)[KP], double& v, double& vn,
                                                 int (&act)[KP], bool& oor) {
  const int K = e.K;
  // 1. v = b + sum_k h_k p_k, ascending k (products are exact: h < 2^15, p has 24 bits)
  double acc = b;
#pragma unroll
  for (int k = 0; k < KP; ++k)
    if (k < K) acc = fadd64(acc, fmul64((double)h[k], (double)p[k]));
  v = acc;
  // 2. clamp (R6)
  int aa[KP];
#pragma unroll
  for (int k = 0; k < KP; ++k) {
    int x = (k < K) ? a[k] : 0;
    if (x > e.max_trade) { x = e.max_trade; oor = true; }
    if (x < -e.max_trade) { x = -e.max_trade; oor = true; }
    aa[k] = x;
    act[k] = x;
  }
  // 3. sells, clipped to holdings: b += (n p) (1 - c)
#pragma unroll
  for (int k = 0; k < KP; ++k) {
    if (k < K && aa[k] < 0) {
      int n = min(-aa[k], h[k]);
      b = fadd64(b, fmul64(fmul64((double)n, (double)p[k]), e.dn));
      h[k] -= n;
    }
  }
  // 4. buys, ascending k, each the largest affordable count at u = p (1 + c)
#pragma unroll
  for (int k = 0; k < KP; ++k) {
    if (k < K && aa[k] > 0) {
      double u = fmul64((double)p[k], e.up);
      int n = affordable(b, u, min(aa[k], FIN_HOLD_MAX - h[k]));
      b = fsub64(b, fmul64((double)n, u));
      h[k] += n;
    }
  }
  // 5. v' = b' + sum_k h'_k p'_k
  acc = b;
#pragma unroll
  for (int k = 0; k < KP; ++k)
    if (k < K) acc = fadd64(acc, fmul64((double)h[k], (double)pn[k]));
  vn = acc;
}

// reward = (v' - v) * scale (exact power-of-two scale), stored fp32
__device__ __forceinline__ float stock_reward(const EnvDev& e, double v, double vn) {
  return (float)fmul64(fsub64(vn, v), e.scale);
}
