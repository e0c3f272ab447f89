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

// P / U: row d of the f64 price table -- close p_k (exact widening of the fp32
// market) and u_k = fl(p_k * up) -- in shared or global memory.  Padding assets
// (k >= K) carry p = u = 0, h = 0 and a = 0, so every loop below runs to the
// compile-time KA with no per-asset predicate: a padded asset adds +0 to the cash
// (b is never -0) and to the sums, which leaves them bit-identical.

// v = b + sum_k h_k p_k, ascending k (each product is exact: h < 2^15, p has 24 bits)
template <int KA>
__device__ __forceinline__ double stock_mark(double b, const int (&h)[KA], const double* P) {
  double acc = b;
#pragma unroll
  for (int k = 0; k < KA; ++k) acc = fadd64(acc, fmul64(nn2d(h[k]), P[k]));
  return acc;
}

// The trade of one step.  a[] holds the requested deltas on entry and the clamped
// deltas (R6) on exit; h[] and b are updated in place.
template <int KA>
__device__ __forceinline__ void stock_trade(const EnvDev& e, double& b, int (&h)[KA], const double* P,
                                            const double* U, int (&a)[KA], bool& oor) {
  // 2. clamp (R6); any clamped entry sets the sticky range flag
  int diff = 0;
#pragma unroll
  for (int k = 0; k < KA; ++k) {
    const int x = min(max(a[k], -e.max_trade), e.max_trade);
    diff |= x ^ a[k];
    a[k] = x;
  }
  oor |= diff != 0;
  // 3. sells, clipped to holdings: b += fl(fl(n p) (1 - c)); n = 0 adds +0
#pragma unroll
  for (int k = 0; k < KA; ++k) {
    const int n = max(min(-a[k], h[k]), 0);
    b = fadd64(b, fmul64(fmul64(nn2d(n), P[k]), e.dn));
    h[k] -= n;
  }
  // 4. buys, ascending k, each the largest affordable count at u (R5); the fast
  //    path (the whole request is affordable) reuses the product it tested
#pragma unroll
  for (int k = 0; k < KA; ++k) {
    const int want = max(min(a[k], FIN_HOLD_MAX - h[k]), 0);
    const double u = U[k];
    double c = fmul64(nn2d(want), u);
    int n = want;
    if (!(c <= b)) {
      n = affordable_slow(b, u, want);
      c = fmul64(nn2d(n), u);
    }
    b = fsub64(b, c);
    h[k] += n;
  }
}

// reward = (v' - v) * scale (exact power-of-two scale), stored fp32
__device__ __forceinline__ float stock_reward(const EnvDev& e, double v, double vn) {
  return (float)fmul64(fsub64(vn, v), e.scale);
}
