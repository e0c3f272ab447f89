// env_crypto.cuh -- the crypto SubEnv transition (single asset, 10-level LOB) as a
// device function, shared by the step kernel (K2) and the fused Q rollout.
//
// PAPER.md P:124 (BTC, second-level LOB), P:129-132 (state / action / reward),
// §5.2.2 P:317-321 (discrete actions), BASELINE configs[3] (actions {-1,0,1},
// position limit +-1, max holding 120 steps).  Readings R24-R28:
// forced exit at tau >= max_hold overrides the action; buys walk the asks and
// sells walk the bids level by level, any remainder past the displayed depth
// fills at the last level; fee multiplies the notional; reward scale 1.
#pragma once
#include "fin_internal.cuh"

#define FIN_C_MID 0
#define FIN_C_ASK_PX 1
#define FIN_C_ASK_SZ 11
#define FIN_C_BID_PX 21
#define FIN_C_BID_SZ 31
#define FIN_C_F0 41
#define FIN_C_LEVELS 10
#define FIN_C_FACTORS 101
#define FIN_C_ROW 144

__device__ __forceinline__ double walk_book(const float* __restrict__ px, const float* __restrict__ sz, double qty) {
  double rem = qty, notional = 0.0;
#pragma unroll
  for (int l = 0; l < FIN_C_LEVELS; ++l) {
    const double size = (double)sz[l];
    const double fill = rem < size ? rem : size;
    notional = fadd64(notional, fmul64(fill, (double)px[l]));
    rem = fsub64(rem, fill);
  }
  if (rem > 0.0) notional = fadd64(notional, fmul64(rem, (double)px[FIN_C_LEVELS - 1]));
  return notional;
}

// One transition.  h: position in {-1,0,1}; tau: consecutive holding steps.
__device__ __forceinline__ void crypto_transition(const EnvDev& e, double& b, int& h, int& tau,
                                                  const float* __restrict__ row, const float* __restrict__ row_next,
                                                  int a, double& v, double& vn, int& delta) {
  int target = h + a;
  target = target > 1 ? 1 : (target < -1 ? -1 : target);
  if (h != 0 && tau >= e.max_hold) target = 0;   // forced exit (R26)
  delta = target - h;
  const double m = (double)row[FIN_C_MID];
  v = fadd64(b, fmul64((double)h, m));
  if (delta > 0) {
    b = fsub64(b, fmul64(walk_book(row + FIN_C_ASK_PX, row + FIN_C_ASK_SZ, (double)delta), e.up));
  } else if (delta < 0) {
    b = fadd64(b, fmul64(walk_book(row + FIN_C_BID_PX, row + FIN_C_BID_SZ, (double)(-delta)), e.dn));
  }
  if (target == 0) tau = 0;
  else if (target == h) tau = tau + 1;
  else tau = 1;
  h = target;
  vn = fadd64(b, fmul64((double)target, (double)row_next[FIN_C_MID]));
}
