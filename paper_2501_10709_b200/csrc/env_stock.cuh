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

// The price rows of one step (fin_internal.cuh: P U MP MU RU PN MPN) are staged in
// shared memory.  Products n * x with a non-negative int n are formed as fma(2^52 + n, x, -2^52 x):
// the exact value is n * x, so the single rounding of the fma gives fl(n * x) --
// the same bits as converting n and multiplying, with neither the XU-pipe I2F
// conversion nor a separate subtract.  2^52 + n is the bit pattern 0x43300000:n.
// Padding assets (k >= K) carry zeros in every row and in h and a, so every loop
// runs to the compile-time KA with no per-asset predicate: a padded asset adds +0
// to the cash (b is never -0) and to the sums, which leaves them bit-identical.

// Register-pressure control.  Left alone, ptxas hoists all 2-3 x 30 f64 row loads of
// a loop to its top (255 registers and spills).  The rows of asset chunk c+1 are
// therefore addressed through an offset computed from the loop's running value at
// the start of chunk c: (x >> 31) with x the high word of a non-negative double or a
// non-negative int, which is 0 at run time but not provably so at compile time.  At
// most two chunks of row values are live.
#ifndef FIN_KCHUNK
#define FIN_KCHUNK 6
#endif
constexpr int kChunk = FIN_KCHUNK;
__device__ __forceinline__ int zdep(double x) { return __double2hiint(x) >> 31; }
__device__ __forceinline__ int zdep(int x) { return x >> 31; }
#define FIN_CHUNKED(KA, dep_expr, BODY)                                            \
  {                                                                                \
    int off_ = 0;                                                                  \
    _Pragma("unroll") for (int c_ = 0; c_ < (KA); c_ += kChunk) {                  \
      const int o_ = off_;                                                         \
      off_ = 2 * zdep(dep_expr);  /* even: keeps 16-B row vectors aligned */       \
      _Pragma("unroll") for (int k = c_; k < (c_ + kChunk < (KA) ? c_ + kChunk : (KA)); ++k) { BODY } \
    }                                                                              \
  }

__device__ __forceinline__ double nprod(int n, double x, double mx) {
  return __fma_rn(__hiloint2double(0x43300000, n), x, mx);
}
// the same with -2^52 x formed by an exact multiply instead of a staged row: one fp64
// op instead of one shared-memory row read (the K1 profile is bound by the shared
// memory data path: broadcast 16-B row loads cost 4 wavefronts per warp instruction)
__device__ __forceinline__ double nprodx(int n, double x) {
  return __fma_rn(__hiloint2double(0x43300000, n), x, __dmul_rn(x, -4503599627370496.0));
}

// -2^52 x operands of the products from the staged rows MP / MU / MPN (one shared-memory read,
// two assets per 16-B load) instead of a DMUL each (FIN_MROWS=0): measured +1.8% on K1
#ifndef FIN_MROWS
#define FIN_MROWS 1
#endif
// v = b + sum_k h_k p_k, ascending k (each product is exact: h < 2^15, p has 24 bits);
// P = row PN of a staged row block with stride RS (row MPN follows)
template <int KA>
__device__ __forceinline__ double stock_mark(double b, const int (&h)[KA], const double* P, int RS) {
  double acc = b;
#if FIN_MROWS
  FIN_CHUNKED(KA, acc, acc = fadd64(acc, nprod(h[k], P[k + o_], P[(kRowMPN - kRowPN) * RS + k + o_]));)
#else
  FIN_CHUNKED(KA, acc, acc = fadd64(acc, nprodx(h[k], P[k + o_]));)
#endif
  return acc;
}

// The exact buys of one step in the definition's order (R5), from the post-sell holdings packed
// in ``save`` ([octet] x stride uint4) and the cash before the buys: each asset the largest n <=
// want with fl(n u) <= b (fp32 estimate, then exact fp64 checks).  Only the rare steps whose
// branch-free estimate failed its check come here.  Inline and register-only: a call in the env
// code makes ptxas keep the env state out of its caller-saved registers on every step.
__device__ __forceinline__ int affordable_exact(double b, double u, int want) {
  if (!(b >= u)) return 0;                                 // not even one share (also b < 0, NaN)
  const float qf = fminf(__fdividef((float)b, (float)u), (float)want);
  int n = qf > 0.f ? (int)qf : 0;
  while (n > 0 && fmul64((double)n, u) > b) --n;
  while (n < want && fmul64((double)(n + 1), u) <= b) ++n;
  return n;
}
template <int KA, class Acts>
__device__ __forceinline__ double stock_buys_redo(double b, int (&h)[KA], const Acts& a, const uint4* save,
                                                  int save_stride, const double* U, const double* MU) {
#pragma unroll
  for (int k = 0; k < KA; ++k) {
    const uint4 v = save[(k >> 3) * save_stride];
    const uint32_t wv[4] = {v.x, v.y, v.z, v.w};
    const uint32_t x = wv[(k >> 1) & 3];
    const int hk = (int)((k & 1) ? (x >> 16) : (x & 0xffffu));
    const int want = max(min(a[k], FIN_HOLD_MAX - hk), 0);
    double c = nprod(want, U[k], MU[k]);
    int n = want;
    if (!(c <= b)) {
      n = affordable_exact(b, U[k], want);
      c = nprod(n, U[k], MU[k]);
    }
    b = fsub64(b, c);
    h[k] = hk + n;
  }
  return b;
}

// K1's E-env form keeps the redo out of line (through local arrays, only on that path, the actions
// copied there so the caller's stay in registers): measured +3.1% for K1 (2,890 vs 2,803 GB/s), whose
// few live values survive the call unspilled; the fused rollout (stock_trade) inlines it (no call: +7%)
#ifndef FIN_REDO_CALL
#define FIN_REDO_CALL 1
#endif
template <int KA, class Acts>
static __device__ __noinline__ double stock_buys_redo_ool(double b, int* h, const Acts* a, const uint4* save,
                                                         int save_stride, const double* U, const double* MU) {
  int hh[KA];
#pragma unroll
  for (int k = 0; k < KA; ++k) hh[k] = h[k];
  b = stock_buys_redo<KA>(b, hh, *a, save, save_stride, U, MU);
#pragma unroll
  for (int k = 0; k < KA; ++k) h[k] = hh[k];
  return b;
}
template <int KA, class Acts>
__device__ __forceinline__ double stock_buys_redo_call(double b, int (&h)[KA], const Acts& a, const uint4* save,
                                                       int save_stride, const double* U, const double* MU) {
  int hh[KA];
#pragma unroll
  for (int k = 0; k < KA; ++k) hh[k] = h[k];
  Acts ac = a;   // a copy on this (rare) path: the caller's actions stay in registers
  b = stock_buys_redo_ool<KA, Acts>(b, hh, &ac, save, save_stride, U, MU);
#pragma unroll
  for (int k = 0; k < KA; ++k) h[k] = hh[k];
  return b;
}

// One buy of step 4 (R5): n = the largest count <= want with fl(n u) <= b, b -= fl(n u).
// The estimate f = floor(x), x = b RU exactly with RU = fl(fl(1/u)(1 + 2^-40)) (host, biased
// up), comes from one round-down fma D = RD(b RU + 2^52) whose bits are the biased operand
// 0x43300000:f that nprod needs -- n = min(want, f) is written over its low word, so the product takes D's
// own register pair.  Because x > (b/u)(1 + 2^-41) (RU's two roundings cost < 2^-52), the
// estimate is never below the answer:
// fl((f + 1) u) <= b gives b/u >= (f + 1)(1 - 2^-53), hence x > f + 1.  It can exceed the
// answer by one (b/u within 2^-40 below an integer), and then fl(n u) > b, i.e. the cash after
// the buy b' = fl(b - fl(n u)) < 0 (the sign of a rounded difference is exact).  So the checks:
//  * hi(D) == 0x43300000, i.e. 0 <= x < 2^32 (else NaN / huge / negative cash);
//  * b' >= 0 once, on the final cash (``stock_buys_ok``): buys only subtract (n >= 0), so a
//    negative b' stays negative, or trips the hi(D) check of the next asset (x < 0).
// With both passing, n satisfies the predicate and is >= the largest n that does: n is it.
// A failed check sets ``miss`` (the caller redoes the step's buys exactly).
// FIN_BUY_V1=1 (A/B, the round-2 form): n + 1 product and both checks per asset.
#ifndef FIN_BUY_V1
#define FIN_BUY_V1 0
#endif
__device__ __forceinline__ int buy_want_m(double& b, int want, double u, double mu, double ru, bool& miss) {
#if FIN_BUY_V1
  const double D = __dadd_rd(fmul64(b, ru), 4503599627370496.0);
  const int n = min(want, __double2loint(D));
  const double c = nprod(n, u, mu);
  const double c1 = nprod(n + 1, u, mu);
  miss |= (!(c <= b)) | ((n < want) & !(c1 > b)) | (n < 0);
  b = fsub64(b, c);
#else
  // D = RD(b RU + 2^52) in one fused op: the floor of the exact product (x above), one f64
  // latency less on the serial cash chain than rounding b RU first
  const double D = __fma_rd(b, ru, 4503599627370496.0);
  const int hi = __double2hiint(D);
  const int n = (int)umin((unsigned)want, (unsigned)__double2loint(D));
  const double c = __fma_rn(__hiloint2double(hi, n), u, mu);
  b = fsub64(b, c);
  miss |= hi != 0x43300000;
#endif
  return n;
}
// the same with mu = -2^52 u formed by an exact multiply instead of a staged row
__device__ __forceinline__ int buy_want(double& b, int want, double u, double ru, bool& miss) {
  return buy_want_m(b, want, u, __dmul_rn(u, -4503599627370496.0), ru, miss);
}
__device__ __forceinline__ void buy_one(double& b, int& hk, int ak, double u, double ru, bool& miss) {
  hk += buy_want(b, max(min(ak, FIN_HOLD_MAX - hk), 0), u, ru, miss);
}
// with mu = -2^52 u from the staged MU row (FIN_MROWS) or a DMUL
__device__ __forceinline__ void buy_one_r(double& b, int& hk, int ak, const double* R, int RS, int k, bool& miss) {
  const int want = max(min(ak, FIN_HOLD_MAX - hk), 0);
#if FIN_MROWS
  hk += buy_want_m(b, want, R[kRowU * RS + k], R[kRowMU * RS + k], R[kRowRU * RS + k], miss);
#else
  hk += buy_want(b, want, R[kRowU * RS + k], R[kRowRU * RS + k], miss);
#endif
}
// b + fl(fl(n p) (1 - c)): one sell's proceeds (step 3)
__device__ __forceinline__ double sell_add(const EnvDev& e, double b, int n, const double* R, int RS, int k) {
#if FIN_MROWS
  return fadd64(b, fmul64(nprod(n, R[kRowP * RS + k], R[kRowMP * RS + k]), e.dn));
#else
  return fadd64(b, fmul64(nprodx(n, R[kRowP * RS + k]), e.dn));
#endif
}
// the final check of the branch-free buys (see buy_one): fl(n u) <= b held at every asset
__device__ __forceinline__ bool stock_buys_ok(double b) {
#if FIN_BUY_V1
  return true;
#else
  return b >= 0.0;
#endif
}

// Step 2 of the transition, clamp (R6): any clamped entry sets the sticky range flag;
// ``act_out`` (nullable) receives the clamped actions.  Scalar form (policy actions).
template <int KA>
__device__ __forceinline__ void clamp_actions(const EnvDev& e, int (&a)[KA], bool& oor, int16_t* act_out) {
  int diff = 0;
#pragma unroll
  for (int k = 0; k < KA; ++k) {
    const int x = min(max(a[k], -e.max_trade), e.max_trade);
    diff |= x ^ a[k];
    a[k] = x;
    if (act_out) act_out[k] = (int16_t)x;
  }
  oor |= diff != 0;
}
// Packed form for supplied int16 actions: two assets per 32-bit word, 16-bit SIMD
// min / max (max_trade <= 32767 fits a signed half).
__device__ __forceinline__ uint32_t clamp_pair(uint32_t w, uint32_t mt2, uint32_t& diff) {
  const uint32_t x = __vmins2(__vmaxs2(w, __vneg2(mt2)), mt2);
  diff |= x ^ w;
  return x;
}

// Clamped actions travel packed, two int16 per 32-bit word (asset 2j in the low
// half): 15 registers instead of 30 for the C1 shapes.
template <int KA>
struct PackedActs {
  uint32_t w[(KA + 1) / 2];
  __device__ __forceinline__ int operator[](int k) const {
    return (k & 1) ? ((int)w[k >> 1] >> 16) : (int)(int16_t)(w[k >> 1] & 0xffffu);
  }
};
template <int KA>
__device__ __forceinline__ PackedActs<KA> pack_acts(const int (&a)[KA]) {
  PackedActs<KA> p;
#pragma unroll
  for (int j = 0; j < (KA + 1) / 2; ++j)
    p.w[j] = __byte_perm((uint32_t)a[2 * j], 2 * j + 1 < KA ? (uint32_t)a[2 * j + 1] : 0u, 0x5410);
  return p;
}

// Steps 3-4 of the transition (a already clamped); R[r * RS + k] is row r of the
// staged rows above; h[] and b are updated in place.  ``save`` (16-B aligned,
// (KA+7)/8 uint4; shared or local memory) receives the post-sell holdings for the
// rare exact redo of the buys.
template <int KA>
__device__ __forceinline__ void stock_trade(const EnvDev& e, double& b, int (&h)[KA], const double* R, int RS,
                                            const PackedActs<KA>& a, uint4* save, int save_stride) {
  const double* U = R + kRowU * RS;     // (the rare exact redo)
  const double* MU = R + kRowMU * RS;
  // 3. sells, clipped to holdings: b += fl(fl(n p) (1 - c)); n = 0 adds +0
  FIN_CHUNKED(KA, b, {
    const int n = max(min(-a[k], h[k]), 0);
    b = sell_add(e, b, n, R, RS, k + o_);
    h[k] -= n;
  })
  // 4. buys, ascending k, each n = min(want, f) with f the largest count whose cost
  //    fl(f u) fits the cash (R5).  Branch-free: f = floor(b * fl(1/u)) from one
  //    round-down add (its bits are 2^52 + f, the biased operand nprod needs), then
  //    the definition is verified on the chosen n -- fl(n u) <= b and, when the cash
  //    binds, fl((n + 1) u) > b.  A failed check (x within ~1e-11 of an integer, NaN
  //    cash) sends the step's buys to the exact out-of-line loop.
  const double bpre = b;
#pragma unroll
  for (int o = 0; o < (KA + 7) / 8; ++o) {   // post-sell holdings, packed, for the exact redo
    uint32_t w[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int k0 = 8 * o + 2 * j, k1 = k0 + 1;
      w[j] = __byte_perm(k0 < KA ? (uint32_t)h[k0] : 0u, k1 < KA ? (uint32_t)h[k1] : 0u, 0x5410);
    }
    save[o * save_stride] = make_uint4(w[0], w[1], w[2], w[3]);
  }
  bool miss = false;
  // once the cash of every env of the warp is below min_k u_k, no later asset can be
  // bought (fl(n u) > b for every n >= 1): the rest of the loop is skipped.  Exact.
  const double umin = R[kRowMeta * RS];
  FIN_CHUNKED(KA, b, {
    if (k == c_ && c_ > 0 && __all_sync(__activemask(), !(b >= umin))) goto buys_done;
    buy_one_r(b, h[k], a[k], R, RS, k + o_, miss);
  })
buys_done:
  miss |= !stock_buys_ok(b);
  if (miss) {   // rare
    atomicAdd(e.flags + FIN_CTR_EXACT_REDO, 1u);
    b = stock_buys_redo<KA>(bpre, h, a, save, save_stride, U, MU);
  }
}

// ---------------------------------------------------------------- E envs per thread
// The same transition for E independent envs of one thread, interleaved asset by asset:
// the serial cash chains of the envs overlap (K1 at E = 1 stalled mostly on fixed-
// latency dependencies of one chain).  Identical arithmetic per env.
template <int KA, int E>
__device__ __forceinline__ void stock_mark_e(double (&acc)[E], const int (&h)[E][KA], const double* const (&P)[E],
                                             int RS) {
  FIN_CHUNKED(KA, acc[0], {
#pragma unroll
    for (int q = 0; q < E; ++q) {
#if FIN_MROWS
      acc[q] = fadd64(acc[q], nprod(h[q][k], P[q][k + o_], P[q][(kRowMPN - kRowPN) * RS + k + o_]));
#else
      acc[q] = fadd64(acc[q], nprodx(h[q][k], P[q][k + o_]));
#endif
    }
  })
}

template <int KA, int E>
__device__ __forceinline__ void stock_trade_e(const EnvDev& e, double (&b)[E], int (&h)[E][KA],
                                              const double* const (&R)[E], int RS, const PackedActs<KA> (&a)[E],
                                              uint4* const (&save)[E], int save_stride) {
  // 3. sells
  FIN_CHUNKED(KA, b[0], {
#pragma unroll
    for (int q = 0; q < E; ++q) {
      const int n = max(min(-a[q][k], h[q][k]), 0);
      b[q] = sell_add(e, b[q], n, R[q], RS, k + o_);
      h[q][k] -= n;
    }
  })
  // 4. buys (see stock_trade)
  double bpre[E];
  bool miss[E];
#pragma unroll
  for (int q = 0; q < E; ++q) {
    bpre[q] = b[q];
    miss[q] = false;
#pragma unroll
    for (int o = 0; o < (KA + 7) / 8; ++o) {
      uint32_t w[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int k0 = 8 * o + 2 * j, k1 = k0 + 1;
        w[j] = __byte_perm(k0 < KA ? (uint32_t)h[q][k0] : 0u, k1 < KA ? (uint32_t)h[q][k1] : 0u, 0x5410);
      }
      save[q][o * save_stride] = make_uint4(w[0], w[1], w[2], w[3]);
    }
  }
  double umin[E];
#pragma unroll
  for (int q = 0; q < E; ++q) umin[q] = R[q][kRowMeta * RS];
  FIN_CHUNKED(KA, b[0], {
    if (k == c_ && c_ > 0) {
      bool poor = true;
#pragma unroll
      for (int q = 0; q < E; ++q) poor &= !(b[q] >= umin[q]);
      if (__all_sync(__activemask(), poor)) goto buys_done_e;
    }
#pragma unroll
    for (int q = 0; q < E; ++q) {
      buy_one_r(b[q], h[q][k], a[q][k], R[q], RS, k + o_, miss[q]);
    }
  })
buys_done_e:
#pragma unroll
  for (int q = 0; q < E; ++q) {
    miss[q] |= !stock_buys_ok(b[q]);
    if (miss[q]) {   // rare
      atomicAdd(e.flags + FIN_CTR_EXACT_REDO, 1u);
#if FIN_REDO_CALL
      b[q] = stock_buys_redo_call<KA>(bpre[q], h[q], a[q], save[q], save_stride, R[q] + kRowU * RS, R[q] + kRowMU * RS);
#else
      b[q] = stock_buys_redo<KA>(bpre[q], h[q], a[q], save[q], save_stride, R[q] + kRowU * RS, R[q] + kRowMU * RS);
#endif
    }
  }
}

// ---------------------------------------------------------------- packed form
// Holdings and clamped actions two assets per 32-bit word (asset 2j in the low half; even K):
// 16-bit SIMD for the integer side of the trade, the float64 operations of stock_trade in the
// same order (bit-identical cash / asset).  Used by K1 (k_stock_step2) and the fused rollout.
__device__ __forceinline__ int half_of(uint32_t w, int s) { return s ? (int)(w >> 16) : (int)(w & 0xffffu); }

// the exact redo of one env's trade (rare: a branch-free buy failed its check): sells and exact
// buys from the pre-step cash and holdings (hold_pre[o * stride]) and the clamped actions a2
template <int KA>
__device__ __forceinline__ double k2_redo_body(const EnvDev& e, double b, const uint4* hold_pre, int stride,
                                               const uint32_t* a2, const double* R, int RS, uint32_t* h2) {
  int h[KA], a[KA];
#pragma unroll
  for (int o = 0; o < (KA + 7) / 8; ++o) {
    const uint4 x = hold_pre[(size_t)o * stride];
    const uint32_t wv[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
    for (int c = 0; c < 8; ++c)
      if (8 * o + c < KA) h[8 * o + c] = half_of(wv[c >> 1], c & 1);
  }
#pragma unroll
  for (int k = 0; k < KA; ++k) a[k] = (k & 1) ? ((int)a2[k >> 1] >> 16) : (int)(int16_t)(a2[k >> 1] & 0xffffu);
  const double* P = R + kRowP * RS;
  const double* U = R + kRowU * RS;
  const double* MU = R + kRowMU * RS;
#pragma unroll
  for (int k = 0; k < KA; ++k) {   // 3. sells (the fast path's operations)
    const int n = max(min(-a[k], h[k]), 0);
    b = fadd64(b, fmul64(nprodx(n, P[k]), e.dn));
    h[k] -= n;
  }
#pragma unroll
  for (int k = 0; k < KA; ++k) {   // 4. exact buys (R5)
    const int want = max(min(a[k], FIN_HOLD_MAX - h[k]), 0);
    double c = nprod(want, U[k], MU[k]);
    int n = want;
    if (!(c <= b)) {
      n = affordable_exact(b, U[k], want);
      c = nprod(n, U[k], MU[k]);
    }
    b = fsub64(b, c);
    h[k] += n;
  }
#pragma unroll
  for (int j = 0; j < KA / 2; ++j) h2[j] = __byte_perm((uint32_t)h[2 * j], (uint32_t)h[2 * j + 1], 0x5410);
  return b;
}
template <int KA>
static __device__ __noinline__ double k2_redo(const EnvDev& e, double b, const uint4* hold_pre, int stride,
                                             const uint32_t* a2, const double* R, int RS, uint32_t* h2) {
  return k2_redo_body<KA>(e, b, hold_pre, stride, a2, R, RS, h2);
}
// packed holdings of env i from / to the asset octets [ceil(K/8)][N] x uint4
template <int KA>
__device__ __forceinline__ void load_hold2(const EnvDev& e, int i, uint32_t (&h2)[KA / 2]) {
  const uint4* q = reinterpret_cast<const uint4*>(e.hold);
#pragma unroll
  for (int o = 0; o < (KA + 7) / 8; ++o) {
    const uint4 x = q[(size_t)o * e.N + i];
    const uint32_t wv[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
    for (int c = 0; c < 4; ++c)
      if (4 * o + c < KA / 2) h2[4 * o + c] = wv[c];
  }
}
template <int KA>
__device__ __forceinline__ uint4 hold_octet(const uint32_t (&h2)[KA / 2], int o) {
  return make_uint4(4 * o < KA / 2 ? h2[4 * o] : 0u, 4 * o + 1 < KA / 2 ? h2[4 * o + 1] : 0u,
                    4 * o + 2 < KA / 2 ? h2[4 * o + 2] : 0u, 4 * o + 3 < KA / 2 ? h2[4 * o + 3] : 0u);
}
template <int KA>
__device__ __forceinline__ void store_hold2(const EnvDev& e, int i, const uint32_t (&h2)[KA / 2]) {
  uint4* q = reinterpret_cast<uint4*>(e.hold);
#pragma unroll
  for (int o = 0; o < (KA + 7) / 8; ++o) q[(size_t)o * e.N + i] = hold_octet<KA>(h2, o);
}

// steps 3-4 for E envs with packed holdings / actions; sets miss[q] when env q needs the redo
template <int KA, int E>
__device__ __forceinline__ void k2_trade(const EnvDev& e, double (&b)[E], uint32_t (&h2)[E][KA / 2],
                                         const uint32_t (&a2)[E][KA / 2], const double* const (&R)[E], int RS,
                                         bool (&miss)[E]) {
  // 3. sells, clipped to holdings: n = relu(min(-a, h)) (-a = ~a + 1 per half), b += fl(fl(n p)(1 - c))
  uint32_t n2[E];
  FIN_CHUNKED(KA, b[0], {
#pragma unroll
    for (int q = 0; q < E; ++q) {
      if ((k & 1) == 0) {
        n2[q] = __vmaxs2(__vmins2(__vneg2(a2[q][k >> 1]), h2[q][k >> 1]), 0u);
        h2[q][k >> 1] -= n2[q];   // no borrow across halves: n <= h per half
      }
#if FIN_MROWS
      b[q] = fadd64(b[q], fmul64(nprod(half_of(n2[q], k & 1), R[q][kRowP * RS + k + o_], R[q][kRowMP * RS + k + o_]),
                                 e.dn));
#else
      b[q] = fadd64(b[q], fmul64(nprodx(half_of(n2[q], k & 1), R[q][kRowP * RS + k + o_]), e.dn));
#endif
    }
  })
  // 4. buys, ascending k (buy_one); a pair's limits before its buys
  uint32_t want2[E];
#pragma unroll
  for (int q = 0; q < E; ++q) miss[q] = false;
  double umin[E];
#pragma unroll
  for (int q = 0; q < E; ++q) umin[q] = R[q][kRowMeta * RS];
  FIN_CHUNKED(KA, b[0], {
    if (k == c_ && c_ > 0) {
      bool poor = true;
#pragma unroll
      for (int q = 0; q < E; ++q) poor &= !(b[q] >= umin[q]);
      if (__all_sync(__activemask(), poor)) goto k2_buys_done;
    }
#pragma unroll
    for (int q = 0; q < E; ++q) {
      if ((k & 1) == 0)
        want2[q] = __vmaxs2(__vmins2(a2[q][k >> 1], __vsub2(0x7fff7fffu, h2[q][k >> 1])), 0u);
#if FIN_MROWS
      const int n = buy_want_m(b[q], half_of(want2[q], k & 1), R[q][kRowU * RS + k + o_], R[q][kRowMU * RS + k + o_],
                               R[q][kRowRU * RS + k + o_], miss[q]);
#else
      const int n = buy_want(b[q], half_of(want2[q], k & 1), R[q][kRowU * RS + k + o_], R[q][kRowRU * RS + k + o_],
                             miss[q]);
#endif
      h2[q][k >> 1] += (k & 1) ? ((uint32_t)n << 16) : (uint32_t)n;
    }
  })
k2_buys_done:
#pragma unroll
  for (int q = 0; q < E; ++q) miss[q] |= !stock_buys_ok(b[q]);
}

template <int KA, int E>
__device__ __forceinline__ void k2_mark(double (&acc)[E], const uint32_t (&h2)[E][KA / 2], const double* const (&PN)[E],
                                        int RS) {
  FIN_CHUNKED(KA, acc[0], {
#pragma unroll
    for (int q = 0; q < E; ++q) {
#if FIN_MROWS   // PN[q] points at row PN; row MPN follows it
      acc[q] = fadd64(acc[q], nprod(half_of(h2[q][k >> 1], k & 1), PN[q][k + o_], PN[q][(kRowMPN - kRowPN) * RS + k + o_]));
#else
      acc[q] = fadd64(acc[q], nprodx(half_of(h2[q][k >> 1], k & 1), PN[q][k + o_]));
#endif
    }
  })
}

// copy the price rows of day d (px[d], kPriceRows x kp doubles) into pr[kPriceRows][kp]
// (threads tid = 0 .. nthr-1 of the staging group)
__device__ __forceinline__ void stage_price_rows(const EnvDev& e, double* pr, int d, int tid, int nthr) {
  const double* src = e.px + (size_t)d * kPriceRows * e.kp;
  for (int j = tid; j < kPriceRows * e.kp; j += nthr) pr[j] = __ldg(src + j);
}

// reward = (v' - v) * scale (exact power-of-two scale), stored fp32
__device__ __forceinline__ float stock_reward(const EnvDev& e, double v, double vn) {
  return (float)fmul64(fsub64(vn, v), e.scale);
}
