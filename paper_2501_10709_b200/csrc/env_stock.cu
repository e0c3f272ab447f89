// env_stock.cu -- stock VecEnv kernels: reset, single step (K1), replay rollout
// (K4), state get/set.  PAPER.md §4.2: reset / step / reward over
// all SubEnvs; the paper vmaps them in PyTorch on an A100, here each is
// one hand-written sm_100a kernel over the SoA state.
//
// K1 / K4 layout of work: one env per thread, 128-thread blocks
// (one window block of envs, so the block normally sits on one market day).
//  * state: coalesced SoA; holdings as 16-byte asset octets (hold_at), kept packed two
//    assets per 32-bit word in registers by the default (even K) kernels k_stock_step2 /
//    k_stock_replay2, which run the 16-bit SIMD / exact-f64 trade of env_stock.cuh k2_trade.
//  * actions [N][K] int16 (caller layout, 60 B per env at K = 30): each warp copies
//    its contiguous rows into shared memory with 16-byte cp.async, one slice / step
//    ahead, then every thread reads its row as 32-bit words (stride K/2 words:
//    conflict-free for odd K/2).
//  * prices: the f64 price-row block of a day (px, fin_internal.cuh) is prefetched per
//    warp for the day predicted from lane 0's env; a warp whose envs sit elsewhere reads
//    the L2-resident table (the padded-K replay k_stock_replay stages per block and day).
//  * arithmetic: exact f64 in the oracle's order, int -> f64 on the fp64 pipe.
// K1 / K4: row values of a whole step's assets in one chunk (ptxas schedules the loads freely;
// A/B at 6 / 8 / 10 / 12 / 15 / 30 assets per chunk: 30 best, K1 +3%, K4 +4% over 6)
#ifndef FIN_KCHUNK
#define FIN_KCHUNK 30
#endif
#include "env_stock.cuh"
#include "group_stage.cuh"
#include "sm100.cuh"

#include <algorithm>

namespace {

constexpr int kThreads = 256;       // reset / get / set
constexpr int kStep = 128;          // K1 / K4 block: 4 warps
constexpr int kBar = 1;             // named barrier of group_apply (0 is __syncthreads)

__device__ __forceinline__ MetricAcc load_metric(const EnvDev& e, int i) {
  MetricAcc m;
  m.v0 = e.m_v0[i]; m.vprev = e.m_vprev[i]; m.peak = e.m_peak[i]; m.mdd = e.m_mdd[i];
  m.mean = e.m_mean[i]; m.m2 = e.m_m2[i]; m.n = e.m_n[i];
  return m;
}
__device__ __forceinline__ void store_metric(const EnvDev& e, int i, const MetricAcc& m) {
  e.m_v0[i] = m.v0; e.m_vprev[i] = m.vprev; e.m_peak[i] = m.peak; e.m_mdd[i] = m.mdd;
  e.m_mean[i] = m.mean; e.m_m2[i] = m.m2; e.m_n[i] = m.n;
}

__global__ void k_stock_reset(EnvDev e, const uint8_t* __restrict__ mask) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= e.N) return;
  if (mask && !mask[i]) return;
  e.cash[i] = e.cash0;
  e.vcur[i] = e.cash0;
  uint4* q = reinterpret_cast<uint4*>(e.hold);
  for (int o = 0; o < (e.K + 7) / 8; ++o) q[(size_t)o * e.N + i] = make_uint4(0u, 0u, 0u, 0u);
  e.t_ep[i] = 0;
  e.window[i] = window_of(e, e.env_offset + i);
  for (int m = 0; m < e.ou_slots; ++m)
    for (int k = 0; k < e.K; ++k) e.ou[((size_t)m * e.K + k) * e.N + i] = 0.f;
  MetricAcc a;
  metric_start(a, e.cash0);
  store_metric(e, i, a);
}

// ------------------------------------------------------------------ K1 / K4 pieces
// KA: compile-time asset count (EXACT: KA == K) or bound (K <= KA, padding zeros).
template <int KA>
struct StepSmem {
  uint4 save[(KA + 7) / 8][kStep];          // per-thread post-sell holdings (exact buy redo)
  alignas(16) double pr[2][kPriceRows * ((KA + 3) / 4 * 4)];   // price rows, [buffer]
  GroupSlots gs;
  uint64_t rows[2];
  int pred[2];
  alignas(16) int16_t act[2][4][32 * KA];   // [buffer][warp] action rows
  // K4: each env's episode-metric and aggregate accumulators between steps ([field][thread]):
  // touched once per step / episode, and out of the registers the trade needs (FIN_K4_ACC_SM)
  double met[6][kStep];
  double agg[FIN_AGG_LEN][kStep];
};
#ifndef FIN_K4_ACC_SM
#define FIN_K4_ACC_SM 1
#endif
template <int KA>
__device__ __forceinline__ void met_put(StepSmem<KA>& sm, int tid, const MetricAcc& m) {
  sm.met[0][tid] = m.v0; sm.met[1][tid] = m.vprev; sm.met[2][tid] = m.peak;
  sm.met[3][tid] = m.mdd; sm.met[4][tid] = m.mean; sm.met[5][tid] = m.m2;
}
__device__ __forceinline__ void met_put_k4(double (*met)[kStep], int tid, const MetricAcc& m) {
  met[0][tid] = m.v0; met[1][tid] = m.vprev; met[2][tid] = m.peak;
  met[3][tid] = m.mdd; met[4][tid] = m.mean; met[5][tid] = m.m2;
}
__device__ __forceinline__ void met_get_k4(const double (*met)[kStep], int tid, MetricAcc& m) {
  m.v0 = met[0][tid]; m.vprev = met[1][tid]; m.peak = met[2][tid];
  m.mdd = met[3][tid]; m.mean = met[4][tid]; m.m2 = met[5][tid];
}
template <int KA>
__device__ __forceinline__ void met_get(const StepSmem<KA>& sm, int tid, MetricAcc& m) {
  m.v0 = sm.met[0][tid]; m.vprev = sm.met[1][tid]; m.peak = sm.met[2][tid];
  m.mdd = sm.met[3][tid]; m.mean = sm.met[4][tid]; m.m2 = sm.met[5][tid];
}

// copy this warp's action rows [n_valid][K] (contiguous in the caller's [N][K]) to shared
__device__ __forceinline__ void slab_load(int16_t* dst, const int16_t* src, int n_valid, int K, int lane, bool vec) {
  const int elems = n_valid * K;
  if (vec) {   // n_valid == 32 and src 16-B aligned: 64 K bytes = 4 K vectors
    for (int j = lane; j < 4 * K; j += 32) sm100::cp_async16(dst + 8 * j, src + 8 * j);
  } else {
    for (int j = lane; j < elems; j += 32) dst[j] = src[j];
  }
  sm100::cp_async_commit();
}

// this thread's action row from shared memory, clamped (R6; sets oor, writes act_out)
template <int KA, bool EXACT>
__device__ __forceinline__ void slab_read(const EnvDev& e, const int16_t* slab, int lane, int K, bool live,
                                          PackedActs<KA>& a, bool& oor, int16_t* act_out) {
  if constexpr (EXACT && (KA % 2 == 0)) {
    const uint32_t* w = reinterpret_cast<const uint32_t*>(slab) + lane * (KA / 2);
    const uint32_t mt2 = (uint32_t)e.max_trade * 0x10001u;
    uint32_t diff = 0;
#pragma unroll
    for (int j = 0; j < KA / 2; ++j) {
      a.w[j] = clamp_pair(live ? w[j] : 0u, mt2, diff);
      if (act_out) reinterpret_cast<uint32_t*>(act_out)[j] = a.w[j];   // K even: 4-B aligned rows
    }
    oor |= diff != 0;
  } else {
    int x[KA];
#pragma unroll
    for (int k = 0; k < KA; ++k) x[k] = (live && k < K) ? (int)slab[lane * K + k] : 0;
    clamp_actions<KA>(e, x, oor, nullptr);
    if (act_out)
      for (int k = 0; k < K; ++k) act_out[k] = (int16_t)x[k];
    a = pack_acts<KA>(x);
  }
}

template <int KA>
__device__ __forceinline__ void write_hold_row(const EnvDev& e, const TrajDev& o, size_t ti, const int (&h)[KA]) {
  if (o.hold) {
#pragma unroll
    for (int k = 0; k < KA; ++k)
      if (k < e.K) o.hold[ti * e.K + k] = (int16_t)h[k];
  }
}

// K1: one step of every env with supplied actions [N][K].
//
// Persistent and software-pipelined: each block walks tiles of 128 envs (stride
// gridDim.x), and each of its 4 warps runs its own pipeline over its 32-env slice of
// those tiles: while the warp steps slice j, its lanes have already issued the 16-byte
// cp.async copies of slice j + gridDim.x's state (cash, asset, clock, window, holdings
// octets) and action rows into the other shared-memory buffer, plus the price-row block
// of the day PREDICTED for that slice (envs step in lockstep and their windows advance
// together, so the next slice's window is this slice's shifted by the difference of
// their initial assignments, R10).  A wrong prediction only sends the warp to the
// L2-resident row table.  No barrier but __syncwarp: no warp ever waits for another.
// Round 2 had one producer thread per block issuing 1-D bulk copies: its warp carried
// ~340 extra instructions per tile (uniform-operand set-up of ten bulk copies, the 64-bit
// divisions of the prediction), and the warps of the other SM sub-partitions waited on
// its refills (ncu: 22% of the warp samples on the full-barrier wait).
// Results go straight from registers to global memory (coalesced stores).
template <int KA>
struct K1Slice {   // one warp's 32 envs of a tile
  double cash[32];
  double v[32];
  int32_t t[32];
  int32_t w[32];
  uint4 hold[(KA + 7) / 8][32];
  alignas(16) int16_t act[32 * KA];
};
#ifndef FIN_K1_LDS
#define FIN_K1_LDS 1   // shared-typed trade path when every env of the warp is on the predicted day
#endif
#ifndef FIN_K1_NBUF
#define FIN_K1_NBUF 2   // slice buffers: NBUF - 1 slices in flight ahead of the one being stepped
#endif
constexpr int kK1Buf = FIN_K1_NBUF;
constexpr int kK1W = kStep / 32;   // warps per K1 block
template <int KA>
struct K1Smem {
  K1Slice<KA> sl[kK1Buf][kK1W];
  uint4 save[(KA + 7) / 8][kStep];   // [octet][thread]: conflict-free 16-B stores
  alignas(16) double pr[kK1Buf][kK1W][kPriceRows * ((KA + 3) / 4 * 4)];
};

// all lanes of a warp: cp.async the slice of 32 envs starting at env i (state + action rows)
template <int KA>
__device__ __forceinline__ void k1_fetch(const EnvDev& e, const int16_t* actions, int K, K1Slice<KA>& S, int i,
                                         int lane) {
  {  // cash | asset: 16 + 16 chunks (the two arrays are adjacent in the slice)
    const double* src = lane < 16 ? e.cash + i + 2 * lane : e.vcur + i + 2 * (lane - 16);
    sm100::cp_async16(S.cash + 2 * lane, src);
  }
  if (lane < 16) {  // clock | window: 8 + 8 chunks
    const int32_t* src = lane < 8 ? e.t_ep + i + 4 * lane : e.window + i + 4 * (lane - 8);
    sm100::cp_async16(S.t + 4 * lane, src);
  }
  const uint4* hq = reinterpret_cast<const uint4*>(e.hold);
#pragma unroll
  for (int o = 0; o < (KA + 7) / 8; ++o)
    if (8 * o < K) sm100::cp_async16(&S.hold[o][lane], hq + (size_t)o * e.N + i + lane);
  const uint4* aq = reinterpret_cast<const uint4*>(actions + (size_t)i * K);   // 32 K int16 = 4 K chunks
  uint4* ad = reinterpret_cast<uint4*>(S.act);
#pragma unroll
  for (int c = 0; c < (4 * KA + 31) / 32; ++c)
    if (32 * c + lane < 4 * K) sm100::cp_async16(ad + 32 * c + lane, aq + 32 * c + lane);
}
// all lanes: cp.async the price-row block of day d (kPriceRows x kp doubles) into pr
__device__ __forceinline__ void k1_fetch_rows(const EnvDev& e, double* pr, int d, int lane) {
  FIN_CHECK(d >= 0 && d + 1 < e.rows);
  const int chunks = kPriceRows * e.kp / 2;
  const double* src = e.px + (size_t)d * kPriceRows * e.kp;
  for (int c = lane; c < chunks; c += 32) sm100::cp_async16(pr + 2 * c, src + 2 * c);
}
__device__ __forceinline__ bool day_ok(const EnvDev& e, int d) { return d >= 0 && d + 1 < e.rows; }

#ifndef FIN_K1_E
#define FIN_K1_E 1      // envs per thread (2 and 4 measured slower, round 1; the per-warp pipelines need 1)
#endif
#ifndef FIN_K1_MINB
#define FIN_K1_MINB 3   // resident K1 blocks per SM (4: 128 registers, measured slower)
#endif
constexpr int kK1Threads = kStep;
template <int KA, bool EXACT>
__global__ void __launch_bounds__(kK1Threads, FIN_K1_MINB)
    k_stock_step(EnvDev e, const int16_t* __restrict__ actions, TrajDev o, int tma_ok) {
  static_assert(FIN_K1_E == 1, "K1's per-warp pipelines step one env per thread");
  extern __shared__ __align__(16) uint8_t k1_smem[];   // dynamic: > 48 KB static limit
  K1Smem<KA>& sm = *reinterpret_cast<K1Smem<KA>*>(k1_smem);
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, r0 = wid * 32;
  const int K = EXACT ? KA : e.K;
  const int n_tiles = (e.N + kStep - 1) / kStep;
  const int n_full = tma_ok ? e.N / kStep : 0;   // tiles served by the cp.async pipeline
  const int RS = EXACT ? (KA + 3) / 4 * 4 : e.kp;   // staged row stride (= kp)
  const int G = gridDim.x;
  // window shift between a slice and the one (NBUF - 1) G tiles later (exact when the window
  // block divides that env distance, R10; otherwise a prediction that may miss)
  const int dW = (int)(((int64_t)kStep * G * (kK1Buf - 1) / e.wblock) % e.W);
  // predicted day of the rows of the slices in flight, oldest first (-1: none; the same in every
  // lane); a shift register, so it stays in registers
  int pred[kK1Buf];
#pragma unroll
  for (int q = 0; q < kK1Buf; ++q) pred[q] = -1;
  // prologue: the warp's slices of the block's first NBUF - 1 tiles, rows of each slice's actual day
#pragma unroll
  for (int q = 0; q + 1 < kK1Buf; ++q) {
    const int jq = blockIdx.x + q * G;
    if (jq < n_tiles) {
      const int i0 = jq * kStep + r0;
      if (jq < n_full) k1_fetch<KA>(e, actions, K, sm.sl[q][wid], i0, lane);
      const int ir = min(i0, e.N - 1);
      const int dq = day_of(e, __ldg(e.window + ir), __ldg(e.t_ep + ir));
      if (day_ok(e, dq)) {
        k1_fetch_rows(e, sm.pr[q][wid], dq, lane);
        pred[q] = dq;
      }
    }
    sm100::cp_async_commit();
  }
  bool oor = false;
  int it = 0;
  for (int j = blockIdx.x; j < n_tiles; j += G, ++it) {
    const int sb = it % kK1Buf;
    const int ps = pred[0];
    const int jn = j + (kK1Buf - 1) * G;           // tile whose slice is fetched this iteration
    const int sn = (it + kK1Buf - 1) % kK1Buf;      // ... into the slot of tile j - G
    const bool tma = j < n_full;
    K1Slice<KA>& S = sm.sl[sb][wid];
    sm100::cp_async_wait<kK1Buf - 2>();            // this lane's copies of slot sb landed
    __syncwarp();                                  // ... and every lane's
    const int r = r0 + lane;   // env row in the tile
    const int i = j * kStep + r;
    const bool live = i < e.N;
    int t = 0, w = 0;
    double b = 0.0, v = 0.0;
    int h[1][KA];
    PackedActs<KA> a[1];
#pragma unroll
    for (int k = 0; k < KA; ++k) h[0][k] = 0;
    if (tma) {
      t = S.t[lane];
      w = S.w[lane];
      b = S.cash[lane];
      v = S.v[lane];
#pragma unroll
      for (int oc = 0; oc < (KA + 7) / 8; ++oc) {
        const uint4 x = S.hold[oc][lane];
        const uint32_t wv[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
        for (int c = 0; c < 8; ++c)
          if (8 * oc + c < KA) h[0][8 * oc + c] = (int)((c & 1) ? (wv[c >> 1] >> 16) : (wv[c >> 1] & 0xffffu));
      }
      slab_read<KA, EXACT>(e, S.act, lane, K, true, a[0], oor, o.actions ? o.actions + (size_t)i * K : nullptr);
    } else if (live) {   // ragged last tile / unaligned actions: direct loads
      t = e.t_ep[i];
      w = e.window[i];
      b = e.cash[i];
      v = e.vcur[i];
      load_hold<KA>(e, i, h[0]);
      int x[KA];
#pragma unroll
      for (int k = 0; k < KA; ++k) x[k] = (k < K) ? (int)actions[(size_t)i * K + k] : 0;
      clamp_actions<KA>(e, x, oor, nullptr);
      if (o.actions)
        for (int k = 0; k < K; ++k) o.actions[(size_t)i * K + k] = (int16_t)x[k];
      a[0] = pack_acts<KA>(x);
    } else {
#pragma unroll
      for (int c = 0; c < (KA + 1) / 2; ++c) a[0].w[c] = 0u;
    }
    const bool stepping = live && t < e.L;
    if (live && !stepping) {  // done env, autoreset = 0: ignored
      set_flag(e, FIN_FLAG_EPISODE_DONE);
      if (o.reward) o.reward[i] = 0.f;
      if (o.done) o.done[i] = 1;
    }
    const int d = day_of(e, w, t);
    FIN_CHECK(!live || (i >= 0 && i < e.N && w >= 0 && w < e.W));
    const bool bad = stepping && (d < 0 || d + 1 >= e.rows);
    if (bad) set_flag(e, FIN_FLAG_BAD_INDEX);
    const bool go = stepping && !bad;
    if (!go) {   // steps with no trade: leaves b and h untouched
#pragma unroll
      for (int c = 0; c < (KA + 1) / 2; ++c) a[0].w[c] = 0u;
    }
    // fetch (all lanes): slice jn's state into the slot of tile j - G (read in the previous
    // iteration, before the __syncwarp above) and the rows of its predicted day -- lane 0's
    // window shifted by dW at lane 0's clock
    {
      const int t0 = __shfl_sync(0xffffffffu, t, 0), w0 = __shfl_sync(0xffffffffu, w, 0);
      int pn = -1;
      if (jn < n_tiles) {
        if (jn < n_full) k1_fetch<KA>(e, actions, K, sm.sl[sn][wid], jn * kStep + r0, lane);
        int wn = w0 + dW;
        if (wn >= e.W) wn -= e.W;
        const int dn = day_of(e, wn, t0);
        if (day_ok(e, dn)) {
          k1_fetch_rows(e, sm.pr[sn][wid], dn, lane);
          pn = dn;
        }
      }
      sm100::cp_async_commit();
#pragma unroll
      for (int q = 0; q + 2 < kK1Buf; ++q) pred[q] = pred[q + 1];
      pred[kK1Buf - 2] = pn;
    }
    const bool staged = !go || d == ps;
    const double* R[1] = {static_cast<const double*>(__builtin_assume_aligned(
        staged ? sm.pr[sb][wid] : e.px + (size_t)d * kPriceRows * e.kp, 16))};
    uint4* sv[1] = {&sm.save[0][tid]};
    double bb[1] = {b}, vn[1];
#if FIN_K1_LDS
    // the normal case (every env of the warp on the predicted day): the rows are addressed
    // from the shared array itself, so they are read with shared loads, not generic ones
    if (__all_sync(0xffffffffu, staged)) {
      const double* Rs[1] = {sm.pr[sb][wid]};
      stock_trade_e<KA, 1>(e, bb, h, Rs, RS, a, sv, kStep);
      vn[0] = bb[0];
      const double* PNs[1] = {sm.pr[sb][wid] + kRowPN * RS};
      stock_mark_e<KA, 1>(vn, h, PNs, RS);
    } else
#endif
    {
      stock_trade_e<KA, 1>(e, bb, h, R, RS, a, sv, kStep);
      vn[0] = bb[0];
      const double* PN[1] = {R[0] + kRowPN * RS};
      stock_mark_e<KA, 1>(vn, h, PN, RS);
    }
    b = bb[0];
    if (go) {
      double vnext = vn[0];
      t += 1;
      const bool done = (t == e.L);
      if (o.reward) o.reward[i] = stock_reward(e, v, vn[0]);
      if (o.done) o.done[i] = done ? 1 : 0;
      if (o.cash) o.cash[i] = b;
      if (o.asset) o.asset[i] = vn[0];
      write_hold_row<KA>(e, o, (size_t)i, h[0]);
      if (done && e.autoreset) {
        b = e.cash0;
        vnext = e.cash0;
#pragma unroll
        for (int k = 0; k < KA; ++k) h[0][k] = 0;
        t = 0;
        if (e.wadv) w = (w + 1) % e.W;
      }
      e.cash[i] = b;
      e.vcur[i] = vnext;
      store_hold<KA>(e, i, h[0]);
      e.t_ep[i] = t;
      if (e.wadv) e.window[i] = w;
    }
  }
  sm100::cp_async_wait<0>();
  if (oor) set_flag(e, FIN_FLAG_ACTION_RANGE);
}

// ---------------------------------------------------------------- K1, packed form (default)
// The same step with holdings / actions kept packed two assets per 32-bit word (asset 2j in
// the low half), for even compile-time K (K = 30, the C1 shape; K = 4):
//  * 16-bit SIMD for the integer side: sells n = relu(min(-a, h)) and h -= n for two assets
//    in three instructions; the buy limit want = relu(min(a, 32767 - h)) of a pair before
//    its buys (an asset's limit depends on its own holding only);
//  * no holdings unpack / repack at load and store, and no post-sell save for the redo (the
//    rare exact redo recomputes the env's whole trade from its pre-step state, still in the
//    slice buffer), so 3 blocks of 4 warps keep 162 registers and 54 KB of shared memory;
//  * E envs per thread (FIN_K2_E; both read the same staged row values).
// Every float64 operation is the one of stock_trade, in the same order, so cash / asset are
// bit-identical.
#ifndef FIN_K1_PACKED
#define FIN_K1_PACKED 1
#endif
#ifndef FIN_K2_E
#define FIN_K2_E 1      // envs per thread of the packed K1 (2: 226 registers, 2 warps per
#endif                  // scheduler, 5% slower despite 19% fewer instructions per env-step)
#ifndef FIN_K2_MINB
#define FIN_K2_MINB 3   // resident blocks per SM (E = 1: 4 forces 128 registers, 7% slower)
#endif
constexpr int kK2E = FIN_K2_E;
constexpr int kK2Threads = kStep / kK2E;
constexpr int kK2W = kK2Threads / 32;
constexpr int kK2Slice = kStep / kK2W;   // 32 E envs per warp slice
template <int KA>
struct K2Slice {
  double cash[kK2Slice];
  double v[kK2Slice];
  int32_t t[kK2Slice];
  int32_t w[kK2Slice];
  uint4 hold[(KA + 7) / 8][kK2Slice];
  alignas(16) int16_t act[kK2Slice * KA];
};
template <int KA>
struct K2Smem {
  K2Slice<KA> sl[kK1Buf][kK2W];
  alignas(16) double pr[kK1Buf][kK2W][kPriceRows * ((KA + 3) / 4 * 4)];
};
template <int KA>
__device__ __forceinline__ void k2_fetch(const EnvDev& e, const int16_t* actions, K2Slice<KA>& S, int i, int lane) {
  FIN_CHECK(i >= 0 && i + kK2Slice <= e.N && (i & 1) == 0);   // whole slices of full tiles, 16-B aligned
  constexpr int NS = kK2Slice, H = NS / 2;   // cash | asset: NS / 2 + NS / 2 chunks
#pragma unroll
  for (int c = 0; c < kK2E; ++c) {
    const int x = 32 * c + lane;
    const double* src = x < H ? e.cash + i + 2 * x : e.vcur + i + 2 * (x - H);
    sm100::cp_async16(S.cash + 2 * x, src);
  }
  if (lane < NS / 2) {  // clock | window: NS / 4 + NS / 4 chunks
    const int32_t* src = lane < NS / 4 ? e.t_ep + i + 4 * lane : e.window + i + 4 * (lane - NS / 4);
    sm100::cp_async16(S.t + 4 * lane, src);
  }
  const uint4* hq = reinterpret_cast<const uint4*>(e.hold);
#pragma unroll
  for (int o = 0; o < (KA + 7) / 8; ++o) {
#pragma unroll
    for (int c = 0; c < kK2E; ++c)
      sm100::cp_async16(&S.hold[o][lane + 32 * c], hq + (size_t)o * e.N + i + lane + 32 * c);
  }
  const uint4* aq = reinterpret_cast<const uint4*>(actions + (size_t)i * KA);   // NS KA int16 = NS KA / 8 chunks
  uint4* ad = reinterpret_cast<uint4*>(S.act);
#pragma unroll
  for (int c = 0; c < (NS * KA / 8 + 31) / 32; ++c)
    if (32 * c + lane < NS * KA / 8) sm100::cp_async16(ad + 32 * c + lane, aq + 32 * c + lane);
}

template <int KA>
__global__ void __launch_bounds__(kK2Threads, FIN_K2_MINB)
    k_stock_step2(EnvDev e, const int16_t* __restrict__ actions, TrajDev o, int tma_ok) {
  constexpr int E = kK2E, KP = KA / 2;
  static_assert(KA % 2 == 0, "packed K1: even K");
  extern __shared__ __align__(16) uint8_t k2_smem[];
  K2Smem<KA>& sm = *reinterpret_cast<K2Smem<KA>*>(k2_smem);
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, r0 = wid * kK2Slice;
  const int n_tiles = (e.N + kStep - 1) / kStep;
  const int n_full = tma_ok ? e.N / kStep : 0;
  constexpr int RS = (KA + 3) / 4 * 4;
  const int G = gridDim.x;
  const int dW = (int)(((int64_t)kStep * G * (kK1Buf - 1) / e.wblock) % e.W);
  const uint32_t mt2 = (uint32_t)e.max_trade * 0x10001u;
  int pred[kK1Buf];
#pragma unroll
  for (int q = 0; q < kK1Buf; ++q) pred[q] = -1;
#pragma unroll
  for (int q = 0; q + 1 < kK1Buf; ++q) {
    const int jq = blockIdx.x + q * G;
    if (jq < n_tiles) {
      const int i0 = jq * kStep + r0;
      if (jq < n_full) k2_fetch<KA>(e, actions, sm.sl[q][wid], i0, lane);
      const int ir = min(i0, e.N - 1);
      const int dq = day_of(e, __ldg(e.window + ir), __ldg(e.t_ep + ir));
      if (day_ok(e, dq)) {
        k1_fetch_rows(e, sm.pr[q][wid], dq, lane);
        pred[q] = dq;
      }
    }
    sm100::cp_async_commit();
  }
  bool oor = false;
  int it = 0;
  for (int j = blockIdx.x; j < n_tiles; j += G, ++it) {
    const int sb = it % kK1Buf;
    const int ps = pred[0];
    const int jn = j + (kK1Buf - 1) * G;
    const int sn = (it + kK1Buf - 1) % kK1Buf;
    const bool tma = j < n_full;
    K2Slice<KA>& S = sm.sl[sb][wid];
    sm100::cp_async_wait<kK1Buf - 2>();
    __syncwarp();
    int t[E], w[E], d[E], idx[E], gi[E];
    bool live[E], go[E];
    double b[E], v[E];
    uint32_t h2[E][KP], a2[E][KP];
    uint32_t diff = 0;
#pragma unroll
    for (int q = 0; q < E; ++q) {
      idx[q] = lane + 32 * q;              // env row in the warp's slice
      gi[q] = j * kStep + r0 + idx[q];
      live[q] = gi[q] < e.N;
      t[q] = 0; w[q] = 0; b[q] = 0.0; v[q] = 0.0;
#pragma unroll
      for (int c = 0; c < KP; ++c) { h2[q][c] = 0u; a2[q][c] = 0u; }
      if (tma) {
        t[q] = S.t[idx[q]];
        w[q] = S.w[idx[q]];
        b[q] = S.cash[idx[q]];
        v[q] = S.v[idx[q]];
#pragma unroll
        for (int oc = 0; oc < (KA + 7) / 8; ++oc) {
          const uint4 x = S.hold[oc][idx[q]];
          const uint32_t wv[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
          for (int c = 0; c < 4; ++c)
            if (4 * oc + c < KP) h2[q][4 * oc + c] = wv[c];
        }
        const uint32_t* aw = reinterpret_cast<const uint32_t*>(S.act) + idx[q] * KP;
#pragma unroll
        for (int c = 0; c < KP; ++c) a2[q][c] = aw[c];
      } else if (live[q]) {   // ragged last tile / unaligned actions: direct loads
        const int i = gi[q];
        t[q] = e.t_ep[i];
        w[q] = e.window[i];
        b[q] = e.cash[i];
        v[q] = e.vcur[i];
        const uint4* hq = reinterpret_cast<const uint4*>(e.hold);
#pragma unroll
        for (int oc = 0; oc < (KA + 7) / 8; ++oc) {
          const uint4 x = hq[(size_t)oc * e.N + i];
          const uint32_t wv[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
          for (int c = 0; c < 4; ++c)
            if (4 * oc + c < KP) h2[q][4 * oc + c] = wv[c];
        }
#pragma unroll
        for (int c = 0; c < KP; ++c)
          a2[q][c] = __byte_perm((uint32_t)(uint16_t)actions[(size_t)i * KA + 2 * c],
                                 (uint32_t)(uint16_t)actions[(size_t)i * KA + 2 * c + 1], 0x5410);
      }
      // 2. clamp (R6), two assets per instruction
#pragma unroll
      for (int c = 0; c < KP; ++c) a2[q][c] = clamp_pair(a2[q][c], mt2, diff);
      if (o.actions && live[q]) {
#pragma unroll
        for (int c = 0; c < KP; ++c) reinterpret_cast<uint32_t*>(o.actions + (size_t)gi[q] * KA)[c] = a2[q][c];
      }
      const bool stepping = live[q] && t[q] < e.L;
      if (live[q] && !stepping) {  // done env, autoreset = 0: ignored
        set_flag(e, FIN_FLAG_EPISODE_DONE);
        if (o.reward) o.reward[gi[q]] = 0.f;
        if (o.done) o.done[gi[q]] = 1;
      }
      d[q] = day_of(e, w[q], t[q]);
      FIN_CHECK(!live[q] || (gi[q] >= 0 && gi[q] < e.N && w[q] >= 0 && w[q] < e.W && t[q] >= 0));
      FIN_CHECK(!tma || (idx[q] >= 0 && idx[q] < kK2Slice && gi[q] < e.N));
      const bool bad = stepping && (d[q] < 0 || d[q] + 1 >= e.rows);
      if (bad) set_flag(e, FIN_FLAG_BAD_INDEX);
      go[q] = stepping && !bad;
      if (!go[q]) {
#pragma unroll
        for (int c = 0; c < KP; ++c) a2[q][c] = 0u;
      }
    }
    oor |= diff != 0;
    {  // fetch slice jn and the rows of its predicted day (see k_stock_step)
      const int t0 = __shfl_sync(0xffffffffu, t[0], 0), w0 = __shfl_sync(0xffffffffu, w[0], 0);
      int pn = -1;
      if (jn < n_tiles) {
        if (jn < n_full) k2_fetch<KA>(e, actions, sm.sl[sn][wid], jn * kStep + r0, lane);
        int wn = w0 + dW;
        if (wn >= e.W) wn -= e.W;
        const int dn = day_of(e, wn, t0);
        if (day_ok(e, dn)) {
          k1_fetch_rows(e, sm.pr[sn][wid], dn, lane);
          pn = dn;
        }
      }
      sm100::cp_async_commit();
#pragma unroll
      for (int q = 0; q + 2 < kK1Buf; ++q) pred[q] = pred[q + 1];
      pred[kK1Buf - 2] = pn;
    }
    bool staged = true;
    const double* R[E];
#pragma unroll
    for (int q = 0; q < E; ++q) {
      const bool st = !go[q] || d[q] == ps;
      staged &= st;
      R[q] = static_cast<const double*>(__builtin_assume_aligned(
          st ? sm.pr[sb][wid] : e.px + (size_t)d[q] * kPriceRows * e.kp, 16));
    }
    double bb[E], vn[E];
    bool miss[E];
#pragma unroll
    for (int q = 0; q < E; ++q) bb[q] = b[q];
    if (__all_sync(0xffffffffu, staged)) {   // shared-typed row reads
      const double* Rs[E];
      const double* PNs[E];
#pragma unroll
      for (int q = 0; q < E; ++q) Rs[q] = sm.pr[sb][wid];
      k2_trade<KA, E>(e, bb, h2, a2, Rs, RS, miss);
#pragma unroll
      for (int q = 0; q < E; ++q) { vn[q] = bb[q]; PNs[q] = sm.pr[sb][wid] + kRowPN * RS; }
      k2_mark<KA, E>(vn, h2, PNs, RS);
    } else {
      k2_trade<KA, E>(e, bb, h2, a2, R, RS, miss);
      const double* PN[E];
#pragma unroll
      for (int q = 0; q < E; ++q) { vn[q] = bb[q]; PN[q] = R[q] + kRowPN * RS; }
      k2_mark<KA, E>(vn, h2, PN, RS);
    }
#pragma unroll
    for (int q = 0; q < E; ++q) {
      if (miss[q]) {   // rare: redo env q's trade exactly from its pre-step state
        atomicAdd(e.flags + FIN_CTR_EXACT_REDO, 1u);
        const uint4* hp = tma ? &S.hold[0][idx[q]] : reinterpret_cast<const uint4*>(e.hold) + gi[q];
        uint32_t ac[KP];
#pragma unroll
        for (int c = 0; c < KP; ++c) ac[c] = a2[q][c];
        uint32_t hn[KP];
        bb[q] = k2_redo<KA>(e, b[q], hp, tma ? kK2Slice : e.N, ac, R[q], RS, hn);
#pragma unroll
        for (int c = 0; c < KP; ++c) h2[q][c] = hn[c];
        vn[q] = bb[q];
        const double* PNq[1] = {R[q] + kRowPN * RS};
        double acc[1] = {bb[q]};
        uint32_t hq1[1][KP];
#pragma unroll
        for (int c = 0; c < KP; ++c) hq1[0][c] = hn[c];
        k2_mark<KA, 1>(acc, hq1, PNq, RS);
        vn[q] = acc[0];
      }
    }
#pragma unroll
    for (int q = 0; q < E; ++q) {
      if (!go[q]) continue;
      const int i = gi[q];
      double bq = bb[q], vnext = vn[q];
      int tq = t[q] + 1, wq = w[q];
      const bool done = (tq == e.L);
      if (o.reward) o.reward[i] = stock_reward(e, v[q], vn[q]);
      if (o.done) o.done[i] = done ? 1 : 0;
      if (o.cash) o.cash[i] = bq;
      if (o.asset) o.asset[i] = vn[q];
      if (o.hold) {
#pragma unroll
        for (int c = 0; c < KP; ++c) reinterpret_cast<uint32_t*>(o.hold + (size_t)i * KA)[c] = h2[q][c];
      }
      uint32_t hs[KP];
#pragma unroll
      for (int c = 0; c < KP; ++c) hs[c] = h2[q][c];
      if (done && e.autoreset) {
        bq = e.cash0;
        vnext = e.cash0;
#pragma unroll
        for (int c = 0; c < KP; ++c) hs[c] = 0u;
        tq = 0;
        if (e.wadv) wq = (wq + 1) % e.W;
      }
      e.cash[i] = bq;
      e.vcur[i] = vnext;
      uint4* hq = reinterpret_cast<uint4*>(e.hold);
#pragma unroll
      for (int oc = 0; oc < (KA + 7) / 8; ++oc) {
        const uint32_t w0_ = 4 * oc < KP ? hs[4 * oc] : 0u, w1_ = 4 * oc + 1 < KP ? hs[4 * oc + 1] : 0u;
        const uint32_t w2_ = 4 * oc + 2 < KP ? hs[4 * oc + 2] : 0u, w3_ = 4 * oc + 3 < KP ? hs[4 * oc + 3] : 0u;
        hq[(size_t)oc * e.N + i] = make_uint4(w0_, w1_, w2_, w3_);
      }
      e.t_ep[i] = tq;
      if (e.wadv) e.window[i] = wq;
    }
  }
  sm100::cp_async_wait<0>();
  if (oor) set_flag(e, FIN_FLAG_ACTION_RANGE);
}

// thread 0: publish the prediction, then bulk-copy the price rows of day d into pr
// (completing on bar); with no usable prediction the barrier phase completes at once (K4)
__device__ __forceinline__ void rows_issue(const EnvDev& e, double* pr, uint64_t* bar, int* pred, int d) {
  if (d >= 0 && d + 1 < e.rows) {
    *pred = d;
    const uint32_t bytes = kPriceRows * e.kp * 8;
    sm100::mbar_arrive_expect_tx(bar, bytes);
    sm100::bulk_g2s(pr, e.px + (size_t)d * kPriceRows * e.kp, bytes, bar);
  } else {
    *pred = -1;
    sm100::mbar_arrive(bar);
  }
}

// K4: T steps with supplied actions [T][N][K]; the env state (cash, holdings,
// episode clock, window, metric accumulators) lives in registers for all T, and the
// pre-trade asset v of a step is the previous step's post-trade asset v' (the same
// sum over the same holdings and prices), or b0 after a reset.
#ifndef FIN_K4_MINB
#define FIN_K4_MINB 3   // measured best of 2, 3, 4 (scripts/k4_sweep.sh)
#endif
template <int KA, bool EXACT>
__global__ void __launch_bounds__(kStep, FIN_K4_MINB) k_stock_replay(EnvDev e, const int16_t* __restrict__ actions, int T,
                                                        TrajDev o, int vec_ok) {
  __shared__ StepSmem<KA> sm;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int i = blockIdx.x * kStep + tid;
  const bool live = i < e.N;
  const int K = EXACT ? KA : e.K, N = e.N;
  AggAcc agg;
  agg_init(agg);
  int t = 0, w = 0;
  double b = 0.0;
  int h[KA];
#pragma unroll
  for (int k = 0; k < KA; ++k) h[k] = 0;
  MetricAcc m;
  metric_start(m, 0.0);
  double vc = 0.0;   // pre-trade asset of the next step (the cached v, then each post-trade v)
  if (live) {
    t = e.t_ep[i];
    w = e.window[i];
    b = e.cash[i];
    vc = e.vcur[i];
    load_hold<KA>(e, i, h);
    m = load_metric(e, i);
  }
  if (FIN_K4_ACC_SM) {
    met_put(sm, tid, m);
#pragma unroll
    for (int j = 0; j < FIN_AGG_LEN; ++j) sm.agg[j][tid] = agg.s[j];
  }
  const int i0 = blockIdx.x * kStep + wid * 32;
  const int nv = max(0, min(32, N - i0));
  const bool vec = vec_ok && nv == 32;
  if (nv > 0) slab_load(sm.act[0][wid], actions + (size_t)i0 * K, nv, K, lane, vec);
  const int RS = EXACT ? (KA + 3) / 4 * 4 : e.kp;   // staged row stride (= kp)
  if (tid == 0) {
    sm100::mbar_init(&sm.rows[0], 1);
    sm100::mbar_init(&sm.rows[1], 1);
    sm100::fence_mbar_init();
  }
  gs_init(&sm.gs, tid, kBar);
  __syncthreads();
  if (tid == 0) rows_issue(e, sm.pr[0], &sm.rows[0], &sm.pred[0], day_of(e, w, t));   // thread 0 is live
  __syncthreads();
  uint32_t rphase = 0;
  int cnt = 0, round = 0;
  double rsum = 0.0;
  bool oor = false, bad = false;
  for (int s = 0; s < T; ++s) {
    if (s + 1 < T && nv > 0)
      slab_load(sm.act[(s + 1) & 1][wid], actions + ((size_t)(s + 1) * N + i0) * K, nv, K, lane, vec);
    if (s + 1 < T && nv > 0) sm100::cp_async_wait<1>();
    else sm100::cp_async_wait<0>();
    __syncwarp();
    PackedActs<KA> a;
    const size_t ti = (size_t)s * N + i;
    FIN_CHECK(s >= 0 && s < T && (!live || i < N));
    slab_read<KA, EXACT>(e, sm.act[s & 1][wid], lane, K, live, a, oor,
                         (o.actions && live) ? o.actions + ti * K : nullptr);
    const bool stepping = live && !bad && t < e.L;
    if (live && !bad && !stepping) {
      set_flag(e, FIN_FLAG_EPISODE_DONE);
      if (o.reward) o.reward[ti] = 0.f;
      if (o.done) o.done[ti] = 1;
    }
    const int d = day_of(e, w, t);
    if (stepping && (d < 0 || d + 1 >= e.rows)) bad = true;
    const int sb = s & 1;
    // rows of step s+1, predicted from thread 0's env (lockstep): the next day, or the
    // first day of its (possibly advanced) window after a reset
    if (tid == 0 && s + 1 < T) {
      const int w1 = (e.wadv && t + 1 >= e.L) ? (w + 1) % e.W : w;
      rows_issue(e, sm.pr[sb ^ 1], &sm.rows[sb ^ 1], &sm.pred[sb ^ 1],
                 t + 1 < e.L ? d + 1 : (e.autoreset ? day_of(e, w1, 0) : -1));
    }
    double* pr = sm.pr[sb];
    sm100::mbar_wait(&sm.rows[sb], (rphase >> sb) & 1u);   // rows landed (or no prediction)
    rphase ^= 1u << sb;
    if (tid == 0) sm.gs.staged = sm.pred[sb];
    group_apply(
        &sm.gs, round, d, stepping && !bad, tid, kBar, [&](int dd) { stage_price_rows(e, pr, dd, tid, kStep); },
        [&]() {
          const double v = vc;
          stock_trade<KA>(e, b, h, pr, RS, a, &sm.save[0][tid], kStep);
          const double vn = stock_mark<KA>(b, h, pr + kRowPN * RS, RS);
          vc = vn;
          t += 1;
          const bool done = (t == e.L);
          const float r = stock_reward(e, v, vn);
          rsum += (double)r;
          if (o.reward) o.reward[ti] = r;
          if (o.done) o.done[ti] = done ? 1 : 0;
          if (o.cash) o.cash[ti] = b;
          if (o.asset) o.asset[ti] = vn;
          write_hold_row<KA>(e, o, ti, h);
          if (FIN_K4_ACC_SM) met_get(sm, tid, m);
          metric_push(m, vn);
          if (done) {
            double em[3];
            metric_finish(m, 252.0, 0.0, em);
            if (o.ep_metrics && cnt < o.ep_capacity) {
              double* dst = o.ep_metrics + ((size_t)cnt * N + i) * 3;
              dst[0] = em[0]; dst[1] = em[1]; dst[2] = em[2];
            }
            ++cnt;
            if (FIN_K4_ACC_SM) {
              AggAcc ag;
#pragma unroll
              for (int j = 0; j < FIN_AGG_LEN; ++j) ag.s[j] = sm.agg[j][tid];
              agg_episode(ag, em);
#pragma unroll
              for (int j = 0; j < FIN_AGG_LEN; ++j) sm.agg[j][tid] = ag.s[j];
            } else {
              agg_episode(agg, em);
            }
            if (e.autoreset) {
              b = e.cash0;
#pragma unroll
              for (int k = 0; k < KA; ++k) h[k] = 0;
              t = 0;
              vc = e.cash0;
              if (e.wadv) w = (w + 1) % e.W;
              metric_start(m, e.cash0);
            }
          }
          if (FIN_K4_ACC_SM) met_put(sm, tid, m);
        });
  }
  if (FIN_K4_ACC_SM) {
    met_get(sm, tid, m);
#pragma unroll
    for (int j = 0; j < FIN_AGG_LEN; ++j) agg.s[j] = sm.agg[j][tid];
  }
  if (live) {
    if (oor) set_flag(e, FIN_FLAG_ACTION_RANGE);
    if (bad) set_flag(e, FIN_FLAG_BAD_INDEX);
    e.cash[i] = b;
    e.vcur[i] = vc;
    store_hold<KA>(e, i, h);
    e.t_ep[i] = t;
    e.window[i] = w;
    store_metric(e, i, m);
    if (o.ep_count) o.ep_count[i] = cnt;
  }
  agg.s[FIN_AGG_SUM_REWARD] = rsum;
  if (o.agg_partial) agg_block_write(agg, o.agg_partial + (size_t)blockIdx.x * FIN_AGG_LEN);
}

// asset (v = b + sum h p at the env's current day) through the same f64 table
__device__ __forceinline__ double asset_now(const EnvDev& e, int i) {
  int d = day_of(e, e.window[i], e.t_ep[i]);
  if (d >= e.rows) d = e.rows - 1;
  const double* p = e.px + (size_t)d * kPriceRows * e.kp + kRowP * e.kp;
  double v = e.cash[i];
  for (int k = 0; k < e.K; ++k) v = fadd64(v, fmul64(nn2d(e.hold[hold_at(e.N, k, i)]), p[k]));
  return v;
}

__global__ void k_stock_get_state(EnvDev e, double* cash, int16_t* hold, double* asset, int32_t* t_ep,
                                  int32_t* window) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= e.N) return;
  const int K = e.K;
  if (cash) cash[i] = e.cash[i];
  if (t_ep) t_ep[i] = e.t_ep[i];
  if (window) window[i] = e.window[i];
  if (hold)
    for (int k = 0; k < K; ++k) hold[(size_t)i * K + k] = e.hold[hold_at(e.N, k, i)];
  if (asset) asset[i] = asset_now(e, i);
}

__global__ void k_stock_set_state(EnvDev e, const double* cash, const int16_t* hold, const int32_t* t_ep,
                                  const int32_t* window) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= e.N) return;
  const int K = e.K;
  if (cash) e.cash[i] = cash[i];
  if (hold)
    for (int k = 0; k < K; ++k) e.hold[hold_at(e.N, k, i)] = hold[(size_t)i * K + k];
  if (t_ep) e.t_ep[i] = t_ep[i];
  if (window) e.window[i] = window[i];
  // cached asset and online metrics restart at the current equity
  const double v = asset_now(e, i);
  e.vcur[i] = v;
  MetricAcc m;
  metric_start(m, v);
  store_metric(e, i, m);
}

// One warp per aggregate component: lanes stride over the partial rows, then a fixed
// shuffle tree (deterministic order) -- the serial per-component loop cost ~36 us per
// rollout (512 partial rows of dependent-chain loads).
__global__ void k_agg_finalize(const double* __restrict__ partial, int n_blocks, double* agg) {
  const int j = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (j >= FIN_AGG_LEN) return;
  const bool sum = j < FIN_AGG_NSUM;
  double s = sum ? 0.0 : __longlong_as_double(0x7ff0000000000000ULL);
  for (int b = lane; b < n_blocks; b += 32) {
    const double x = __ldg(partial + (size_t)b * FIN_AGG_LEN + j);
    s = sum ? s + x : fmin(s, x);
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    const double o = __shfl_down_sync(0xffffffffu, s, off);
    s = sum ? s + o : fmin(s, o);
  }
  if (lane == 0) agg[j] = s;
}

inline int blocks_for(int n, int threads = kThreads) { return (n + threads - 1) / threads; }

// 16-byte cp.async of whole action rows needs a 16-B aligned base and, for the
// per-step slabs of K4, a 16-B multiple per step (N K int16)
inline int vec_ok(const void* p, long long elems_per_step) {
  return ((reinterpret_cast<uintptr_t>(p) & 15u) == 0 && (elems_per_step % 8) == 0) ? 1 : 0;
}

}  // namespace

namespace fin {

int num_sms();

// K = 30 (C1) and K = 4 (C0) are compiled exactly; any other K runs in the next
// power-of-two bound with zero padding.
// K4, packed form (default for even K): the replay with K1's round-2 structure -- holdings and
// actions two assets per word (k2_trade), each warp prefetching its own next step (action slab
// + the rows of the day predicted from lane 0's env) with cp.async, no block barrier (round 2's
// K4 staged the rows once per block and day behind a named barrier, thread 0 issuing them).
#ifndef FIN_K4_PACKED
#define FIN_K4_PACKED 1
#endif
template <int KA>
struct K4Smem {
  alignas(16) int16_t act[2][4][32 * KA];
  alignas(16) double pr[2][4][kPriceRows * ((KA + 3) / 4 * 4)];
  uint4 save[(KA + 7) / 8][kStep];   // pre-step holdings of the rare exact redo
  double met[6][kStep];
  double agg[FIN_AGG_LEN][kStep];
};
template <int KA>
__global__ void __launch_bounds__(kStep, FIN_K4_MINB) k_stock_replay2(EnvDev e, const int16_t* __restrict__ actions,
                                                                     int T, TrajDev o, int vec_ok) {
  constexpr int KP = KA / 2;
  constexpr int RS = (KA + 3) / 4 * 4;
  static_assert(KA % 2 == 0, "packed K4: even K");
  extern __shared__ __align__(16) uint8_t k4_smem[];   // dynamic: > 48 KB static limit
  K4Smem<KA>& sm = *reinterpret_cast<K4Smem<KA>*>(k4_smem);
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int i = blockIdx.x * kStep + tid;
  const bool live = i < e.N;
  const int N = e.N;
  int t = 0, w = 0, mn = 0;
  double b = 0.0, vc = 0.0;
  uint32_t h2[KP];
#pragma unroll
  for (int c = 0; c < KP; ++c) h2[c] = 0u;
  {
    MetricAcc m;
    metric_start(m, 0.0);
    if (live) {
      t = e.t_ep[i];
      w = e.window[i];
      b = e.cash[i];
      vc = e.vcur[i];
      load_hold2<KA>(e, i, h2);
      m = load_metric(e, i);
    }
    met_put_k4(sm.met, tid, m);
    mn = m.n;
#pragma unroll
    for (int j = 0; j < FIN_AGG_LEN; ++j) sm.agg[j][tid] = 0.0;
    AggAcc a0;
    agg_init(a0);
#pragma unroll
    for (int j = 0; j < FIN_AGG_LEN; ++j) sm.agg[j][tid] = a0.s[j];
  }
  const int i0 = blockIdx.x * kStep + wid * 32;
  const int nv = max(0, min(32, N - i0));
  const bool vec = vec_ok && nv == 32;
  const uint32_t mt2 = (uint32_t)e.max_trade * 0x10001u;
  // fetch (all lanes, one cp.async group): step s's action slab of this warp + the rows of day ds
  auto fetch = [&](int s, int ds) {
    FIN_CHECK(s >= 0 && s < T && (nv == 0 || i0 + nv <= N));
    if (nv > 0) {
      const int16_t* src = actions + ((size_t)s * N + i0) * KA;
      int16_t* dst = sm.act[s & 1][wid];
      if (vec) {
        for (int j = lane; j < 4 * KA; j += 32) sm100::cp_async16(dst + 8 * j, src + 8 * j);
      } else {
        for (int j = lane; j < nv * KA; j += 32) dst[j] = src[j];
      }
    }
    if (day_ok(e, ds)) k1_fetch_rows(e, sm.pr[s & 1][wid], ds, lane);
    sm100::cp_async_commit();
  };
  int pred_cur;
  {
    const int t0 = __shfl_sync(0xffffffffu, t, 0), w0 = __shfl_sync(0xffffffffu, w, 0);
    const int d0 = day_of(e, w0, t0);
    pred_cur = day_ok(e, d0) ? d0 : -1;
    fetch(0, pred_cur);
  }
  int cnt = 0;
  double rsum = 0.0;
  bool oor = false, bad = false;
  for (int s = 0; s < T; ++s) {
    const size_t ti = (size_t)s * N + i;
    const int d = day_of(e, w, t);
    const bool stepping = live && !bad && t < e.L;
    FIN_CHECK(!live || (i < N && w >= 0 && w < e.W && t >= 0 && t <= e.L));
    // prefetch step s+1: its slab and the rows of lane 0's next day (d + 1, or the first day of
    // its (possibly advanced) window after a reset)
    int pred_next = -1;
    if (s + 1 < T) {
      const int t0 = __shfl_sync(0xffffffffu, t, 0), w0 = __shfl_sync(0xffffffffu, w, 0);
      const int d0 = __shfl_sync(0xffffffffu, d, 0);
      const int w1 = (e.wadv && t0 + 1 >= e.L) ? (w0 + 1) % e.W : w0;
      const int dn = t0 + 1 < e.L ? d0 + 1 : (e.autoreset ? day_of(e, w1, 0) : -1);
      pred_next = day_ok(e, dn) ? dn : -1;
      fetch(s + 1, pred_next);
      sm100::cp_async_wait<1>();
    } else {
      sm100::cp_async_wait<0>();
    }
    __syncwarp();
    uint32_t a2[1][KP];
    uint32_t diff = 0;
    {
      const uint32_t* aw = reinterpret_cast<const uint32_t*>(sm.act[s & 1][wid]) + lane * KP;
#pragma unroll
      for (int c = 0; c < KP; ++c) a2[0][c] = clamp_pair(live ? aw[c] : 0u, mt2, diff);
    }
    oor |= diff != 0;
    if (o.actions && live) {
#pragma unroll
      for (int c = 0; c < KP; ++c) reinterpret_cast<uint32_t*>(o.actions + ti * KA)[c] = a2[0][c];
    }
    if (live && !bad && !stepping) {
      set_flag(e, FIN_FLAG_EPISODE_DONE);
      if (o.reward) o.reward[ti] = 0.f;
      if (o.done) o.done[ti] = 1;
    }
    if (stepping && !day_ok(e, d)) bad = true;
    const bool go = stepping && !bad;
    if (!go) {
#pragma unroll
      for (int c = 0; c < KP; ++c) a2[0][c] = 0u;
    }
    const bool st_ok = !go || d == pred_cur;
    const double* R1[1] = {static_cast<const double*>(__builtin_assume_aligned(
        st_ok ? sm.pr[s & 1][wid] : e.px + (size_t)(go ? d : 0) * kPriceRows * e.kp, 16))};
    const MetricRcp mr = metric_rcps(sm.met[1][tid], sm.met[2][tid], mn);
#pragma unroll
    for (int oc = 0; oc < (KA + 7) / 8; ++oc) sm.save[oc][tid] = hold_octet<KA>(h2, oc);
    double bb[1] = {b};
    uint32_t hh[1][KP];
#pragma unroll
    for (int c = 0; c < KP; ++c) hh[0][c] = h2[c];
    bool miss[1];
    if (__all_sync(0xffffffffu, st_ok)) {
      const double* Rs[1] = {sm.pr[s & 1][wid]};
      k2_trade<KA, 1>(e, bb, hh, a2, Rs, RS, miss);
    } else {
      k2_trade<KA, 1>(e, bb, hh, a2, R1, RS, miss);
    }
    if (miss[0]) {   // rare: the exact trade from the pre-step state
      atomicAdd(e.flags + FIN_CTR_EXACT_REDO, 1u);
      uint32_t ac[KP];
#pragma unroll
      for (int c = 0; c < KP; ++c) ac[c] = a2[0][c];
      bb[0] = k2_redo<KA>(e, b, &sm.save[0][tid], kStep, ac, R1[0], RS, hh[0]);
    }
    pred_cur = pred_next;
    if (go) {
      const double v = vc;
      b = bb[0];
#pragma unroll
      for (int c = 0; c < KP; ++c) h2[c] = hh[0][c];
      double acc[1] = {b};
      const double* PN1[1] = {R1[0] + kRowPN * RS};
      k2_mark<KA, 1>(acc, hh, PN1, RS);
      const double vn = acc[0];
      vc = vn;
      t += 1;
      const bool done = (t == e.L);
      const float r = stock_reward(e, v, vn);
      rsum += (double)r;
      if (o.reward) o.reward[ti] = r;
      if (o.done) o.done[ti] = done ? 1 : 0;
      if (o.cash) o.cash[ti] = b;
      if (o.asset) o.asset[ti] = vn;
      if (o.hold) {
#pragma unroll
        for (int c = 0; c < KP; ++c) reinterpret_cast<uint32_t*>(o.hold + ti * KA)[c] = h2[c];
      }
      MetricAcc m;
      met_get_k4(sm.met, tid, m);
      m.n = mn;
      metric_push_pre(m, vn, mr);
      if (done) {
        double em[3];
        metric_finish(m, 252.0, 0.0, em);
        if (o.ep_metrics && cnt < o.ep_capacity) {
          double* dst = o.ep_metrics + ((size_t)cnt * N + i) * 3;
          dst[0] = em[0]; dst[1] = em[1]; dst[2] = em[2];
        }
        ++cnt;
        AggAcc ag;
#pragma unroll
        for (int j = 0; j < FIN_AGG_LEN; ++j) ag.s[j] = sm.agg[j][tid];
        agg_episode(ag, em);
#pragma unroll
        for (int j = 0; j < FIN_AGG_LEN; ++j) sm.agg[j][tid] = ag.s[j];
        if (e.autoreset) {
          b = e.cash0;
#pragma unroll
          for (int c = 0; c < KP; ++c) h2[c] = 0u;
          t = 0;
          vc = e.cash0;
          if (e.wadv) w = (w + 1) % e.W;
          metric_start(m, e.cash0);
        }
      }
      met_put_k4(sm.met, tid, m);
      mn = m.n;
    }
  }
  MetricAcc m;
  met_get_k4(sm.met, tid, m);
  m.n = mn;
  AggAcc agg;
#pragma unroll
  for (int j = 0; j < FIN_AGG_LEN; ++j) agg.s[j] = sm.agg[j][tid];
  if (live) {
    if (oor) set_flag(e, FIN_FLAG_ACTION_RANGE);
    if (bad) set_flag(e, FIN_FLAG_BAD_INDEX);
    e.cash[i] = b;
    e.vcur[i] = vc;
    store_hold2<KA>(e, i, h2);
    e.t_ep[i] = t;
    e.window[i] = w;
    store_metric(e, i, m);
    if (o.ep_count) o.ep_count[i] = cnt;
  }
  agg.s[FIN_AGG_SUM_REWARD] = rsum;
  if (o.agg_partial) agg_block_write(agg, o.agg_partial + (size_t)blockIdx.x * FIN_AGG_LEN);
}

#define FIN_DISPATCH_K(K, KERNEL, GRID, STREAM, ...)                                         \
  do {                                                                                       \
    if ((K) == 30) KERNEL<30, true><<<GRID, kStep, 0, STREAM>>>(__VA_ARGS__);                \
    else if ((K) == 4) KERNEL<4, true><<<GRID, kStep, 0, STREAM>>>(__VA_ARGS__);             \
    else if ((K) <= 8) KERNEL<8, false><<<GRID, kStep, 0, STREAM>>>(__VA_ARGS__);            \
    else if ((K) <= 16) KERNEL<16, false><<<GRID, kStep, 0, STREAM>>>(__VA_ARGS__);          \
    else KERNEL<32, false><<<GRID, kStep, 0, STREAM>>>(__VA_ARGS__);                         \
  } while (0)

cudaError_t launch_stock_reset(const EnvDev& e, const uint8_t* mask, cudaStream_t s) {
  k_stock_reset<<<blocks_for(e.N), kThreads, 0, s>>>(e, mask);
  return cudaGetLastError();
}

// persistent grid for K1: resident blocks per SM (occupancy API) x SMs, capped by the tiles
template <int KA, bool EXACT>
int k1_grid(int N) {
  static int per_sm = 0;
  if (per_sm == 0) {
    cudaFuncSetAttribute(k_stock_step<KA, EXACT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)sizeof(K1Smem<KA>));
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_stock_step<KA, EXACT>, kK1Threads,
                                                      sizeof(K1Smem<KA>)) != cudaSuccess)
      per_sm = 1;
  }
  if (per_sm < 1) per_sm = 1;
  const int tiles = (N + kStep - 1) / kStep;
  return std::min(tiles, per_sm * num_sms());
}

// persistent grid for the packed K1: resident blocks per SM x SMs, capped by the tiles
template <int KA>
int k2_grid(int N) {
  static int per_sm = 0;
  if (per_sm == 0) {
    cudaFuncSetAttribute(k_stock_step2<KA>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(K2Smem<KA>));
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_stock_step2<KA>, kK2Threads, sizeof(K2Smem<KA>)) !=
        cudaSuccess)
      per_sm = 1;
  }
  if (per_sm < 1) per_sm = 1;
  const int tiles = (N + kStep - 1) / kStep;
  return std::min(tiles, per_sm * num_sms());
}
#define K2_LAUNCH(KA) \
  k_stock_step2<KA><<<k2_grid<KA>(e.N), kK2Threads, sizeof(K2Smem<KA>), s>>>(e, actions, o, v)

cudaError_t launch_stock_step(const EnvDev& e, const int16_t* actions, const TrajDev& o, cudaStream_t s) {
  const int v = vec_ok(actions, 8);   // bulk copies of whole 128-env tiles: 256 K bytes each
#define FIN_K1(KA, EX) \
  k_stock_step<KA, EX><<<k1_grid<KA, EX>(e.N), kK1Threads, sizeof(K1Smem<KA>), s>>>(e, actions, o, v)
#if FIN_K1_PACKED
  if (e.K == 30) K2_LAUNCH(30);
  else if (e.K == 4) K2_LAUNCH(4);
#else
  if (e.K == 30) FIN_K1(30, true);
  else if (e.K == 4) FIN_K1(4, true);
#endif
  else if (e.K <= 8) FIN_K1(8, false);
  else if (e.K <= 16) FIN_K1(16, false);
  else FIN_K1(32, false);
#undef FIN_K1
  return cudaGetLastError();
}

cudaError_t launch_stock_replay(const EnvDev& e, const int16_t* actions, int T, const TrajDev& o, int* n_blocks,
                                cudaStream_t s) {
  *n_blocks = blocks_for(e.N, kStep);
  const int v = vec_ok(actions, (long long)e.N * e.K);
#if FIN_K4_PACKED
  if (e.K == 30 || e.K == 4) {
    if (e.K == 30) {
      static const bool attr30 = cudaFuncSetAttribute(k_stock_replay2<30>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                      (int)sizeof(K4Smem<30>)) == cudaSuccess;
      (void)attr30;
      k_stock_replay2<30><<<blocks_for(e.N, kStep), kStep, sizeof(K4Smem<30>), s>>>(e, actions, T, o, v);
    } else {
      k_stock_replay2<4><<<blocks_for(e.N, kStep), kStep, sizeof(K4Smem<4>), s>>>(e, actions, T, o, v);
    }
    return cudaGetLastError();
  }
#endif
  FIN_DISPATCH_K(e.K, k_stock_replay, blocks_for(e.N, kStep), s, e, actions, T, o, v);
  return cudaGetLastError();
}

cudaError_t launch_stock_get_state(const EnvDev& e, double* cash, int16_t* hold, double* asset, int32_t* t_ep,
                                   int32_t* window, cudaStream_t s) {
  k_stock_get_state<<<blocks_for(e.N), kThreads, 0, s>>>(e, cash, hold, asset, t_ep, window);
  return cudaGetLastError();
}

cudaError_t launch_stock_set_state(const EnvDev& e, const double* cash, const int16_t* hold, const int32_t* t_ep,
                                   const int32_t* window, cudaStream_t s) {
  k_stock_set_state<<<blocks_for(e.N), kThreads, 0, s>>>(e, cash, hold, t_ep, window);
  return cudaGetLastError();
}

cudaError_t launch_agg_finalize(const double* partial, int n_blocks, double* agg, cudaStream_t s) {
  k_agg_finalize<<<1, 32 * FIN_AGG_LEN, 0, s>>>(partial, n_blocks, agg);
  return cudaGetLastError();
}

}  // namespace fin
