// rollout_tc.cuh -- the warp-specialised tcgen05 rollout kernel template (K3/K5/K7).
//
// One CTA owns TILES tiles of 128 SubEnvs (UMMA M = 128: TMEM lane r <-> env r of
// a tile) for all T steps; env state stays in registers.  Per step and per
// ensemble member the policy MLP (BASELINE configs[1..3])
// runs as three tcgen05.mma GEMMs  D = A * W^T  with A (activations, bf16,
// K-major core-matrix layout in smem) and W (bf16 weights, streamed by 1-D bulk
// TMA into a ring of smem stages, or resident) accumulating fp32 in TMEM.  Every
// streamed weight stage feeds the MMAs of all TILES tiles, so L2 weight traffic
// per env-step is divided by TILES.
//
// Warp roles (128 + 128 * TILES threads, whole warpgroups so registers can move
// between them with setmaxnreg):
//   warp 0        producer: streams weight stages global(L2) -> smem ring (cp.async.bulk)
//   warp 1        TMEM allocator + MMA issuer (one elected lane)
//   warps 2, 3    idle (complete the first warpgroup)
//   warps 4..     one "env" warpgroup per tile: per-tile staging of the shared market
//                 row, observation rows, TMEM epilogues (bias, ReLU, bf16), action
//                 sampling / ensemble averaging, the env transition (trade, reward,
//                 done / reset) and online metrics -- thread r of a warpgroup owns env
//                 r of its tile (warp w reads TMEM lanes 32*(w%4)..+31).
// Synchronisation (mbarriers): w_full / w_empty per ring slot (TMA <-> MMA),
// a_full (all env threads -> MMA: A operands written, TMEM columns free), d_full
// (MMA commit -> env: accumulators ready).  A tile's A buffer holds the
// observation for layer 1 and is overwritten by the hidden activations (the
// layer's MMAs have completed when d_full fires), so the observation is rebuilt
// for every ensemble member from the per-step staging area.
#pragma once
#include <cstdio>
#include <cstdlib>
#include <type_traits>

#include "fin_internal.cuh"
#include "sm100.cuh"
#include "tc_plan.cuh"

namespace tc {

constexpr int kTileM = 128;
constexpr int kRing = 4;   // max weight-ring slots (barrier storage); a launch may use fewer
constexpr int kSmemLimit = 232448;  // 227 KB per CTA

struct TcParams {
  EnvDev e;
  TrajDev o;
  const uint8_t* wpack[FIN_MAX_MEMBERS];  // packed member weights (TcPlan layout)
  const float* bias[FIN_MAX_MEMBERS];     // [HID + HID + OUT_PAD] fp32 per member
  uint8_t bias_nz[FIN_MAX_MEMBERS];       // bit l: member m, layer l has a non-zero bias.  Adding an
                                          // exactly-zero bias is the identity (up to the sign of a
                                          // zero), so the epilogue skips those loads and adds
  int8_t ou_slot[FIN_MAX_MEMBERS];        // DDPG members: OU state slot (else -1)
  int32_t n_ddpg;                         // DDPG members in this call
  int32_t kinds[FIN_MAX_MEMBERS];
  float mw[FIN_MAX_MEMBERS];              // member weights (weighted mode)
  int32_t M;
  float inv_m;                            // fl(1 / M), host division
  int32_t weighted;
  int32_t T;
  int32_t noise_mode;
  uint64_t noise_seed;
  const float* noise;                     // supplied noise
  const uint32_t* noise_ready;            // streamed supplied noise: finished producer blocks per step, or null
  uint32_t noise_ready_target;            // producer blocks (step t is complete at this count)
  // fin_ensemble_act: compute the (ensemble) action only, no env transition
  int32_t act_only;
  int32_t commit_ou;                      // fin_ensemble_act: advance the DDPG OU states (else left untouched)
  float* mean_out;                        // [N][K] averaged continuous action
  uint16_t* hid_out;                      // bf16 hidden activations (probe [B][2][HID])
  const float* z1s;                       // factored layer 1: shared term [M][rows][HID] (or probe [B][HID])
  int32_t z1s_rows;
  unsigned long long* trace;              // debug: clock64 timeline of block 0 ([T][16]) or null
  // K7 probe
  const uint16_t* x_in;
  float* z_out;
  int32_t B, in_dim, out_dim;
  int32_t tiles_per_cta;                  // set by launch(): aggregate partial rows per CTA
  // Dynamic chunk schedule (Ops::kSegments, one tile per CTA).  The T
  // steps of every tile are cut into n_chunks chunks [chunk_t0[k], chunk_t0[k + 1]) of
  // decreasing length; work item i = chunk i / n_tiles of tile i % n_tiles (chunk-major).
  // Each CTA's producer warp claims items with one atomicAdd on q_ctr (zeroed before the
  // launch) and hands them to the MMA warp and the env warpgroup through a 2-slot
  // shared-memory queue; an item (tile, k > 0) starts once seg_flag[tile] says chunk k - 1
  // is done (flag = epoch << 8 | chunks done).  Blocking chains strictly decrease in claim
  // order, so the schedule cannot deadlock, resident or not.  q_ctr null: one tile per CTA,
  // all T steps.
  uint32_t* q_ctr;
  uint32_t* seg_flag;
  uint32_t seg_epoch;
  int32_t n_tiles, n_chunks;
  int32_t chunk_t0[17];
  int32_t seg_grid;                       // CTAs of the chunk schedule (2 per SM)
  unsigned long long* seg_prof;           // debug (FIN_SEG_PROF): [grid][16] globaltimer stamps, or null
};

#ifndef FIN_PIPE_KICK
#define FIN_PIPE_KICK 0   // 1: column-split resident plans issue each layer's MMAs in two halves (kPipeKick; A/B: C3 3.56 vs 3.28 us, off)
#endif
#ifndef FIN_PREPARE_LAYER
#define FIN_PREPARE_LAYER 0   // Ops::prepare runs after the kick of layer FIN_PREPARE_LAYER + 1
#endif

// debug timeline (fin_debug_trace): block 0 only, one slot per event.  Compiled in only
// with -DFIN_TRACE (FIN_NVCC_FLAGS=-DFIN_TRACE): the per-event predicates alone cost ~4%
// of the headline rollout (A/B, round 1), so production builds carry none.
#ifndef FIN_TRACE
#define FIN_TR(cond, t, slot) \
  do {                        \
  } while (0)
#else
#define FIN_TR(cond, t, slot)                                                                  \
  do {                                                                                         \
    if (p.trace && blockIdx.x == 0 && (cond)) p.trace[(size_t)(t) * 32 + (slot)] = clock64(); \
  } while (0)
#endif

__device__ __forceinline__ uint32_t cm_off(int r, int kchunk, int kt8) {
  return (uint32_t)(((r >> 3) * kt8 + kchunk) * 128 + (r & 7) * 16);
}

// plain (non-volatile, no memory clobber) 16-byte shared store: ordered by the
// proxy fence / barriers that follow, free to be scheduled with the loads before it
__device__ __forceinline__ void sts128(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d));
}

// Shared-memory carve-up (dynamic smem, 1024-B aligned base).  The bias region is
// sized for the launch's member count.
template <class Plan, bool RESIDENT, int TILES, class Ops, int RING = kRing>
struct Smem {
  static constexpr int kA = kTileM * (Plan::kIn > Plan::kHidMax ? Plan::kIn : Plan::kHidMax) * 2;  // per tile
  static constexpr int kFixed = TILES * kA + TILES * Ops::kStageBytes + 512;  // + barriers, flags
  static constexpr int kBiasPerMember = Plan::kBiasFloats * 4;
  static constexpr int kStaticSmem = 512;  // agg_group_write scratch etc.
  // members whose weights fit resident in shared memory (resident plans only)
  static constexpr int kResMembers =
      RESIDENT ? ((kSmemLimit - kStaticSmem - kFixed) / (Plan::kMemberBytes + kBiasPerMember) < FIN_MAX_MEMBERS
                      ? (kSmemLimit - kStaticSmem - kFixed) / (Plan::kMemberBytes + kBiasPerMember)
                      : FIN_MAX_MEMBERS)
               : FIN_MAX_MEMBERS;
  __host__ __device__ static constexpr int w_bytes(int M) {
    return RESIDENT ? Plan::kMemberBytes * M : RING * Plan::kStageBytes;
  }
  // members whose biases are staged in shared memory (Ops::kStageBias = false: none, the
  // epilogues read them from L2 -- the ensemble kernels, where the smem is needed elsewhere)
  __host__ __device__ static constexpr int staged(int M) {
    return !Ops::kStageBias ? 0 : (M < FIN_STAGE_MEMBERS ? M : FIN_STAGE_MEMBERS);
  }
  __host__ __device__ static constexpr int total(int M) { return kFixed + w_bytes(M) + staged(M) * kBiasPerMember; }
  __host__ __device__ static constexpr int max_members() {   // resident plans: weights of M members in smem
    return RESIDENT ? (kSmemLimit - kStaticSmem - kFixed - FIN_STAGE_MEMBERS * kBiasPerMember) / Plan::kMemberBytes
                    : FIN_MAX_MEMBERS;
  }
};

// ---------------------------------------------------------------------------------
// The kernel.  Ops supplies the env-side behaviour (see rollout_stock.cu etc.):
//   struct Ops {
//     static constexpr int kStageBytes;             // per-tile staging area
//     struct State;
//     init(State&, p, env, row)
//     stage(State&, p, env, row, t, stage_ptr, bar_id)   per step, all 128 threads of a tile
//     build_obs(State&, p, env, row, t, m, x_addr, stage_ptr)
//     hidden_ptr(State&, p, env, t, m, l, hid) -> uint16_t* or nullptr
//     consume(State&, p, env, t, m, const float* z)
//     finish_step(State&, p, env, t, stage_ptr, a_tile)   (a_tile: the tile's A operand, free during the
//                                                        env step -- scratch for the env side)
//     finalize(State&, p, env, group_tid, bar_id)
//   };
// RING: weight-ring slots; MINB: CTAs per SM (MINB = 2 runs two independent tiles per
// SM whose env phases overlap each other's MMA / weight-streaming phases).
// SPLIT > 1 (one tile per CTA: the latency-bound crypto rollout and, round 2, the small-N
// stock rollout): SPLIT warpgroups share each hidden layer's epilogue by columns (warpgroup w
// takes chunk range w of the layer's 16-column chunks); the first runs everything else.  A
// factored layer 1 (stock): the first warpgroup publishes each row's addend pointer in shared
// memory past the plan's layout (named barrier kSplitBar0, arrive / sync) before the layer's
// MMAs; the launch adds 1 KB.
template <class Plan, bool RESIDENT, int TILES, class Ops, int RING = kRing, int MINB = 1, int SPLIT = 1>
__global__ void __launch_bounds__(128 + 128 * TILES * SPLIT, MINB) k_tc_rollout(const __grid_constant__ TcParams p) {
  static_assert(SPLIT == 1 || (TILES == 1 && Ops::kSplitOK), "column-split epilogues: 1 tile");
  static_assert((Plan::kHidMax / 16) % SPLIT == 0, "chunks must divide among the warpgroups");
  using S = Smem<Plan, RESIDENT, TILES, Ops, RING>;
  extern __shared__ __align__(1024) uint8_t smem[];
  const int M = p.M;
  const int T = p.T;
  constexpr int NS = Plan::kStages;
  constexpr int kTc = Plan::kHidMax > Plan::kOut ? Plan::kHidMax : Plan::kOut;   // TMEM columns per tile
  // Column-split resident plans (kPipeKick, see run_epi): the next layer's MMAs start while the
  // epilogue still reads this layer's accumulator, so consecutive layers alternate between two
  // accumulator banks of kTc columns
  constexpr bool kPipeKick = SPLIT > 1 && RESIDENT && FIN_PIPE_KICK;
  constexpr int kBanks = kPipeKick ? 2 : 1;
  static_assert(TILES * kTc * kBanks <= 512, "TMEM holds 512 fp32 columns");
  constexpr uint32_t kTmemCols =
      (TILES * kTc * kBanks <= 128) ? 128 : (TILES * kTc * kBanks <= 256 ? 256 : 512);
  static_assert(TILES * kTc <= 512, "TMEM holds 512 fp32 columns");

  uint8_t* sA = smem;                                           // TILES x kA
  uint8_t* sStage = sA + TILES * S::kA;                         // TILES x Ops::kStageBytes
  uint64_t* bars = reinterpret_cast<uint64_t*>(sStage + TILES * Ops::kStageBytes);
  uint64_t* w_full = bars;
  uint64_t* w_empty = bars + kRing;
  uint64_t* a_full = bars + 2 * kRing;
  uint64_t* d_full = bars + 2 * kRing + 1;          // [TILES]: one per tile
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * kRing + 1 + TILES);
  uint64_t* q_full = bars + 16;                                  // [2] item published (1 arrival)
  uint64_t* q_empty = bars + 18;                                 // [2] item read (MMA warp + env group)
  int4* q_item = reinterpret_cast<int4*>(bars + 32);             // [2] {tile, t0, t1, k} (tile < 0: end)
  // Resident weights: each tile's thread 0 issues its own MMAs right after the tile's
  // epilogue barrier (the issue code sits in the env warps' hot path; a separate MMA
  // warp woken per layer cost ~1,000 cycles per layer in the C3 timeline, mostly
  // instruction fetch of a code path that runs once per layer).  Streamed weights keep
  // the MMA warp: its stages feed both tiles.
  constexpr bool kEnvIssue = RESIDENT;
  uint8_t* sW = reinterpret_cast<uint8_t*>(bars) + 512;
  float* sBias = reinterpret_cast<float*>(sW + S::w_bytes(M));

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  // dynamic chunk schedule: item queue in shared memory (2 slots), filled by the producer
  constexpr bool kSeg = Ops::kSegments && TILES == 1 && SPLIT == 1;
  const bool segd = kSeg && p.q_ctr != nullptr;

  // ---- one-time setup
  for (int j = threadIdx.x; j < S::staged(M) * Plan::kBiasFloats; j += blockDim.x) {
    const int m = j / Plan::kBiasFloats, q = j % Plan::kBiasFloats;
    sBias[j] = p.bias[m] ? p.bias[m][q] : 0.f;
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < kRing; ++s) {
      sm100::mbar_init(&w_full[s], 1);
      sm100::mbar_init(&w_empty[s], 1);
    }
    sm100::mbar_init(a_full, 128 * TILES);
    for (int tl = 0; tl < TILES; ++tl) sm100::mbar_init(&d_full[tl], 1);
    for (int s = 0; s < 2; ++s) {
      sm100::mbar_init(&q_full[s], 1);
      sm100::mbar_init(&q_empty[s], 2);
    }
    sm100::fence_mbar_init();
  }
  if (warp == 1) {
    sm100::tmem_alloc(tmem_slot, kTmemCols);
    sm100::tmem_relinquish();
  }
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  // register split (one CTA per SM, two tiles): the producer / MMA warpgroup needs few
  // registers, the env warpgroups hold each env's whole state for all T steps.  Each
  // role's code sits inside the branch that resized its registers, so ptxas allocates
  // it against the new budget.
  // (two tiles, one CTA per SM: 4 x 40 + 8 x 232 warps' worth = 64 K registers; one tile, two
  // CTAs per SM: each CTA 4 x 40 + 4 x 216 of its 128-per-thread launch allocation)
  // (the column-split streamed-weight stock tile, 1 CTA per SM: 4 x 40 + 8 x 232 as two tiles)
  constexpr bool kSplit2 = TILES == 1 && SPLIT == 2 && MINB == 1 && !RESIDENT;
  constexpr bool kSplitRegs = (TILES == 2 && MINB == 1) || (TILES == 1 && MINB == 2) || kSplit2;
#ifndef FIN_DUAL_LOW_REGS
#define FIN_DUAL_LOW_REGS 32   // producer / MMA warpgroup registers in the dual layout (A/B: 32 +0.4% vs 40, 48 -0.4%)
#endif
  // dual layout (one tile, two CTAs per SM): 128 x (low + env) = 32 K registers per CTA
  constexpr uint32_t kLowRegs = (TILES == 2 || kSplit2) ? 40 : FIN_DUAL_LOW_REGS;
  constexpr uint32_t kEnvRegs = (TILES == 2 || kSplit2) ? 232 : 256 - kLowRegs;
  if (warp < 4) {
  if constexpr (kSplitRegs) asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(kLowRegs) : "memory");
  if (warp == 0) {
    // ============================ producer ============================
    if (lane == 0) {
      if (RESIDENT) {
        uint32_t total = (uint32_t)(Plan::kMemberBytes * M);
        sm100::mbar_arrive_expect_tx(&w_full[0], total);
        for (int m = 0; m < M; ++m)
          for (int s = 0; s < NS; ++s)
            sm100::bulk_g2s(sW + m * Plan::kMemberBytes + Plan::offset_of(s), p.wpack[m] + Plan::offset_of(s),
                            (uint32_t)Plan::bytes_of(s), &w_full[0]);
      } else {
        const uint64_t pol = sm100::l2_policy_evict_last();
        uint32_t it = 0;
        uint32_t qi = 0;
        for (;;) {
          int n_steps = T;
          if (segd) {   // claim the next work item and publish it to the MMA warp and the env group
            const uint32_t i = atomicAdd(p.q_ctr, 1u);
            const uint32_t n_items = (uint32_t)p.n_tiles * (uint32_t)p.n_chunks;
            int4 item = make_int4(-1, 0, 0, 0);
            if (i < n_items) {
              const int k = (int)(i / (uint32_t)p.n_tiles), tl = (int)(i % (uint32_t)p.n_tiles);
              item = make_int4(tl, p.chunk_t0[k], p.chunk_t0[k + 1], k);
            }
            const uint32_t qs = qi & 1u;
            sm100::mbar_wait(&q_empty[qs], ((qi >> 1) & 1u) ^ 1u);
            q_item[qs] = item;
            sm100::mbar_arrive(&q_full[qs]);   // (release: the item store is visible to the waiters)
            ++qi;
            if (item.x < 0) break;
            n_steps = item.z - item.y;
          }
          for (int t = 0; t < n_steps; ++t)
            for (int m = 0; m < M; ++m)
#pragma unroll
              for (int s = 0; s < NS; ++s, ++it) {   // unrolled: per-stage plan values fold to constants
                const uint32_t slot = it % RING, ph = (it / RING) & 1;
                sm100::mbar_wait_fast(&w_empty[slot], ph ^ 1);
                FIN_TR(m == 0 && (s == 0 || s == NS - 1), t, s == 0 ? 30 : 31);
                FIN_TR(m == 0 && s < 16, T + t, 16 + s);   // per-stage detail rows (trace [2T][32])
                sm100::mbar_arrive_expect_tx(&w_full[slot], (uint32_t)Plan::bytes_of(s));
                sm100::bulk_g2s_hint(sW + slot * Plan::kStageBytes, p.wpack[m] + Plan::offset_of(s),
                                     (uint32_t)Plan::bytes_of(s), &w_full[slot], pol);
              }
          if (!segd) break;
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ============================ MMA issuer ============================
    if (lane == 0 && !kEnvIssue) {
      uint32_t it = 0, a_use = 0;
      if (RESIDENT) sm100::mbar_wait(&w_full[0], 0);
      const uint32_t aa = sm100::smem_u32(sA), wa = sm100::smem_u32(sW);
      uint32_t qi = 0;
      for (;;) {
      int n_steps = T;
      if (segd) {
        const uint32_t qs = qi & 1u;
        sm100::mbar_wait(&q_full[qs], (qi >> 1) & 1u);
        const int4 item = q_item[qs];
        sm100::mbar_arrive(&q_empty[qs]);
        ++qi;
        if (item.x < 0) break;
        n_steps = item.z - item.y;
      }
      for (int t = 0; t < n_steps; ++t) {
        for (int m = 0; m < M; ++m) {
#pragma unroll
          for (int l = 0; l < Plan::kNL; ++l) {
            sm100::mbar_wait_fast(a_full, a_use & 1);
            ++a_use;
            FIN_TR(m == 0, t, 9 + 2 * l);
            sm100::tc_fence_after();
            const uint32_t a_sbo = (uint32_t)(Plan::kdim(l) / 8) * 128u;
            const uint32_t idesc = sm100::make_idesc_bf16(kTileM, Plan::nrows(l));
            // layer 1 of a kL1Init member: the accumulator starts at the day's shared-input term
            // (a uniform tile's image copied here, a mixed tile's rows stored by its env threads)
            const bool l1init = Ops::kL1Init && l == 0;   // accumulator pre-set by the env threads
#pragma unroll
            for (int s = Plan::first_stage(l); s < Plan::first_stage(l) + Plan::nstages(l); ++s) {
              uint32_t b_base;
              if (RESIDENT) {
                b_base = wa + (uint32_t)(m * Plan::kMemberBytes + Plan::offset_of(s));
              } else {
                const uint32_t slot = it % RING, ph = (it / RING) & 1;
                FIN_TR(m == 0 && s < 16, 2 * T + t, s);
                sm100::mbar_wait_fast(&w_full[slot], ph);
                FIN_TR(m == 0 && s == Plan::first_stage(l), t, 26 + l);
                FIN_TR(m == 0 && l == 1 && s == Plan::first_stage(1) + Plan::nstages(1) - 1, t, 29);
                FIN_TR(m == 0 && s < 16, T + t, s);
                sm100::tc_fence_after();
                b_base = wa + slot * (uint32_t)Plan::kStageBytes;
              }
              const int j0 = Plan::j0_of(s), nks = Plan::nks_of(s);
              const uint32_t b_sbo = (uint32_t)(nks * 2) * 128u;  // Kt/8 * 128 with Kt = 16 nks
#pragma unroll
              for (int tile = 0; tile < TILES; ++tile) {
                const uint32_t a_base = aa + (uint32_t)(tile * S::kA);
                const uint32_t d_tmem = tmem + (uint32_t)(tile * kTc);
                // descriptors of k-step 0; each further k-step advances both start
                // addresses by 256 B = 16 units of the descriptor's address field
                const uint64_t ad0 = sm100::make_sdesc(a_base + (uint32_t)j0 * 256u, 128u, a_sbo);
                const uint64_t bd0 = sm100::make_sdesc(b_base, 128u, b_sbo);
                for (int j = 0; j < nks; ++j)
                  sm100::mma_bf16(d_tmem, ad0 + (uint64_t)(16 * j), bd0 + (uint64_t)(16 * j), idesc,
                                  (l1init || (j0 + j) > 0) ? 1u : 0u);
              }
              FIN_TR(m == 0 && s < 16, 2 * T + t, 16 + s);
              if (!RESIDENT) {
                sm100::mma_commit(&w_empty[it % RING]);
                ++it;
              }
            }
            sm100::mma_commit(d_full);   // TILES == 1 or 2 share one phase when the MMA warp issues
            if (TILES > 1) sm100::mma_commit(&d_full[1]);
            FIN_TR(m == 0, t, 10 + 2 * l);
          }
        }
      }
      if (!segd) break;
      }
    }
    __syncwarp();
  }
  } else {
    if constexpr (kSplitRegs) asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(kEnvRegs) : "memory");
    // ============================ env warpgroups ============================
    const int part = SPLIT > 1 ? ((warp - 4) >> 2) : 0;   // column share of the epilogues (SPLIT > 1)
    const int tile = SPLIT > 1 ? 0 : ((warp - 4) >> 2);
    const int q = warp & 3;                 // TMEM lane quarter this warp may access
    const int row = q * 32 + lane;          // env row of the tile == TMEM lane
    const int gtid = (warp - 4 - (tile + part) * 4) * 32 + lane;   // thread index within its warpgroup
    const int env = (blockIdx.x * TILES + tile) * kTileM + row;
    const uint32_t t_lane0 = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(tile * kTc * kBanks);
    uint32_t t_lane = t_lane0;   // this layer's accumulator bank (kPipeKick: layer l in bank l % 2)
    auto bank_of = [&](int l) -> uint32_t { return kBanks > 1 ? (uint32_t)((l & 1) * kTc) : 0u; };
    const uint32_t xa = sm100::smem_u32(sA + tile * S::kA);
    uint8_t* stg = sStage + tile * Ops::kStageBytes;
    const int bar_id = 1 + tile;
    constexpr int kSplitBar = 1 + TILES;     // the warpgroups of a column-split tile meet here
    constexpr int kSplitBar0 = 2 + TILES;    // ... and here for the layer-1 addend pointers
    // (SPLIT > 1) per-row layer-1 addend pointers, past the plan's shared-memory layout
    const float** sAdd = reinterpret_cast<const float**>(smem + S::total(M));
    // Hidden-layer epilogue of chunks [c0, c1): D -> +bias (+ addend) -> ReLU -> bf16 -> A
    // (K-major core matrices).  16 columns per TMEM load: half the registers of 32-column
    // chunks (the env state lives in registers across the whole rollout).  One loop per
    // addend combination (uniform branch), so an absent addend costs no issue slots.
    auto epi = [&](auto has_b, auto has_add, const float* bl, const float* add, uint4* hlog, int ncol, int c0,
                   int c1, int cs) {
      constexpr bool HB = decltype(has_b)::value, HA = decltype(has_add)::value;
      // addend b (+ z1s for the factored layer 1) of chunk c, 128-bit broadcast loads
      auto addend = [&](int c, float (&ad)[16]) {
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4) {
          float4 x = make_float4(0.f, 0.f, 0.f, 0.f);
          if constexpr (HB) x = reinterpret_cast<const float4*>(bl + c * 16)[q4];
          if constexpr (HA) {
            const float4 y = reinterpret_cast<const float4*>(add + c * 16)[q4];
            if constexpr (HB) {
              x.x += y.x; x.y += y.y; x.z += y.z; x.w += y.w;
            } else {
              x = y;
            }
          }
          ad[4 * q4] = x.x; ad[4 * q4 + 1] = x.y; ad[4 * q4 + 2] = x.z; ad[4 * q4 + 3] = x.w;
        }
      };
      // chunk c's accumulators v -> + addend -> ReLU -> bf16 -> A operand (and the log)
      auto proc = [&](int c, const uint32_t (&v)[16], const float (&ad)[16]) {
        uint32_t pk[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {   // ReLU + bf16 in one cvt.rn.relu.bf16x2
          if constexpr (HB || HA)
            pk[j] = sm100::pack_bf16_relu(__uint_as_float(v[2 * j]) + ad[2 * j],
                                          __uint_as_float(v[2 * j + 1]) + ad[2 * j + 1]);
          else
            pk[j] = sm100::pack_bf16_relu(__uint_as_float(v[2 * j]), __uint_as_float(v[2 * j + 1]));
        }
#pragma unroll
        for (int g = 0; g < 2; ++g)
          sts128(xa + cm_off(row, c * 2 + g, ncol / 8), pk[4 * g], pk[4 * g + 1], pk[4 * g + 2], pk[4 * g + 3]);
        if (hlog) {
#pragma unroll
          for (int g = 0; g < 2; ++g)
            hlog[c * 2 + g] = make_uint4(pk[4 * g], pk[4 * g + 1], pk[4 * g + 2], pk[4 * g + 3]);
        }
      };
      if constexpr (Ops::kEpiPipe) {
      // (Ops::kEpiPipe, the light-state crypto rollout: 2.7% faster there, 6.5% slower in
      // the register-heavy stock rollout -- A/B round 1) two chunk buffers: the TMEM load of
      // chunk c + 1 is in flight while chunk c is processed (tcgen05.wait::ld waits for every outstanding load of the thread, so
      // each wait sits after the other buffer's processing); chunk counts are even
      uint32_t va[16], vb[16];
      float ad[16];
      sm100::tmem_ld16(t_lane + (uint32_t)(c0 * 16), va);
      sm100::tmem_wait_ld();
#pragma unroll 1
      for (int c = c0; c < c1; c += 2 * cs) {
        sm100::tmem_ld16(t_lane + (uint32_t)((c + cs) * 16), vb);
        addend(c, ad);
        proc(c, va, ad);
        sm100::tmem_wait_ld();
        if (c + 2 * cs < c1) sm100::tmem_ld16(t_lane + (uint32_t)((c + 2 * cs) * 16), va);
        addend(c + cs, ad);
        proc(c + cs, vb, ad);
        sm100::tmem_wait_ld();
      }
      } else {
#pragma unroll 1
      for (int c = c0; c < c1; c += cs) {
        uint32_t v[16];
        sm100::tmem_ld16(t_lane + (uint32_t)(c * 16), v);
        // the addend loads are issued while the TMEM load is in flight
        float ad[16];
        addend(c, ad);
        sm100::tmem_wait_ld();
        proc(c, v, ad);
      }
      }
    };
    auto run_epi = [&](const float* bl, const float* add, uint4* hlog, int ncol, int c0, int c1, int cs = 1) {
      using T1 = std::true_type;
      using F0 = std::false_type;
      // (bl is uniform; add is null for every thread or for none -- Ops contract)
      if (bl && add) epi(T1{}, T1{}, bl, add, hlog, ncol, c0, c1, cs);
      else if (bl) epi(T1{}, F0{}, bl, add, hlog, ncol, c0, c1, cs);
      else if (add) epi(F0{}, T1{}, bl, add, hlog, ncol, c0, c1, cs);
      else epi(F0{}, F0{}, bl, add, hlog, ncol, c0, c1, cs);
    };
    // Column-split resident plans (kPipeKick): each warpgroup takes the chunks c = part (mod SPLIT)
    // and the next layer's MMAs are issued in two halves -- k-steps [0, K/2) as soon as the first
    // half of every warpgroup's chunks is in the A operand, the rest after the second half -- so
    // the issue of the first half (and its tensor work) overlaps the second half of the epilogue.
    // Same k-step order, so the same accumulation as one issue after the whole epilogue.
    static_assert(!kPipeKick || ((Plan::kH1 / 16) / 2) % SPLIT == 0, "halves must divide among the warpgroups");
    // this layer's width = the next layer's K (a compile-time constant when all hidden
    // layers have one width, as in the BASELINE nets: the runtime bound cost ~10%)
    constexpr bool kUniformHid = Plan::hid(0) == Plan::hid(1) && (Plan::kNH < 3 || Plan::hid(2) == Plan::hid(0));
    bool is_helper = false;
    if constexpr (SPLIT > 1) {
    if (part > 0) {
      // ======================= epilogue helper (column share `part`) =======================
      is_helper = true;
      uint32_t d_use = 0;
      for (int t = 0; t < T; ++t) {
        for (int m = 0; m < M; ++m) {
          const float* bias = (Ops::kStageBias && m < FIN_STAGE_MEMBERS) ? sBias + m * Plan::kBiasFloats : p.bias[m];
#pragma unroll 1
          for (int l = 0; l < Plan::kNH; ++l) {
            sm100::mbar_wait(&d_full[0], d_use & 1);
            ++d_use;
            sm100::tc_fence_after();
            const float* bl = ((p.bias_nz[m] >> l) & 1u) ? bias + Plan::bias_off(l) : nullptr;
            const int ncol = kUniformHid ? Plan::kH1 : Plan::nrows(l);
            const int cpp = (ncol / 16) / SPLIT;
            uint4* hlog = reinterpret_cast<uint4*>(Ops::helper_hidden_ptr(p, env, t, m, l, Plan::kHidMax));
            const float* add = nullptr;
            if constexpr (Ops::kSplitAddend) {
              if (l == 0) {
                sm100::named_bar_sync(kSplitBar0, 128 * SPLIT);
                add = sAdd[row];
              }
            }
            t_lane = t_lane0 + bank_of(l);
            if constexpr (kPipeKick) {
              const int nch = ncol / 16;
              for (int h = 0; h < 2; ++h) {
                run_epi(bl, nullptr, hlog, ncol, h * (nch / 2) + part, (h + 1) * (nch / 2), SPLIT);
                sm100::fence_proxy_async_smem();
                sm100::tc_fence_before();
                sm100::named_bar_sync(kSplitBar, 128 * SPLIT);
              }
            } else {
              run_epi(bl, add, hlog, ncol, part * cpp, (part + 1) * cpp);
              sm100::fence_proxy_async_smem();
              sm100::tc_fence_before();
              sm100::named_bar_sync(kSplitBar, 128 * SPLIT);
            }
          }
          // the output layer's phase (read by the first warpgroup only) must still be waited
          // for: parity waits only tell the current phase from the previous one
          sm100::mbar_wait(&d_full[0], d_use & 1);
          ++d_use;
        }
      }
    }
    }
    if (!is_helper) {
    typename Ops::State st;
    uint32_t d_use = 0;
    bool w_ready = false;   // resident weights landed (env-issued MMAs)
    int t_cur = 0;          // (the timeline's step index inside kick)
    // A operand of layer l of member m written by this thread: hand it to the tensor core
    auto kick = [&](int m, int l, int half = -1) {   // half 0 / 1: kPipeKick's k-step halves (commit after 1)
      sm100::fence_proxy_async_smem();
      sm100::tc_fence_before();
      if constexpr (kEnvIssue) {
        if (SPLIT > 1 && l > 0) sm100::named_bar_sync(kSplitBar, 128 * SPLIT);   // the helpers' columns too
        else sm100::named_bar_sync(bar_id, 128);
        if (gtid == 0) {
          FIN_TR(tile == 0 && m == 0 && l == 0, t_cur, 25);
          if (!w_ready) {
            sm100::mbar_wait(&w_full[0], 0);
            w_ready = true;
          }
          sm100::tc_fence_after();
          const uint32_t a_sbo = (uint32_t)(Plan::kdim(l) / 8) * 128u;
          const uint32_t idesc = sm100::make_idesc_bf16(kTileM, Plan::nrows(l));
          const uint32_t a_base = sm100::smem_u32(sA) + (uint32_t)(tile * S::kA);
          const uint32_t d_tmem = tmem + (uint32_t)(tile * kTc * kBanks) + bank_of(l);
          // layer 1 of a tile whose envs share the step's row (Ops::kL1Bcast): k-steps >= 1 read
          // one 8-row core-matrix column per k-group with SBO = 0, so every 8-row group of the
          // tile sees the same shared inputs (same operand values, same MMA sequence)
          uint32_t bc = 0;
          if constexpr (Ops::kL1Bcast) bc = l == 0 ? Ops::l1_bcast(st, stg) : 0u;
          const bool l1init = Ops::kL1Init && l == 0;   // accumulator pre-set by the env threads
          for (int s = Plan::first_stage(l); s < Plan::first_stage(l) + Plan::nstages(l); ++s) {
            const uint32_t b_base = sm100::smem_u32(sW) + (uint32_t)(m * Plan::kMemberBytes + Plan::offset_of(s));
            const int j0 = Plan::j0_of(s), nks = Plan::nks_of(s);
            const uint32_t b_sbo = (uint32_t)(nks * 2) * 128u;
            const uint64_t ad0 = sm100::make_sdesc(a_base + (uint32_t)j0 * 256u, 128u, a_sbo);
            const uint64_t bd0 = sm100::make_sdesc(b_base, 128u, b_sbo);
            const int ks = Plan::ksteps(l);
            const int jlo = half == 1 ? ks / 2 : 0, jhi = half == 0 ? ks / 2 : ks;
            for (int j = 0; j < nks; ++j) {
              if (half >= 0 && (j0 + j < jlo || j0 + j >= jhi)) continue;
              uint64_t ad = ad0 + (uint64_t)(16 * j);
              if (bc && j0 + j > 0) ad = sm100::make_sdesc(bc + (uint32_t)(j0 + j - 1) * 256u, 128u, 0u);
              sm100::mma_bf16(d_tmem, ad, bd0 + (uint64_t)(16 * j), idesc, (l1init || (j0 + j) > 0) ? 1u : 0u);
            }
          }
          FIN_TR(tile == 0 && m == 0 && l == 0, t_cur, 26);
          if (half != 0) sm100::mma_commit(&d_full[tile]);
        }
      } else {
        if (SPLIT > 1 && l > 0) sm100::named_bar_sync(kSplitBar, 128 * SPLIT);   // the helpers' columns too
        sm100::mbar_arrive(a_full);
      }
    };
    // one work item = steps [t_begin, t_end) of one tile (without the chunk schedule: this
    // CTA's tile, all T steps)
    uint32_t qi = 0;
    for (int si = 0;; ++si) {
    int4 sg = make_int4(blockIdx.x * TILES + tile, 0, T, 0);
    if constexpr (kSeg) {
      if (segd) {
        const uint32_t qs = qi & 1u;
        sm100::mbar_wait(&q_full[qs], (qi >> 1) & 1u);
        sg = q_item[qs];
        ++qi;
        sm100::named_bar_sync(bar_id, 128);          // every thread has read the slot
        if (gtid == 0) sm100::mbar_arrive(&q_empty[qs]);
        if (sg.x < 0) break;
      }
    }
    const int env = sg.x * kTileM + row;
    const int t_begin = sg.y, t_end = sg.z;
    FIN_CHECK(!segd || (sg.x >= 0 && sg.x < p.n_tiles && sg.w >= 0 && sg.w < p.n_chunks));
    FIN_CHECK(0 <= t_begin && t_begin < t_end && t_end <= T);
    if constexpr (kSeg) {
      if (p.seg_prof && gtid == 0 && si < 5) {
        p.seg_prof[blockIdx.x * 16 + 3 * si] = sm100::globaltimer();
        uint32_t smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        p.seg_prof[blockIdx.x * 16 + 15] = smid;
      }
      if (segd) {
        if (sg.w > 0) {   // chunk k > 0: wait until the tile's chunk k - 1 is written back
          if (gtid == 0) {
            const uint32_t need = (p.seg_epoch << 8) | (uint32_t)sg.w;
            while (sm100::ld_acquire_gpu(p.seg_flag + sg.x) < need) __nanosleep(128);
          }
          sm100::named_bar_sync(bar_id, 128);
        }
        Ops::init_seg(st, p, env, row, t_begin, t_end);
      } else {
        Ops::init(st, p, env, row);
      }
      if (p.seg_prof && gtid == 0 && si < 5) p.seg_prof[blockIdx.x * 16 + 3 * si + 1] = sm100::globaltimer();
    } else {
      Ops::init(st, p, env, row);
    }
    for (int t = t_begin; t < t_end; ++t) {
      t_cur = t;
      FIN_TR(row == 0 && tile == 0, t, 0);
      Ops::stage(st, p, env, gtid, t, stg, bar_id);
      for (int m = 0; m < M; ++m) {
        if constexpr (Ops::kL1Bcast && kEnvIssue) Ops::build_obs_bcast(st, p, env, row, t, m, xa, stg);
        else Ops::build_obs(st, p, env, row, t, m, xa, stg);
        if constexpr (Ops::kL1Init) Ops::l1_init_rows(st, p, t_lane0, stg);
        if constexpr (SPLIT > 1 && Ops::kSplitAddend) {
          sAdd[row] = Ops::l1_addend(st, p, m, stg);
          sm100::named_bar_arrive(kSplitBar0, 128 * SPLIT);
        }
        kick(m, 0);
        FIN_TR(row == 0 && tile == 0 && m == 0, t, 1);
        // biases of the first FIN_STAGE_MEMBERS members in shared memory, the rest from L2
        const float* bias = (Ops::kStageBias && m < FIN_STAGE_MEMBERS) ? sBias + m * Plan::kBiasFloats : p.bias[m];
        // hidden layers: D -> +bias -> ReLU -> bf16 -> A (K-major core matrices)
#pragma unroll 1
        for (int l = 0; l < Plan::kNH; ++l) {
          sm100::mbar_wait(&d_full[tile], d_use & 1);
          ++d_use;
          FIN_TR(row == 0 && tile == 0 && m == 0, t, 2 + 2 * l);
          sm100::tc_fence_after();
          const float* bl = ((p.bias_nz[m] >> l) & 1u) ? bias + Plan::bias_off(l) : nullptr;
          const int ncol = kUniformHid ? Plan::kH1 : Plan::nrows(l);
          // factored layer 1: + shared-input term of the env's day (smem or global row)
          const float* add = l == 0 ? Ops::l1_addend(st, p, m, stg) : nullptr;
          // debug / parity log of the bf16 hidden activations (teacher-forced layer checks)
          uint4* hlog = reinterpret_cast<uint4*>(Ops::hidden_ptr(st, p, env, t, m, l, Plan::kHidMax));
          t_lane = t_lane0 + bank_of(l);
          if constexpr (kPipeKick) {
            const int nch = ncol / 16;
            run_epi(bl, add, hlog, ncol, 0, nch / 2, SPLIT);
            kick(m, l + 1, 0);
            run_epi(bl, add, hlog, ncol, nch / 2, nch, SPLIT);
            kick(m, l + 1, 1);
          } else {
            run_epi(bl, add, hlog, ncol, 0, (ncol / 16) / SPLIT);
            kick(m, l + 1);
          }
          // work that does not depend on the network output (e.g. the step's noise)
          // overlaps the largest MMA (layer 2) instead of following the last one
          if (l == (Plan::kNH > FIN_PREPARE_LAYER ? FIN_PREPARE_LAYER : Plan::kNH - 1)) Ops::prepare(st, p, env, t, m);
          FIN_TR(row == 0 && tile == 0 && m == 0, t, 3 + 2 * l);
        }
        // output layer
        sm100::mbar_wait(&d_full[tile], d_use & 1);
        ++d_use;
        FIN_TR(row == 0 && tile == 0 && m == 0, t, 6);
        sm100::tc_fence_after();
        float z[Plan::kOut];
        t_lane = t_lane0 + bank_of(Plan::kNH);
#pragma unroll
        for (int c = 0; c < Plan::kOut / 16; ++c) {
          uint32_t v[16];
          sm100::tmem_ld16(t_lane + (uint32_t)(c * 16), v);
          sm100::tmem_wait_ld();
          if ((p.bias_nz[m] >> Plan::kNH) & 1u) {
#pragma unroll
            for (int j = 0; j < 16; ++j)
              z[c * 16 + j] = __uint_as_float(v[j]) + bias[Plan::bias_off(Plan::kNH) + c * 16 + j];
          } else {
#pragma unroll
            for (int j = 0; j < 16; ++j) z[c * 16 + j] = __uint_as_float(v[j]);
          }
        }
        sm100::tc_fence_before();
        Ops::consume(st, p, env, t, m, z);
        FIN_TR(row == 0 && tile == 0 && m == 0, t, 7);
      }
      Ops::finish_step(st, p, env, t, stg, sA + tile * S::kA);
      FIN_TR(row == 0 && tile == 0, t, 8);
    }
    if constexpr (kSeg) {
      if (p.seg_prof && gtid == 0 && si < 5) p.seg_prof[blockIdx.x * 16 + 3 * si + 2] = sm100::globaltimer();
      if (segd) {
        Ops::finalize_seg(st, p, env, gtid, bar_id, sg.x, t_end);
        if (t_end < T) {   // publish the tile's state for the item that runs its next chunk
          sm100::named_bar_sync(bar_id, 128);
          if (gtid == 0) {
            __threadfence();
            sm100::st_release_gpu(p.seg_flag + sg.x, (p.seg_epoch << 8) | (uint32_t)(sg.w + 1));
          }
        }
      } else {
        Ops::finalize(st, p, env, gtid, bar_id, tile);
      }
    } else {
      Ops::finalize(st, p, env, gtid, bar_id, tile);
    }
    if (!segd) break;
    }   // work items
    }   // first warpgroup
  }
  __syncthreads();
  if (warp == 1) {
    sm100::tc_fence_after();
    sm100::tmem_dealloc(tmem, kTmemCols);
  }
}

template <class Plan, bool RESIDENT, int TILES, class Ops, int RING = kRing, int MINB = 1, int SPLIT = 1>
cudaError_t launch(const TcParams& p, int n_envs, cudaStream_t s, int seg_grid = 0) {
  using Sm = Smem<Plan, RESIDENT, TILES, Ops, RING>;
  auto kern = k_tc_rollout<Plan, RESIDENT, TILES, Ops, RING, MINB, SPLIT>;
  const int bytes = Sm::total(p.M) + (SPLIT > 1 ? 1024 : 0);   // (SPLIT: the addend pointers)
  if (MINB > 1 && bytes * MINB > kSmemLimit) return cudaErrorInvalidConfiguration;
  if (bytes > kSmemLimit) return cudaErrorInvalidConfiguration;
  cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (err != cudaSuccess) return err;
  // all of the SM's shared memory as shared memory (the occupancy that cooperative launches
  // check assumes the function's preferred carveout; MINB CTAs need the maximum)
  err = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
  if (err != cudaSuccess) return err;
  const int per_cta = kTileM * TILES;
  TcParams q = p;
  q.tiles_per_cta = TILES;
  if (seg_grid > 0 && p.q_ctr) {
    // chunk schedule: MINB CTAs per SM pull work items until the queue is empty
    kern<<<seg_grid, 128 + 128 * TILES * SPLIT, bytes, s>>>(q);
    return cudaGetLastError();
  }
  q.q_ctr = nullptr;
  kern<<<(n_envs + per_cta - 1) / per_cta, 128 + 128 * TILES * SPLIT, bytes, s>>>(q);
  return cudaGetLastError();
}

}  // namespace tc
