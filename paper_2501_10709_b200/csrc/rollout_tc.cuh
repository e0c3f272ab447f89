// rollout_tc.cuh -- the warp-specialised tcgen05 rollout kernel template (K3/K5/K7).
//
// One CTA owns a tile of 128 SubEnvs (UMMA M = 128: TMEM lane r <-> env r of the
// tile) for all T steps; env state stays in registers.  Per step and per
// ensemble member the policy MLP (BASELINE configs[1..3])
// runs as three tcgen05.mma GEMMs  D = A * W^T  with A (activations, bf16,
// K-major core-matrix layout in smem) and W (bf16 weights, streamed by 1-D bulk
// TMA into a ring of smem stages, or resident) accumulating fp32 in TMEM.
//
// Warp roles (192 threads):
//   warp 0       producer: streams weight stages global(L2) -> smem ring (cp.async.bulk)
//   warp 1       TMEM allocator + MMA issuer (one elected lane)
//   warps 2..5   "env" warpgroup: observation build, TMEM epilogues (bias, ReLU,
//                bf16), action sampling / ensemble averaging, the env transition
//                (trade, reward, done / reset) and online metrics -- thread r of
//                the group owns env r (warp w reads TMEM lanes 32*(w%4)..+31).
// Synchronisation (mbarriers): w_full / w_empty per ring slot (TMA <-> MMA),
// a_full (env -> MMA: A operand written, TMEM columns free), d_full (MMA commit ->
// env: accumulator ready).  Layer l+1's MMAs start when the epilogue of layer l
// has written its activations; the producer prefetches across layers and steps.
#pragma once
#include "fin_internal.cuh"
#include "sm100.cuh"
#include "tc_plan.cuh"

namespace tc {

constexpr int kTileM = 128;
constexpr int kThreads = 192;
constexpr int kEnvWarp0 = 2;
constexpr int kRing = 4;

struct TcParams {
  EnvDev e;
  TrajDev o;
  const uint8_t* wpack[FIN_MAX_MEMBERS];  // packed member weights (TcPlan layout)
  const float* bias[FIN_MAX_MEMBERS];     // [HID + HID + OUT_PAD] fp32 per member
  int32_t kinds[FIN_MAX_MEMBERS];
  float mw[FIN_MAX_MEMBERS];              // member weights (weighted mode)
  int32_t M;
  int32_t weighted;
  int32_t T;
  int32_t noise_mode;
  uint64_t noise_seed;
  const float* noise;                     // supplied noise
  // fin_ensemble_act: compute the (ensemble) action only, no env transition
  int32_t act_only;
  float* mean_out;                        // [N][K] averaged continuous action
  uint16_t* hid_out;                      // bf16 hidden activations (probe [B][2][HID]; rollout [T][M][N][2][HID])
  // K7 probe
  const uint16_t* x_in;
  float* z_out;
  int32_t B, in_dim, out_dim;
};

__device__ __forceinline__ uint32_t cm_off(int r, int kchunk, int kt8) {
  return (uint32_t)(((r >> 3) * kt8 + kchunk) * 128 + (r & 7) * 16);
}

// Shared-memory carve-up (dynamic smem, 1024-B aligned base).
constexpr int kSmemBudget = 232448 - 2048;  // 227 KB per CTA, minus static smem of the env ops

template <class Plan, bool RESIDENT>
struct Smem {
  static constexpr int kX = kTileM * Plan::kIn * 2;
  static constexpr int kH = kTileM * Plan::kHid * 2;
  static constexpr int kBias = FIN_MAX_MEMBERS * Plan::kBiasFloats * 4;
  static constexpr int kFree = kSmemBudget - kX - kH - kBias - 256;
  // members whose weights fit resident in shared memory (resident plans only)
  static constexpr int kResMembers = RESIDENT ? (kFree / Plan::kMemberBytes < FIN_MAX_MEMBERS
                                                     ? kFree / Plan::kMemberBytes : FIN_MAX_MEMBERS)
                                              : FIN_MAX_MEMBERS;
  static_assert(!RESIDENT || kResMembers >= 1, "resident network does not fit in shared memory");
  static constexpr int kW = RESIDENT ? Plan::kMemberBytes * kResMembers : kRing * Plan::kStageBytes;
  static constexpr int oX = 0, oH = oX + kX, oW = oH + kH, oBias = oW + kW, oBar = oBias + kBias;
  static constexpr int kBars = 2 * kRing + 2;
  static constexpr int kTotal = oBar + kBars * 8 + 16;
};

// ---------------------------------------------------------------------------------
// The kernel.  Ops supplies the env-side behaviour (see rollout_stock.cu etc.):
//   struct Ops {
//     struct State;
//     __device__ static void init(State&, const TcParams&, int env, int row);
//     __device__ static void build_obs(State&, const TcParams&, int env, int row, int t, uint32_t x_addr);
//     __device__ static void consume(State&, const TcParams&, int env, int t, int m, const float* z);
//     __device__ static uint16_t* hidden_ptr(State&, const TcParams&, int env, int t, int m, int l, int hid);
//     __device__ static void finish_step(State&, const TcParams&, int env, int t);
//     __device__ static void finalize(State&, const TcParams&, int env);
//   };
template <class Plan, bool RESIDENT, class Ops>
__global__ void __launch_bounds__(kThreads, 1) k_tc_rollout(const __grid_constant__ TcParams p) {
  using S = Smem<Plan, RESIDENT>;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sX = smem + S::oX;
  uint8_t* sH = smem + S::oH;
  uint8_t* sW = smem + S::oW;
  float* sBias = reinterpret_cast<float*>(smem + S::oBias);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + S::oBar);
  uint64_t* w_full = bars;
  uint64_t* w_empty = bars + kRing;
  uint64_t* a_full = bars + 2 * kRing;
  uint64_t* d_full = bars + 2 * kRing + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + S::oBar + S::kBars * 8);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int M = p.M;
  const int T = p.T;
  constexpr int NS = Plan::kStages;

  // ---- one-time setup
  for (int j = threadIdx.x; j < M * Plan::kBiasFloats; j += blockDim.x) {
    const int m = j / Plan::kBiasFloats, q = j % Plan::kBiasFloats;
    sBias[j] = p.bias[m] ? p.bias[m][q] : 0.f;
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < kRing; ++s) {
      sm100::mbar_init(&w_full[s], 1);
      sm100::mbar_init(&w_empty[s], 1);
    }
    sm100::mbar_init(a_full, 4 * 32);
    sm100::mbar_init(d_full, 1);
    sm100::fence_mbar_init();
  }
  if (warp == 1) {
    sm100::tmem_alloc(tmem_slot, Plan::kHid <= 128 ? 128 : 256);
    sm100::tmem_relinquish();
  }
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

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
        for (int t = 0; t < T; ++t)
          for (int m = 0; m < M; ++m)
            for (int s = 0; s < NS; ++s, ++it) {
              const uint32_t slot = it % kRing, ph = (it / kRing) & 1;
              sm100::mbar_wait(&w_empty[slot], ph ^ 1);
              sm100::mbar_arrive_expect_tx(&w_full[slot], (uint32_t)Plan::bytes_of(s));
              sm100::bulk_g2s_hint(sW + slot * Plan::kStageBytes, p.wpack[m] + Plan::offset_of(s),
                                   (uint32_t)Plan::bytes_of(s), &w_full[slot], pol);
            }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ============================ MMA issuer ============================
    if (lane == 0) {
      uint32_t it = 0, a_use = 0;
      if (RESIDENT) {
        sm100::mbar_wait(&w_full[0], 0);
      }
      const uint32_t xa = sm100::smem_u32(sX), ha = sm100::smem_u32(sH), wa = sm100::smem_u32(sW);
      for (int t = 0; t < T; ++t) {
        for (int m = 0; m < M; ++m) {
#pragma unroll 1
          for (int l = 0; l < 3; ++l) {
            sm100::mbar_wait(a_full, a_use & 1);
            ++a_use;
            sm100::tc_fence_after();
            const uint32_t a_base = (l == 0) ? xa : ha;
            const uint32_t a_sbo = (uint32_t)(Plan::kdim(l) / 8) * 128u;
            const uint32_t idesc = sm100::make_idesc_bf16(kTileM, Plan::nrows(l));
            for (int s = Plan::first_stage(l); s < Plan::first_stage(l) + Plan::nstages(l); ++s) {
              uint32_t b_base;
              if (RESIDENT) {
                b_base = wa + (uint32_t)(m * Plan::kMemberBytes + Plan::offset_of(s));
              } else {
                const uint32_t slot = it % kRing, ph = (it / kRing) & 1;
                sm100::mbar_wait(&w_full[slot], ph);
                sm100::tc_fence_after();
                b_base = wa + slot * (uint32_t)Plan::kStageBytes;
              }
              const int j0 = Plan::j0_of(s), nks = Plan::nks_of(s);
              const uint32_t b_sbo = (uint32_t)(nks * 2) * 128u;  // Kt/8 * 128 with Kt = 16 nks
              for (int j = 0; j < nks; ++j) {
                const uint64_t ad = sm100::make_sdesc(a_base + (uint32_t)(j0 + j) * 256u, 128u, a_sbo);
                const uint64_t bd = sm100::make_sdesc(b_base + (uint32_t)j * 256u, 128u, b_sbo);
                sm100::mma_bf16(tmem, ad, bd, idesc, (j0 + j) > 0 ? 1u : 0u);
              }
              if (!RESIDENT) {
                sm100::mma_commit(&w_empty[it % kRing]);
                ++it;
              }
            }
            sm100::mma_commit(d_full);
          }
        }
      }
    }
    __syncwarp();
  } else {
    // ============================ env warpgroup ============================
    const int q = warp & 3;                 // TMEM lane quarter this warp may access
    const int row = q * 32 + lane;          // env row of the tile == TMEM lane
    const int env = blockIdx.x * kTileM + row;
    const uint32_t t_lane = tmem + ((uint32_t)(q * 32) << 16);
    const uint32_t xa = sm100::smem_u32(sX), ha = sm100::smem_u32(sH);
    typename Ops::State st;
    Ops::init(st, p, env, row);
    uint32_t d_use = 0;
    for (int t = 0; t < T; ++t) {
      Ops::build_obs(st, p, env, row, t, xa);
      sm100::fence_proxy_async_smem();
      sm100::tc_fence_before();
      sm100::mbar_arrive(a_full);
      for (int m = 0; m < M; ++m) {
        const float* bias = sBias + m * Plan::kBiasFloats;
        // hidden layers: D -> +bias -> ReLU -> bf16 -> H (K-major core matrices)
#pragma unroll 1
        for (int l = 0; l < 2; ++l) {
          sm100::mbar_wait(d_full, d_use & 1);
          ++d_use;
          sm100::tc_fence_after();
          const float* bl = bias + l * Plan::kHid;
          // debug / parity log of the bf16 hidden activations (teacher-forced layer checks)
          uint4* hlog = reinterpret_cast<uint4*>(Ops::hidden_ptr(st, p, env, t, m, l, Plan::kHid));
#pragma unroll 1
          for (int c = 0; c < Plan::kHid / 32; ++c) {
            uint32_t v[32];
            sm100::tmem_ld32(t_lane + (uint32_t)(c * 32), v);
            sm100::tmem_wait_ld();
            uint32_t pk[16];
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              const float a0 = fmaxf(__uint_as_float(v[2 * j]) + bl[c * 32 + 2 * j], 0.f);
              const float a1 = fmaxf(__uint_as_float(v[2 * j + 1]) + bl[c * 32 + 2 * j + 1], 0.f);
              pk[j] = sm100::pack_bf16(a0, a1);
            }
#pragma unroll
            for (int g = 0; g < 4; ++g)
              sm100::st_shared_v4(ha + cm_off(row, c * 4 + g, Plan::kHid / 8), pk[4 * g], pk[4 * g + 1],
                                  pk[4 * g + 2], pk[4 * g + 3]);
            if (hlog) {
#pragma unroll
              for (int g = 0; g < 4; ++g) hlog[c * 4 + g] = make_uint4(pk[4 * g], pk[4 * g + 1], pk[4 * g + 2], pk[4 * g + 3]);
            }
          }
          sm100::fence_proxy_async_smem();
          sm100::tc_fence_before();
          sm100::mbar_arrive(a_full);
        }
        // output layer
        sm100::mbar_wait(d_full, d_use & 1);
        ++d_use;
        sm100::tc_fence_after();
        float z[Plan::kOut];
#pragma unroll
        for (int c = 0; c < Plan::kOut / 16; ++c) {
          uint32_t v[16];
          sm100::tmem_ld16(t_lane + (uint32_t)(c * 16), v);
          sm100::tmem_wait_ld();
#pragma unroll
          for (int j = 0; j < 16; ++j) z[c * 16 + j] = __uint_as_float(v[j]) + bias[2 * Plan::kHid + c * 16 + j];
        }
        sm100::tc_fence_before();
        if (m + 1 < M) sm100::mbar_arrive(a_full);   // X stays valid for the next member
        Ops::consume(st, p, env, t, m, z);
      }
      Ops::finish_step(st, p, env, t);
    }
    Ops::finalize(st, p, env);
  }
  __syncthreads();
  if (warp == 1) {
    sm100::tc_fence_after();
    sm100::tmem_dealloc(tmem, Plan::kHid <= 128 ? 128 : 256);
  }
}

}  // namespace tc
