// tc_plan.cuh -- compile-time weight-streaming plan shared by the host packer
// (api.cu, fin_policy_create) and the tcgen05 kernels, so both agree on the
// packed layout by construction.
//
// An MLP in -> H1 -> H2 [-> H3] -> OUT (BASELINE configs[1]: 301-256-256-30,
// configs[3]: 103-128-128-3; the paper's own 301-64-32-30 and 103-128x3-3) is
// cut into "stages": runs of K-steps (16 input
// features each, the bf16 UMMA K) of one layer, at most STAGE_BYTES each.  A
// stage is stored in global memory exactly as its shared-memory image: the
// SWIZZLE_NONE K-major canonical layout of 8-row x 16-byte core matrices,
//     byte(n, k) = ((n / 8) * (Kt / 8) + k / 8) * 128 + (n % 8) * 16 + (k % 8) * 2
// with Kt = 16 * (k-steps in the stage), so one 1-D bulk copy (cp.async.bulk)
// lands a stage ready for tcgen05.mma (LBO = 128 B, SBO = Kt / 8 * 128 B).
#pragma once

template <int IN_PAD, int H1, int H2, int OUT_PAD, int STAGE_BYTES, int H3 = 0>
struct TcPlan {
  static_assert(IN_PAD % 16 == 0 && H1 % 16 == 0 && H2 % 16 == 0 && H3 % 16 == 0 && OUT_PAD % 16 == 0,
                "dims must be multiples of 16");
  static_assert(H1 <= 256 && H2 <= 256 && H3 <= 256 && OUT_PAD <= 256 && OUT_PAD >= 16, "UMMA N range (M = 128)");
  // hidden layers kNH = 2 (in-H1-H2-out) or 3 (in-H1-H2-H3-out); layers kNL = kNH + 1
  static constexpr int kNH = H3 > 0 ? 3 : 2, kNL = kNH + 1;
  static constexpr int kIn = IN_PAD, kOut = OUT_PAD, kStageBytes = STAGE_BYTES;
  static constexpr int kH1 = H1;   // first hidden width (the factored layer-1 shared term z1s)
  static constexpr int kHidMax = H1 > H2 ? (H1 > H3 ? H1 : H3) : (H2 > H3 ? H2 : H3);
  __host__ __device__ static constexpr int hid(int l) { return l == 0 ? H1 : (l == 1 ? H2 : H3); }
  __host__ __device__ static constexpr int nrows(int l) { return l < kNH ? hid(l) : OUT_PAD; }
  __host__ __device__ static constexpr int kdim(int l) { return l == 0 ? IN_PAD : hid(l - 1); }
  __host__ __device__ static constexpr int ksteps(int l) { return kdim(l) / 16; }
  __host__ __device__ static constexpr int kps(int l) {
    return (STAGE_BYTES / (nrows(l) * 32)) < ksteps(l) ? (STAGE_BYTES / (nrows(l) * 32)) : ksteps(l);
  }
  __host__ __device__ static constexpr int nstages(int l) { return (ksteps(l) + kps(l) - 1) / kps(l); }
  // (loop-free: these run per stage in the producer / MMA warps with a runtime l or s)
  __host__ __device__ static constexpr int first_stage(int l) {
    return (l > 0 ? nstages(0) : 0) + (l > 1 ? nstages(1) : 0) + (l > 2 ? nstages(2) : 0) +
           (l > 3 ? nstages(3) : 0);
  }
  static constexpr int kStages = first_stage(kNL);
  // stage s -> layer, first k-step, number of k-steps, bytes, byte offset in the packed member
  __host__ __device__ static constexpr int layer_of(int s) {
    return (s >= first_stage(1) ? 1 : 0) + (s >= first_stage(2) ? 1 : 0) + (kNL > 3 && s >= first_stage(3) ? 1 : 0);
  }
  __host__ __device__ static constexpr int j0_of(int s) { return (s - first_stage(layer_of(s))) * kps(layer_of(s)); }
  __host__ __device__ static constexpr int nks_of(int s) {
    return (ksteps(layer_of(s)) - j0_of(s)) < kps(layer_of(s)) ? (ksteps(layer_of(s)) - j0_of(s))
                                                               : kps(layer_of(s));
  }
  __host__ __device__ static constexpr int bytes_of(int s) { return nrows(layer_of(s)) * nks_of(s) * 32; }
  // layers are stored back to back; inside a layer every stage but the last is full
  __host__ __device__ static constexpr int layer_base(int l) {
    return (l > 0 ? nrows(0) * kdim(0) * 2 : 0) + (l > 1 ? nrows(1) * kdim(1) * 2 : 0) +
           (l > 2 ? nrows(2) * kdim(2) * 2 : 0) + (l > 3 ? nrows(3) * kdim(3) * 2 : 0);
  }
  __host__ __device__ static constexpr int offset_of(int s) {
    return layer_base(layer_of(s)) + (s - first_stage(layer_of(s))) * kps(layer_of(s)) * nrows(layer_of(s)) * 32;
  }
  // fp32 biases of all layers back to back: [H1 | H2 | (H3) | OUT_PAD]
  __host__ __device__ static constexpr int bias_off(int l) {
    return (l > 0 ? nrows(0) : 0) + (l > 1 ? nrows(1) : 0) + (l > 2 ? nrows(2) : 0) + (l > 3 ? nrows(3) : 0);
  }
  static constexpr int kMemberBytes = layer_base(kNL);
  static constexpr int kBiasFloats = bias_off(kNL);
  static constexpr long kFlopsPerRow = (long)kMemberBytes;   // 2 * sum(nrows * kdim) = bf16 bytes
};

// byte offset of element (n, k) inside a stage image whose K extent is kt elements
__host__ __device__ inline int tc_cm_offset(int n, int k, int kt) {
  return ((n / 8) * (kt / 8) + k / 8) * 128 + (n % 8) * 16 + (k % 8) * 2;
}

// Stock observation split ("layer-1 factorisation").  The stock
// observation x = [b/b0, close_norm_d (K), h/max_trade (K), features_d (I*K)]
// has 1 + K env-private entries (cash, holdings) and K + I*K entries that depend
// only on the market day d.  Layer 1 is computed as
//     z1 = W1_env x_env + z1s[d] + b1,   z1s[d] = W1_shared x_shared(d)
// with W1_env = W1's private columns (a tcgen05 GEMM with K = 1 + K padded to 16) and
// z1s precomputed once per rollout for every market day (float64 accumulation,
// rounded once to fp32).  The result is the same linear map; only the rounding
// order differs, inside the fp32 accumulation bound of the layered parity check.
template <int KA, int IA>
struct StockObs {
  static constexpr int kIn = 1 + 2 * KA + IA * KA;      // 301 for C1
  static constexpr int kEnv = 1 + KA;                   // private entries
  static constexpr int kEnvPad = (kEnv + 15) / 16 * 16;  // UMMA K multiple
  static constexpr int kShared = kIn - kEnv;             // 270 for C1
  // full-observation column of private entry j (0 = cash, 1 + k = holding k)
  __host__ __device__ static constexpr int env_col(int j) { return j == 0 ? 0 : KA + j; }
  // full-observation column of shared entry s (close_norm first, then the features)
  __host__ __device__ static constexpr int shared_col(int s) { return s < KA ? 1 + s : 1 + 2 * KA + (s - KA); }
};

// The network shapes compiled into libfinenv.so (fin_policy_create rejects others).
//   stock C1 policy   301-256-256-30      -> factored layer 1 K = 32 (31 private inputs), (32, 256, 256, 32)
//   stock paper net   301-64-32-30        -> (32, 64, 32, 32): the paper's own PPO/SAC/DDPG net
//   stock small test   25-128-128-4       -> factored layer 1 K = 16 (5 private inputs),   (16, 128, 128, 16)
//   crypto C3 Q-net   103-128-128-3 / -4  -> (112, 128, 128, 16)   (every input is read from the step's row)
//   crypto paper net  103-128-128-128-3 / -4 -> (112, 128, 128, 128, 16): three 128-unit hidden layers
using ObsC1 = StockObs<30, 8>;
using ObsSmall = StockObs<4, 4>;
#ifndef FIN_C1_STAGE
#define FIN_C1_STAGE 16384   // weight-stage bytes of the streamed C1 plan
#endif
using PlanStockC1 = TcPlan<ObsC1::kEnvPad, 256, 256, 32, FIN_C1_STAGE>;
using PlanStockPaper = TcPlan<ObsC1::kEnvPad, 64, 32, 32, 16384>;
using PlanStockSmall = TcPlan<ObsSmall::kEnvPad, 128, 128, 16, 16384>;
using PlanCrypto = TcPlan<112, 128, 128, 16, 32768>;
using PlanCryptoPaper = TcPlan<112, 128, 128, 16, 32768, 128>;
