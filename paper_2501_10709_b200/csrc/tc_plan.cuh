// tc_plan.cuh -- compile-time weight-streaming plan shared by the host packer
// (api.cu, fin_policy_create) and the tcgen05 kernels, so both agree on the
// packed layout by construction.
//
// A 3-layer MLP in -> HID -> HID -> OUT (BASELINE configs[1]: 301-256-256-30,
// configs[3]: 103-128-128-3) is cut into "stages": runs of K-steps (16 input
// features each, the bf16 UMMA K) of one layer, at most STAGE_BYTES each.  A
// stage is stored in global memory exactly as its shared-memory image: the
// SWIZZLE_NONE K-major canonical layout of 8-row x 16-byte core matrices,
//     byte(n, k) = ((n / 8) * (Kt / 8) + k / 8) * 128 + (n % 8) * 16 + (k % 8) * 2
// with Kt = 16 * (k-steps in the stage), so one 1-D bulk copy (cp.async.bulk)
// lands a stage ready for tcgen05.mma (LBO = 128 B, SBO = Kt / 8 * 128 B).
#pragma once

template <int IN_PAD, int HID, int OUT_PAD, int STAGE_BYTES>
struct TcPlan {
  static_assert(IN_PAD % 16 == 0 && HID % 16 == 0 && OUT_PAD % 16 == 0, "dims must be multiples of 16");
  static_assert(HID <= 256 && OUT_PAD <= 256 && OUT_PAD >= 16, "UMMA N range (M = 128)");
  static constexpr int kIn = IN_PAD, kHid = HID, kOut = OUT_PAD, kStageBytes = STAGE_BYTES;
  __host__ __device__ static constexpr int ksteps(int l) { return l == 0 ? IN_PAD / 16 : HID / 16; }
  __host__ __device__ static constexpr int nrows(int l) { return l == 2 ? OUT_PAD : HID; }
  __host__ __device__ static constexpr int kdim(int l) { return l == 0 ? IN_PAD : HID; }
  __host__ __device__ static constexpr int kps(int l) {
    return (STAGE_BYTES / (nrows(l) * 32)) < ksteps(l) ? (STAGE_BYTES / (nrows(l) * 32)) : ksteps(l);
  }
  __host__ __device__ static constexpr int nstages(int l) { return (ksteps(l) + kps(l) - 1) / kps(l); }
  static constexpr int kStages = nstages(0) + nstages(1) + nstages(2);
  __host__ __device__ static constexpr int first_stage(int l) {
    return l == 0 ? 0 : (l == 1 ? nstages(0) : nstages(0) + nstages(1));
  }
  // stage s -> layer, first k-step, number of k-steps, bytes, byte offset in the packed member
  __host__ __device__ static constexpr int layer_of(int s) {
    return s < nstages(0) ? 0 : (s < nstages(0) + nstages(1) ? 1 : 2);
  }
  __host__ __device__ static constexpr int j0_of(int s) { return (s - first_stage(layer_of(s))) * kps(layer_of(s)); }
  __host__ __device__ static constexpr int nks_of(int s) {
    return (ksteps(layer_of(s)) - j0_of(s)) < kps(layer_of(s)) ? (ksteps(layer_of(s)) - j0_of(s))
                                                               : kps(layer_of(s));
  }
  __host__ __device__ static constexpr int bytes_of(int s) { return nrows(layer_of(s)) * nks_of(s) * 32; }
  // layers are stored back to back; inside a layer every stage but the last is full
  __host__ __device__ static constexpr int layer_base(int l) {
    return l == 0 ? 0 : (l == 1 ? HID * IN_PAD * 2 : HID * IN_PAD * 2 + HID * HID * 2);
  }
  __host__ __device__ static constexpr int offset_of(int s) {
    return layer_base(layer_of(s)) + (s - first_stage(layer_of(s))) * kps(layer_of(s)) * nrows(layer_of(s)) * 32;
  }
  static constexpr int kMemberBytes = 2 * (HID * IN_PAD + HID * HID + OUT_PAD * HID);
  static constexpr int kBiasFloats = HID + HID + OUT_PAD;
  static constexpr long kFlopsPerRow = 2L * (HID * (long)IN_PAD + HID * (long)HID + OUT_PAD * (long)HID);
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
//   stock C1 policy  301-256-256-30  -> factored layer 1 K = 32 (31 private inputs), (32, 256, 32)
//   stock small test  25-128-128-4   -> factored layer 1 K = 16 (5 private inputs),   (16, 128, 16)
//   crypto C3 Q-net  103-128-128-3   -> (112, 128, 16)   (every input is read from the step's row)
using ObsC1 = StockObs<30, 8>;
using ObsSmall = StockObs<4, 4>;
#ifndef FIN_C1_STAGE
#define FIN_C1_STAGE 16384   // weight-stage bytes of the streamed C1 plan
#endif
using PlanStockC1 = TcPlan<ObsC1::kEnvPad, 256, 32, FIN_C1_STAGE>;
using PlanStockSmall = TcPlan<ObsSmall::kEnvPad, 128, 16, 16384>;
using PlanCrypto = TcPlan<112, 128, 16, 32768>;
