// api.cu -- the C ABI of libfinenv.so (include/fin.h): argument validation,
// handle / memory management, weight packing, kernel dispatch.  Host code only.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <new>
#include <string>
#include <type_traits>
#include <algorithm>
#include <atomic>
#include <vector>

#include "fin_internal.cuh"
#include "rollout_tc.cuh"
#include "tc_plan.cuh"

namespace fin {
// n_envs rows; *tiles receives the tiles per CTA the launch used (agg partial rows
// = ceil(n_envs / (128 * tiles)) * tiles)
cudaError_t launch_stock_rollout(int net, const tc::TcParams& p, int n_envs, int* tiles, cudaStream_t s);
int stock_seg_grid(int net, const tc::TcParams& p, int n_envs);
int num_sms();
cudaError_t launch_pregen_noise(uint64_t seed, int64_t off, int N, int K, int M, int64_t t0, int T, float* out,
                                cudaStream_t s);
cudaError_t load_stream_noise();
cudaError_t launch_stream_noise(uint64_t seed, int64_t off, int N, int K, int M, int64_t t0, int T, float* out,
                                uint32_t* ready, int blocks, cudaStream_t s);
cudaError_t launch_crypto_market(int64_t steps, uint64_t seed, double sigma, double m0, double phi, float* rows,
                                 cudaStream_t s);
cudaError_t launch_stock_market(int D, int K, uint64_t seed, double mu, double sigma, double s0_lo, double s0_hi,
                                float* ohlcv, cudaStream_t s);
cudaError_t launch_ppo_grad(int B, int in, int H1, int H2, int K, const uint16_t* x, const uint16_t* hid,
                            const float* z, const float* a, const float* logp_old, const float* adv, double sigma,
                            double eps, const float* w2, const float* w3, float* dw1, float* db1, float* dw2,
                            float* db2, float* dw3, float* db3, double* stats, cudaStream_t s);
cudaError_t launch_adam(int64_t n, float* th, float* m, float* v, const float* g, int step, double lr, double b1,
                        double b2, double eps, cudaStream_t s);
cudaError_t launch_dqn_grad(int B, int in, int H1, int H2, int O, const uint16_t* x, const uint16_t* hid,
                            const float* out, const uint8_t* act, const float* rew, const uint8_t* done,
                            const float* qt, const float* qo, double gamma, int dueling, const float* w2,
                            const float* w3, float* dw1, float* db1, float* dw2, float* db2, float* dw3, float* db3,
                            double* stats, cudaStream_t s);
cudaError_t backward(int B, int in, int H1, int H2, int K, const uint16_t* x, const uint16_t* hid, const float* g3,
                     const float* w2, const float* w3, float* dw1, float* db1, float* dw2, float* db2, float* dw3,
                     float* db3, cudaStream_t s);
cudaError_t launch_concat_sa(int B, int S, const uint16_t* x, int K, const float* a, float* out, cudaStream_t s);
cudaError_t launch_squash(int B, int K, const float* z, const float* eps, double sigma, float* a, float* logp,
                          cudaStream_t s);
cudaError_t launch_critic_head(int B, const float* q, const float* r, const uint8_t* done, const float* q1n,
                               const float* q2n, const float* lpn, double gamma, double alpha, float* g, double* stats,
                               cudaStream_t s);
cudaError_t launch_actor_head(int B, int K, const float* a, const float* lp, const float* q1, const float* dq1,
                              const float* q2, const float* dq2, int ldq, double alpha, float* gz, double* stats,
                              cudaStream_t s);
cudaError_t launch_soft_update(int64_t n, float* t, const float* o, double tau, cudaStream_t s);
cudaError_t dense_forward(int B, int in, int H1, int H2, int O, const float* x, const float* w1, const float* b1,
                          const float* w2, const float* b2, const float* w3, const float* b3, float* hid, float* out,
                          cudaStream_t s);
cudaError_t dense_backward(int B, int in, int H1, int H2, int O, const float* x, const float* hid, const float* g3,
                           const float* w1, const float* w2, const float* w3, float* dw1, float* db1, float* dw2,
                           float* db2, float* dw3, float* db3, float* gx, cudaStream_t s);
cudaError_t launch_gather_obs(const EnvDev& e, const uint16_t* priv, int P, const int32_t* day, const int64_t* idx,
                              int B, uint16_t* x, cudaStream_t s);
cudaError_t launch_noise_at(uint64_t seed, int64_t off, int N, int64_t t_base, const int64_t* idx, int B, int K,
                            int member, float* out, cudaStream_t s);
cudaError_t launch_ppo_prepare(int B, int K, const float* z, const float* eps, double sigma, float* a, float* logp,
                               cudaStream_t s);
cudaError_t launch_to_bf16(int64_t n, const float* x, uint16_t* y, cudaStream_t s);
cudaError_t launch_policy_gather(int64_t n_pack, const int32_t* pack_src, const float* const (&w)[4], uint16_t* wpack,
                                 int64_t n_w1s, const int32_t* w1s_src, float* w1s, cudaStream_t s);
cudaError_t launch_gae(const float* rew, const float* val, const uint8_t* done, int T, int N, double gamma,
                       double lam, int normalise, float* adv, float* ret, cudaStream_t s);
cudaError_t launch_kl_diversity(const float* out, int M, int B, int K, int kind, double sigma, double* D,
                                cudaStream_t s);
cudaError_t launch_crypto_rollout(int net, const tc::TcParams& p, int n_envs, int* tiles, cudaStream_t s);
cudaError_t launch_mlp_probe(int net, const tc::TcParams& p, int n_rows, cudaStream_t s);
cudaError_t launch_z1s_market(int net, const float* w1s_t, const float* b1, int H, const EnvDev& e, float* z1s,
                              cudaStream_t s);
cudaError_t launch_z1s_probe(int net, const float* w1s_t, const float* b1, int H, const uint16_t* x, int B, int in_dim,
                             float* z1s,
                             cudaStream_t s);
}  // namespace fin

struct fin_env {
  fin_env_config cfg;
  EnvDev d;
  int device;
  cudaStream_t last_stream;
  void* state_mem;
  float* market_mem;
  double* agg_scratch;
  size_t agg_cap;  // rows of FIN_AGG_LEN
  float* z1s;      // factored layer 1: per-member shared term of every market day [M][rows][HID]
  size_t z1s_cap;  // floats
  std::vector<uint64_t> z1s_key;   // uids of the members z1s holds (empty: none)
  float* ou_mem;   // DDPG OU state [ou_slots][K][N] (grown on demand)
  // dynamic chunk schedule of the fused stock rollout (rollout_tc.cuh TcParams::q_ctr)
  uint32_t* q_ctr;      // work-item counter (zeroed before each launch)
  uint32_t seg_epoch;   // per-call value of the tiles' progress flags
  uint32_t ctr_seg, ctr_seg_fallback;   // rollouts launched with the chunk schedule / refused
  int seg_fallback_err;                 // cudaError_t of the last refusal
  // small-N rollouts: the step noise pre-drawn by k_pregen_noise
  float* noise_mem;     // [T][M][N][K] normals of the last pre-drawn rollout
  size_t noise_cap;     // floats
  uint32_t ctr_pregen;  // rollouts that ran on pre-drawn noise
  uint32_t* noise_ready;   // [ceil(T / FIN_NOISE_GROUP)] streamed mode: producer blocks finished per step group
  size_t ready_cap;
  cudaStream_t noise_side;              // streamed mode: the producer's stream (forked / joined per call)
  cudaEvent_t noise_fork, noise_join;
};

struct fin_policy {
  int32_t kind;
  int32_t net;                 // 0 stock C1, 1 stock small, 2 crypto, 3 stock paper net, 4 crypto paper net
  int32_t n_layers;            // 3 or 4
  int32_t dims[5];
  uint8_t* wpack;              // device, TcPlan layout (stock: layer 1 = private columns only)
  float* bias;                 // device, [H1 | H2 | (H3) | OUT_PAD] (TcPlan::bias_off)
  uint8_t bias_nz;             // bit l: layer l has a non-zero bias (an all-zero bias is skipped)
  float* w1s_t;                // stock: device [S][HID] shared columns of W1 (exact bf16 values), else null
  bool b1_in_z1s;              // factored stock net with a non-zero layer-1 bias: folded into z1s (f64)
  uint64_t uid;                // process-unique id (keys the env's z1s cache; addresses can be reused)
  int32_t* pack_src = nullptr; // device gather table of fin_policy_load: per bf16 of wpack (l << 24 | index) or -1
  int32_t* w1s_src = nullptr;  // ... per float of w1s_t: the index into W1, or -1
  int64_t n_pack = 0, n_w1s = 0;
  cudaEvent_t used;            // recorded on the stream of every call that reads the policy (destroy waits on it)
};

namespace {

uint64_t new_uid() {   // process-unique policy ids (key the envs' z1s caches)
  static std::atomic<uint64_t> next_uid{1};
  return next_uid.fetch_add(1);
}

thread_local std::string g_err;
unsigned long long* g_trace = nullptr;   // fin_debug_trace

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

int cuda_fail(cudaError_t e, const char* what) {
  return fail(FIN_E_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

#define FIN_CUDA(call)                                    \
  do {                                                    \
    cudaError_t _e = (call);                              \
    if (_e != cudaSuccess) return cuda_fail(_e, #call);   \
  } while (0)

inline cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }

int check_device(int ordinal) {
  cudaDeviceProp prop;
  cudaError_t e = cudaGetDeviceProperties(&prop, ordinal);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDeviceProperties");
  if (prop.major != 10 || prop.minor != 0)
    return fail(FIN_E_UNSUPPORTED, "device %d is sm_%d%d; libfinenv.so is built for sm_100a only", ordinal,
                prop.major, prop.minor);
  return FIN_OK;
}

TrajDev to_dev(const fin_traj* o) {
  TrajDev t;
  std::memset(&t, 0, sizeof(t));
  if (!o) return t;
  t.reward = o->reward;
  t.done = o->done;
  t.actions = o->actions;
  t.cash = o->cash;
  t.hold = o->hold;
  t.asset = o->asset;
  t.mlp_out = o->mlp_out;
  t.mlp_hidden = o->mlp_hidden;
  t.ep_metrics = o->ep_metrics;
  t.ep_count = o->ep_count;
  t.ep_capacity = o->ep_metrics ? o->ep_capacity : 0;
  t.agg_partial = nullptr;
  t.obs_private = o->obs_private;
  t.day = o->day;
  return t;
}

int ensure_agg(fin_env* env, size_t rows) {
  if (env->agg_cap >= rows) return FIN_OK;
  if (env->agg_scratch) cudaFree(env->agg_scratch);
  env->agg_scratch = nullptr;
  env->agg_cap = 0;
  FIN_CUDA(cudaMalloc(&env->agg_scratch, rows * FIN_AGG_LEN * sizeof(double)));
  env->agg_cap = rows;
  return FIN_OK;
}


// network id from (n_layers, dims), -1 if not compiled
int net_of(int n_layers, const int32_t* dims) {
  if (n_layers == 3) {
    if (dims[0] == 301 && dims[1] == 256 && dims[2] == 256 && dims[3] == 30) return 0;
    if (dims[0] == 25 && dims[1] == 128 && dims[2] == 128 && dims[3] == 4) return 1;
    if (dims[0] == 103 && dims[1] == 128 && dims[2] == 128 && (dims[3] == 3 || dims[3] == 4)) return 2;
    if (dims[0] == 301 && dims[1] == 64 && dims[2] == 32 && dims[3] == 30) return 3;
  }
  if (n_layers == 4 && dims[0] == 103 && dims[1] == 128 && dims[2] == 128 && dims[3] == 128 &&
      (dims[4] == 3 || dims[4] == 4))
    return 4;
  return -1;
}

// Obs = StockObs<..>: layer 1 keeps only W1's env-private columns (factored layer 1,
// tc_plan.cuh); the shared columns go to w1s (transposed [S][HID], float).
template <class Plan, class Obs>
void pack_member(const int32_t* dims, const uint16_t* const* w, const float* const* bias, std::vector<uint8_t>& wp,
                 std::vector<float>& bp, std::vector<float>* w1s) {
  constexpr bool kFactored = !std::is_void<Obs>::value;
  wp.assign(Plan::kMemberBytes, 0);
  for (int s = 0; s < Plan::kStages; ++s) {
    const int l = Plan::layer_of(s), j0 = Plan::j0_of(s), nks = Plan::nks_of(s);
    const int kt = nks * 16, rows = Plan::nrows(l);
    const int in_l = dims[l], out_l = dims[l + 1];
    uint8_t* base = wp.data() + Plan::offset_of(s);
    for (int n = 0; n < rows; ++n)
      for (int kk = 0; kk < kt; ++kk) {
        int k = j0 * 16 + kk;
        if constexpr (kFactored) {
          if (l == 0) k = k < Obs::kEnv ? Obs::env_col(k) : in_l;  // private column or padding
        }
        const uint16_t v = (n < out_l && k < in_l) ? w[l][(size_t)n * in_l + k] : (uint16_t)0;
        std::memcpy(base + tc_cm_offset(n, kk, kt), &v, 2);
      }
  }
  if constexpr (kFactored) {
    const int H = dims[1];
    w1s->assign((size_t)Obs::kShared * H, 0.f);
    for (int sidx = 0; sidx < Obs::kShared; ++sidx)
      for (int n = 0; n < H; ++n) {
        const uint32_t bits = (uint32_t)w[0][(size_t)n * dims[0] + Obs::shared_col(sidx)] << 16;
        float f;
        std::memcpy(&f, &bits, 4);
        (*w1s)[(size_t)sidx * H + n] = f;
      }
  }
  bp.assign(Plan::kBiasFloats, 0.f);
  for (int l = 0; l < Plan::kNL; ++l) {
    const int off = Plan::bias_off(l);
    if (bias && bias[l])
      for (int n = 0; n < dims[l + 1]; ++n) bp[off + n] = bias[l][n];
  }
}

// the same layout as a gather table (fin_policy_load on the device): src[i] = (l << 24) | (n in_l + k)
// for bf16 i of the image, -1 for padding; w1s_src[sidx H + n] = n in_0 + shared_col(sidx); bias_off[l]
template <class Plan, class Obs>
void index_member(const int32_t* dims, std::vector<int32_t>& src, std::vector<int32_t>& w1s_src,
                  std::vector<int>& bias_off, int& bias_floats) {
  constexpr bool kFactored = !std::is_void<Obs>::value;
  src.assign(Plan::kMemberBytes / 2, -1);
  for (int s = 0; s < Plan::kStages; ++s) {
    const int l = Plan::layer_of(s), j0 = Plan::j0_of(s), nks = Plan::nks_of(s);
    const int kt = nks * 16, rows = Plan::nrows(l);
    const int in_l = dims[l], out_l = dims[l + 1];
    const size_t base = Plan::offset_of(s);
    for (int n = 0; n < rows; ++n)
      for (int kk = 0; kk < kt; ++kk) {
        int k = j0 * 16 + kk;
        if constexpr (kFactored) {
          if (l == 0) k = k < Obs::kEnv ? Obs::env_col(k) : in_l;
        }
        if (n < out_l && k < in_l) src[(base + tc_cm_offset(n, kk, kt)) / 2] = (l << 24) | (n * in_l + k);
      }
  }
  w1s_src.clear();
  if constexpr (kFactored) {
    const int H = dims[1];
    w1s_src.assign((size_t)Obs::kShared * H, -1);
    for (int sidx = 0; sidx < Obs::kShared; ++sidx)
      for (int n = 0; n < H; ++n) w1s_src[(size_t)sidx * H + n] = n * dims[0] + Obs::shared_col(sidx);
  }
  bias_off.assign(Plan::kNL, 0);
  for (int l = 0; l < Plan::kNL; ++l) bias_off[l] = Plan::bias_off(l);
  bias_floats = Plan::kBiasFloats;
}

void index_any(int net, const int32_t* dims, std::vector<int32_t>& src, std::vector<int32_t>& w1s_src,
               std::vector<int>& bias_off, int& bias_floats) {
  if (net == 0) index_member<PlanStockC1, ObsC1>(dims, src, w1s_src, bias_off, bias_floats);
  else if (net == 1) index_member<PlanStockSmall, ObsSmall>(dims, src, w1s_src, bias_off, bias_floats);
  else if (net == 3) index_member<PlanStockPaper, ObsC1>(dims, src, w1s_src, bias_off, bias_floats);
  else if (net == 4) index_member<PlanCryptoPaper, void>(dims, src, w1s_src, bias_off, bias_floats);
  else index_member<PlanCrypto, void>(dims, src, w1s_src, bias_off, bias_floats);
}

void pack_any(int net, const int32_t* dims, const uint16_t* const* w, const float* const* b, std::vector<uint8_t>& wp,
              std::vector<float>& bp, std::vector<float>& w1s) {
  if (net == 0) pack_member<PlanStockC1, ObsC1>(dims, w, b, wp, bp, &w1s);
  else if (net == 1) pack_member<PlanStockSmall, ObsSmall>(dims, w, b, wp, bp, &w1s);
  else if (net == 3) pack_member<PlanStockPaper, ObsC1>(dims, w, b, wp, bp, &w1s);
  else if (net == 4) pack_member<PlanCryptoPaper, void>(dims, w, b, wp, bp, nullptr);
  else pack_member<PlanCrypto, void>(dims, w, b, wp, bp, nullptr);
}

bool finite_all(const float* x, int64_t n) {
  for (int64_t i = 0; i < n; ++i)
    if (!std::isfinite(x[i])) return false;
  return true;
}

}  // namespace

extern "C" {

const char* fin_last_error(void) { return g_err.c_str(); }
int fin_debug_trace(void* device_buffer) {
  g_trace = static_cast<unsigned long long*>(device_buffer);
  return FIN_OK;
}
int fin_abi_version(void) { return FIN_ABI_VERSION; }
int fin_device_check(int32_t ordinal) { return check_device(ordinal); }

int fin_env_create(const fin_env_config* cfg, const float* market, int64_t market_elems, void* stream,
                   fin_env** out) {
  if (!cfg || !market || !out) return fail(FIN_E_CONFIG, "fin_env_create: null argument");
  *out = nullptr;
  const fin_env_config& c = *cfg;
  if (c.task != FIN_STOCK && c.task != FIN_CRYPTO) return fail(FIN_E_CONFIG, "task must be FIN_STOCK or FIN_CRYPTO");
  if (c.num_envs < 1) return fail(FIN_E_CONFIG, "num_envs must be >= 1");
  if (c.num_rows < 2) return fail(FIN_E_CONFIG, "num_rows must be >= 2");
  if (c.episode_len < 1) return fail(FIN_E_CONFIG, "episode_len must be >= 1");
  if (!(c.initial_cash > 0) || !std::isfinite(c.initial_cash)) return fail(FIN_E_CONFIG, "initial_cash must be > 0");
  if (!(c.cost_rate >= 0 && c.cost_rate < 1)) return fail(FIN_E_CONFIG, "cost_rate must be in [0, 1)");
  if (!std::isfinite(c.reward_scale)) return fail(FIN_E_CONFIG, "reward_scale must be finite");
  int dev = 0;
  FIN_CUDA(cudaGetDevice(&dev));
  int rc = check_device(dev);
  if (rc != FIN_OK) return rc;

  EnvDev d;
  std::memset(&d, 0, sizeof(d));
  d.task = c.task;
  d.N = c.num_envs;
  d.rows = c.num_rows;
  d.L = c.episode_len;
  d.autoreset = c.autoreset ? 1 : 0;
  d.cash0 = c.initial_cash;
  d.rcash0 = 1.0 / c.initial_cash;
  d.cost = c.cost_rate;
  d.scale = c.reward_scale;
  d.up = 1.0 + c.cost_rate;
  d.dn = 1.0 - c.cost_rate;
  d.noise_std = c.noise_std;
  d.ou_theta = c.ou_theta;
  d.ou_sigma = c.ou_sigma;
  d.eps = c.epsilon;
  d.seed = c.seed;
  d.env_offset = c.env_offset;
  d.t_global = 0;
  int64_t expect = 0;
  if (c.task == FIN_STOCK) {
    if (c.num_assets < 1 || c.num_assets > FIN_MAX_ASSETS) return fail(FIN_E_CONFIG, "num_assets must be in [1, 32]");
    if (c.num_indicators < 0) return fail(FIN_E_CONFIG, "num_indicators must be >= 0");
    if (c.max_trade < 1 || c.max_trade > FIN_HOLD_MAX) return fail(FIN_E_CONFIG, "max_trade must be in [1, 32767]");
    if (c.num_windows < 1 || c.window_block < 1 || c.window_stride < 0 || c.window_offset < 0 || c.window_base < 0)
      return fail(FIN_E_CONFIG, "window parameters invalid");
    // every window's last transition reads row start + L, which must exist
    const int64_t last = (int64_t)c.window_offset + (int64_t)(c.num_windows - 1) * c.window_stride + c.episode_len;
    if (last >= c.num_rows)
      return fail(FIN_E_CONFIG, "windows exceed the market: last row %lld >= num_rows %d", (long long)last, c.num_rows);
    d.K = c.num_assets;
    d.I = c.num_indicators;
    d.kp = (c.num_assets + 3) / 4 * 4;
    d.row_floats = (2 + c.num_indicators) * d.kp;
    d.wstride = c.window_stride;
    d.woff = c.window_offset;
    d.W = c.num_windows;
    d.wblock = c.window_block;
    d.wbase = c.window_base;
    d.wadv = c.advance_window_on_reset ? 1 : 0;
    d.max_trade = c.max_trade;
    expect = (int64_t)c.num_rows * (2 + c.num_indicators) * c.num_assets;
  } else {
    if (c.num_assets != 1) return fail(FIN_E_CONFIG, "crypto env: num_assets must be 1");
    if (c.pos_limit != 1) return fail(FIN_E_CONFIG, "crypto env: pos_limit must be 1");
    if (c.max_hold < 1) return fail(FIN_E_CONFIG, "crypto env: max_hold must be >= 1");
    if (c.episode_len >= c.num_rows) return fail(FIN_E_CONFIG, "crypto env: episode_len must be < num_rows");
    d.K = 1;
    d.I = 0;
    d.kp = 1;
    d.row_floats = 144;
    d.W = 1;
    d.wblock = 1;
    d.max_trade = 1;
    d.max_hold = c.max_hold;
    expect = (int64_t)c.num_rows * 144;
  }
  d.rmax_trade = 1.f / (float)d.max_trade;
  d.rmax_hold = d.max_hold > 0 ? 1.f / (float)d.max_hold : 0.f;
  if (market_elems != expect)
    return fail(FIN_E_CONFIG, "market_elems %lld != expected %lld", (long long)market_elems, (long long)expect);
  // ---- validate the market: finite, prices > 0
  if (!finite_all(market, market_elems)) return fail(FIN_E_DATA, "market contains non-finite values");
  std::vector<float> padded;
  const float* upload = market;
  if (c.task == FIN_STOCK) {
    const int K = c.num_assets, C = 2 + c.num_indicators;
    for (int r = 0; r < c.num_rows; ++r)
      for (int k = 0; k < K; ++k)
        if (!(market[(size_t)r * C * K + k] > 0.f))
          return fail(FIN_E_DATA, "close price <= 0 at row %d asset %d", r, k);
    padded.assign((size_t)c.num_rows * d.row_floats, 0.f);
    for (int r = 0; r < c.num_rows; ++r)
      for (int ch = 0; ch < C; ++ch)
        for (int k = 0; k < K; ++k)
          padded[(size_t)r * d.row_floats + ch * d.kp + k] = market[((size_t)r * C + ch) * K + k];
    upload = padded.data();
  } else {
    for (int r = 0; r < c.num_rows; ++r) {
      const float* row = market + (size_t)r * 144;
      if (!(row[0] > 0.f)) return fail(FIN_E_DATA, "mid price <= 0 at row %d", r);
      for (int l = 0; l < 10; ++l)
        if (!(row[1 + l] > 0.f) || !(row[21 + l] > 0.f) || row[11 + l] < 0.f || row[31 + l] < 0.f)
          return fail(FIN_E_DATA, "invalid book level at row %d", r);
    }
  }
  fin_env* env = new (std::nothrow) fin_env();
  if (!env) return fail(FIN_E_CONFIG, "out of host memory");
  env->cfg = c;
  env->device = dev;
  env->last_stream = S(stream);
  const size_t N = (size_t)c.num_envs, K = (size_t)d.K;
  // one allocation for all state arrays (8-byte members first)
  const size_t n8 = N * 8;  // cash + 6 metric doubles
  size_t bytes = 8 * n8 * sizeof(double) / 8;   // 8 double arrays
  bytes += N * 4 * sizeof(int32_t);              // t_ep, window, tau, m_n
  bytes += N * FIN_AGG_LEN * sizeof(double) + 16; // per-env aggregate partials
  bytes += N * (sizeof(int32_t) + sizeof(double)) + 32;   // seg_cnt, seg_rsum
  bytes += ((N + 127) / 128) * sizeof(uint32_t) + 16;      // seg_flag
  const size_t KO = (K + 7) / 8;                 // holdings: asset octets (hold_at)
  bytes += KO * 8 * N * sizeof(int16_t);
  bytes += 256;
  cudaError_t e;
  if ((e = cudaMalloc(&env->state_mem, bytes)) != cudaSuccess) { delete env; return cuda_fail(e, "cudaMalloc(state)"); }
  if ((e = cudaMemset(env->state_mem, 0, bytes)) != cudaSuccess) {
    cudaFree(env->state_mem);
    delete env;
    return cuda_fail(e, "cudaMemset(state)");
  }
  uint8_t* p = static_cast<uint8_t*>(env->state_mem);
  auto take = [&](size_t b) { uint8_t* r = p; p += (b + 15) / 16 * 16; return r; };
  d.cash = reinterpret_cast<double*>(take(N * 8));
  d.vcur = reinterpret_cast<double*>(take(N * 8));
  d.m_v0 = reinterpret_cast<double*>(take(N * 8));
  d.m_vprev = reinterpret_cast<double*>(take(N * 8));
  d.m_peak = reinterpret_cast<double*>(take(N * 8));
  d.m_mdd = reinterpret_cast<double*>(take(N * 8));
  d.m_mean = reinterpret_cast<double*>(take(N * 8));
  d.m_m2 = reinterpret_cast<double*>(take(N * 8));
  d.ou = nullptr;      // DDPG OU slots: allocated by the first rollout with DDPG members
  d.ou_slots = 0;
  d.t_ep = reinterpret_cast<int32_t*>(take(N * 4));
  d.window = reinterpret_cast<int32_t*>(take(N * 4));
  d.tau = reinterpret_cast<int32_t*>(take(N * 4));
  d.m_n = reinterpret_cast<int32_t*>(take(N * 4));
  d.hold = reinterpret_cast<int16_t*>(take(KO * 8 * N * 2));
  d.agg_env = reinterpret_cast<double*>(take(N * FIN_AGG_LEN * 8));
  d.seg_rsum = reinterpret_cast<double*>(take(N * 8));
  d.seg_cnt = reinterpret_cast<int32_t*>(take(N * 4));
  d.seg_flag = reinterpret_cast<uint32_t*>(take(((N + 127) / 128) * 4));
  if ((size_t)(p - static_cast<uint8_t*>(env->state_mem)) > bytes) {
    cudaFree(env->state_mem);
    delete env;
    return fail(FIN_E_CONFIG, "internal: state layout overflow");
  }
  // market copy | flags word | (stock) f64 price rows px[rows][kPriceRows][kp]
  // (fin_internal.cuh), each entry one IEEE double operation on the host: p exact,
  // u = fl(p (1 + c)), the -2^52 scalings exact, fl(1 / u); padding assets stay 0
  const size_t mbytes = (size_t)c.num_rows * d.row_floats * sizeof(float);
  std::vector<double> px;
  if (c.task == FIN_STOCK) {
    const double m52 = -4503599627370496.0;
    px.assign((size_t)c.num_rows * kPriceRows * d.kp, 0.0);
    for (int r = 0; r < c.num_rows; ++r)
      for (int k = 0; k < d.K; ++k) {
        double* row = px.data() + (size_t)r * kPriceRows * d.kp;
        const double pk = (double)padded[(size_t)r * d.row_floats + k];
        const double uk = pk * d.up;
        const double pn = r + 1 < c.num_rows ? (double)padded[(size_t)(r + 1) * d.row_floats + k] : 0.0;
        row[kRowP * d.kp + k] = pk;
        row[kRowU * d.kp + k] = uk;
        row[kRowMP * d.kp + k] = pk * m52;
        row[kRowMU * d.kp + k] = uk * m52;
        row[kRowRU * d.kp + k] = (1.0 / uk) * (1.0 + 0x1p-40);   // biased up (env_stock.cuh buy_want)
        row[kRowPN * d.kp + k] = pn;
        row[kRowMPN * d.kp + k] = pn * m52;
        double& umin = row[kRowMeta * d.kp];
        umin = (k == 0 || uk < umin) ? uk : umin;
      }
  }
  const size_t pxbytes = px.size() * sizeof(double);
  if ((e = cudaMalloc(&env->market_mem, mbytes + 64 + pxbytes)) != cudaSuccess) {
    cudaFree(env->state_mem);
    delete env;
    return cuda_fail(e, "cudaMalloc(market)");
  }
  d.flags = reinterpret_cast<uint32_t*>(reinterpret_cast<uint8_t*>(env->market_mem) + mbytes);
  d.market = env->market_mem;
  d.px = pxbytes ? reinterpret_cast<const double*>(reinterpret_cast<uint8_t*>(env->market_mem) + mbytes + 64)
                 : nullptr;
  cudaStream_t s = S(stream);
  e = cudaMemcpyAsync(env->market_mem, upload, mbytes, cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess && pxbytes)
    e = cudaMemcpyAsync(const_cast<double*>(d.px), px.data(), pxbytes, cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess) e = cudaMemsetAsync(d.flags, 0, 64, s);
  env->d = d;
  if (e == cudaSuccess)
    e = (c.task == FIN_STOCK) ? fin::launch_stock_reset(d, nullptr, s) : fin::launch_crypto_reset(d, nullptr, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) {
    cudaFree(env->market_mem);
    cudaFree(env->state_mem);
    delete env;
    return cuda_fail(e, "fin_env_create upload/reset");
  }
  *out = env;
  return FIN_OK;
}

int fin_env_reset(fin_env* env, const uint8_t* mask, void* stream) {
  if (!env) return fail(FIN_E_CONFIG, "null env");
  env->last_stream = S(stream);
  cudaError_t e = env->d.task == FIN_STOCK ? fin::launch_stock_reset(env->d, mask, S(stream))
                                           : fin::launch_crypto_reset(env->d, mask, S(stream));
  if (e != cudaSuccess) return cuda_fail(e, "fin_env_reset");
  return FIN_OK;
}

int fin_env_step(fin_env* env, const int16_t* actions, const fin_traj* out, void* stream) {
  if (!env || !actions) return fail(FIN_E_CONFIG, "fin_env_step: null argument");
  env->last_stream = S(stream);
  TrajDev o = to_dev(out);
  o.ep_metrics = nullptr;
  o.ep_count = nullptr;
  cudaError_t e = env->d.task == FIN_STOCK ? fin::launch_stock_step(env->d, actions, o, S(stream))
                                           : fin::launch_crypto_step(env->d, actions, o, S(stream));
  if (e != cudaSuccess) return cuda_fail(e, "fin_env_step");
  env->d.t_global += 1;
  return FIN_OK;
}

int fin_env_get_state(const fin_env* env, double* cash, int16_t* hold, double* asset, int32_t* t_ep,
                      int32_t* window, void* stream) {
  if (!env) return fail(FIN_E_CONFIG, "null env");
  cudaError_t e;
  if (env->d.task == FIN_STOCK)
    e = fin::launch_stock_get_state(env->d, cash, hold, asset, t_ep, window, S(stream));
  else {
    e = fin::launch_crypto_get_state(env->d, cash, hold, asset, t_ep, S(stream));
    if (e == cudaSuccess && window) e = cudaMemsetAsync(window, 0, sizeof(int32_t) * env->d.N, S(stream));
  }
  if (e != cudaSuccess) return cuda_fail(e, "fin_env_get_state");
  return FIN_OK;
}

int fin_env_set_state(fin_env* env, const double* cash, const int16_t* hold, const int32_t* t_ep,
                      const int32_t* window, const int32_t* tau, void* stream) {
  if (!env) return fail(FIN_E_CONFIG, "null env");
  env->last_stream = S(stream);
  cudaError_t e = env->d.task == FIN_STOCK
                      ? fin::launch_stock_set_state(env->d, cash, hold, t_ep, window, S(stream))
                      : fin::launch_crypto_set_state(env->d, cash, hold, t_ep, tau, S(stream));
  if (e != cudaSuccess) return cuda_fail(e, "fin_env_set_state");
  return FIN_OK;
}

int fin_env_check(fin_env* env, uint32_t* flags) {
  if (!env) return fail(FIN_E_CONFIG, "null env");
  FIN_CUDA(cudaStreamSynchronize(env->last_stream));
  uint32_t f = 0;
  FIN_CUDA(cudaMemcpy(&f, env->d.flags, sizeof(f), cudaMemcpyDeviceToHost));
  FIN_CUDA(cudaMemset(env->d.flags, 0, sizeof(uint32_t)));
  if (flags) *flags = f;
  if (f) return fail(FIN_E_DEVICE_ASYNC, "device flags 0x%x (1 action range, 2 episode done, 4 non-finite, 8 index, 16 noise wait)", f);
  return FIN_OK;
}

int fin_env_counters(fin_env* env, uint32_t* counters, int32_t clear) {
  if (!env || !counters) return fail(FIN_E_CONFIG, "fin_env_counters: null argument");
  FIN_CUDA(cudaStreamSynchronize(env->last_stream));
  FIN_CUDA(cudaMemcpy(counters, env->d.flags + FIN_CTR_EXACT_REDO, FIN_CTR_LEN * sizeof(uint32_t),
                      cudaMemcpyDeviceToHost));
  counters[1] = env->ctr_seg;
  counters[2] = env->ctr_seg_fallback;
  counters[3] = (uint32_t)env->seg_fallback_err;
  counters[4] = env->ctr_pregen;
  if (clear) {
    FIN_CUDA(cudaMemset(env->d.flags + FIN_CTR_EXACT_REDO, 0, FIN_CTR_LEN * sizeof(uint32_t)));
    env->ctr_seg = env->ctr_seg_fallback = env->ctr_pregen = 0;
  }
  return FIN_OK;
}

void fin_env_destroy(fin_env* env) {
  if (!env) return;
  cudaStreamSynchronize(env->last_stream);
  if (env->q_ctr) cudaFree(env->q_ctr);
  if (env->noise_mem) cudaFree(env->noise_mem);
  if (env->noise_ready) cudaFree(env->noise_ready);
  if (env->noise_side) cudaStreamDestroy(env->noise_side);
  if (env->noise_fork) cudaEventDestroy(env->noise_fork);
  if (env->noise_join) cudaEventDestroy(env->noise_join);
  if (env->agg_scratch) cudaFree(env->agg_scratch);
  if (env->z1s) cudaFree(env->z1s);
  if (env->ou_mem) cudaFree(env->ou_mem);
  if (env->market_mem) cudaFree(env->market_mem);
  if (env->state_mem) cudaFree(env->state_mem);
  delete env;
}

int fin_policy_create(int32_t kind, int32_t n_layers, const int32_t* dims, const uint16_t* const* w_bf16,
                      const float* const* bias, void* stream, fin_policy** out) {
  if (!dims || !w_bf16 || !out) return fail(FIN_E_CONFIG, "fin_policy_create: null argument");
  *out = nullptr;
  if (kind < FIN_PPO_GAUSS || kind > FIN_Q_DUELING) return fail(FIN_E_CONFIG, "unknown policy kind %d", kind);
  if (n_layers != 3 && n_layers != 4)
    return fail(FIN_E_UNSUPPORTED, "only 3- and 4-layer networks are compiled (got %d)", n_layers);
  for (int l = 0; l < n_layers; ++l)
    if (!w_bf16[l]) return fail(FIN_E_CONFIG, "weight %d is null", l);
  const int net = net_of(n_layers, dims);
  if (net < 0)
    return fail(FIN_E_UNSUPPORTED,
                "network %d-%d-%d-%d%s not compiled (have 301-256-256-30, 301-64-32-30, 25-128-128-4, "
                "103-128-128-3 / -4, 103-128-128-128-3 / -4)",
                dims[0], dims[1], dims[2], dims[3], n_layers == 4 ? "-.." : "");
  const bool qkind = kind == FIN_Q_ARGMAX || kind == FIN_Q_DUELING;
  const bool qnet = net == 2 || net == 4;
  const int n_out = dims[n_layers];
  if (qnet != qkind) return fail(FIN_E_CONFIG, "Q kinds pair with the 103-128-.. Q-nets");
  if (kind == FIN_Q_ARGMAX && n_out != 3) return fail(FIN_E_CONFIG, "Q_ARGMAX needs 3 outputs");
  if (kind == FIN_Q_DUELING && n_out != 4) return fail(FIN_E_CONFIG, "Q_DUELING needs 4 outputs (A0..A2, V)");
  for (int l = 0; l < n_layers; ++l) {
    if (bias && bias[l] && !finite_all(bias[l], dims[l + 1])) return fail(FIN_E_DATA, "bias %d non-finite", l);
  }
  std::vector<uint8_t> wp;
  std::vector<float> bp, w1s;
  pack_any(net, dims, w_bf16, bias, wp, bp, w1s);
  fin_policy* pol = new (std::nothrow) fin_policy();
  if (!pol) return fail(FIN_E_CONFIG, "out of host memory");
  pol->uid = new_uid();
  pol->kind = kind;
  pol->net = net;
  pol->n_layers = n_layers;
  pol->bias_nz = 0;
  for (int l = 0; l < n_layers; ++l)
    if (bias && bias[l])
      for (int n = 0; n < dims[l + 1]; ++n)
        if (bias[l][n] != 0.f) pol->bias_nz |= 1u << l;
  if (!w1s.empty() && (pol->bias_nz & 1u)) {   // z1s carries b1: epilogues never add it
    pol->b1_in_z1s = true;
    pol->bias_nz &= ~1u;
  }
  for (int l = 0; l < 5; ++l) pol->dims[l] = l <= n_layers ? dims[l] : 0;
  cudaError_t e = cudaMalloc(&pol->wpack, wp.size());
  if (e == cudaSuccess) e = cudaMalloc(&pol->bias, bp.size() * sizeof(float));
  if (e == cudaSuccess && !w1s.empty()) e = cudaMalloc(&pol->w1s_t, w1s.size() * sizeof(float));
  if (e == cudaSuccess) e = cudaMemcpyAsync(pol->wpack, wp.data(), wp.size(), cudaMemcpyHostToDevice, S(stream));
  if (e == cudaSuccess) e = cudaMemcpyAsync(pol->bias, bp.data(), bp.size() * 4, cudaMemcpyHostToDevice, S(stream));
  if (e == cudaSuccess && !w1s.empty())
    e = cudaMemcpyAsync(pol->w1s_t, w1s.data(), w1s.size() * 4, cudaMemcpyHostToDevice, S(stream));
  if (e == cudaSuccess) e = cudaStreamSynchronize(S(stream));
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&pol->used, cudaEventDisableTiming);
  if (e != cudaSuccess) {
    if (pol->wpack) cudaFree(pol->wpack);
    if (pol->bias) cudaFree(pol->bias);
    if (pol->w1s_t) cudaFree(pol->w1s_t);
    delete pol;
    return cuda_fail(e, "fin_policy_create upload");
  }
  *out = pol;
  return FIN_OK;
}

int fin_policy_load(fin_policy* pol, const float* const* w, const float* const* bias, void* stream) {
  if (!pol || !w) return fail(FIN_E_CONFIG, "fin_policy_load: null argument");
  const int L = pol->n_layers;
  for (int l = 0; l < L; ++l)
    if (!w[l]) return fail(FIN_E_CONFIG, "fin_policy_load: weight %d is null", l);
  cudaStream_t s = S(stream);
  // the gather tables of this network's image (built once per handle, host layout code only)
  std::vector<int> boff;
  int bfloats = 0;
  {
    std::vector<int32_t> src, w1s_src;
    index_any(pol->net, pol->dims, src, w1s_src, boff, bfloats);
    if (!pol->pack_src) {
      FIN_CUDA(cudaMalloc(&pol->pack_src, src.size() * sizeof(int32_t)));
      FIN_CUDA(cudaMemcpy(pol->pack_src, src.data(), src.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
      pol->n_pack = (int64_t)src.size();
      if (!w1s_src.empty()) {
        FIN_CUDA(cudaMalloc(&pol->w1s_src, w1s_src.size() * sizeof(int32_t)));
        FIN_CUDA(cudaMemcpy(pol->w1s_src, w1s_src.data(), w1s_src.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
        pol->n_w1s = (int64_t)w1s_src.size();
      }
    }
  }
  // stream-ordered after the last call that read the old image (any stream)
  if (pol->used) FIN_CUDA(cudaStreamWaitEvent(s, pol->used, 0));
  const float* wl[4] = {w[0], w[1], w[2], L > 3 ? w[3] : nullptr};
  cudaError_t e = fin::launch_policy_gather(pol->n_pack, pol->pack_src, wl, reinterpret_cast<uint16_t*>(pol->wpack),
                                            pol->n_w1s, pol->w1s_src, pol->w1s_t, s);
  if (e == cudaSuccess) e = cudaMemsetAsync(pol->bias, 0, (size_t)bfloats * sizeof(float), s);
  uint8_t nz = 0;
  for (int l = 0; l < L && e == cudaSuccess; ++l)
    if (bias && bias[l]) {
      e = cudaMemcpyAsync(pol->bias + boff[l], bias[l], (size_t)pol->dims[l + 1] * sizeof(float),
                          cudaMemcpyDeviceToDevice, s);
      nz |= (uint8_t)(1u << l);   // added whether or not it is all zero (+0 is the identity up to a zero's sign)
    }
  if (e != cudaSuccess) return cuda_fail(e, "fin_policy_load");
  pol->b1_in_z1s = pol->w1s_t != nullptr && (nz & 1u);
  pol->bias_nz = pol->b1_in_z1s ? (uint8_t)(nz & ~1u) : nz;
  if (pol->used) cudaEventRecord(pol->used, s);   // the new image is being written on s
  pol->uid = new_uid();   // envs recompute their z1s term for the new weights
  return FIN_OK;
}

void fin_policy_destroy(fin_policy* pol) {
  if (!pol) return;
  if (pol->used) {   // wait for the last call that read the weights (not for the whole device)
    cudaEventSynchronize(pol->used);
    cudaEventDestroy(pol->used);
  }
  cudaFree(pol->wpack);
  cudaFree(pol->bias);
  if (pol->w1s_t) cudaFree(pol->w1s_t);
  if (pol->pack_src) cudaFree(pol->pack_src);
  if (pol->w1s_src) cudaFree(pol->w1s_src);
  delete pol;
}

}  // extern "C"

namespace {

// host packing of one member's bf16 weights into the tcgen05 image of its plan (fin_policy_create,
// fin_policy_load): layout only, no arithmetic
void pack_any(int net, const int32_t* dims, const uint16_t* const* w, const float* const* b, std::vector<uint8_t>& wp,
              std::vector<float>& bp, std::vector<float>& w1s);
void index_any(int net, const int32_t* dims, std::vector<int32_t>& src, std::vector<int32_t>& w1s_src,
               std::vector<int>& bias_off, int& bias_floats);

// every policy of a call records its `used` event on the call's stream after the launch
void mark_used(const fin_policy* const* members, int n, cudaStream_t s) {
  for (int m = 0; m < n; ++m)
    if (members[m] && members[m]->used) cudaEventRecord(members[m]->used, s);
}

// DDPG OU state: one [K][N] slot per DDPG member, grown on demand (existing slots kept)
int ensure_ou_slots(fin_env* env, int n, cudaStream_t s) {
  if (n <= env->d.ou_slots) return FIN_OK;
  const size_t slot = (size_t)env->d.K * env->d.N * sizeof(float);
  float* mem = nullptr;
  FIN_CUDA(cudaMalloc(&mem, n * slot));
  FIN_CUDA(cudaMemsetAsync(mem, 0, n * slot, s));
  if (env->ou_mem) {
    FIN_CUDA(cudaMemcpyAsync(mem, env->ou_mem, env->d.ou_slots * slot, cudaMemcpyDeviceToDevice, s));
    FIN_CUDA(cudaStreamSynchronize(s));
    cudaFree(env->ou_mem);
  }
  env->ou_mem = mem;
  env->d.ou = mem;
  env->d.ou_slots = n;
  return FIN_OK;
}

int fill_members(fin_env* env, const fin_policy* const* members, int32_t n, const float* member_w,
                 tc::TcParams& p, int* net_out, cudaStream_t s) {
  if (!members || n < 1 || n > FIN_MAX_MEMBERS) return fail(FIN_E_CONFIG, "n_members must be in [1, %d]", FIN_MAX_MEMBERS);
  int net = -1, n_ddpg = 0;
  for (int m = 0; m < n; ++m) {
    if (!members[m]) return fail(FIN_E_CONFIG, "member %d is null", m);
    if (net >= 0 && members[m]->net != net) return fail(FIN_E_CONFIG, "members must share one network shape");
    net = members[m]->net;
    p.wpack[m] = members[m]->wpack;
    p.bias[m] = members[m]->bias;
    p.bias_nz[m] = members[m]->bias_nz;
    p.kinds[m] = members[m]->kind;
    p.ou_slot[m] = members[m]->kind == FIN_DDPG_OU ? (int8_t)(n_ddpg++) : (int8_t)-1;
    p.mw[m] = member_w ? member_w[m] : 1.f;
  }
  p.n_ddpg = n_ddpg;
  if (n_ddpg > 0) {
    const int rc = ensure_ou_slots(env, n_ddpg, s);
    if (rc != FIN_OK) return rc;
  }
  if (env->d.task == FIN_STOCK) {
    if (net == 2 || net == 4) return fail(FIN_E_CONFIG, "stock env needs a stock policy");
    const int need_k = net == 1 ? 4 : 30, need_i = net == 1 ? 4 : 8;
    if (env->d.K != need_k || env->d.I != need_i)
      return fail(FIN_E_UNSUPPORTED, "policy network expects K=%d, I=%d; env has K=%d, I=%d", need_k, need_i,
                  env->d.K, env->d.I);
  } else {
    if (net != 2 && net != 4) return fail(FIN_E_CONFIG, "crypto env takes Q_ARGMAX / Q_DUELING members");
    if (member_w) return fail(FIN_E_CONFIG, "crypto ensembles vote: member_w must be NULL");
  }
  p.M = n;
  p.inv_m = 1.f / (float)n;
  p.weighted = member_w ? 1 : 0;
  *net_out = net;
  return FIN_OK;
}

// Factored stock layer 1: the shared-input term of every market day for every member
// (z1s = W1_shared q(x_shared(d)), tc_plan.cuh; 1008 x 270 x 256 FMAs).  Kept per env
// and recomputed only when the member list changes (policies and the env's market copy
// are immutable after creation; policies are keyed by their process-unique uid).
int prepare_z1s(fin_env* env, const fin_policy* const* members, int n, int net, tc::TcParams& p, cudaStream_t s) {
  if (env->d.task != FIN_STOCK) return FIN_OK;
  const int H = members[0]->dims[1];
  std::vector<uint64_t> key(n);
  for (int m = 0; m < n; ++m) key[m] = members[m]->uid;
  if (env->z1s && key == env->z1s_key) {
    p.z1s = env->z1s;
    p.z1s_rows = env->d.rows;
    return FIN_OK;
  }
  env->z1s_key.clear();
  const size_t need = (size_t)n * env->d.rows * H;
  if (env->z1s_cap < need) {
    if (env->z1s) cudaFree(env->z1s);
    env->z1s = nullptr;
    env->z1s_cap = 0;
    FIN_CUDA(cudaMalloc(&env->z1s, need * sizeof(float)));
    env->z1s_cap = need;
  }
  for (int m = 0; m < n; ++m) {
    cudaError_t e = fin::launch_z1s_market(net, members[m]->w1s_t, members[m]->b1_in_z1s ? members[m]->bias : nullptr,
                                           H, env->d, env->z1s + (size_t)m * env->d.rows * H, s);
    if (e != cudaSuccess) return cuda_fail(e, "z1s precompute");
  }
  env->z1s_key = key;
  p.z1s = env->z1s;
  p.z1s_rows = env->d.rows;
  return FIN_OK;
}

// The dynamic chunk schedule (rollout_tc.cuh TcParams::q_ctr): the T steps
// of every tile are cut into chunks of decreasing length -- a quarter of the remaining
// steps, between 8 and max(64, T / 8) -- so the last rounds of work items are short and
// the CTAs (whose speeds differ by a few percent) finish together.
int chunk_plan(int T, int32_t* t0, int max_chunks) {
  int n = 0, pos = 0;
  const int cap = T / 8 > 64 ? T / 8 : 64;
  while (pos < T && n < max_chunks - 1) {
    const int rem = T - pos;
    int c = rem / 4;
    c = c < 8 ? 8 : (c > cap ? cap : c);
    if (c > rem) c = rem;
    t0[n++] = pos;
    pos += c;
  }
  if (pos < T) t0[n++] = pos;   // (cap reached: one last chunk takes the rest)
  t0[n] = T;
  return n;
}

int prepare_chunks(fin_env* env, int n_tiles, int T, int grid, tc::TcParams& p) {
  if (!env->q_ctr) FIN_CUDA(cudaMalloc(&env->q_ctr, 64));
  p.n_chunks = chunk_plan(T, p.chunk_t0, 17);
  p.n_tiles = n_tiles;
  p.q_ctr = env->q_ctr;
  p.seg_flag = env->d.seg_flag;
  if (++env->seg_epoch >= (1u << 24)) {   // epoch << 8 would wrap: clear the flags, restart at 1
    FIN_CUDA(cudaMemsetAsync(env->d.seg_flag, 0, ((env->d.N + 127) / 128) * sizeof(uint32_t), env->last_stream));
    env->seg_epoch = 1;
  }
  p.seg_epoch = env->seg_epoch;
  p.seg_grid = grid;
  FIN_CUDA(cudaMemsetAsync(env->q_ctr, 0, sizeof(uint32_t), env->last_stream));
  return FIN_OK;
}

int fill_noise(const fin_noise* noise, tc::TcParams& p) {
  if (!noise) {
    p.noise_mode = FIN_NOISE_NONE;
    return FIN_OK;
  }
  if (noise->mode < FIN_NOISE_PHILOX || noise->mode > FIN_NOISE_NONE) return fail(FIN_E_CONFIG, "bad noise mode");
  if (noise->mode == FIN_NOISE_SUPPLIED && !noise->supplied) return fail(FIN_E_CONFIG, "supplied noise is null");
  p.noise_mode = noise->mode;
  p.noise_seed = noise->seed;
  p.noise = noise->supplied;
  return FIN_OK;
}

// Small N (fewer tiles than SMs: the fused rollout is latency-bound on each tile's serial step
// chain): the rollout's Philox normals are drawn by a separate kernel and read
// as supplied noise, taking the Philox / Box-Muller work off the chain -- bitwise the in-kernel
// draws (same counters, same philox_normals8_v).  "Streamed" (FIN_PREGEN=2): the
// producer k_stream_noise runs on the idle SMs concurrently with the rollout (a side stream
// forked after the flag reset and joined after the rollout) and publishes each finished group of
// 8 steps in noise_ready[t / 8]; used when the idle SMs number at least half the tiles (A/B,
// scripts/pregen_ab.py, N x 256 steps: +8.0% at N = 64, +7.3% at 2,048, +5.4% at 8,192, +5.0% at
// 12,288 = 96 tiles; -10.7% at 16,384, whose 20 idle SMs cannot keep up).  FIN_PREGEN=1: the whole
// buffer drawn before the rollout (k_pregen_noise; A/B: +10.9% at N = 64, +6.5% at 2,048 x 30
// (streamed +3.1%), -0.8% at 8,192 x 256); FIN_PREGEN=0: in-kernel draws.  Large N keeps the in-kernel draws,
// which ride on issue slots the env phases leave idle.
constexpr size_t kPregenCapBytes = size_t(1) << 30;
struct NoisePlan {
  int mode = 0;   // 0 none, 1 drawn before the rollout, 2 streamed (producer launched after it)
  int blocks = 0;
  size_t elems = 0;
};
int plan_noise(fin_env* env, tc::TcParams& p, int n_tiles, int T, cudaStream_t s, NoisePlan& np) {
  np = NoisePlan();
  if (env->d.task != FIN_STOCK || p.act_only) return FIN_OK;
  const int free_sms = fin::num_sms() - n_tiles;
  if (free_sms < 0) return FIN_OK;   // more tiles than SMs: the large-N layouts
  const size_t groups = ((size_t)T + FIN_NOISE_GROUP - 1) / FIN_NOISE_GROUP;
  if (env->ready_cap < groups) {
    if (env->noise_ready) cudaFree(env->noise_ready);   // synchronises: no rollout still reads it
    env->noise_ready = nullptr;
    env->ready_cap = 0;
    FIN_CUDA(cudaMalloc(&env->noise_ready, groups * sizeof(uint32_t)));
    env->ready_cap = groups;
  }
  const size_t elems = (size_t)T * p.M * env->d.N * env->d.K;
  const char* force = getenv("FIN_PREGEN");
  // Philox noise, default: drawn before the rollout up to 2,048 env-members (its cost ~N T / 7,700 us
  // against a gain of ~T us: it pays below ~7,700 envs, and beats streaming where the producer's
  // start-up shows, e.g. T = 30), streamed while the idle SMs number at least half the tiles,
  // else in-kernel.  Mode 4 (and any supplied / no noise): the small-N kernel with every step
  // complete from the start (target 0) -- its column-split epilogues without a noise pass.
  int mode = 4;
  if (p.noise_mode == FIN_NOISE_PHILOX)
    mode = force ? atoi(force) : (2 * free_sms < n_tiles ? 4 : (size_t)p.M * env->d.N <= 2048 ? 1 : 2);
  if (mode == 2 && free_sms < 1) mode = 4;   // the producer needs SMs the rollout's tiles leave free
  if (mode == 2 && getenv("FIN_SEG_PROF")) mode = 1;   // that debug path synchronises right after the launch
  if (mode != 4 && elems * sizeof(float) > kPregenCapBytes) mode = 4;
  if (mode < 1 || mode > 4) return FIN_OK;   // 0: in-kernel draws, one env warpgroup (A/B);
                                             // 3 (A/B only): the streamed path with the producer run first
  if (mode == 4) {
    p.noise_ready = env->noise_ready;
    p.noise_ready_target = 0;
    return FIN_OK;
  }
  if (env->noise_cap < elems) {
    if (env->noise_mem) cudaFree(env->noise_mem);   // synchronises: no rollout still reads it
    env->noise_mem = nullptr;
    env->noise_cap = 0;
    FIN_CUDA(cudaMalloc(&env->noise_mem, elems * sizeof(float)));
    env->noise_cap = elems;
  }
  if (mode == 1) {
    cudaError_t e = fin::launch_pregen_noise(p.noise_seed, env->d.env_offset, env->d.N, env->d.K, p.M,
                                             env->d.t_global, T, env->noise_mem, s);
    if (e != cudaSuccess) return cuda_fail(e, "fin_rollout pre-drawn noise");
    // the small-N (STREAM) kernel with every step complete from the start (target 0): its
    // column-split epilogues, no waits
    p.noise_ready = env->noise_ready;
    p.noise_ready_target = 0;
  } else {
    cudaError_t le = fin::load_stream_noise();   // before the rollout that will wait on it
    if (le != cudaSuccess) return cuda_fail(le, "fin_rollout streamed noise (load)");
    if (!env->noise_side) {
      FIN_CUDA(cudaStreamCreateWithFlags(&env->noise_side, cudaStreamNonBlocking));
      FIN_CUDA(cudaEventCreateWithFlags(&env->noise_fork, cudaEventDisableTiming));
      FIN_CUDA(cudaEventCreateWithFlags(&env->noise_join, cudaEventDisableTiming));
    }
    FIN_CUDA(cudaMemsetAsync(env->noise_ready, 0, groups * sizeof(uint32_t), s));
    FIN_CUDA(cudaEventRecord(env->noise_fork, s));   // the producer waits for the reset only
    const size_t per_t = (size_t)p.M * env->d.N * ((env->d.K + 7) / 8);
    const size_t need = (per_t + 511) / 512;   // 512-thread blocks, one per idle SM
    np.blocks = (int)std::min<size_t>(need, (size_t)std::max(free_sms, 1));
    p.noise_ready = env->noise_ready;
    p.noise_ready_target = (uint32_t)np.blocks;
    if (mode == 3) {
      cudaError_t e3 = fin::launch_stream_noise(p.noise_seed, env->d.env_offset, env->d.N, env->d.K, p.M,
                                                env->d.t_global, T, env->noise_mem, env->noise_ready, np.blocks, s);
      if (e3 != cudaSuccess) return cuda_fail(e3, "fin_rollout streamed noise");
    }
  }
  p.noise_mode = FIN_NOISE_SUPPLIED;
  p.noise = env->noise_mem;
  np.mode = mode;
  np.elems = elems;
  ++env->ctr_pregen;
  return FIN_OK;
}

// streamed mode, after the rollout's launch (so its tiles take their SMs first): the producer
// on the side stream, then the caller's stream joins it
int launch_noise_producer(fin_env* env, const tc::TcParams& p, const NoisePlan& np, int T, cudaStream_t s) {
  if (np.mode != 2) return FIN_OK;
  FIN_CUDA(cudaStreamWaitEvent(env->noise_side, env->noise_fork, 0));
  cudaError_t e = fin::launch_stream_noise(p.noise_seed, env->d.env_offset, env->d.N, env->d.K, p.M,
                                           env->d.t_global, T, env->noise_mem, env->noise_ready, np.blocks,
                                           env->noise_side);
  if (e != cudaSuccess) return cuda_fail(e, "fin_rollout streamed noise");
  FIN_CUDA(cudaEventRecord(env->noise_join, env->noise_side));
  FIN_CUDA(cudaStreamWaitEvent(s, env->noise_join, 0));
  return FIN_OK;
}

}  // namespace

extern "C" {

int fin_rollout(fin_env* env, const fin_policy* const* members, int32_t n_members, const float* member_w, int32_t T,
                const fin_noise* noise, const fin_traj* out, void* stream) {
  if (!env) return fail(FIN_E_CONFIG, "null env");
  if (T < 0) return fail(FIN_E_CONFIG, "T must be >= 0");
  if (T == 0) return FIN_OK;
  tc::TcParams p;
  std::memset(&p, 0, sizeof(p));
  int net = -1;
  int rc = fill_members(env, members, n_members, member_w, p, &net, S(stream));
  if (rc != FIN_OK) return rc;
  rc = fill_noise(noise, p);
  if (rc != FIN_OK) return rc;
  rc = prepare_z1s(env, members, n_members, net, p, S(stream));
  if (rc != FIN_OK) return rc;
  const int n_tiles = (env->d.N + tc::kTileM - 1) / tc::kTileM;
  NoisePlan np;
  rc = plan_noise(env, p, n_tiles, T, S(stream), np);
  if (rc != FIN_OK) return rc;
  p.e = env->d;
  p.o = to_dev(out);
  p.T = T;
  p.trace = g_trace;
  if (out && out->agg) {
    rc = ensure_agg(env, (size_t)n_tiles + 2);
    if (rc != FIN_OK) return rc;
    p.o.agg_partial = env->agg_scratch;
  }
  env->last_stream = S(stream);
  if (env->d.task == FIN_STOCK) {
    const int grid = fin::stock_seg_grid(net, p, env->d.N);
    if (grid > 0) {
      rc = prepare_chunks(env, n_tiles, T, grid, p);
      if (rc != FIN_OK) return rc;
    }
    if (getenv("FIN_SEG_PROF")) {
      p.seg_grid = grid > 0 ? grid : n_tiles;
      FIN_CUDA(cudaMalloc(&p.seg_prof, (size_t)p.seg_grid * 16 * 8));
      FIN_CUDA(cudaMemset(p.seg_prof, 0, (size_t)p.seg_grid * 16 * 8));
    }
  }
  int tiles = 1;
  cudaError_t e = env->d.task == FIN_STOCK ? fin::launch_stock_rollout(net, p, env->d.N, &tiles, S(stream))
                                           : fin::launch_crypto_rollout(net, p, env->d.N, &tiles, S(stream));
  if (p.seg_prof) {   // debug: per-CTA segment timeline -> file FIN_SEG_PROF
    cudaStreamSynchronize(S(stream));
    std::vector<unsigned long long> h((size_t)p.seg_grid * 16);
    cudaMemcpy(h.data(), p.seg_prof, h.size() * 8, cudaMemcpyDeviceToHost);
    cudaFree(p.seg_prof);
    if (FILE* f = fopen(getenv("FIN_SEG_PROF"), "wb")) {
      fwrite(h.data(), 8, h.size(), f);
      fclose(f);
    }
  }
  if (p.q_ctr) {
    if (e == cudaSuccess) {
      ++env->ctr_seg;
    } else {   // the balanced grid is not co-resident (cooperative launch refused): one tile per CTA
      (void)cudaGetLastError();
      ++env->ctr_seg_fallback;
      env->seg_fallback_err = (int)e;
      p.q_ctr = nullptr;
      e = fin::launch_stock_rollout(net, p, env->d.N, &tiles, S(stream));
    }
  }
  if (e == cudaSuccess) {
    rc = launch_noise_producer(env, p, np, T, S(stream));
    if (rc != FIN_OK) return rc;
  }
  mark_used(members, n_members, S(stream));
  if (e != cudaSuccess) return cuda_fail(e, "fin_rollout launch");
  if (out && out->agg) {
    const int rows = (env->d.N + tc::kTileM * tiles - 1) / (tc::kTileM * tiles) * tiles;
    e = fin::launch_agg_finalize(env->agg_scratch, rows, out->agg, S(stream));
    if (e != cudaSuccess) return cuda_fail(e, "fin_rollout agg");
  }
  env->d.t_global += T;
  return FIN_OK;
}

int fin_rollout_actions(fin_env* env, const int16_t* actions, int32_t T, const fin_traj* out, void* stream) {
  if (!env || !actions) return fail(FIN_E_CONFIG, "fin_rollout_actions: null argument");
  if (T < 0) return fail(FIN_E_CONFIG, "T must be >= 0");
  if (T == 0) return FIN_OK;
  if (env->d.task != FIN_STOCK) return fail(FIN_E_UNSUPPORTED, "fin_rollout_actions: stock envs only");
  TrajDev o = to_dev(out);
  const int nb = (env->d.N + 255) / 256;
  if (out && out->agg) {
    int rc = ensure_agg(env, (size_t)nb);
    if (rc != FIN_OK) return rc;
    o.agg_partial = env->agg_scratch;
  }
  env->last_stream = S(stream);
  int n_blocks = 0;
  cudaError_t e = fin::launch_stock_replay(env->d, actions, T, o, &n_blocks, S(stream));
  if (e != cudaSuccess) return cuda_fail(e, "fin_rollout_actions launch");
  if (out && out->agg) {
    e = fin::launch_agg_finalize(env->agg_scratch, n_blocks, out->agg, S(stream));
    if (e != cudaSuccess) return cuda_fail(e, "fin_rollout_actions agg");
  }
  env->d.t_global += T;
  return FIN_OK;
}

int fin_ensemble_act(fin_env* env, const fin_policy* const* members, int32_t n_members, const float* member_w,
                     const fin_noise* noise, int16_t* actions, float* mean_action, int32_t commit_ou,
                     void* stream) {
  if (!env || !actions) return fail(FIN_E_CONFIG, "fin_ensemble_act: null argument");
  if (env->d.task != FIN_STOCK) return fail(FIN_E_UNSUPPORTED, "fin_ensemble_act: stock envs only");
  tc::TcParams p;
  std::memset(&p, 0, sizeof(p));
  int net = -1;
  int rc = fill_members(env, members, n_members, member_w, p, &net, S(stream));
  if (rc != FIN_OK) return rc;
  rc = fill_noise(noise, p);
  if (rc != FIN_OK) return rc;
  rc = prepare_z1s(env, members, n_members, net, p, S(stream));
  if (rc != FIN_OK) return rc;
  p.e = env->d;   // supplied noise is read as [1][M][N][K]; Philox uses the env's current step
  p.T = 1;
  p.act_only = 1;
  p.commit_ou = commit_ou != 0;
  p.mean_out = mean_action;
  p.o.actions = actions;
  env->last_stream = S(stream);
  int tiles = 1;
  cudaError_t e = fin::launch_stock_rollout(net, p, env->d.N, &tiles, S(stream));
  mark_used(members, n_members, S(stream));
  if (e != cudaSuccess) return cuda_fail(e, "fin_ensemble_act launch");
  return FIN_OK;
}

int fin_episode_metrics(const double* equity, const uint8_t* done, int32_t T, int32_t N, double reset_equity,
                        double periods_per_year, double rf, double* ep_metrics, int32_t ep_capacity,
                        int32_t* ep_count, double* agg, void* stream) {
  if (!equity || !done) return fail(FIN_E_CONFIG, "fin_episode_metrics: null argument");
  if (T < 1 || N < 1) return fail(FIN_E_CONFIG, "T and N must be >= 1");
  if (!(periods_per_year > 0)) return fail(FIN_E_CONFIG, "periods_per_year must be > 0");
  double* partial = nullptr;
  const int env_blocks = (N + 127) / 128;
  const size_t max_rows = (size_t)env_blocks * 4096;
  cudaStream_t s = S(stream);
  if (agg) FIN_CUDA(cudaMallocAsync(&partial, max_rows * FIN_AGG_LEN * sizeof(double), s));
  int n_blocks = 0;
  cudaError_t e = fin::launch_episode_metrics(equity, done, T, N, reset_equity, periods_per_year, rf, ep_metrics,
                                              ep_metrics ? ep_capacity : 0, ep_count, partial, &n_blocks, s);
  if (e != cudaSuccess) return cuda_fail(e, "fin_episode_metrics launch");
  if (agg) {
    e = fin::launch_agg_finalize(partial, n_blocks, agg, s);
    cudaFreeAsync(partial, s);
    if (e != cudaSuccess) return cuda_fail(e, "fin_episode_metrics agg");
  }
  return FIN_OK;
}

int fin_mlp_forward(const fin_policy* pol, const uint16_t* x, int32_t B, float* z, uint16_t* hidden, void* stream) {
  if (!pol || !x || !z) return fail(FIN_E_CONFIG, "fin_mlp_forward: null argument");
  if (B < 1) return fail(FIN_E_CONFIG, "B must be >= 1");
  tc::TcParams p;
  std::memset(&p, 0, sizeof(p));
  p.wpack[0] = pol->wpack;
  p.bias[0] = pol->bias;
  p.kinds[0] = pol->kind;
  p.bias_nz[0] = pol->bias_nz;
  p.M = 1;
  p.inv_m = 1.f;
  p.T = 1;
  p.x_in = x;
  p.z_out = z;
  p.hid_out = hidden;
  p.B = B;
  p.in_dim = pol->dims[0];
  p.out_dim = pol->dims[pol->n_layers];
  float* z1s = nullptr;
  cudaStream_t s = S(stream);
  cudaError_t e = cudaSuccess;
  if (pol->w1s_t) {  // factored stock net: shared-input term of each probe row
    e = cudaMallocAsync(&z1s, sizeof(float) * (size_t)B * pol->dims[1], s);
    if (e == cudaSuccess)
      e = fin::launch_z1s_probe(pol->net, pol->w1s_t, pol->b1_in_z1s ? pol->bias : nullptr, pol->dims[1], x, B,
                                pol->dims[0], z1s, s);
    p.z1s = z1s;
  }
  if (e == cudaSuccess) e = fin::launch_mlp_probe(pol->net, p, B, s);
  if (pol->used) cudaEventRecord(pol->used, s);
  if (z1s) cudaFreeAsync(z1s, s);
  if (e != cudaSuccess) return cuda_fail(e, "fin_mlp_forward launch");
  return FIN_OK;
}

int fin_market_prepare(const float* ohlcv, int32_t D, int32_t K, int32_t warmup, const int32_t* indicators,
                       int32_t I, double magnitude, uint64_t seed, float* market, double* raw, void* stream) {
  if (!ohlcv || !market || !raw || (I > 0 && !indicators)) return fail(FIN_E_CONFIG, "fin_market_prepare: null argument");
  if (K < 1 || warmup < 0 || D - warmup < 1) return fail(FIN_E_CONFIG, "need K >= 1 and D > warmup >= 0");
  if (I < 0 || I > 16) return fail(FIN_E_CONFIG, "I must be in [0, 16]");
  for (int i = 0; i < I; ++i)
    if (indicators[i] < FIN_IND_MACD || indicators[i] > FIN_IND_SMA60)
      return fail(FIN_E_CONFIG, "unknown indicator id %d", indicators[i]);
  if (!(magnitude >= 0.0 && magnitude <= 0.1)) return fail(FIN_E_CONFIG, "magnitude must be in [0, 0.1]");
  cudaError_t e = fin::launch_market_prepare(ohlcv, D, K, warmup, indicators, I, magnitude, seed, market, raw,
                                             S(stream));
  if (e != cudaSuccess) return cuda_fail(e, "fin_market_prepare launch");
  return FIN_OK;
}

int fin_crypto_market(int64_t steps, uint64_t seed, double sigma, double m0, double phi, float* rows, void* stream) {
  if (!rows) return fail(FIN_E_CONFIG, "fin_crypto_market: null rows");
  if (steps < 1 || steps > (int64_t)1 << 31) return fail(FIN_E_CONFIG, "steps must be in [1, 2^31]");
  if (!(sigma >= 0.0) || !std::isfinite(sigma)) return fail(FIN_E_CONFIG, "sigma must be finite and >= 0");
  if (!(m0 > 0.0) || !std::isfinite(m0)) return fail(FIN_E_CONFIG, "m0 must be finite and > 0");
  if (!(phi >= 0.0 && phi < 1.0)) return fail(FIN_E_CONFIG, "phi must be in [0, 1)");
  cudaError_t e = fin::launch_crypto_market(steps, seed, sigma, m0, phi, rows, S(stream));
  if (e != cudaSuccess) return cuda_fail(e, "fin_crypto_market launch");
  return FIN_OK;
}

int fin_stock_market(int32_t days, int32_t K, uint64_t seed, double mu, double sigma, double s0_lo, double s0_hi,
                     float* ohlcv, void* stream) {
  if (!ohlcv) return fail(FIN_E_CONFIG, "fin_stock_market: null ohlcv");
  if (days < 1 || days > (1 << 24)) return fail(FIN_E_CONFIG, "days must be in [1, 2^24]");
  if (K < 1 || K > 4096) return fail(FIN_E_CONFIG, "K must be in [1, 4096]");
  if (!std::isfinite(mu)) return fail(FIN_E_CONFIG, "mu must be finite");
  if (!(sigma >= 0.0) || !std::isfinite(sigma)) return fail(FIN_E_CONFIG, "sigma must be finite and >= 0");
  if (!(s0_lo > 0.0 && s0_lo < s0_hi) || !std::isfinite(s0_hi))
    return fail(FIN_E_CONFIG, "need 0 < s0_lo < s0_hi < inf");
  cudaError_t e = fin::launch_stock_market(days, K, seed, mu, sigma, s0_lo, s0_hi, ohlcv, S(stream));
  if (e != cudaSuccess) return cuda_fail(e, "fin_stock_market launch");
  return FIN_OK;
}

int fin_ppo_grad(int32_t B, int32_t in_dim, int32_t h1, int32_t h2, int32_t k_out, const uint16_t* x,
                 const uint16_t* hidden, const float* z, const float* a, const float* logp_old, const float* adv,
                 double sigma, double clip_eps, const float* w2, const float* w3, float* dw1, float* db1, float* dw2,
                 float* db2, float* dw3, float* db3, double* stats, void* stream) {
  if (!x || !hidden || !z || !a || !logp_old || !adv || !w2 || !w3 || !dw1 || !db1 || !dw2 || !db2 || !dw3 || !db3 ||
      !stats)
    return fail(FIN_E_CONFIG, "fin_ppo_grad: null argument");
  if (B < 1 || in_dim < 1 || in_dim > 4096 || h1 < 1 || h1 > 1024 || h2 < 1 || h2 > 1024 || k_out < 1 || k_out > 64)
    return fail(FIN_E_CONFIG, "fin_ppo_grad: bad sizes");
  if (!(sigma > 0.0) || !std::isfinite(sigma) || !(clip_eps >= 0.0 && clip_eps < 1.0))
    return fail(FIN_E_CONFIG, "fin_ppo_grad: need sigma > 0 and 0 <= clip_eps < 1");
  cudaError_t e = fin::launch_ppo_grad(B, in_dim, h1, h2, k_out, x, hidden, z, a, logp_old, adv, sigma, clip_eps, w2, w3,
                                       dw1, db1, dw2, db2, dw3, db3, stats, S(stream));
  if (e != cudaSuccess) return cuda_fail(e, "fin_ppo_grad launch");
  return FIN_OK;
}

int fin_dqn_grad(int32_t B, int32_t in_dim, int32_t h1, int32_t h2, int32_t k_out, const uint16_t* x,
                 const uint16_t* hidden, const float* out, const uint8_t* action, const float* reward,
                 const uint8_t* done, const float* q_next_target, const float* q_next_online, double gamma,
                 int32_t dueling, const float* w2, const float* w3, float* dw1, float* db1, float* dw2, float* db2,
                 float* dw3, float* db3, double* stats, void* stream) {
  if (!x || !hidden || !out || !action || !reward || !done || !q_next_target || !w2 || !w3 || !dw1 || !db1 || !dw2 ||
      !db2 || !dw3 || !db3 || !stats)
    return fail(FIN_E_CONFIG, "fin_dqn_grad: null argument");
  if (B < 1 || in_dim < 1 || in_dim > 4096 || h1 < 1 || h1 > 1024 || h2 < 1 || h2 > 1024 || k_out < 2 || k_out > 8)
    return fail(FIN_E_CONFIG, "fin_dqn_grad: bad sizes");
  if (dueling && k_out < 3) return fail(FIN_E_CONFIG, "fin_dqn_grad: a dueling head needs >= 2 actions + V");
  if (!(gamma >= 0.0 && gamma <= 1.0)) return fail(FIN_E_CONFIG, "fin_dqn_grad: gamma must be in [0, 1]");
  cudaError_t e = fin::launch_dqn_grad(B, in_dim, h1, h2, k_out, x, hidden, out, action, reward, done, q_next_target,
                                       q_next_online, gamma, dueling, w2, w3, dw1, db1, dw2, db2, dw3, db3, stats,
                                       S(stream));
  if (e != cudaSuccess) return cuda_fail(e, "fin_dqn_grad launch");
  return FIN_OK;
}

static bool dense_sizes_ok(int32_t B, int32_t in, int32_t h1, int32_t h2, int32_t out) {
  return B >= 1 && in >= 1 && in <= 8192 && h1 >= 1 && h1 <= 4096 && h2 >= 1 && h2 <= 4096 && out >= 1 && out <= 4096;
}

int fin_dense_forward(int32_t B, int32_t in_dim, int32_t h1, int32_t h2, int32_t out_dim, const float* x,
                      const float* w1, const float* b1, const float* w2, const float* b2, const float* w3,
                      const float* b3, float* hidden, float* out, void* stream) {
  if (!x || !w1 || !b1 || !w2 || !b2 || !w3 || !b3 || !out) return fail(FIN_E_CONFIG, "fin_dense_forward: null argument");
  if (!dense_sizes_ok(B, in_dim, h1, h2, out_dim)) return fail(FIN_E_CONFIG, "fin_dense_forward: bad sizes");
  cudaError_t e = fin::dense_forward(B, in_dim, h1, h2, out_dim, x, w1, b1, w2, b2, w3, b3, hidden, out, S(stream));
  if (e != cudaSuccess) return cuda_fail(e, "fin_dense_forward launch");
  return FIN_OK;
}

int fin_dense_backward(int32_t B, int32_t in_dim, int32_t h1, int32_t h2, int32_t out_dim, const float* x,
                       const float* hidden, const float* g_out, const float* w1, const float* w2, const float* w3,
                       float* dw1, float* db1, float* dw2, float* db2, float* dw3, float* db3, float* g_x, void* stream) {
  if (!x || !hidden || !g_out || !w1 || !w2 || !w3) return fail(FIN_E_CONFIG, "fin_dense_backward: null argument");
  const int np = (dw1 != nullptr) + (db1 != nullptr) + (dw2 != nullptr) + (db2 != nullptr) + (dw3 != nullptr) +
                 (db3 != nullptr);
  if (np != 0 && np != 6) return fail(FIN_E_CONFIG, "fin_dense_backward: pass all six gradient tensors or none");
  if (np == 0 && !g_x) return fail(FIN_E_CONFIG, "fin_dense_backward: nothing to compute");
  if (!dense_sizes_ok(B, in_dim, h1, h2, out_dim)) return fail(FIN_E_CONFIG, "fin_dense_backward: bad sizes");
  cudaError_t e = fin::dense_backward(B, in_dim, h1, h2, out_dim, x, hidden, g_out, w1, w2, w3, dw1, db1, dw2, db2, dw3,
                                      db3, g_x, S(stream));
  if (e != cudaSuccess) return cuda_fail(e, "fin_dense_backward launch");
  return FIN_OK;
}

int fin_concat_obs_action(int32_t B, int32_t in_s, const uint16_t* x, int32_t K, const float* a, float* out,
                          void* stream) {
  if (!x || (!a && K > 0) || !out) return fail(FIN_E_CONFIG, "fin_concat_obs_action: null argument");
  if (B < 1 || in_s < 1 || K < 0) return fail(FIN_E_CONFIG, "fin_concat_obs_action: bad sizes");
  cudaError_t e = fin::launch_concat_sa(B, in_s, x, K, a, out, S(stream));
  if (e != cudaSuccess) return cuda_fail(e, "fin_concat_obs_action launch");
  return FIN_OK;
}

int fin_squash(int32_t B, int32_t K, const float* z, const float* eps, double sigma, float* a, float* logp,
               void* stream) {
  if (!z || !a) return fail(FIN_E_CONFIG, "fin_squash: null argument");
  if (B < 1 || K < 1) return fail(FIN_E_CONFIG, "fin_squash: bad sizes");
  if (eps && !(sigma > 0.0 && std::isfinite(sigma))) return fail(FIN_E_CONFIG, "fin_squash: need sigma > 0");
  if (logp && !eps) return fail(FIN_E_CONFIG, "fin_squash: the log-density needs eps");
  cudaError_t e = fin::launch_squash(B, K, z, eps, sigma, a, logp, S(stream));
  if (e != cudaSuccess) return cuda_fail(e, "fin_squash launch");
  return FIN_OK;
}

int fin_critic_head(int32_t B, const float* q, const float* reward, const uint8_t* done, const float* q1_next,
                    const float* q2_next, const float* logp_next, double gamma, double alpha, float* g_q,
                    double* stats, void* stream) {
  if (!q || !reward || !done || !q1_next || !g_q || !stats) return fail(FIN_E_CONFIG, "fin_critic_head: null argument");
  if (B < 1) return fail(FIN_E_CONFIG, "fin_critic_head: B must be >= 1");
  if (!(gamma >= 0.0 && gamma <= 1.0) || !(alpha >= 0.0 && std::isfinite(alpha)))
    return fail(FIN_E_CONFIG, "fin_critic_head: need 0 <= gamma <= 1 and alpha >= 0");
  cudaError_t e = fin::launch_critic_head(B, q, reward, done, q1_next, q2_next, logp_next, gamma, alpha, g_q, stats,
                                          S(stream));
  if (e != cudaSuccess) return cuda_fail(e, "fin_critic_head launch");
  return FIN_OK;
}

int fin_actor_head(int32_t B, int32_t K, const float* a, const float* logp, const float* q1, const float* dq1,
                   const float* q2, const float* dq2, int32_t ld_dq, double alpha, float* g_z, double* stats,
                   void* stream) {
  if (!a || !q1 || !dq1 || !g_z || !stats) return fail(FIN_E_CONFIG, "fin_actor_head: null argument");
  if (B < 1 || K < 1 || ld_dq < K) return fail(FIN_E_CONFIG, "fin_actor_head: bad sizes");
  if ((q2 == nullptr) != (dq2 == nullptr)) return fail(FIN_E_CONFIG, "fin_actor_head: q2 and dq2 go together");
  if (q2 && !logp) return fail(FIN_E_CONFIG, "fin_actor_head: twin critics are SAC's (pass logp)");
  if (!(alpha >= 0.0 && std::isfinite(alpha))) return fail(FIN_E_CONFIG, "fin_actor_head: need alpha >= 0");
  cudaError_t e = fin::launch_actor_head(B, K, a, logp, q1, dq1, q2, dq2, ld_dq, alpha, g_z, stats, S(stream));
  if (e != cudaSuccess) return cuda_fail(e, "fin_actor_head launch");
  return FIN_OK;
}

int fin_policy_backward(int32_t B, int32_t in_dim, int32_t h1, int32_t h2, int32_t k_out, const uint16_t* x,
                        const uint16_t* hidden, const float* g_z, const float* w2, const float* w3, float* dw1,
                        float* db1, float* dw2, float* db2, float* dw3, float* db3, void* stream) {
  if (!x || !hidden || !g_z || !w2 || !w3 || !dw1 || !db1 || !dw2 || !db2 || !dw3 || !db3)
    return fail(FIN_E_CONFIG, "fin_policy_backward: null argument");
  if (B < 1 || in_dim < 1 || in_dim > 4096 || h1 < 1 || h1 > 1024 || h2 < 1 || h2 > 1024 || k_out < 1 || k_out > 64)
    return fail(FIN_E_CONFIG, "fin_policy_backward: bad sizes");
  cudaError_t e = fin::backward(B, in_dim, h1, h2, k_out, x, hidden, g_z, w2, w3, dw1, db1, dw2, db2, dw3, db3,
                                S(stream));
  if (e != cudaSuccess) return cuda_fail(e, "fin_policy_backward launch");
  return FIN_OK;
}

int fin_soft_update(int64_t n, float* target, const float* online, double tau, void* stream) {
  if (!target || !online) return fail(FIN_E_CONFIG, "fin_soft_update: null argument");
  if (n < 1 || !(tau >= 0.0 && tau <= 1.0)) return fail(FIN_E_CONFIG, "fin_soft_update: need n >= 1, 0 <= tau <= 1");
  cudaError_t e = fin::launch_soft_update(n, target, online, tau, S(stream));
  if (e != cudaSuccess) return cuda_fail(e, "fin_soft_update launch");
  return FIN_OK;
}

int fin_env_clock(const fin_env* env, int64_t* t_global) {
  if (!env || !t_global) return fail(FIN_E_CONFIG, "fin_env_clock: null argument");
  *t_global = env->d.t_global;
  return FIN_OK;
}

int fin_gather_observations(const fin_env* env, const uint16_t* obs_private, const int32_t* day, const int64_t* idx,
                            int32_t B, uint16_t* x, void* stream) {
  if (!env || !obs_private || !day || !idx || !x) return fail(FIN_E_CONFIG, "fin_gather_observations: null argument");
  if (env->d.task != FIN_STOCK) return fail(FIN_E_UNSUPPORTED, "fin_gather_observations: stock envs only");
  if (B < 1) return fail(FIN_E_CONFIG, "fin_gather_observations: B must be >= 1");
  const int P = (env->d.K + 1 + 15) / 16 * 16;
  cudaError_t e = fin::launch_gather_obs(env->d, obs_private, P, day, idx, B, x, S(stream));
  if (e != cudaSuccess) return cuda_fail(e, "fin_gather_observations launch");
  return FIN_OK;
}

int fin_rollout_noise(const fin_env* env, uint64_t seed, int64_t t_base, const int64_t* idx, int32_t B, int32_t member,
                      float* out, void* stream) {
  if (!env || !idx || !out) return fail(FIN_E_CONFIG, "fin_rollout_noise: null argument");
  if (B < 1 || member < 0 || member >= FIN_MAX_MEMBERS) return fail(FIN_E_CONFIG, "fin_rollout_noise: bad sizes");
  cudaError_t e = fin::launch_noise_at(seed, env->d.env_offset, env->d.N, t_base, idx, B, env->d.K, member, out,
                                       S(stream));
  if (e != cudaSuccess) return cuda_fail(e, "fin_rollout_noise launch");
  return FIN_OK;
}

int fin_ppo_prepare(int32_t B, int32_t K, const float* z_old, const float* eps, double sigma, float* a, float* logp_old,
                    void* stream) {
  if (!z_old || !eps || !a || !logp_old) return fail(FIN_E_CONFIG, "fin_ppo_prepare: null argument");
  if (B < 1 || K < 1 || !(sigma > 0.0)) return fail(FIN_E_CONFIG, "fin_ppo_prepare: bad arguments");
  cudaError_t e = fin::launch_ppo_prepare(B, K, z_old, eps, sigma, a, logp_old, S(stream));
  if (e != cudaSuccess) return cuda_fail(e, "fin_ppo_prepare launch");
  return FIN_OK;
}

int fin_adam_step(int64_t n, float* theta, float* m, float* v, const float* grad, int32_t step, double lr,
                  double beta1, double beta2, double eps, void* stream) {
  if (!theta || !m || !v || !grad) return fail(FIN_E_CONFIG, "fin_adam_step: null argument");
  if (n < 1 || step < 1) return fail(FIN_E_CONFIG, "fin_adam_step: need n >= 1 and step >= 1");
  if (!(beta1 >= 0.0 && beta1 < 1.0 && beta2 >= 0.0 && beta2 < 1.0 && eps > 0.0 && lr >= 0.0))
    return fail(FIN_E_CONFIG, "fin_adam_step: bad hyper-parameters");
  cudaError_t e = fin::launch_adam(n, theta, m, v, grad, step, lr, beta1, beta2, eps, S(stream));
  if (e != cudaSuccess) return cuda_fail(e, "fin_adam_step launch");
  return FIN_OK;
}

int fin_gae(const float* reward, const float* value, const uint8_t* done, int32_t T, int32_t N, double gamma,
            double lambda, int32_t normalise, float* adv, float* ret, void* stream) {
  if (!reward || !value || !done || !adv || !ret) return fail(FIN_E_CONFIG, "fin_gae: null argument");
  if (T < 1 || N < 1) return fail(FIN_E_CONFIG, "fin_gae: need T >= 1 and N >= 1");
  if (!(gamma >= 0.0 && gamma <= 1.0) || !(lambda >= 0.0 && lambda <= 1.0))
    return fail(FIN_E_CONFIG, "fin_gae: gamma and lambda must be in [0, 1]");
  cudaError_t e = fin::launch_gae(reward, value, done, T, N, gamma, lambda, normalise, adv, ret, S(stream));
  if (e != cudaSuccess) return cuda_fail(e, "fin_gae launch");
  return FIN_OK;
}

int fin_kl_diversity(const float* outputs, int32_t M, int32_t B, int32_t K, int32_t kind, double sigma, double* D,
                     void* stream) {
  if (!outputs || !D) return fail(FIN_E_CONFIG, "fin_kl_diversity: null argument");
  if (M < 1 || M > FIN_MAX_MEMBERS || B < 1 || K < 1) return fail(FIN_E_CONFIG, "fin_kl_diversity: bad sizes");
  if (kind != 0 && kind != 1) return fail(FIN_E_CONFIG, "fin_kl_diversity: kind must be 0 or 1");
  if (kind == 0 && !(sigma > 0.0 && std::isfinite(sigma))) return fail(FIN_E_CONFIG, "fin_kl_diversity: sigma > 0");
  cudaError_t e = fin::launch_kl_diversity(outputs, M, B, K, kind, sigma, D, S(stream));
  if (e != cudaSuccess) return cuda_fail(e, "fin_kl_diversity launch");
  return FIN_OK;
}

int fin_member_weights(const double* aggs, int32_t M, double threshold, double temperature, float* w,
                       double* sharpe, void* stream) {
  if (!aggs || !w) return fail(FIN_E_CONFIG, "fin_member_weights: null argument");
  if (M < 1 || M > FIN_MAX_MEMBERS) return fail(FIN_E_CONFIG, "M must be in [1, %d]", FIN_MAX_MEMBERS);
  if (!(temperature > 0.0) || !std::isfinite(temperature)) return fail(FIN_E_CONFIG, "temperature must be > 0");
  if (std::isnan(threshold)) return fail(FIN_E_CONFIG, "threshold is NaN");
  cudaError_t e = fin::launch_member_weights(aggs, M, threshold, temperature, w, sharpe, S(stream));
  if (e != cudaSuccess) return cuda_fail(e, "fin_member_weights launch");
  return FIN_OK;
}

int fin_philox_normals(uint64_t seed, int64_t env_offset, int32_t N, int32_t K, int32_t member, int64_t t_global,
                       float* out, void* stream) {
  if (!out || N < 1 || K < 1) return fail(FIN_E_CONFIG, "fin_philox_normals: bad argument");
  cudaError_t e = fin::launch_philox_normals(seed, env_offset, N, K, member, t_global, out, S(stream));
  if (e != cudaSuccess) return cuda_fail(e, "fin_philox_normals launch");
  return FIN_OK;
}

}  // extern "C"
