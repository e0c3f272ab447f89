/*
 * fin.h -- C ABI of libfinenv.so, the B200-native rollout hot path of
 * arXiv 2501.10709 ("Revisiting Ensemble Methods for Stock Trading and Crypto
 * Trading Tasks at ACM ICAIF FinRL Contests 2023/2024").
 *
 * Citations: "P:n" = line n of the paper text; "S:n" = SPEC.md line n;
 * "Rn" = reading n of DESIGN.md §3 (where the paper is silent or ambiguous).
 *
 * What the library computes (§3.1, §4.2, §4.3):
 *   N independent trading sub-environments (SubEnvs) stepping in lockstep.  Per
 *   step: policy-MLP forward, action sampling / clipping, buy/sell execution with
 *   transaction cost and cash/holding constraints, total asset v_t = b_t + p_t^T h_t
 *   and reward R = v_{t+1} - v_t, done / auto-reset; the stock
 *   ensemble's averaging of PPO/SAC/DDPG actions and per-episode
 *   metrics: cumulative return, Sharpe (Eq. 6), max drawdown.
 *
 * Conventions (all entry points):
 *   - Every pointer is a DEVICE pointer on the handle's device unless marked (host).
 *   - Return value: FIN_OK (0) or an FIN_E_* code; fin_last_error() gives the text
 *     (thread-local).  No C++ exception crosses the ABI.
 *   - Asynchrony: calls enqueue on ``stream`` (a cudaStream_t passed as void*;
 *     NULL = legacy default stream) and do not synchronise, except
 *     fin_env_create (one sync after the market upload), fin_policy_create (one
 *     sync after packing), fin_env_check and fin_env_destroy.
 *   - Device-detected conditions (action outside +-max_trade -> clamped; stepping a
 *     done env with autoreset = 0 -> the env is left unchanged; non-finite
 *     policy output or noise) set bits of a sticky per-handle error word, reported
 *     by fin_env_check() as FIN_E_DEVICE_ASYNC (bits in *flags).
 *   - Ownership: the caller owns every pointer it passes; the library owns the
 *     handle's SoA state, its padded copy of the market and the packed weights.
 *     Caller buffers may be freed as soon as the create call returns.
 *   - Threading: one handle is driven by one host thread / one stream at a time.
 *   - Layouts: caller-visible trajectory tensors use the paper's [T][N][D] order
 *     (P:242-273); the handle's internal state is SoA ([K][N]) for coalescing.
 *   - Multi-GPU: the library links no NCCL.  Each rank creates its handle with
 *     ``env_offset`` = global id of its local env 0 (window assignment and Philox
 *     streams are keyed by the global id, so results do not depend on the
 *     partition) and the caller all-reduces the FIN_AGG_* partials.
 */
#ifndef FIN_H_
#define FIN_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FIN_ABI_VERSION 1

/* status codes; 1/2/3 mirror SPEC's exit codes */
enum {
  FIN_OK = 0,
  FIN_E_CONFIG = 1,        /* invalid argument / configuration (host-side check) */
  FIN_E_DATA = 2,          /* market data invalid: non-finite, price <= 0, shape */
  FIN_E_NUMERIC = 3,       /* reserved: host-detected numeric failure */
  FIN_E_CUDA = 4,          /* a CUDA runtime call failed */
  FIN_E_EPISODE_DONE = 5,  /* reserved */
  FIN_E_UNSUPPORTED = 6,   /* device is not sm_100 / shape outside the compiled kernels */
  FIN_E_DEVICE_ASYNC = 7   /* sticky device error word non-zero (see FIN_FLAG_*) */
};

/* sticky device error bits (fin_env_check) */
enum {
  FIN_FLAG_ACTION_RANGE = 1,   /* |action| > max_trade: clamped (R6) */
  FIN_FLAG_EPISODE_DONE = 2,   /* step of a done env with autoreset = 0: ignored */
  FIN_FLAG_NONFINITE = 4,      /* non-finite MLP output / noise: action forced to 0 */
  FIN_FLAG_BAD_INDEX = 8,      /* market row index out of range: env left unchanged */
  FIN_FLAG_NOISE_WAIT = 16     /* small-N rollout: the streamed pre-drawn noise of a step did not
                                  arrive within ~8 s (the step used whatever the buffer held) */
};

enum { FIN_STOCK = 0, FIN_CRYPTO = 1 };

/* policy member kinds: C1 / C2 members (BASELINE configs[1,2]) and the C3 Q-nets.
 * FIN_Q_ARGMAX: DQN or Double DQN (identical at inference: greedy on Q), net
 * 103-128-128-3; FIN_Q_DUELING: Dueling DQN, net 103-128-128-4 whose outputs
 * are the advantage head A_0..A_2 then V (Q = V + A - mean A; its greedy action is the
 * argmax of A). */
enum { FIN_PPO_GAUSS = 0, FIN_SAC_SQUASH = 1, FIN_DDPG_OU = 2, FIN_Q_ARGMAX = 3, FIN_Q_DUELING = 4 };

/* most ensemble members in one call (PAPER.md P:445 Ensemble-3: 30) */
#define FIN_MAX_MEMBERS_API 32

/* noise modes for fin_rollout / fin_ensemble_act */
enum { FIN_NOISE_PHILOX = 0, FIN_NOISE_SUPPLIED = 1, FIN_NOISE_NONE = 2 };

/* per-rank aggregate vector written by fin_rollout / fin_episode_metrics.
 * Entries [0, FIN_AGG_NSUM) are reduced with SUM across ranks, the rest with MIN. */
enum {
  FIN_AGG_EPISODES = 0,     /* number of completed episodes */
  FIN_AGG_SUM_CUM = 1,      /* sum of cumulative returns */
  FIN_AGG_SUM_SHARPE = 2,   /* sum of finite Sharpe ratios */
  FIN_AGG_N_SHARPE = 3,     /* number of finite Sharpe ratios */
  FIN_AGG_SUM_MDD = 4,      /* sum of max drawdowns */
  FIN_AGG_SUM_REWARD = 5,   /* sum of rewards over all transitions */
  FIN_AGG_NSUM = 6,
  FIN_AGG_MIN_MDD = 6,      /* worst (most negative) drawdown */
  FIN_AGG_LEN = 8           /* index 7 = MIN of cumulative return */
};

typedef struct fin_env fin_env;
typedef struct fin_policy fin_policy;

/* Environment configuration (host struct).  Stock: P:123, P:129-132, P:148,
 * BASELINE configs[0,1,2,4]; crypto: P:124, BASELINE configs[3]. */
typedef struct {
  int32_t task;             /* FIN_STOCK or FIN_CRYPTO */
  int32_t num_envs;         /* N >= 1 local envs */
  int32_t num_assets;       /* K: stock 1..32; crypto must be 1 */
  int32_t num_indicators;   /* I (stock): market has 2+I channels; crypto: ignored */
  int32_t num_rows;         /* market rows (days / seconds) */
  int32_t episode_len;      /* L_ep steps per episode (R9); done on the L_ep-th step */
  int32_t window_stride;    /* stock window w starts at window_offset + w*window_stride (R10) */
  int32_t window_offset;
  int32_t num_windows;      /* W >= 1 */
  int32_t window_block;     /* envs [j*block, (j+1)*block) (global ids) share window j+base */
  int32_t window_base;
  int32_t advance_window_on_reset;  /* C2 test mode: w <- (w+1) mod W on reset */
  int32_t max_trade;        /* stock: |a_k| <= max_trade shares (R6) */
  int32_t max_hold;         /* crypto: forced exit after max_hold steps (R26) */
  int32_t pos_limit;        /* crypto: |position| <= pos_limit (must be 1) */
  int32_t autoreset;        /* 1: reset on done (BASELINE "reset on done") */
  double initial_cash;      /* b_0 */
  double cost_rate;         /* fee per side (0.001 = 0.1%, R4) */
  double reward_scale;      /* stock 2^-12 (R8), crypto 1 */
  float noise_std;          /* Gaussian policy std (0.1, configs[1]) */
  float ou_theta, ou_sigma; /* DDPG OU noise (0.15, 0.2, configs[2]) */
  float epsilon;            /* crypto epsilon-greedy (0.005) */
  uint64_t seed;            /* Philox key for production-mode noise */
  int64_t env_offset;       /* global id of local env 0 */
} fin_env_config;

/* Create an env handle.  ``market`` (host) holds num_rows rows:
 *   stock  float32 [num_rows][2 + I][K]: channel 0 raw close (execution/marking),
 *          channel 1 normalised close (observation), 2.. indicators (observation);
 *   crypto float32 [num_rows][144]: [mid, ask_px[10], ask_sz[10], bid_px[10],
 *          bid_sz[10], f[101], pad[2]].
 * market_elems must equal the product of those dims.  Validates (FIN_E_DATA on
 * non-finite values or close/mid <= 0), uploads a padded copy, resets all envs
 * and synchronises once.  Window ranges must stay inside the market. */
int fin_env_create(const fin_env_config* cfg /*host*/, const float* market /*host*/,
                   int64_t market_elems, void* stream, fin_env** out /*host*/);

/* reset: b = initial_cash, h = 0, t_ep = 0, online metric state cleared;
 * mask [N] u8 selects envs (NULL = all).  The window index is re-derived from the
 * global id (R10). */
int fin_env_reset(fin_env* env, const uint8_t* mask, void* stream);

/* Trajectory outputs, [T][N][...] (paper order P:242-273); NULL field = not written.
 * Transition fields hold PRE-reset values of the transition (the state right
 * after the trade and the mark at the next row), before any auto-reset.
 *   reward   f32 [T][N]      R = (v' - v) * reward_scale (R8)
 *   done     u8  [T][N]
 *   actions  i16 [T][N][K]   executed share deltas h' - h (stock) / position delta (crypto)
 *   cash     f64 [T][N]      b after the trade
 *   hold     i16 [T][N][K]   holdings after the trade (crypto: position in {-1,0,1})
 *   asset    f64 [T][N]      v' = b' + p_{t+1}^T h'
 *   mlp_out  f32 [T][M][N][Kout]  raw network outputs z (debug / parity)
 *   mlp_hidden bf16 bits [T][M][N][2][HID]  both hidden activations (debug / parity)
 *   ep_metrics f64 [E][N][3] (cum, sharpe, mdd) of the episodes completed during the
 *            call, in completion order; ep_count i32 [N] counts them (written; may
 *            exceed E, extra episodes are counted but not stored)
 *   agg      f64 [FIN_AGG_LEN] per-rank partials (overwritten)
 *   obs_private bf16 bits [T][N][P] (stock policy rollouts) the env-private observation entries
 *            the network consumed -- [b / b0, h_1 / max_trade .. h_K / max_trade, 0 pad], P = K + 1
 *            rounded up to 16 -- and day i32 [T][N] the market day of the step: with the market they
 *            rebuild the full observation (fin_gather_observations) for the learner */
typedef struct {
  float* reward;
  uint8_t* done;
  int16_t* actions;
  double* cash;
  int16_t* hold;
  double* asset;
  float* mlp_out;
  uint16_t* mlp_hidden;
  double* ep_metrics;
  int32_t* ep_count;
  int32_t ep_capacity;      /* E */
  double* agg;
  uint16_t* obs_private;
  int32_t* day;
} fin_traj;

/* One VecEnv step with supplied integer actions [N][K] i16 (stock share
 * deltas; crypto position deltas in {-1,0,1}).  ``out`` uses T = 1.  Episode metrics
 * are not produced by this call (use fin_rollout_actions or fin_episode_metrics). */
int fin_env_step(fin_env* env, const int16_t* actions, const fin_traj* out /*host*/, void* stream);

/* State snapshot: cash f64 [N], hold i16 [N][K] (crypto: position), asset
 * f64 [N] = b + p_t^T h at the current row, t_ep i32 [N], window i32 [N].  Any
 * pointer may be NULL. */
int fin_env_get_state(const fin_env* env, double* cash, int16_t* hold, double* asset,
                      int32_t* t_ep, int32_t* window, void* stream);

/* Overwrite state (teacher forcing / resume).  hold [N][K]; crypto: hold = position,
 * tau = holding time (NULL = 0).  Online metric state restarts at the current equity. */
int fin_env_set_state(fin_env* env, const double* cash, const int16_t* hold, const int32_t* t_ep,
                      const int32_t* window, const int32_t* tau, void* stream);

/* Synchronise the handle's last stream and return FIN_E_DEVICE_ASYNC if any sticky
 * flag is set (written to *flags, host, may be NULL); clears the word. */
int fin_env_check(fin_env* env, uint32_t* flags /*host*/);

/* Event counters of the handle (host array counters[FIN_CTR_LEN], u32; synchronises the
 * handle's last stream; clear != 0 zeroes them afterwards):
 *   [0] stock steps whose buys took the exact out-of-line affordability path (R5: the
 *       fast floor estimate failed its check -- cash at or within ~1e-11 of a multiple
 *       of the unit cost); for tests, which prove the slow path ran;
 *   [1] fused stock rollouts launched with the balanced persistent schedule;
 *   [2] rollouts where that cooperative launch was refused and one tile per CTA ran instead;
 *   [3] the cudaError_t of the last refusal (0: none);
 *   [4] fused stock rollouts whose Philox noise was drawn by a separate kernel (small N: tiles
 *       at most twice the idle SMs; streamed on those SMs while the rollout runs; the same
 *       normals, bitwise, as the in-kernel draws). */
enum { FIN_CTR_LEN = 5 };
int fin_env_counters(fin_env* env, uint32_t* counters /*host*/, int32_t clear);

void fin_env_destroy(fin_env* env);

/* Create a policy / Q network (BASELINE configs[1,3]).
 * kind: FIN_* member kind.  dims (host) = {in, h1, ..., out}, n_layers linear
 * layers (currently 3: in <= 304, h1 = h2 in {128, 256}, out <= 32).  w_bf16[l]
 * (host array of HOST pointers) = bf16 bit patterns [dims[l+1]][dims[l]];
 * bias[l] (host pointers) = f32 [dims[l+1]] or NULL for zero.  Hidden layers use
 * ReLU (R15); inputs and hidden activations are bf16, accumulation fp32.
 * The library pads and packs a device copy in the tcgen05 K-major layout. */
int fin_policy_create(int32_t kind, int32_t n_layers, const int32_t* dims /*host*/,
                      const uint16_t* const* w_bf16 /*host*/, const float* const* bias /*host*/,
                      void* stream, fin_policy** out /*host*/);
/* Waits for the policy's last use (the event recorded on the stream of the most recent
 * call that read it; not a device-wide synchronisation), then frees it.  A caller that
 * used one policy on several streams concurrently synchronises those streams first. */
void fin_policy_destroy(fin_policy* policy);

/* Noise source.  PHILOX: counter-based Philox4x32-10 keyed by ``seed`` and the
 * global env id; SUPPLIED: ``supplied`` f32 [T][M][N][K] N(0,1)
 * (stock) or [T][N][2] U[0,1) (crypto epsilon-greedy: u_explore, u_action);
 * NONE: zero noise / greedy. */
typedef struct {
  int32_t mode;
  uint64_t seed;
  const float* supplied;
} fin_noise;

/* Fused rollout of T steps (the producer of P:139-146 / P:241-278): per step the
 * members' MLPs on the current observation (tcgen05 tensor cores), sampling /
 * ensemble combination, trade execution, reward, done / auto-reset, online episode
 * metrics.  members (host array) has n_members in [1, 32] policies of identical
 * shape.  Stock: kinds PPO/SAC/DDPG, executed action = uniform mean of
 * the members' continuous actions, or the member_w (host, M floats) weighted sum
 * (the Sharpe-softmax weights of fin_member_weights); each DDPG member keeps its own
 * OU state (slot i = the i-th DDPG member of the list).  Crypto: kinds
 * Q_ARGMAX / Q_DUELING, executed action = plurality vote of the members' greedy
 * actions (ties to hold, then the lowest index), then epsilon-greedy; member_w
 * must be NULL.  mlp_out / mlp_hidden logs are [T][M][N][.].  No host round-trip. */
int fin_rollout(fin_env* env, const fin_policy* const* members /*host*/, int32_t n_members,
                const float* member_w /*host*/, int32_t T, const fin_noise* noise /*host*/,
                const fin_traj* out /*host*/, void* stream);

/* Replay rollout: T steps with supplied actions [T][N][K] i16, state kept on chip;
 * online episode metrics as in fin_rollout. */
int fin_rollout_actions(fin_env* env, const int16_t* actions, int32_t T, const fin_traj* out /*host*/,
                        void* stream);

/* Ensemble action on the current state without stepping: writes
 * actions i16 [N][K] and, if non-NULL, mean_action f32 [N][K] (the averaged
 * continuous action before rounding).  Noise uses step index t_global of the env
 * (supplied noise is read as [1][M][N][K]).  The env (cash, holdings, clock, metrics)
 * is never modified.  Each DDPG member's OU state x (R19, R-OU-M) is updated-then-used
 * for the action as in a rollout step; the updated x is written back to the env only
 * if commit_ou != 0 (commit_ou = 0: the call is a pure function of the env state, so
 * repeated calls return the same actions).  Same behaviour for one or several DDPG
 * members. */
int fin_ensemble_act(fin_env* env, const fin_policy* const* members /*host*/, int32_t n_members,
                     const float* member_w /*host*/, const fin_noise* noise /*host*/,
                     int16_t* actions, float* mean_action, int32_t commit_ou, void* stream);

/* Episode metrics from a stored equity log (Eq. 6): equity f64 [T+1][N]
 * (row 0 = equity at the start, row t = v' of transition t), done u8 [T][N] (an
 * episode ends at a done transition; the next starts at equity row... the reset
 * value ``reset_equity``).  Segmented warp-shuffle scans over time.
 * Writes ep_metrics f64 [E][N][3], ep_count i32 [N], agg f64 [FIN_AGG_LEN] (or NULL). */
int fin_episode_metrics(const double* equity, const uint8_t* done, int32_t T, int32_t N,
                        double reset_equity, double periods_per_year, double rf,
                        double* ep_metrics, int32_t ep_capacity, int32_t* ep_count, double* agg,
                        void* stream);

/* Standalone policy forward for parity / profiling: x bf16 bits [B][dims[0]],
 * z f32 [B][dims[n_layers]], hidden (or NULL) bf16 bits [B][2][dims[1]]. */
int fin_mlp_forward(const fin_policy* policy, const uint16_t* x, int32_t B, float* z, uint16_t* hidden,
                    void* stream);

/* Production-noise probe: normals f32 [N][K] for member m at step t_global,
 * exactly as fin_rollout draws them (Philox4x32-10 + Box-Muller). */
int fin_philox_normals(uint64_t seed, int64_t env_offset, int32_t N, int32_t K, int32_t member,
                       int64_t t_global, float* out, void* stream);

/* Market preparation on the device (the step before the rollout; P:290, P:338;
 * readings R11, R12, R-PERTURB): from raw OHLCV f32 [D][5][K] (open, high, low, close,
 * volume; the first ``warmup`` of the D days are hidden warm-up), build the stock market
 * tensor f32 [D - warmup][2 + I][K] that fin_env_create takes: c = 0 close, c = 1
 * close / close[first stored day], c = 2 + i indicator ``indicators[i]`` (host array of
 * FIN_IND_*, I <= 16) z-scored per (asset, indicator) over the stored days.  Every
 * price of asset k is first scaled by c_k = 1 + magnitude (2 u_k - 1), u_k a Philox
 * uniform of (seed, k) (magnitude 0: no perturbation).  Float64 arithmetic in the
 * definitions' order.  ``raw`` (f64 [I][K][D - warmup], caller scratch) receives the
 * stored indicator series before the z-score; the call needs it (no allocation). */
enum { FIN_IND_MACD = 0, FIN_IND_BOLL_UB = 1, FIN_IND_BOLL_LB = 2, FIN_IND_RSI30 = 3, FIN_IND_CCI30 = 4,
       FIN_IND_DX30 = 5, FIN_IND_SMA30 = 6, FIN_IND_SMA60 = 7 };
int fin_market_prepare(const float* ohlcv, int32_t D, int32_t K, int32_t warmup, const int32_t* indicators /*host*/,
                       int32_t I, double magnitude, uint64_t seed, float* market, double* raw, void* stream);

/* Crypto market generation on the device (the synthetic stand-in
 * for the paper's BTC LOB series, with the shapes of BASELINE configs[3]; reading
 * R-CGEN, formulas in oracle/crypto_market.py): writes ``rows`` (device, f32
 * [steps + 1][144], the layout fin_env_create takes for FIN_CRYPTO: mid, ask px / size,
 * bid px / size over 10 levels, 101 factors, 2 pad) for steps 0 .. steps of a GBM mid
 * (``sigma`` per step from ``m0``), a 10-level book (lognormal half-spread and level
 * gaps, Exp(1) sizes) and 101 stationary AR(1) factors (coefficient ``phi``), all drawn
 * from Philox4x32-10 keyed by ``seed``.  Float64 arithmetic, one f32 rounding per value.
 * Needs steps >= 1, sigma >= 0, m0 > 0, 0 <= phi < 1.  Allocates stream-ordered scratch
 * (8 (steps + 1) bytes + chunk carries) and frees it on the stream. */
int fin_crypto_market(int64_t steps, uint64_t seed, double sigma, double m0, double phi, float* rows, void* stream);

/* Stock OHLCV generation on the device (the synthetic stand-in for the
 * paper's daily bars, with BASELINE configs[0]'s GBM; reading R-SGEN, formulas in
 * oracle/stock_market.py): writes ``ohlcv`` (device, f32 [days][5][K]: open, high, low,
 * close, volume -- the input of fin_market_prepare) for a GBM close per asset, S0 ~
 * U(s0_lo, s0_hi), drift mu and volatility sigma per day, open = previous close, high / low =
 * max / min(open, close) (1 +- (0.5 sigma)|Z|), volume LogNormal(ln 1e6, 0.5); random numbers
 * from Philox4x32-10 keyed by ``seed`` (streams 11..15).  Float64 arithmetic, one f32 rounding
 * per value.  Needs days >= 1, 1 <= K <= 4096, sigma >= 0, 0 < s0_lo < s0_hi.  Allocates
 * stream-ordered scratch (16 (days + 1) K bytes) and frees it on the stream. */
int fin_stock_market(int32_t days, int32_t K, uint64_t seed, double mu, double sigma, double s0_lo, double s0_hi,
                     float* ohlcv, void* stream);

/* The learner's policy-gradient step (Eq. 3-4, P:176-195 -- the
 * Monte-Carlo gradient estimate grad J = (1/N) sum_i sum_t R grad log pi(a_t | s_t) -- in PPO's
 * clipped-surrogate form; reading R-PPO, formulas in oracle/learn.py) for the
 * Gaussian policy of a 3-layer ReLU MLP (mean tanh(z), fixed std ``sigma``).  Per sample s of
 * the batch (device arrays): x bf16 bits [B][in_dim] the observation, hidden bf16 bits
 * [B][2][max(h1, h2)] and z f32 [B][k_out] the hidden activations and outputs of the CURRENT
 * weights (fin_mlp_forward), a f32 [B][k_out] the pre-clip continuous action the rollout drew,
 * logp_old f32 [B] its log-density under the rollout's policy, adv f32 [B] its advantage (e.g.
 * fin_gae, normalised).  Weights (device f32, the values the forward used, [out][in]): w2
 * [h2][h1], w3 [k_out][h2].  Writes the gradients of the loss -L (L = the mean clipped surrogate,
 * ratio clip 1 +- clip_eps) to dw1 [h1][in_dim], db1 [h1], dw2 [h2][h1], db2 [h2], dw3
 * [k_out][h2], db3 [k_out] (device f32) and stats (device f64 [4]: L, mean ratio, clipped
 * fraction, B).  float64 head, fp32 contractions, deterministic.  Allocates stream-ordered
 * scratch (~4 B (k_out + h1 + h2) + split partials) and frees it on the stream. */
int fin_ppo_grad(int32_t B, int32_t in_dim, int32_t h1, int32_t h2, int32_t k_out, const uint16_t* x,
                 const uint16_t* hidden, const float* z, const float* a, const float* logp_old, const float* adv,
                 double sigma, double clip_eps, const float* w2, const float* w3, float* dw1, float* db1, float* dw2,
                 float* db2, float* dw3, float* db3, double* stats, void* stream);

/* The DQN family's gradient step (the crypto members of P:317-321 / P:346;
 * SPEC S:362-391; reading R-DQN, formulas in oracle/learn.py): for B transitions (s, a, r, done,
 * s') of a 3-layer ReLU Q-net (device): x bf16 bits [B][in_dim], hidden bf16 bits
 * [B][2][max(h1, h2)] and out f32 [B][k_out] of the online net at s (fin_mlp_forward), action u8
 * [B] (0 .. number of actions - 1), reward f32 [B], done u8 [B], q_next_target f32 [B][k_out] the
 * target net's outputs at s', q_next_online f32 [B][k_out] the online net's at s' for Double DQN
 * (NULL: DQN).  dueling != 0: outputs are (A_0 .. A_{n-1}, V) and Q = V + A - mean A.  Target y =
 * r + gamma (1 - done) max_a Q_target(s', a) (Double: Q_target(s', argmax_a Q_online(s', a))),
 * loss L = mean (Q(s, a) - y)^2 with y held fixed; writes dL/dtheta (device f32, as fin_ppo_grad)
 * and stats (device f64 [4]: L, mean Q(s, a), mean y, B).  Weights w2 / w3 as in fin_ppo_grad. */
int fin_dqn_grad(int32_t B, int32_t in_dim, int32_t h1, int32_t h2, int32_t k_out, const uint16_t* x,
                 const uint16_t* hidden, const float* out, const uint8_t* action, const float* reward,
                 const uint8_t* done, const float* q_next_target, const float* q_next_online, double gamma,
                 int32_t dueling, const float* w2, const float* w3, float* dw1, float* db1, float* dw2, float* db2,
                 float* dw3, float* db3, double* stats, void* stream);

/* The DDPG / SAC updates (the stock ensemble's other members, P:78, P:300,
 * P:343; reading R-AC, formulas in oracle/learn.py).  A critic Q(s, a) is a
 * 3-layer ReLU MLP in float32 on the concatenated input [x(s); a] with a linear output (learner-
 * only; the actor is the rollout's policy).  All arrays are device memory; every call is
 * stream-ordered, allocates stream-ordered scratch and frees it on the stream; bad arguments
 * return FIN_E_CONFIG before any launch.
 *
 * fin_dense_forward: x f32 [B][in_dim] -> hidden f32 [B][h1 + h2] (h1 = ReLU(W1 x + b1) then h2 =
 *   ReLU(W2 h1 + b2) per row; NULL: not stored) and out f32 [B][out_dim] = W3 h2 + b3; weights f32
 *   [out][in] row-major, biases f32 [out].  fp32 CUDA-core contractions (deterministic).
 * fin_dense_backward: from g_out = dL/d out f32 [B][out_dim] and the forward's x / hidden: the
 *   parameter gradients dw1 [h1][in_dim], db1, dw2 [h2][h1], db2, dw3 [out_dim][h2], db3 (all six
 *   or none) and / or g_x = dL/dx f32 [B][in_dim] (NULL: skipped); ReLU derivative 1 where the
 *   activation is > 0.  Split-K over the batch with partials summed in a fixed order.
 * fin_concat_obs_action: out f32 [B][in_s + K] = [x (bf16 bits [B][in_s], widened); a f32 [B][K]]
 *   (K = 0, a NULL: the widened observation alone -- the input of a value net V(s)).
 * fin_squash: a f32 [B][K] = tanh(z + sigma eps) (eps NULL: tanh z, DDPG's mu(s)); logp f32 [B]
 *   (needs eps; NULL: skipped) = sum_k [-eps^2 / 2 - ln(sigma sqrt(2 pi)) - ln(1 - tanh(u)^2)], the
 *   last term in the stable form 2 (ln 2 - u - softplus(-2 u)); float64 arithmetic.
 * fin_critic_head: y = r + gamma (1 - done) (min(q1_next, q2_next) - alpha logp_next) (q2_next /
 *   logp_next NULL: omitted -- DDPG), the loss L = mean (q - y)^2 with y held fixed, g_q f32 [B] =
 *   dL/dq = 2 (q - y) / B, stats f64 [4] = (L, mean q, mean y, B); float64 head.  SAC calls it
 *   once per critic with the same next-state inputs.
 * fin_actor_head: DDPG (logp NULL, q2 / dq2 NULL): L = -mean q1, g_z = -(1/B) dq1 (1 - a^2).  SAC
 *   (logp = log pi(a|s) of the reparameterised sample a = tanh(z + sigma eps)): per sample the
 *   smaller critic m (Q1 on ties), L = mean (alpha logp - q_m), g_z = (1/B) (2 alpha a - dq_m (1 -
 *   a^2)).  dq rows (dQ/da, e.g. the last K columns of fin_dense_backward's g_x) have stride ld_dq
 *   >= K.  stats f64 [4] = (L, mean q_m, mean logp, B).  The actor's parameter gradients follow
 *   from fin_policy_backward with g_z.
 * fin_policy_backward: the backward pass of fin_ppo_grad from a given g_z = dL/dz f32 [B][k_out]
 *   through the policy MLP (inputs and hidden activations of fin_mlp_forward; weights as there).
 * fin_soft_update: target[i] = f32(tau online[i] + (1 - tau) target[i]) with the products and the
 *   sum in float64 (0 <= tau <= 1). */
int fin_dense_forward(int32_t B, int32_t in_dim, int32_t h1, int32_t h2, int32_t out_dim, const float* x,
                      const float* w1, const float* b1, const float* w2, const float* b2, const float* w3,
                      const float* b3, float* hidden, float* out, void* stream);
int fin_dense_backward(int32_t B, int32_t in_dim, int32_t h1, int32_t h2, int32_t out_dim, const float* x,
                       const float* hidden, const float* g_out, const float* w1, const float* w2, const float* w3,
                       float* dw1, float* db1, float* dw2, float* db2, float* dw3, float* db3, float* g_x, void* stream);
int fin_concat_obs_action(int32_t B, int32_t in_s, const uint16_t* x, int32_t K, const float* a, float* out,
                          void* stream);
int fin_squash(int32_t B, int32_t K, const float* z, const float* eps, double sigma, float* a, float* logp,
               void* stream);
int fin_critic_head(int32_t B, const float* q, const float* reward, const uint8_t* done, const float* q1_next,
                    const float* q2_next, const float* logp_next, double gamma, double alpha, float* g_q,
                    double* stats, void* stream);
int fin_actor_head(int32_t B, int32_t K, const float* a, const float* logp, const float* q1, const float* dq1,
                   const float* q2, const float* dq2, int32_t ld_dq, double alpha, float* g_z, double* stats,
                   void* stream);
int fin_policy_backward(int32_t B, int32_t in_dim, int32_t h1, int32_t h2, int32_t k_out, const uint16_t* x,
                        const uint16_t* hidden, const float* g_z, const float* w2, const float* w3, float* dw1,
                        float* db1, float* dw2, float* db2, float* dw3, float* db3, void* stream);
int fin_soft_update(int64_t n, float* target, const float* online, double tau, void* stream);

/* The learner's view of a rollout's samples (NEXT-4).  A sample is idx = t N + env (step t of
 * the call, local env).  fin_env_clock: the handle's global step counter (host out) -- record it
 * before a rollout: its Philox noise of step t is drawn at t_global + t.
 * fin_gather_observations (stock): x bf16 bits [B][1 + 2K + I K] (device) = the full observation
 * P:129 of each sample, rebuilt from the rollout's obs_private / day logs (fin_traj) and the
 * market: [b / b0, close_norm (K), h / max_trade (K), features indicator-major (I K)], the
 * shared entries bf16 of the market value -- the network input the rollout used.
 * fin_rollout_noise: out f32 [B][K] = the rollout's Philox normals of member ``member`` at the
 * samples (seed and t_base = the rollout's noise seed and starting clock).
 * fin_ppo_prepare: from the rollout policy's outputs z_old f32 [B][K] and its noise eps, the
 * Gaussian sample a = tanh(z_old) + sigma eps (f32) and its log-density log pi_old(a) f32 [B]
 * (float64 arithmetic; R17 / R-PPO), the inputs of fin_ppo_grad. */
int fin_env_clock(const fin_env* env, int64_t* t_global /*host*/);
int fin_gather_observations(const fin_env* env, const uint16_t* obs_private, const int32_t* day, const int64_t* idx,
                            int32_t B, uint16_t* x, void* stream);
int fin_rollout_noise(const fin_env* env, uint64_t seed, int64_t t_base, const int64_t* idx, int32_t B, int32_t member,
                      float* out, void* stream);
int fin_ppo_prepare(int32_t B, int32_t K, const float* z_old, const float* eps, double sigma, float* a, float* logp_old,
                    void* stream);

/* Replace a policy's weights (same network) with device f32 values w[l] [dims[l+1]][dims[l]]
 * and optional biases b[l] [dims[l+1]] (host arrays of DEVICE pointers; NULL bias = 0): gathered
 * into the tcgen05 image on the device (bf16 round to nearest even) through a per-handle index
 * table of the layout (built and uploaded by the first call, synchronously); stream-ordered after
 * the policy's last use (its event), no host synchronisation.  A given bias is added even if it is
 * all zero (fin_policy_create skips all-zero biases: the results differ at most in the sign of a
 * zero output).  Non-finite values are not checked here (rollouts flag FIN_FLAG_NONFINITE).  The
 * policy gets a new id, so envs recompute their cached layer-1 term.  The caller orders the next
 * use on another stream after this one. */
int fin_policy_load(fin_policy* policy, const float* const* w, const float* const* b, void* stream);

/* One Adam step (Kingma & Ba) on n parameters (device f32 theta, m, v updated in place; grad the
 * loss gradient): m = b1 m + (1 - b1) g, v = b2 v + (1 - b2) g^2, theta -= lr mhat / (sqrt(vhat) +
 * eps), mhat / vhat bias-corrected with the 1-based ``step``.  Needs n >= 1, step >= 1, 0 <= b1, b2
 * < 1, eps > 0, lr >= 0. */
int fin_adam_step(int64_t n, float* theta, float* m, float* v, const float* grad, int32_t step, double lr,
                  double beta1, double beta2, double eps, void* stream);

/* Generalised advantage estimation over a rollout's trajectory (
 * SPEC S:392-395; reading R-GAE, formulas in oracle/learn.py): from reward f32 [T][N],
 * value f32 [T+1][N] (row T = the bootstrap value of the last state) and done u8 [T][N]
 * (device), writes adv and ret f32 [T][N] (device): delta_t = r_t + gamma V_{t+1} (1 - d_t)
 * - V_t, A_t = delta_t + gamma lambda (1 - d_t) A_{t+1}, A_T = 0, R_t = A_t + V_t, float64
 * per env in this order (bit-identical to the oracle before the f32 rounding).
 * ``normalise`` != 0: adv is then replaced by (A - mean) / std over all T N entries
 * (population std of the float64 advantages, deterministic merge; A - mean if std = 0);
 * ret keeps the unnormalised A + V.  Needs T >= 1, N >= 1, 0 <= gamma, lambda <= 1. */
int fin_gae(const float* reward, const float* value, const uint8_t* done, int32_t T, int32_t N, double gamma,
            double lambda, int32_t normalise, float* adv, float* ret, void* stream);

/* The KL diversity term of Eq. 5: from M
 * members' outputs f32 [M][B][K] on the same B states (device) writes D f64 [M][M]
 * (device), D[i][j] = mean over the states of KL(pi_j || pi_i) (D[i][i] = 0); member i's
 * loss term is lambda sum_{j != i} D[i][j].  kind 0: diagonal Gaussians N(out, sigma^2)
 * (PPO, and DDPG wrapped with sigma): sum_k (mu_j - mu_i)^2 / (2 sigma^2); kind 1:
 * categorical softmax(out) (the DQN family's Q-values).  Float64, deterministic. */
int fin_kl_diversity(const float* outputs, int32_t M, int32_t B, int32_t K, int32_t kind, double sigma, double* D,
                     void* stream);

/* Ensemble weights from validation statistics (Eq. 6; reading R-GATE):
 * aggs f64 [M][FIN_AGG_LEN] = the aggregate vector of one validation fin_rollout per
 * member (deterministic: FIN_NOISE_NONE), all-reduced over ranks.  Member Sharpe =
 * aggs[m][FIN_AGG_SUM_SHARPE] / aggs[m][FIN_AGG_N_SHARPE] (NaN if that count is 0).  Members below ``threshold`` (or NaN) are discarded; the rest get
 * softmax(Sharpe / temperature); if all are discarded the best finite Sharpe gets 1.
 * Writes w f32 [M] (device) and, if non-NULL, sharpe f64 [M] (device). */
int fin_member_weights(const double* aggs, int32_t M, double threshold, double temperature, float* w,
                       double* sharpe, void* stream);

/* Debug: record a clock64 timeline of block 0 of subsequent fin_rollout calls into
 * ``device_buffer`` (u64 [T][16]; NULL disables).  Not for production use. */
int fin_debug_trace(void* device_buffer);

/* thread-local text for the last non-OK status of this thread */
const char* fin_last_error(void);

/* ABI version, device check: FIN_OK if device ``ordinal`` is sm_100 (else UNSUPPORTED) */
int fin_abi_version(void);
int fin_device_check(int32_t ordinal);

#ifdef __cplusplus
}
#endif
#endif /* FIN_H_ */
