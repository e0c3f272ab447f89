"""Thin Python binding of libfinenv.so (include/fin.h) -- argument marshalling only.

Every function here has the name of the C entry point it calls and does nothing
but convert arguments (torch tensors -> device pointers, NumPy arrays -> host
pointers, ``torch.cuda.Stream`` -> ``cudaStream_t``) and turn a non-OK status
into :class:`FinError`.  All arithmetic of the hot path runs in the CUDA kernels
of the library; there is no CPU fallback -- importing this module on a machine
without the built library raises.

PyTorch is used only for device memory and streams (tensors are allocated by the
caller).  Before a call, the binding checks that every tensor it passes is at least
as large as the call's shapes require (include/fin.h states them), so a short tensor
raises ValueError instead of becoming an out-of-bounds device write.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FIN_LIB_PATH") or os.path.join(_HERE, "libfinenv.so")   # override: A/B runs

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build it with `python -m paper_2501_10709_b200.build` "
        "(nvcc, sm_100a). There is no CPU fallback.")
_lib = C.CDLL(LIB_PATH)

# ----------------------------------------------------------------- constants (fin.h)
FIN_OK, FIN_E_CONFIG, FIN_E_DATA, FIN_E_NUMERIC, FIN_E_CUDA, FIN_E_EPISODE_DONE, FIN_E_UNSUPPORTED, \
    FIN_E_DEVICE_ASYNC = range(8)
FIN_FLAG_ACTION_RANGE, FIN_FLAG_EPISODE_DONE, FIN_FLAG_NONFINITE, FIN_FLAG_BAD_INDEX = 1, 2, 4, 8
FIN_STOCK, FIN_CRYPTO = 0, 1
FIN_PPO_GAUSS, FIN_SAC_SQUASH, FIN_DDPG_OU, FIN_Q_ARGMAX, FIN_Q_DUELING = 0, 1, 2, 3, 4
FIN_MAX_MEMBERS = 32
FIN_IND_MACD, FIN_IND_BOLL_UB, FIN_IND_BOLL_LB, FIN_IND_RSI30, FIN_IND_CCI30, FIN_IND_DX30, FIN_IND_SMA30, \
    FIN_IND_SMA60 = range(8)
FIN_IND_NAMES = ("macd", "boll_ub", "boll_lb", "rsi30", "cci30", "dx30", "sma30", "sma60")
FIN_NOISE_PHILOX, FIN_NOISE_SUPPLIED, FIN_NOISE_NONE = 0, 1, 2
FIN_AGG_EPISODES, FIN_AGG_SUM_CUM, FIN_AGG_SUM_SHARPE, FIN_AGG_N_SHARPE, FIN_AGG_SUM_MDD, \
    FIN_AGG_SUM_REWARD = range(6)
FIN_AGG_NSUM = 6
FIN_AGG_MIN_MDD = 6
FIN_AGG_MIN_CUM = 7
FIN_AGG_LEN = 8

# every symbol include/fin.h declares (checked by tests/test_abi.py)
EXPORTS = ("fin_env_create", "fin_env_reset", "fin_env_step", "fin_env_get_state", "fin_env_set_state",
           "fin_env_check", "fin_env_destroy", "fin_policy_create", "fin_policy_destroy", "fin_rollout",
           "fin_rollout_actions", "fin_ensemble_act", "fin_episode_metrics", "fin_mlp_forward",
           "fin_philox_normals", "fin_member_weights", "fin_market_prepare", "fin_crypto_market", "fin_gae", "fin_kl_diversity", "fin_last_error", "fin_abi_version", "fin_device_check",
           "fin_debug_trace", "fin_env_counters", "fin_stock_market", "fin_ppo_grad", "fin_adam_step",
           "fin_env_clock", "fin_gather_observations", "fin_rollout_noise", "fin_ppo_prepare", "fin_policy_load",
           "fin_dqn_grad", "fin_dense_forward", "fin_dense_backward", "fin_concat_obs_action", "fin_squash",
           "fin_critic_head", "fin_actor_head", "fin_policy_backward", "fin_soft_update")


class FinError(RuntimeError):
    def __init__(self, code: int, where: str, msg: str):
        super().__init__(f"{where}: status {code}: {msg}")
        self.code = code


class fin_env_config(C.Structure):
    _fields_ = [("task", C.c_int32), ("num_envs", C.c_int32), ("num_assets", C.c_int32),
                ("num_indicators", C.c_int32), ("num_rows", C.c_int32), ("episode_len", C.c_int32),
                ("window_stride", C.c_int32), ("window_offset", C.c_int32), ("num_windows", C.c_int32),
                ("window_block", C.c_int32), ("window_base", C.c_int32), ("advance_window_on_reset", C.c_int32),
                ("max_trade", C.c_int32), ("max_hold", C.c_int32), ("pos_limit", C.c_int32),
                ("autoreset", C.c_int32), ("initial_cash", C.c_double), ("cost_rate", C.c_double),
                ("reward_scale", C.c_double), ("noise_std", C.c_float), ("ou_theta", C.c_float),
                ("ou_sigma", C.c_float), ("epsilon", C.c_float), ("seed", C.c_uint64), ("env_offset", C.c_int64)]


class fin_traj(C.Structure):
    _fields_ = [("reward", C.c_void_p), ("done", C.c_void_p), ("actions", C.c_void_p), ("cash", C.c_void_p),
                ("hold", C.c_void_p), ("asset", C.c_void_p), ("mlp_out", C.c_void_p),
                ("mlp_hidden", C.c_void_p), ("ep_metrics", C.c_void_p),
                ("ep_count", C.c_void_p), ("ep_capacity", C.c_int32), ("agg", C.c_void_p),
                ("obs_private", C.c_void_p), ("day", C.c_void_p)]


class fin_noise(C.Structure):
    _fields_ = [("mode", C.c_int32), ("seed", C.c_uint64), ("supplied", C.c_void_p)]


_P = C.c_void_p
_sig = {
    "fin_env_create": ([C.POINTER(fin_env_config), _P, C.c_int64, _P, C.POINTER(_P)], C.c_int),
    "fin_env_reset": ([_P, _P, _P], C.c_int),
    "fin_env_step": ([_P, _P, C.POINTER(fin_traj), _P], C.c_int),
    "fin_env_get_state": ([_P, _P, _P, _P, _P, _P, _P], C.c_int),
    "fin_env_set_state": ([_P, _P, _P, _P, _P, _P, _P], C.c_int),
    "fin_env_check": ([_P, C.POINTER(C.c_uint32)], C.c_int),
    "fin_env_destroy": ([_P], None),
    "fin_env_counters": ([_P, _P, C.c_int32], C.c_int),
    "fin_policy_create": ([C.c_int32, C.c_int32, C.POINTER(C.c_int32), C.POINTER(_P), C.POINTER(_P), _P,
                           C.POINTER(_P)], C.c_int),
    "fin_policy_destroy": ([_P], None),
    "fin_rollout": ([_P, C.POINTER(_P), C.c_int32, _P, C.c_int32, C.POINTER(fin_noise), C.POINTER(fin_traj), _P],
                    C.c_int),
    "fin_rollout_actions": ([_P, _P, C.c_int32, C.POINTER(fin_traj), _P], C.c_int),
    "fin_ensemble_act": ([_P, C.POINTER(_P), C.c_int32, _P, C.POINTER(fin_noise), _P, _P, C.c_int32, _P],
                         C.c_int),
    "fin_episode_metrics": ([_P, _P, C.c_int32, C.c_int32, C.c_double, C.c_double, C.c_double, _P, C.c_int32, _P,
                             _P, _P], C.c_int),
    "fin_mlp_forward": ([_P, _P, C.c_int32, _P, _P, _P], C.c_int),
    "fin_philox_normals": ([C.c_uint64, C.c_int64, C.c_int32, C.c_int32, C.c_int32, C.c_int64, _P, _P], C.c_int),
    "fin_member_weights": ([_P, C.c_int32, C.c_double, C.c_double, _P, _P, _P], C.c_int),
    "fin_gae": ([_P, _P, _P, C.c_int32, C.c_int32, C.c_double, C.c_double, C.c_int32, _P, _P, _P], C.c_int),
    "fin_kl_diversity": ([_P, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_double, _P, _P], C.c_int),
    "fin_crypto_market": ([C.c_int64, C.c_uint64, C.c_double, C.c_double, C.c_double, _P, _P], C.c_int),
    "fin_ppo_grad": ([C.c_int32] * 5 + [_P] * 6 + [C.c_double, C.c_double] + [_P] * 10, C.c_int),
    "fin_adam_step": ([C.c_int64, _P, _P, _P, _P, C.c_int32, C.c_double, C.c_double, C.c_double, C.c_double, _P],
                      C.c_int),
    "fin_env_clock": ([_P, _P], C.c_int),
    "fin_dqn_grad": ([C.c_int32] * 5 + [_P] * 8 + [C.c_double, C.c_int32] + [_P] * 10, C.c_int),
    "fin_gather_observations": ([_P, _P, _P, _P, C.c_int32, _P, _P], C.c_int),
    "fin_rollout_noise": ([_P, C.c_uint64, C.c_int64, _P, C.c_int32, C.c_int32, _P, _P], C.c_int),
    "fin_ppo_prepare": ([C.c_int32, C.c_int32, _P, _P, C.c_double, _P, _P, _P], C.c_int),
    "fin_policy_load": ([_P, C.POINTER(_P), C.POINTER(_P), _P], C.c_int),
    "fin_stock_market": ([C.c_int32, C.c_int32, C.c_uint64, C.c_double, C.c_double, C.c_double, C.c_double, _P, _P],
                         C.c_int),
    "fin_market_prepare": ([_P, C.c_int32, C.c_int32, C.c_int32, C.POINTER(C.c_int32), C.c_int32, C.c_double,
                            C.c_uint64, _P, _P, _P], C.c_int),
    "fin_dense_forward": ([C.c_int32] * 5 + [_P] * 10, C.c_int),
    "fin_dense_backward": ([C.c_int32] * 5 + [_P] * 14, C.c_int),
    "fin_concat_obs_action": ([C.c_int32, C.c_int32, _P, C.c_int32, _P, _P, _P], C.c_int),
    "fin_squash": ([C.c_int32, C.c_int32, _P, _P, C.c_double, _P, _P, _P], C.c_int),
    "fin_critic_head": ([C.c_int32] + [_P] * 6 + [C.c_double, C.c_double, _P, _P, _P], C.c_int),
    "fin_actor_head": ([C.c_int32, C.c_int32] + [_P] * 6 + [C.c_int32, C.c_double, _P, _P, _P], C.c_int),
    "fin_policy_backward": ([C.c_int32] * 5 + [_P] * 12, C.c_int),
    "fin_soft_update": ([C.c_int64, _P, _P, C.c_double, _P], C.c_int),
    "fin_last_error": ([], C.c_char_p),
    "fin_abi_version": ([], C.c_int),
    "fin_device_check": ([C.c_int32], C.c_int),
    "fin_debug_trace": ([_P], C.c_int),
}
for _name, (_args, _res) in _sig.items():
    _f = getattr(_lib, _name)
    _f.argtypes = _args
    _f.restype = _res


def _check(rc: int, where: str):
    if rc != FIN_OK:
        raise FinError(rc, where, _lib.fin_last_error().decode())


# ----------------------------------------------------------------- marshalling helpers
def _ptr(t, dtype=None, what=""):
    """Device pointer of a CUDA tensor (or None).  Checks dtype, device and contiguity."""
    if t is None:
        return None
    import torch
    if not isinstance(t, torch.Tensor):
        raise TypeError(f"{what}: expected a torch.Tensor")
    if not t.is_cuda:
        raise ValueError(f"{what}: tensor must live on the GPU (no CPU fallback)")
    if dtype is not None and t.dtype != dtype:
        raise TypeError(f"{what}: dtype {t.dtype}, expected {dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{what}: tensor must be contiguous")
    return t.data_ptr()


def _ptr_rows(t, dtype, what=""):
    """Device pointer of a 2-D CUDA tensor view whose rows are contiguous (any row stride)."""
    if t is None:
        return None
    import torch
    if not isinstance(t, torch.Tensor) or not t.is_cuda or t.dtype != dtype or t.dim() != 2 or t.stride(1) != 1:
        raise ValueError(f"{what}: expected a 2-D {dtype} CUDA tensor with contiguous rows")
    return t.data_ptr()


def _stream(stream):
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


def make_traj(reward=None, done=None, actions=None, cash=None, hold=None, asset=None, mlp_out=None,
              mlp_hidden=None, ep_metrics=None, ep_count=None, agg=None, obs_private=None, day=None) -> fin_traj:
    import torch
    tr = fin_traj()
    tr.reward = _ptr(reward, torch.float32, "reward")
    tr.done = _ptr(done, torch.uint8, "done")
    tr.actions = _ptr(actions, torch.int16, "actions")
    tr.cash = _ptr(cash, torch.float64, "cash")
    tr.hold = _ptr(hold, torch.int16, "hold")
    tr.asset = _ptr(asset, torch.float64, "asset")
    tr.mlp_out = _ptr(mlp_out, torch.float32, "mlp_out")
    tr.mlp_hidden = _ptr(mlp_hidden, torch.int16, "mlp_hidden")
    tr.ep_metrics = _ptr(ep_metrics, torch.float64, "ep_metrics")
    tr.ep_count = _ptr(ep_count, torch.int32, "ep_count")
    tr.ep_capacity = int(ep_metrics.shape[0]) if ep_metrics is not None else 0
    tr.agg = _ptr(agg, torch.float64, "agg")
    tr.obs_private = _ptr(obs_private, torch.int16, "obs_private")
    tr.day = _ptr(day, torch.int32, "day")
    # the tensors stay referenced by the struct (lifetime) and are size-checked per call
    tr._t = dict(reward=reward, done=done, actions=actions, cash=cash, hold=hold, asset=asset, mlp_out=mlp_out,
                 mlp_hidden=mlp_hidden, ep_metrics=ep_metrics, ep_count=ep_count, agg=agg, obs_private=obs_private,
                 day=day)
    return tr


def make_noise(mode: int = FIN_NOISE_NONE, seed: int = 0, supplied=None) -> fin_noise:
    import torch
    n = fin_noise()
    n.mode = mode
    n.seed = seed
    n.supplied = _ptr(supplied, torch.float32, "noise") if supplied is not None else None
    if mode == FIN_NOISE_SUPPLIED and supplied is None:
        raise ValueError("FIN_NOISE_SUPPLIED needs a supplied tensor")
    n._supplied = supplied
    return n


def _need(t, numel: int, what: str):
    """Raise ValueError if tensor ``t`` (None = not passed) holds fewer than ``numel`` elements."""
    if t is not None and t.numel() < numel:
        raise ValueError(f"{what}: tensor has {t.numel()} elements, the call writes/reads {numel}")


def _need_noise(nz: fin_noise, T: int, M: int, N: int, K: int, crypto: bool = False):
    if nz.mode == FIN_NOISE_SUPPLIED:
        s = getattr(nz, "_supplied", None)
        if s is None:
            raise ValueError("supplied noise: build the fin_noise with make_noise(..., supplied=tensor)")
        _need(s, T * N * 2 if crypto else T * M * N * K, "supplied noise " + ("[T][N][2]" if crypto else "[T][M][N][K]"))


def _need_traj(tr: fin_traj, T: int, N: int, K: int, M: int = 1, out_dim: int = 0, hid: int = 0):
    """Size checks of the trajectory tensors against fin.h's [T][N][...] shapes."""
    t = getattr(tr, "_t", None)
    if t is None:
        if any(getattr(tr, f) for f, _ in fin_traj._fields_ if f != "ep_capacity"):
            raise ValueError("fin_traj must be built with make_traj (its tensors are size-checked)")
        return
    _need(t["reward"], T * N, "reward [T][N]")
    _need(t["done"], T * N, "done [T][N]")
    _need(t["actions"], T * N * K, "actions [T][N][K]")
    _need(t["cash"], T * N, "cash [T][N]")
    _need(t["hold"], T * N * K, "hold [T][N][K]")
    _need(t["asset"], T * N, "asset [T][N]")
    _need(t["mlp_out"], T * M * N * out_dim, "mlp_out [T][M][N][Kout]")
    _need(t["mlp_hidden"], T * M * N * 2 * hid, "mlp_hidden [T][M][N][2][HID]")
    _need(t["ep_metrics"], int(t["ep_metrics"].shape[0]) * N * 3 if t["ep_metrics"] is not None else 0,
          "ep_metrics [E][N][3]")
    _need(t["ep_count"], N, "ep_count [N]")
    _need(t["agg"], FIN_AGG_LEN, "agg [FIN_AGG_LEN]")
    _need(t["obs_private"], T * N * ((K + 1 + 15) // 16 * 16), "obs_private [T][N][P]")
    _need(t["day"], T * N, "day [T][N]")


def env_config(**kw) -> fin_env_config:
    """fin_env_config with the BASELINE defaults (stock task, C1 constants)."""
    c = fin_env_config()
    defaults = dict(task=FIN_STOCK, num_envs=1, num_assets=30, num_indicators=8, num_rows=2, episode_len=1,
                    window_stride=5, window_offset=0, num_windows=1, window_block=128, window_base=0,
                    advance_window_on_reset=0, max_trade=100, max_hold=120, pos_limit=1, autoreset=1,
                    initial_cash=1e6, cost_rate=1e-3, reward_scale=2.0 ** -12, noise_std=0.1, ou_theta=0.15,
                    ou_sigma=0.2, epsilon=0.005, seed=0, env_offset=0)
    defaults.update(kw)
    for k, v in defaults.items():
        setattr(c, k, v)
    return c


# ----------------------------------------------------------------- entry points
class Env:
    """Owning wrapper of a ``fin_env*`` (destroyed with the object)."""

    def __init__(self, handle, cfg: fin_env_config):
        self.handle = handle
        self.cfg = cfg

    @property
    def N(self):
        return self.cfg.num_envs

    @property
    def K(self):
        return self.cfg.num_assets

    def __del__(self, _destroy=_lib.fin_env_destroy):  # bound early: module globals vanish at exit
        h, self.handle = getattr(self, "handle", None), None
        if h:
            _destroy(h)


class Policy:
    def __init__(self, handle, kind, dims):
        self.handle = handle
        self.kind = kind
        self.dims = tuple(dims)

    def __del__(self, _destroy=_lib.fin_policy_destroy):
        h, self.handle = getattr(self, "handle", None), None
        if h:
            _destroy(h)


def fin_abi_version() -> int:
    return _lib.fin_abi_version()


def fin_device_check(ordinal: int = 0) -> None:
    _check(_lib.fin_device_check(ordinal), "fin_device_check")


def fin_debug_trace(buf=None) -> None:
    """Debug timeline of block 0 (u64 [T][16] CUDA tensor, int64 dtype) or None to disable."""
    import torch
    _check(_lib.fin_debug_trace(_ptr(buf, torch.int64, "trace")), "fin_debug_trace")


def fin_last_error() -> str:
    return _lib.fin_last_error().decode()


def fin_env_create(cfg: fin_env_config, market: np.ndarray, stream=None) -> Env:
    m = np.ascontiguousarray(market, dtype=np.float32)
    h = _P()
    _check(_lib.fin_env_create(C.byref(cfg), m.ctypes.data_as(_P), m.size, _stream(stream), C.byref(h)),
           "fin_env_create")
    return Env(h, cfg)


def fin_env_reset(env: Env, mask=None, stream=None) -> None:
    import torch
    _check(_lib.fin_env_reset(env.handle, _ptr(mask, torch.uint8, "mask"), _stream(stream)), "fin_env_reset")


def fin_env_step(env: Env, actions, traj: fin_traj | None = None, stream=None) -> None:
    import torch
    tr = traj if traj is not None else fin_traj()
    _need(actions, env.N * env.K, "actions [N][K]")
    _need_traj(tr, 1, env.N, env.K)
    _check(_lib.fin_env_step(env.handle, _ptr(actions, torch.int16, "actions"), C.byref(tr), _stream(stream)),
           "fin_env_step")


def fin_env_get_state(env: Env, cash=None, hold=None, asset=None, t_ep=None, window=None, stream=None) -> None:
    import torch
    _check(_lib.fin_env_get_state(env.handle, _ptr(cash, torch.float64, "cash"), _ptr(hold, torch.int16, "hold"),
                                  _ptr(asset, torch.float64, "asset"), _ptr(t_ep, torch.int32, "t_ep"),
                                  _ptr(window, torch.int32, "window"), _stream(stream)), "fin_env_get_state")


def fin_env_set_state(env: Env, cash=None, hold=None, t_ep=None, window=None, tau=None, stream=None) -> None:
    import torch
    _check(_lib.fin_env_set_state(env.handle, _ptr(cash, torch.float64, "cash"), _ptr(hold, torch.int16, "hold"),
                                  _ptr(t_ep, torch.int32, "t_ep"), _ptr(window, torch.int32, "window"),
                                  _ptr(tau, torch.int32, "tau"), _stream(stream)), "fin_env_set_state")


def fin_env_check(env: Env) -> int:
    """Returns the sticky device flags (0 = clean); raises FinError on a CUDA failure."""
    f = C.c_uint32(0)
    rc = _lib.fin_env_check(env.handle, C.byref(f))
    if rc not in (FIN_OK, FIN_E_DEVICE_ASYNC):
        _check(rc, "fin_env_check")
    return int(f.value)


def fin_env_counters(env: Env, clear: bool = False) -> dict:
    """Event counters of the handle (synchronises): exact_redo = stock steps whose buys
    took the exact out-of-line affordability path; balanced_rollouts / balanced_refused =
    fused stock rollouts launched with the balanced persistent schedule / refused it;
    pregen_rollouts = fused stock rollouts that ran on noise pre-drawn by a separate kernel."""
    c = (C.c_uint32 * 5)()
    _check(_lib.fin_env_counters(env.handle, C.cast(c, _P), int(bool(clear))), "fin_env_counters")
    return {"exact_redo": int(c[0]), "balanced_rollouts": int(c[1]), "balanced_refused": int(c[2]),
            "balanced_refused_err": int(c[3]), "pregen_rollouts": int(c[4])}


def fin_env_destroy(env: Env) -> None:
    h, env.handle = env.handle, None
    if h:
        _lib.fin_env_destroy(h)


def fin_policy_create(kind: int, layers, stream=None) -> Policy:
    """layers = [(W_bits uint16 [out][in] (host), bias float32 [out] or None), ...]."""
    dims = [int(layers[0][0].shape[1])] + [int(w.shape[0]) for w, _ in layers]
    ws = [np.ascontiguousarray(w, dtype=np.uint16) for w, _ in layers]
    bs = [None if b is None else np.ascontiguousarray(b, dtype=np.float32) for _, b in layers]
    n = len(layers)
    dims_c = (C.c_int32 * (n + 1))(*dims)
    w_c = (_P * n)(*[w.ctypes.data_as(_P) for w in ws])
    b_c = (_P * n)(*[None if b is None else b.ctypes.data_as(_P) for b in bs])
    h = _P()
    _check(_lib.fin_policy_create(kind, n, dims_c, w_c, b_c, _stream(stream), C.byref(h)), "fin_policy_create")
    return Policy(h, kind, dims)


def fin_policy_destroy(pol: Policy) -> None:
    h, pol.handle = pol.handle, None
    if h:
        _lib.fin_policy_destroy(h)


def _members(members):
    arr = (_P * len(members))(*[m.handle for m in members])
    return arr


def _weights(member_w, n_members: int):
    if member_w is None:
        return None, None
    w = np.ascontiguousarray(member_w, dtype=np.float32).reshape(-1)
    if w.size != n_members:
        raise ValueError(f"member_w has {w.size} weights for {n_members} members")
    return w, w.ctypes.data_as(_P)


def fin_rollout(env: Env, members, T: int, noise: fin_noise | None = None, traj: fin_traj | None = None,
                member_w=None, stream=None) -> None:
    nz = noise if noise is not None else make_noise(FIN_NOISE_NONE)
    tr = traj if traj is not None else fin_traj()
    keep, wp = _weights(member_w, len(members))
    crypto = env.cfg.task == FIN_CRYPTO
    M = len(members)
    if M:
        d = members[0].dims
        _need_traj(tr, T, env.N, env.K, M, out_dim=d[-1], hid=d[1])
    _need_noise(nz, T, M, env.N, env.K, crypto)
    _check(_lib.fin_rollout(env.handle, _members(members), len(members), wp, T, C.byref(nz), C.byref(tr),
                            _stream(stream)), "fin_rollout")


def fin_rollout_actions(env: Env, actions, T: int, traj: fin_traj | None = None, stream=None) -> None:
    import torch
    tr = traj if traj is not None else fin_traj()
    _need(actions, T * env.N * env.K, "actions [T][N][K]")
    _need_traj(tr, T, env.N, env.K)
    _check(_lib.fin_rollout_actions(env.handle, _ptr(actions, torch.int16, "actions"), T, C.byref(tr),
                                    _stream(stream)), "fin_rollout_actions")


def fin_ensemble_act(env: Env, members, actions, mean_action=None, noise: fin_noise | None = None, member_w=None,
                     commit_ou: bool = False, stream=None) -> None:
    import torch
    nz = noise if noise is not None else make_noise(FIN_NOISE_NONE)
    keep, wp = _weights(member_w, len(members))
    N, K = env.N, env.K
    _need(actions, N * K, "actions [N][K]")
    _need(mean_action, N * K, "mean_action [N][K]")
    _need_noise(nz, 1, len(members), N, K)
    _check(_lib.fin_ensemble_act(env.handle, _members(members), len(members), wp, C.byref(nz),
                                 _ptr(actions, torch.int16, "actions"), _ptr(mean_action, torch.float32, "mean"),
                                 int(bool(commit_ou)), _stream(stream)), "fin_ensemble_act")


def fin_episode_metrics(equity, done, reset_equity: float, periods_per_year: float = 252.0, rf: float = 0.0,
                        ep_metrics=None, ep_count=None, agg=None, stream=None) -> None:
    import torch
    T = int(done.shape[0])
    N = int(done.shape[1])
    cap = int(ep_metrics.shape[0]) if ep_metrics is not None else 0
    _check(_lib.fin_episode_metrics(_ptr(equity, torch.float64, "equity"), _ptr(done, torch.uint8, "done"), T, N,
                                    reset_equity, periods_per_year, rf, _ptr(ep_metrics, torch.float64, "ep_metrics"),
                                    cap, _ptr(ep_count, torch.int32, "ep_count"), _ptr(agg, torch.float64, "agg"),
                                    _stream(stream)), "fin_episode_metrics")


def fin_mlp_forward(policy: Policy, x_bf16_bits, z, hidden=None, stream=None) -> None:
    import torch
    B = int(x_bf16_bits.shape[0])
    _check(_lib.fin_mlp_forward(policy.handle, _ptr(x_bf16_bits, torch.int16, "x"), B, _ptr(z, torch.float32, "z"),
                                _ptr(hidden, torch.int16, "hidden"), _stream(stream)), "fin_mlp_forward")


def fin_philox_normals(seed: int, env_offset: int, out, member: int, t_global: int, stream=None) -> None:
    import torch
    N, K = int(out.shape[0]), int(out.shape[1])
    _check(_lib.fin_philox_normals(seed, env_offset, N, K, member, t_global, _ptr(out, torch.float32, "out"),
                                   _stream(stream)), "fin_philox_normals")


def fin_member_weights(aggs, w, sharpe=None, threshold: float = 0.0, temperature: float = 1.0,
                       stream=None) -> None:
    """aggs f64 [M][FIN_AGG_LEN] (device) -> w f32 [M] (device), sharpe f64 [M] (device, optional)."""
    import torch
    M = int(aggs.shape[0])
    _check(_lib.fin_member_weights(_ptr(aggs, torch.float64, "aggs"), M, float(threshold), float(temperature),
                                   _ptr(w, torch.float32, "w"), _ptr(sharpe, torch.float64, "sharpe"),
                                   _stream(stream)), "fin_member_weights")


def fin_market_prepare(ohlcv, warmup: int, indicators, market, raw, magnitude: float = 0.0, seed: int = 0,
                       stream=None) -> None:
    """ohlcv f32 [D][5][K] (device) -> market f32 [D-warmup][2+I][K] (device); raw f64
    [I][K][D-warmup] (device scratch).  indicators: FIN_IND_* ids or names."""
    import torch
    D, _, K = (int(v) for v in ohlcv.shape)
    ids = [FIN_IND_NAMES.index(i) if isinstance(i, str) else int(i) for i in indicators]
    arr = (C.c_int32 * max(1, len(ids)))(*ids)
    _check(_lib.fin_market_prepare(_ptr(ohlcv, torch.float32, "ohlcv"), D, K, int(warmup), arr, len(ids),
                                   float(magnitude), int(seed), _ptr(market, torch.float32, "market"),
                                   _ptr(raw, torch.float64, "raw"), _stream(stream)), "fin_market_prepare")


def fin_crypto_market(steps: int, seed: int, rows, sigma: float = 1e-4, m0: float = 5e4, phi: float = 0.9,
                      stream=None) -> None:
    """Generate the crypto market tensor rows f32 [steps + 1][144] (device) on the GPU."""
    import torch
    if tuple(rows.shape) != (steps + 1, 144):
        raise ValueError("rows must be [steps + 1][144]")
    _check(_lib.fin_crypto_market(int(steps), int(seed), float(sigma), float(m0), float(phi),
                                  _ptr(rows, torch.float32, "rows"), _stream(stream)), "fin_crypto_market")


def fin_stock_market(days: int, K: int, seed: int, ohlcv, mu: float = 2e-4, sigma: float = 0.02,
                     s0_lo: float = 50.0, s0_hi: float = 150.0, stream=None) -> None:
    """Generate the stock OHLCV tensor ohlcv f32 [days][5][K] (device) on the GPU."""
    import torch
    if tuple(ohlcv.shape) != (days, 5, K):
        raise ValueError("ohlcv must be [days][5][K]")
    _check(_lib.fin_stock_market(int(days), int(K), int(seed), float(mu), float(sigma), float(s0_lo), float(s0_hi),
                                 _ptr(ohlcv, torch.float32, "ohlcv"), _stream(stream)), "fin_stock_market")


def fin_dqn_grad(x_bf16_bits, hidden, out, action, reward, done, q_next_target, w2, w3, grads, stats,
                 q_next_online=None, gamma: float = 0.99, dueling: bool = False, stream=None) -> None:
    """DQN / Double DQN (q_next_online given) / Dueling gradient step (include/fin.h); grads as in
    fin_ppo_grad; stats f64 [4] (L, mean Q(s, a), mean y, B)."""
    import torch
    B, in_dim = int(x_bf16_bits.shape[0]), int(x_bf16_bits.shape[1])
    k_out = int(out.shape[1])
    h2, h1 = int(w2.shape[0]), int(w2.shape[1])
    if tuple(w3.shape) != (k_out, h2) or tuple(q_next_target.shape) != (B, k_out) or int(hidden.shape[0]) != B:
        raise ValueError("fin_dqn_grad: inconsistent shapes")
    if q_next_online is not None and tuple(q_next_online.shape) != (B, k_out):
        raise ValueError("fin_dqn_grad: q_next_online must be [B][k_out]")
    _need(hidden, B * 2 * max(h1, h2), "hidden [B][2][H]")
    for t, w in ((action, "action"), (reward, "reward"), (done, "done")):
        _need(t, B, w)
    f32 = torch.float32
    p = [_ptr(t, f32, "grad") for pair in grads for t in pair]
    _check(_lib.fin_dqn_grad(B, in_dim, h1, h2, k_out, _ptr(x_bf16_bits, torch.int16, "x"),
                             _ptr(hidden, torch.int16, "hidden"), _ptr(out, f32, "out"),
                             _ptr(action, torch.uint8, "action"), _ptr(reward, f32, "reward"),
                             _ptr(done, torch.uint8, "done"), _ptr(q_next_target, f32, "q_next_target"),
                             _ptr(q_next_online, f32, "q_next_online"), float(gamma), int(bool(dueling)),
                             _ptr(w2, f32, "w2"), _ptr(w3, f32, "w3"), *p, _ptr(stats, torch.float64, "stats"),
                             _stream(stream)), "fin_dqn_grad")


# ---------------------------------------------------------------- actor-critic updates (R-AC)
def _grad_shapes(dims):
    return [((dims[1], dims[0]), (dims[1],)), ((dims[2], dims[1]), (dims[2],)), ((dims[3], dims[2]), (dims[3],))]


def _check_grads(grads, dims, where):
    for (dw, db), (sw, sb) in zip(grads, _grad_shapes(dims)):
        if tuple(dw.shape) != sw or tuple(db.shape) != sb:
            raise ValueError(f"{where}: gradient shapes must be {_grad_shapes(dims)}")


def fin_dense_forward(x, layers, out, hidden=None, stream=None) -> None:
    """Critic forward (include/fin.h): x f32 [B][in], layers = [(W f32 [out][in], b f32 [out])] x 3
    (device), out f32 [B][O], hidden f32 [B][h1 + h2] or None."""
    import torch
    B, in_dim = int(x.shape[0]), int(x.shape[1])
    dims = [in_dim] + [int(w.shape[0]) for w, _ in layers]
    if len(layers) != 3 or any(tuple(w.shape) != (dims[i + 1], dims[i]) or tuple(b.shape) != (dims[i + 1],)
                               for i, (w, b) in enumerate(layers)):
        raise ValueError("fin_dense_forward: three layers [out][in] / [out] chained from x's width")
    if tuple(out.shape) != (B, dims[3]):
        raise ValueError("fin_dense_forward: out must be [B][O]")
    _need(hidden, B * (dims[1] + dims[2]), "hidden [B][h1 + h2]")
    f32 = torch.float32
    wb = [_ptr(t, f32, "layer") for pair in layers for t in pair]
    _check(_lib.fin_dense_forward(B, *dims, _ptr(x, f32, "x"), *wb, _ptr(hidden, f32, "hidden"), _ptr(out, f32, "out"),
                                  _stream(stream)), "fin_dense_forward")


def fin_dense_backward(x, hidden, g_out, weights, grads=None, g_x=None, stream=None) -> None:
    """Critic backward: weights = [W1, W2, W3] f32 (device), grads = [(dw, db)] x 3 or None, g_x f32
    [B][in] or None."""
    import torch
    B, in_dim = int(x.shape[0]), int(x.shape[1])
    dims = [in_dim] + [int(w.shape[0]) for w in weights]
    if len(weights) != 3 or any(tuple(w.shape) != (dims[i + 1], dims[i]) for i, w in enumerate(weights)):
        raise ValueError("fin_dense_backward: three weights [out][in] chained from x's width")
    if tuple(g_out.shape) != (B, dims[3]):
        raise ValueError("fin_dense_backward: g_out must be [B][O]")
    _need(hidden, B * (dims[1] + dims[2]), "hidden [B][h1 + h2]")
    if grads is not None:
        _check_grads(grads, dims, "fin_dense_backward")
    if g_x is not None and tuple(g_x.shape) != (B, in_dim):
        raise ValueError("fin_dense_backward: g_x must be [B][in]")
    f32 = torch.float32
    p = [None] * 6 if grads is None else [_ptr(t, f32, "grad") for pair in grads for t in pair]
    _check(_lib.fin_dense_backward(B, *dims, _ptr(x, f32, "x"), _ptr(hidden, f32, "hidden"), _ptr(g_out, f32, "g_out"),
                                   *[_ptr(w, f32, "w") for w in weights], *p, _ptr(g_x, f32, "g_x"),
                                   _stream(stream)), "fin_dense_backward")


def fin_concat_obs_action(x_bf16_bits, a, out, stream=None) -> None:
    """out f32 [B][S + K] = [x (bf16 bits [B][S]); a f32 [B][K]] (a None: the widened x alone)."""
    import torch
    B, S = int(x_bf16_bits.shape[0]), int(x_bf16_bits.shape[1])
    K = 0 if a is None else int(a.shape[1])
    if (a is not None and int(a.shape[0]) != B) or tuple(out.shape) != (B, S + K):
        raise ValueError("fin_concat_obs_action: a [B][K], out [B][S + K]")
    _check(_lib.fin_concat_obs_action(B, S, _ptr(x_bf16_bits, torch.int16, "x"), K, _ptr(a, torch.float32, "a"),
                                      _ptr(out, torch.float32, "out"), _stream(stream)), "fin_concat_obs_action")


def fin_squash(z, a, eps=None, logp=None, sigma: float = 0.1, stream=None) -> None:
    """a = tanh(z + sigma eps) (eps None: tanh z) and log pi(a|s) into logp [B] (needs eps)."""
    import torch
    B, K = int(z.shape[0]), int(z.shape[1])
    _need(a, B * K, "a [B][K]")
    _need(eps, B * K, "eps [B][K]")
    _need(logp, B, "logp [B]")
    f32 = torch.float32
    _check(_lib.fin_squash(B, K, _ptr(z, f32, "z"), _ptr(eps, f32, "eps"), float(sigma), _ptr(a, f32, "a"),
                           _ptr(logp, f32, "logp"), _stream(stream)), "fin_squash")


def fin_critic_head(q, reward, done, q1_next, g_q, stats, q2_next=None, logp_next=None, gamma: float = 0.99,
                    alpha: float = 0.2, stream=None) -> None:
    """Critic target and squared TD loss: g_q f32 [B] = dL/dq; stats f64 [4] (L, mean q, mean y, B)."""
    import torch
    B = int(q.numel())
    for t, w in ((reward, "reward"), (done, "done"), (q1_next, "q1_next"), (g_q, "g_q"), (q2_next, "q2_next"),
                 (logp_next, "logp_next")):
        _need(t, B, w)
    _need(stats, 4, "stats")
    f32 = torch.float32
    _check(_lib.fin_critic_head(B, _ptr(q, f32, "q"), _ptr(reward, f32, "reward"), _ptr(done, torch.uint8, "done"),
                                _ptr(q1_next, f32, "q1_next"), _ptr(q2_next, f32, "q2_next"),
                                _ptr(logp_next, f32, "logp_next"), float(gamma), float(alpha), _ptr(g_q, f32, "g_q"),
                                _ptr(stats, torch.float64, "stats"), _stream(stream)), "fin_critic_head")


def fin_actor_head(a, q1, dq1, g_z, stats, logp=None, q2=None, dq2=None, alpha: float = 0.2, stream=None) -> None:
    """DDPG (logp None) or SAC actor head: g_z f32 [B][K] = dL/dz; dq1 / dq2 [B][ld] views whose first
    K columns are dQ/da (e.g. g_x[:, S:]); stats f64 [4] (L, mean q_min, mean logp, B)."""
    import torch
    B, K = int(a.shape[0]), int(a.shape[1])
    ld = int(dq1.stride(0))
    for d in (dq1, dq2):
        if d is not None and (int(d.shape[0]) != B or int(d.shape[1]) != K or int(d.stride(1)) != 1 or int(d.stride(0)) != ld):
            raise ValueError("fin_actor_head: dq1 / dq2 must be [B][K] row views with one row stride")
    for t, w in ((q1, "q1"), (q2, "q2"), (logp, "logp")):
        _need(t, B, w)
    _need(g_z, B * K, "g_z [B][K]")
    f32 = torch.float32
    _check(_lib.fin_actor_head(B, K, _ptr(a, f32, "a"), _ptr(logp, f32, "logp"), _ptr(q1, f32, "q1"),
                               _ptr_rows(dq1, f32, "dq1"), _ptr(q2, f32, "q2"), _ptr_rows(dq2, f32, "dq2"), ld, float(alpha),
                               _ptr(g_z, f32, "g_z"), _ptr(stats, torch.float64, "stats"), _stream(stream)),
           "fin_actor_head")


def fin_policy_backward(x_bf16_bits, hidden, g_z, w2, w3, grads, stream=None) -> None:
    """The policy MLP's backward from g_z f32 [B][k_out] (fin_ppo_grad's pass)."""
    import torch
    B, in_dim = int(x_bf16_bits.shape[0]), int(x_bf16_bits.shape[1])
    k_out = int(g_z.shape[1])
    h2, h1 = int(w2.shape[0]), int(w2.shape[1])
    if tuple(w3.shape) != (k_out, h2) or int(g_z.shape[0]) != B or int(hidden.shape[0]) != B:
        raise ValueError("fin_policy_backward: inconsistent shapes")
    _need(hidden, B * 2 * max(h1, h2), "hidden [B][2][H]")
    _check_grads(grads, (in_dim, h1, h2, k_out), "fin_policy_backward")
    f32 = torch.float32
    p = [_ptr(t, f32, "grad") for pair in grads for t in pair]
    _check(_lib.fin_policy_backward(B, in_dim, h1, h2, k_out, _ptr(x_bf16_bits, torch.int16, "x"),
                                    _ptr(hidden, torch.int16, "hidden"), _ptr(g_z, f32, "g_z"), _ptr(w2, f32, "w2"),
                                    _ptr(w3, f32, "w3"), *p, _stream(stream)), "fin_policy_backward")


def fin_soft_update(target, online, tau: float = 0.005, stream=None) -> None:
    """target <- f32(tau online + (1 - tau) target) (float64 arithmetic), flat f32 device tensors."""
    import torch
    n = int(target.numel())
    _need(online, n, "online")
    _check(_lib.fin_soft_update(n, _ptr(target, torch.float32, "target"), _ptr(online, torch.float32, "online"),
                                float(tau), _stream(stream)), "fin_soft_update")


def fin_env_clock(env: Env) -> int:
    t = C.c_int64(0)
    _check(_lib.fin_env_clock(env.handle, C.byref(t)), "fin_env_clock")
    return int(t.value)


def fin_gather_observations(env: Env, obs_private, day, idx, x, stream=None) -> None:
    """x int16 (bf16 bits) [B][1 + 2K + IK] <- the samples idx int64 [B] (t N + env) of a rollout's logs."""
    import torch
    B = int(idx.numel())
    K, I = env.cfg.num_assets, env.cfg.num_indicators
    if tuple(x.shape) != (B, 1 + 2 * K + I * K):
        raise ValueError("x must be [B][1 + 2K + I K]")
    _check(_lib.fin_gather_observations(env.handle, _ptr(obs_private, torch.int16, "obs_private"),
                                        _ptr(day, torch.int32, "day"), _ptr(idx, torch.int64, "idx"), B,
                                        _ptr(x, torch.int16, "x"), _stream(stream)), "fin_gather_observations")


def fin_rollout_noise(env: Env, seed: int, t_base: int, idx, out, member: int = 0, stream=None) -> None:
    import torch
    B = int(idx.numel())
    _need(out, B * env.K, "out [B][K]")
    _check(_lib.fin_rollout_noise(env.handle, int(seed), int(t_base), _ptr(idx, torch.int64, "idx"), B, int(member),
                                  _ptr(out, torch.float32, "out"), _stream(stream)), "fin_rollout_noise")


def fin_ppo_prepare(z_old, eps, a, logp_old, sigma: float = 0.1, stream=None) -> None:
    import torch
    B, K = int(z_old.shape[0]), int(z_old.shape[1])
    for t, n, w in ((eps, B * K, "eps"), (a, B * K, "a"), (logp_old, B, "logp_old")):
        _need(t, n, w)
    f32 = torch.float32
    _check(_lib.fin_ppo_prepare(B, K, _ptr(z_old, f32, "z_old"), _ptr(eps, f32, "eps"), float(sigma), _ptr(a, f32, "a"),
                                _ptr(logp_old, f32, "logp_old"), _stream(stream)), "fin_ppo_prepare")


def fin_policy_load(pol: Policy, weights, biases=None, stream=None) -> None:
    """weights / biases: lists of f32 device tensors [out][in] / [out] (biases None = zero)."""
    import torch
    n = len(pol.dims) - 1
    if len(weights) != n or (biases is not None and len(biases) != n):
        raise ValueError(f"fin_policy_load: {n} layers expected")
    for l, w in enumerate(weights):
        if tuple(w.shape) != (pol.dims[l + 1], pol.dims[l]):
            raise ValueError(f"weight {l} must be [{pol.dims[l + 1]}][{pol.dims[l]}]")
    w_c = (_P * n)(*[_ptr(w, torch.float32, "w") for w in weights])
    b_c = (_P * n)(*([None] * n if biases is None else [_ptr(b, torch.float32, "b") for b in biases]))
    _check(_lib.fin_policy_load(pol.handle, w_c, b_c, _stream(stream)), "fin_policy_load")


def fin_ppo_grad(x_bf16_bits, hidden, z, a, logp_old, adv, w2, w3, grads, stats, sigma: float = 0.1,
                 clip_eps: float = 0.2, stream=None) -> None:
    """PPO policy-gradient step (include/fin.h): grads = [(dw1, db1), (dw2, db2), (dw3, db3)] f32
    device tensors receive d(-L)/dtheta; stats f64 [4] (L, mean ratio, clipped fraction, B)."""
    import torch
    B, in_dim = int(x_bf16_bits.shape[0]), int(x_bf16_bits.shape[1])
    k_out = int(z.shape[1])
    h2, h1 = int(w2.shape[0]), int(w2.shape[1])
    if tuple(w3.shape) != (k_out, h2) or tuple(a.shape) != (B, k_out) or int(hidden.shape[0]) != B:
        raise ValueError("fin_ppo_grad: inconsistent shapes")
    _need(hidden, B * 2 * max(h1, h2), "hidden [B][2][H]")
    _need(logp_old, B, "logp_old [B]")
    _need(adv, B, "adv [B]")
    shapes = [((h1, in_dim), (h1,)), ((h2, h1), (h2,)), ((k_out, h2), (k_out,))]
    for (dw, db), (sw, sb) in zip(grads, shapes):
        if tuple(dw.shape) != sw or tuple(db.shape) != sb:
            raise ValueError(f"fin_ppo_grad: gradient shapes must be {shapes}")
    f32 = torch.float32
    p = [_ptr(t, f32, "grad") for pair in grads for t in pair]
    _check(_lib.fin_ppo_grad(B, in_dim, h1, h2, k_out, _ptr(x_bf16_bits, torch.int16, "x"),
                             _ptr(hidden, torch.int16, "hidden"), _ptr(z, f32, "z"), _ptr(a, f32, "a"),
                             _ptr(logp_old, f32, "logp_old"), _ptr(adv, f32, "adv"), float(sigma), float(clip_eps),
                             _ptr(w2, f32, "w2"), _ptr(w3, f32, "w3"), *p, _ptr(stats, torch.float64, "stats"),
                             _stream(stream)), "fin_ppo_grad")


def fin_adam_step(theta, m, v, grad, step: int, lr: float = 3e-4, beta1: float = 0.9, beta2: float = 0.999,
                  eps: float = 1e-8, stream=None) -> None:
    """One Adam step on flat f32 device tensors (theta, m, v updated in place)."""
    import torch
    n = int(theta.numel())
    for t, w in ((m, "m"), (v, "v"), (grad, "grad")):
        _need(t, n, w)
    f32 = torch.float32
    _check(_lib.fin_adam_step(n, _ptr(theta, f32, "theta"), _ptr(m, f32, "m"), _ptr(v, f32, "v"),
                              _ptr(grad, f32, "grad"), int(step), float(lr), float(beta1), float(beta2), float(eps),
                              _stream(stream)), "fin_adam_step")


def fin_gae(reward, value, done, adv, ret, gamma: float = 0.99, lam: float = 0.95, normalise: bool = False,
            stream=None) -> None:
    """GAE over reward / done [T][N] and value [T+1][N] (device) -> adv, ret [T][N] (device)."""
    import torch
    T, N = int(reward.shape[0]), int(reward.shape[1])
    if tuple(value.shape) != (T + 1, N) or tuple(done.shape) != (T, N):
        raise ValueError("value must be [T+1][N] and done [T][N]")
    _check(_lib.fin_gae(_ptr(reward, torch.float32, "reward"), _ptr(value, torch.float32, "value"),
                        _ptr(done, torch.uint8, "done"), T, N, float(gamma), float(lam), int(bool(normalise)),
                        _ptr(adv, torch.float32, "adv"), _ptr(ret, torch.float32, "ret"), _stream(stream)), "fin_gae")


def fin_kl_diversity(outputs, D, kind: int = 0, sigma: float = 0.1, stream=None) -> None:
    """outputs f32 [M][B][K] (device) -> D f64 [M][M] (device), D[i][j] = mean KL(pi_j || pi_i)."""
    import torch
    M, B, K = (int(x) for x in outputs.shape)
    _check(_lib.fin_kl_diversity(_ptr(outputs, torch.float32, "outputs"), M, B, K, int(kind), float(sigma),
                                 _ptr(D, torch.float64, "D"), _stream(stream)), "fin_kl_diversity")
