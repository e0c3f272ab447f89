"""Time the HBM-bound kernels at working sets far above the 126 MB L2 and print
achieved algorithmic GB/s (DESIGN.md §4.2 / §4.4).  Also used as the ncu target.

    python scripts/prof_hbm.py [k1|k4|k6|all] [reps]

K1 ``fin_env_step``      N = 2^22 envs,          213 B / env-step
K4 ``fin_rollout_actions`` N = 2^20, T = 32,     60 + 5 B / env-step + state / T
K6 ``fin_episode_metrics`` T = 2048, N = 2^18,   9 B / env-step (equity f64 + done u8)
"""
import json
import os
import statistics
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2501_10709_b200 import fin  # noqa: E402
from synth import market  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "all"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
flush_r = torch.ones(256 << 18, dtype=torch.float32, device="cuda")


def flush_l2():
    """Write 256 MiB, then read another 256 MiB: the written lines are evicted (and
    written back) by the read pass, so the timed kernel starts on a clean L2."""
    flush.zero_()
    flush_r.sum()
M = market.stock_c1(rows=1008)
res = {}


MODE = os.environ.get("FIN_TIMING", "flush")   # flush | b2b


def timed(fn, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    if MODE == "b2b":   # back-to-back launches over a working set far above L2
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            fn()
        b.record()
        torch.cuda.synchronize()
        return a.elapsed_time(b) / reps
    ts = []
    for _ in range(reps):
        flush_l2()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts)


def env(N, L=30):
    cfg = fin.env_config(num_envs=N, num_assets=30, num_indicators=8, num_rows=1008, episode_len=L,
                         window_stride=5, num_windows=195, window_block=128)
    return fin.fin_env_create(cfg, M.market)


if which in ("k1", "all"):
    N = int(os.environ.get("FIN_K1_N", 1 << 22))
    e = env(N)
    g = torch.Generator(device="cuda").manual_seed(5)
    acts = torch.randint(-100, 101, (N, 30), device="cuda", generator=g, dtype=torch.int16)
    rew = torch.zeros(N, dtype=torch.float32, device="cuda")
    dn = torch.zeros(N, dtype=torch.uint8, device="cuda")
    tr = fin.make_traj(reward=rew, done=dn)
    ms = timed(lambda: fin.fin_env_step(e, acts, tr))
    B = 229   # state in+out incl. the cached asset v (2 x 8 B), actions 60, reward 4, done 1
    res["k1"] = {"N": N, "ms": ms, "bytes_per_env_step": B, "gbs": B * N / ms / 1e6, "env_steps_s": N / ms * 1e3}
    del e, acts

if which in ("k4", "all"):
    N, T = 1 << 20, 32
    e = env(N)
    g = torch.Generator(device="cuda").manual_seed(6)
    acts = torch.randint(-100, 101, (T, N, 30), device="cuda", generator=g, dtype=torch.int16)
    rew = torch.zeros((T, N), dtype=torch.float32, device="cuda")
    dn = torch.zeros((T, N), dtype=torch.uint8, device="cuda")
    tr = fin.make_traj(reward=rew, done=dn)
    ms = timed(lambda: fin.fin_rollout_actions(e, acts, T, tr))
    # per env-step: actions 60 + reward 4 + done 1; per env per call: state in + out
    # (cash 8, hold 60, t_ep 4, window 4, 6 f64 + 1 i32 metric accumulators 52) x 2
    B = N * T * 65 + N * 2 * (8 + 60 + 4 + 4 + 52)
    res["k4"] = {"N": N, "T": T, "ms": ms, "bytes": B, "gbs": B / ms / 1e6, "env_steps_s": N * T / ms * 1e3}
    del e, acts, rew, dn

if which in ("k6", "all"):
    T, N = 2048, 1 << 18
    g = torch.Generator(device="cuda").manual_seed(7)
    # lockstep episodes of 30 steps, as the rollouts produce them (dones of a tile coincide)
    done = torch.zeros((T, N), dtype=torch.uint8, device="cuda")
    done[29::30] = 1
    equity = 1e6 * torch.exp(torch.cumsum(0.01 * torch.randn((T + 1, N), device="cuda", generator=g,
                                                               dtype=torch.float64), 0))
    E = 160
    epm = torch.zeros((E, N, 3), dtype=torch.float64, device="cuda")
    cnt = torch.zeros(N, dtype=torch.int32, device="cuda")
    ms = timed(lambda: fin.fin_episode_metrics(equity, done, 1e6, ep_metrics=epm, ep_count=cnt))
    B = T * N * 9 + N * 8 + int(cnt.sum().item()) * 24 + N * 4   # reads + episode rows + counts
    res["k6"] = {"N": N, "T": T, "ms": ms, "bytes_alg": B, "gbs": B / ms / 1e6, "env_steps_s": N * T / ms * 1e3}

print(json.dumps(res))
