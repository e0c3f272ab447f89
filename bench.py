"""Benchmark of the rollout hot path (BASELINE.json metric: env-steps/sec, whole box).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--no-extras]

One "step" = one fin_rollout over the headline workload: the C1 30-stock env
(K=30, I=8, obs 301) with the 301-256-256-30 bf16 Gaussian policy, N = 65,536
envs per GPU, horizon T = 256 with reset on done (BASELINE configs[1] env and
policy at the configs[4] sweep's largest per-GPU size; the metric is quoted at
2048-65536 envs).  A step runs every §8(a) row: market-row staging, observation,
tcgen05 MLP, sampling/clipping, trade execution, reward, done/reset, online
episode metrics, and the per-rank aggregate (all-reduced over NCCL when N > 1).

Timing: W untimed warm-up steps, then K steps, each bracketed by CUDA events on
the launching stream; L2 is flushed (256 MiB write) between timed steps outside
the events; barrier + synchronize on both sides; max over ranks.  ``e2e`` repeats
the measurement through the C ABI with host buffers: the step's input state is
copied from pinned host memory and the trajectory (reward, done) and aggregate are
read back inside the timed region.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N_HEAD = 65536
T_HEAD = 256
K_ASSETS = 30
N_IND = 8
ROWS = 1008
L_EP = 30
MLP_FLOP_PER_ENV_STEP = 2 * (301 * 256 + 256 * 256 + 256 * 30)    # 300,544: the unfactored MLP
# tensor-core work the fused kernel performs per env-step with the factored layer 1
# (DESIGN.md §4.3): 31 env-private inputs in layer 1, layers 2 and 3 unchanged
FLOP_PER_ENV_STEP = 2 * (31 * 256 + 256 * 256 + 256 * 30)          # 162,304
Z1S_FLOP_PER_ROLLOUT = 2 * 270 * 256 * ROWS   # fp64 CUDA-core precompute of the per-day layer-1 term
# K1 algorithmic bytes per env-step: read cash 8 + holdings 60 + clock 4 + action 60,
# write cash 8 + holdings 60 + clock 4 + reward 4 + done 1 = 209 B.  The kernel moves 237 B: it also
# reads and writes the cached asset v (8 + 8), reads the window (4), and the holdings travel as
# 16-B asset octets (2 pad assets: 4 + 4) -- DESIGN.md 4.2.
STEP_BYTES_ALGO = 8 + 60 + 4 + 60 + 8 + 60 + 4 + 4 + 1                  # 209
STEP_BYTES_MOVED = STEP_BYTES_ALGO + 8 + 8 + 4 + 4 + 4                    # 237
# K3 HBM bytes per env-step the fused rollout must write (reward f32 + done u8; state is on chip)
ROLLOUT_HBM_BYTES = 5
METRIC = "env-steps/sec (whole box) at 2048-65536 envs, 1/2/4/8 B200; % HBM roofline"
WORKLOAD = "C1 30-stock env + 301-256-256-30 bf16 policy, 65536 envs/GPU, horizon 256, reset on done"


def peaks():
    p = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "source": "fallback"}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            m = json.load(f)
        p.update({k: m[k] for k in ("hbm_gbs", "bf16_tflops", "bf16_tflops_sustained") if k in m})
        p["source"] = "measured"
    except Exception:
        pass
    return p


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled while the timed region runs."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == 6:
                self.rows.append(parts)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        reasons = sorted({n for r in self.rows for n, v in zip(names, r[2:]) if v.lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def dist_info():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def _free_port() -> int:
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def self_launch(args) -> int | None:
    """``--gpus N`` (N > 1) outside a torch.distributed launcher: re-exec this script as
    N ranks (one process per GPU) under torch.distributed.run on 127.0.0.1 and return its
    exit code.  Inside a launcher, WORLD_SIZE must equal N.  Returns None when this
    process is a rank (or N = 1) and should run the benchmark itself."""
    world_env = os.environ.get("WORLD_SIZE")
    if world_env is not None:
        if int(world_env) != args.gpus:
            sys.stderr.write(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world_env}\n")
            return 2
        return None
    if args.gpus <= 1:
        return None
    import torch
    have = torch.cuda.device_count()
    if have < args.gpus:
        print(json.dumps({"metric": METRIC, "error": f"--gpus {args.gpus} but {have} CUDA devices visible",
                          "n_gpus": args.gpus}), flush=True)
        return 1
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def nccl_env():
    """NCCL's own INIT log (communicator size, transports, NVLS) on every rank's output."""
    os.environ.setdefault("NCCL_DEBUG", "INFO")
    os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")


# ------------------------------------------------------------------ oracle (CPU) timing
_SHARD_CACHE = {}


def _oracle_shard(args):
    n_envs, T, env_offset = args
    os.environ["OMP_NUM_THREADS"] = "1"
    from oracle import rollout as orol
    from oracle import stock as ostock
    from synth import inputs, market
    from synth import policy as spol
    if "m" not in _SHARD_CACHE:   # fixtures built once per worker process (not timed work)
        _SHARD_CACHE["m"] = market.stock_c1(rows=ROWS)
        _SHARD_CACHE["layers"] = spol.kaiming_bf16(spol.STOCK_DIMS, 0)
    m = _SHARD_CACHE["m"]
    cfg = ostock.StockEnvConfig(num_envs=n_envs, num_assets=K_ASSETS, num_indicators=N_IND, num_rows=ROWS,
                                episode_len=L_EP, window_stride=5, num_windows=195, window_block=128,
                                env_offset=env_offset)
    layers = _SHARD_CACHE["layers"]
    noise = inputs.supplied_noise(T, 1, n_envs, K_ASSETS, seed=23 + env_offset)
    t0 = time.perf_counter()
    orol.stock_policy_rollout(cfg, m.market, [layers], [orol.PPO_GAUSS], noise, T)
    return time.perf_counter() - t0


def _oracle_c0(_):
    """C0 in full (SURVEY d.5 (i)): K=4, I=4, 8 envs x 64 steps of supplied actions, no policy."""
    os.environ["OMP_NUM_THREADS"] = "1"
    from oracle import stock as ostock
    from synth import inputs, market
    m = market.stock_c0()
    cfg = ostock.StockEnvConfig(num_envs=8, num_assets=4, num_indicators=4, num_rows=m.rows, episode_len=64)
    acts = inputs.stock_actions(64, 8, 4, seed=12)
    t0 = time.perf_counter()
    ostock.run_actions(cfg, m.market, acts)
    return time.perf_counter() - t0


def _oracle_c3(args):
    """A C3 slice (SURVEY d.5 (iii)): n envs x T steps of the crypto env with the f64 Q-net."""
    n_envs, T = args
    os.environ["OMP_NUM_THREADS"] = "1"
    from oracle import crypto as ocry
    from oracle import rollout as orol
    from synth import market
    from synth import policy as spol
    rows = market.crypto_market(T, seed=41)
    cfg = ocry.CryptoEnvConfig(num_envs=n_envs, episode_len=T)
    layers = spol.kaiming_bf16(spol.CRYPTO_DIMS, 4)
    t0 = time.perf_counter()
    orol.crypto_q_rollout(cfg, rows, layers, T)
    return time.perf_counter() - t0


def oracle_slices():
    """the oracle on ONE core -- the C1 slice (64 envs x 30 steps with the
    f64 MLP), C0 in full, a C3 slice -- env-steps/s each."""
    for v in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
        os.environ[v] = "1"
    import multiprocessing as mp
    res = {"cores": 1}
    with mp.get_context("spawn").Pool(1) as pool:
        pool.map(_oracle_c0, [0])   # worker start-up and imports, not timed
        s = pool.map(_oracle_shard, [(64, 30, 0)])[0]
        res["c1_slice_64envs_x_30"] = 64 * 30 / s
        s = pool.map(_oracle_c0, [0])[0]
        res["c0_full_8envs_x_64"] = 8 * 64 / s
        s = pool.map(_oracle_c3, [(64, 1000)])[0]
        res["c3_slice_64envs_x_1000"] = 64 * 1000 / s
    return res


def oracle_rate(n_envs_per_core=2560, T=30, cores=None):
    """Oracle env-steps/s on the host's cores (multiprocessing over env shards)."""
    import multiprocessing as mp
    for v in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
        os.environ[v] = "1"
    if cores is None:
        cores = len(os.sched_getaffinity(0))
    t0 = time.perf_counter()
    with mp.get_context("spawn").Pool(cores) as pool:
        pool.map(_oracle_shard, [(n_envs_per_core, T, 128 * c) for c in range(cores)])
    wall = time.perf_counter() - t0
    steps = n_envs_per_core * T * cores
    return steps / wall, cores, f"{cores} shards x {n_envs_per_core} envs x {T} steps (one C1 episode) of the " \
                                f"headline workload (float64 oracle incl. 301-256-256-30 MLP), wall {wall:.1f}s"


# ------------------------------------------------------------------ GPU arm
def make_env(fin, N, env_offset, T_ep=L_EP):
    from synth import market
    m = market.stock_c1(rows=ROWS)
    cfg = fin.env_config(num_envs=N, num_assets=K_ASSETS, num_indicators=N_IND, num_rows=ROWS, episode_len=T_ep,
                         window_stride=5, num_windows=195, window_block=128, env_offset=env_offset, seed=23)
    return fin.fin_env_create(cfg, m.market)


class L2Flush:
    """Write 256 MiB, then read another 256 MiB: the written lines are evicted (and
    written back) by the read pass, so the next timed region starts on a clean L2
    that holds none of the step's inputs (126 MB L2)."""

    def __init__(self, torch):
        self.w = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
        self.r = torch.ones(64 << 20, dtype=torch.float32, device="cuda")

    def zero_(self):
        self.w.zero_()
        self.r.sum()


def time_rollouts(fin, torch, env, pol, N, T, steps, warmup, flush=None, allreduce=None, clocks_index=None):
    """Returns (per-step ms list (kernel events), launches per step, agg)."""
    stream = torch.cuda.current_stream()
    z = lambda s, d: torch.zeros(s, dtype=d, device="cuda")  # noqa: E731
    reward, done, agg = z((T, N), torch.float32), z((T, N), torch.uint8), z(8, torch.float64)
    traj = fin.make_traj(reward=reward, done=done, agg=agg)
    noise = fin.make_noise(fin.FIN_NOISE_PHILOX, 1234)
    for _ in range(warmup):
        fin.fin_rollout(env, [pol], T, noise, traj, stream=stream)
    torch.cuda.synchronize()
    times = []
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    for i in range(steps):
        if flush is not None:
            flush.zero_()
        ev[i][0].record(stream)
        fin.fin_rollout(env, [pol], T, noise, traj, stream=stream)
        if allreduce is not None:
            allreduce(agg)
        ev[i][1].record(stream)
    torch.cuda.synchronize()
    times = [a.elapsed_time(b) for a, b in ev]
    return times, agg


def run_ours(args):
    import torch
    rank, world, local = dist_info()
    torch.cuda.set_device(local)
    if world > 1:
        import datetime

        import torch.distributed as dist
        nccl_env()
        dist.init_process_group("nccl", device_id=torch.device("cuda", local),
                                timeout=datetime.timedelta(minutes=30))
    from paper_2501_10709_b200 import fin
    from synth import policy as spol
    fin.fin_device_check(local)
    N, T = N_HEAD, T_HEAD
    env = make_env(fin, N, env_offset=rank * N)
    pol = fin.fin_policy_create(fin.FIN_PPO_GAUSS, spol.kaiming_bf16(spol.STOCK_DIMS, 0))
    flush = L2Flush(torch)

    from paper_2501_10709_b200 import dist as fdist

    def allreduce(agg):   # the one collective of the path: per-rank FIN_AGG_* partials (NCCL)
        fdist.allreduce_agg(agg)

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()
        torch.cuda.synchronize()

    barrier()
    with ClockSampler(local) as cs:
        times, agg = time_rollouts(fin, torch, env, pol, N, T, args.steps, args.warmup, flush, allreduce)
    barrier()
    total_ms = fdist.max_over_ranks(sum(times), device="cuda")
    units = N * T * world * args.steps
    value = units / (total_ms / 1e3)
    ms_per_step = total_ms / args.steps
    kern_ms = statistics.mean(times)      # whole fin_rollout call (z1s prep + rollout + agg): conservative
    flops = FLOP_PER_ENV_STEP * N * T
    pk = peaks()
    achieved = flops / (kern_ms / 1e3) / 1e12
    out = {"metric": METRIC, "value": value, "unit": "env-steps/s", "n_gpus": world, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
           "vs_baseline": None, "dtype": "bf16 MLP (fp32 accum) + f64 env", "data": "synthetic",
           "config": {"workload": WORKLOAD, "envs_per_gpu": N, "horizon": T, "episode_len": L_EP,
                      "global_envs": N * world, "parallelism": f"env-sharded dp{world}",
                      "l2": "flushed between timed steps (256 MiB write + 256 MiB read, outside the events)",
                      "noise": "philox"},
           "gpu_launches": 2 * args.steps,   # per rollout: fused rollout + aggregate finalize, plus one
                                             # memset of the chunk queue's counter (the layer-1
                                             # shared term is cached per env: computed by the first call)
           "roofline": {"bound": "tensor", "achieved": achieved, "peak": pk["bf16_tflops"],
                        "unit": "TFLOP/s", "frac": achieved / pk["bf16_tflops"], "traffic": None,
                        "kernel": "k_tc_rollout<PlanStockC1> (fused rollout)",
                        "flop_per_env_step": FLOP_PER_ENV_STEP,
                        "frac_of_sustained": achieved / pk["bf16_tflops_sustained"],
                        "note": "tensor FLOPs the kernel executes (factored layer 1, DESIGN.md 4.3); the "
                                "unfactored MLP is %d FLOP/env-step = %.1f TFLOP/s equivalent. Peak: the burst "
                                "bf16 figure (one ~7 ms launch at the max SM clock between L2 flushes)"
                                % (MLP_FLOP_PER_ENV_STEP, MLP_FLOP_PER_ENV_STEP * N * T / (kern_ms / 1e3) / 1e12),
                        "peak_source": pk["source"] + " bf16 burst",
                        "hbm": {"bytes_per_env_step": ROLLOUT_HBM_BYTES,
                                "achieved_gbs": ROLLOUT_HBM_BYTES * N * T / (kern_ms / 1e3) / 1e9,
                                "peak_gbs": pk["hbm_gbs"],
                                "frac": ROLLOUT_HBM_BYTES * N * T / (kern_ms / 1e3) / 1e9 / pk["hbm_gbs"],
                                "note": "BASELINE metric's % HBM roofline for the fused rollout: it writes reward "
                                        "+ done (5 B/env-step), env state stays on chip; the HBM-bound kernels "
                                        "are in extras (K1 / K4 / K6)"}}}
    prof = os.path.join(ROOT, "profiles", "roofline_traffic.json")
    if os.path.exists(prof):
        with open(prof) as f:
            out["roofline"]["traffic"] = json.load(f).get("rollout_bytes_per_launch")
    out["clocks"] = cs.summary()
    if world > 1:
        out["nccl"] = nccl_info(torch, world)
    # ---- e2e through the C ABI with host buffers (every rank, max over ranks)
    out["e2e"] = e2e(fin, torch, env, pol, N, T, max(4, args.steps), allreduce, world)
    del env
    # ---- the C4 sweep at this G (every rank, max over ranks)
    out["c4_sweep"] = c4_sweep(fin, torch, pol, world, allreduce, barrier)
    if rank == 0 and world == 1 and not args.no_extras:
        out["extras"] = extras(fin, torch, pol)
    if rank == 0 and world == 1:
        rate, cores, sample = oracle_rate()
        out["cpu_baseline"] = {"value": rate, "unit": "env-steps/s", "cores": cores, "kind": "oracle", "sample": sample,
                               "one_core": oracle_slices()}
        out["cpu_baseline"]["gpu_over_oracle"] = {"all_cores": value / rate,
                                                  "one_core_c1": value / out["cpu_baseline"]["one_core"]["c1_slice_64envs_x_30"],
                                                  "note": "GPU / oracle speedups, labelled (the oracle is a deliberately "
                                                          "plain float64 program)"}
        out["paper_context"] = {"note": "paper numbers are from one NVIDIA A100 with real data and PPO/DQN training "
                                        "(P:380, P:336); context only",
                                "stock_samples_per_s_2048_envs_A100": 8813.81, "stock_speedup_2048_vs_1": 47.73,
                                "crypto_samples_per_s_2048_envs_A100": 114885.98, "crypto_speedup_2048_vs_1": 1746.25}
        print(json.dumps(out), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


def nccl_info(torch, world):
    """The communicator as NCCL and torch see it after the timed all-reduces."""
    import torch.distributed as dist
    info = {"backend": dist.get_backend(), "world_size": dist.get_world_size(), "nccl_version":
            ".".join(str(v) for v in torch.cuda.nccl.version()), "nccl_debug": os.environ.get("NCCL_DEBUG")}
    ranks = torch.tensor([dist.get_rank()], dtype=torch.int64, device="cuda")
    seen = [torch.zeros_like(ranks) for _ in range(world)]
    dist.all_gather(seen, ranks)
    info["ranks_seen"] = [int(s.item()) for s in seen]
    return info


def c4_sweep(fin, torch, pol, world, allreduce, barrier):
    """BASELINE configs[4]: N/GPU in {1, 64, 2048, 16384, 65536} at T = 256 on this box's G
    GPUs (G = world size): every rank runs its shard (env_offset = rank * N), the per-rollout
    aggregate is all-reduced, and the rate is N * T * G / the slowest rank's time."""
    from paper_2501_10709_b200 import dist as fdist
    rank = int(os.environ.get("RANK", 0))
    res = {"G": world, "T": T_HEAD, "env_steps_per_s": {}}
    flush = L2Flush(torch)
    for N in (1, 64, 2048, 16384, 65536):
        env = make_env(fin, N, rank * N)
        barrier()
        times, _ = time_rollouts(fin, torch, env, pol, N, T_HEAD, 5, 3, flush, allreduce)
        barrier()
        ms = fdist.max_over_ranks(statistics.mean(times), device="cuda")
        res["env_steps_per_s"][str(N)] = N * T_HEAD * world / (ms / 1e3)
        del env
    r = res["env_steps_per_s"]
    res["same_gpu_scaling_2048_vs_1"] = r["2048"] / r["1"]
    res["paper_same_gpu_scaling_2048_vs_1"] = {"crypto_dqn_A100": 1746.25, "stock_ppo_A100": 47.73,
                                               "note": "P:380: GPU(2048 envs) / GPU(1 env) on one A100; context"}
    return res


def e2e(fin, torch, env, pol, N, T, steps, allreduce, world):
    """Same metric through the public C ABI with host buffers (pinned): per step the
    input state goes H2D, the rollout runs, reward / done / agg come back D2H.  The
    copies run on their own streams and overlap the neighbouring steps' rollouts
    (double-buffered trajectories), as a production producer loop would; the timed
    region spans all of it, from the first H2D to the last D2H."""
    z = lambda s, d: torch.zeros(s, dtype=d, device="cuda")  # noqa: E731
    h_cash = torch.full((N,), 1e6, dtype=torch.float64).pin_memory()
    h_hold = torch.zeros((N, K_ASSETS), dtype=torch.int16).pin_memory()
    h_tep = torch.zeros((N,), dtype=torch.int32).pin_memory()
    h_rew = [torch.empty((T, N), dtype=torch.float32).pin_memory() for _ in range(2)]
    h_done = [torch.empty((T, N), dtype=torch.uint8).pin_memory() for _ in range(2)]
    h_agg = [torch.empty(8, dtype=torch.float64).pin_memory() for _ in range(2)]
    d_cash, d_hold, d_tep = [z(N, torch.float64) for _ in range(2)], [z((N, K_ASSETS), torch.int16) for _ in range(2)], \
        [z(N, torch.int32) for _ in range(2)]
    reward, done = [z((T, N), torch.float32) for _ in range(2)], [z((T, N), torch.uint8) for _ in range(2)]
    agg = [z(8, torch.float64) for _ in range(2)]
    trajs = [fin.make_traj(reward=reward[q], done=done[q], agg=agg[q]) for q in range(2)]
    noise = fin.make_noise(fin.FIN_NOISE_PHILOX, 99)
    comp = torch.cuda.current_stream()
    up, down = torch.cuda.Stream(), torch.cuda.Stream()
    h2d_done = [torch.cuda.Event() for _ in range(2)]
    roll_done = [torch.cuda.Event() for _ in range(2)]
    d2h_done = [torch.cuda.Event() for _ in range(2)]

    def one(i):
        q = i & 1
        with torch.cuda.stream(up):          # inputs of step i (buffer q is free once step i-2 is read)
            up.wait_event(d2h_done[q])
            d_cash[q].copy_(h_cash, non_blocking=True)
            d_hold[q].copy_(h_hold, non_blocking=True)
            d_tep[q].copy_(h_tep, non_blocking=True)
            h2d_done[q].record(up)
        comp.wait_event(h2d_done[q])
        comp.wait_event(d2h_done[q])          # trajectory buffer q read back (step i-2)
        fin.fin_env_set_state(env, cash=d_cash[q], hold=d_hold[q], t_ep=d_tep[q], stream=comp)
        fin.fin_rollout(env, [pol], T, noise, trajs[q], stream=comp)
        allreduce(agg[q])
        roll_done[q].record(comp)
        with torch.cuda.stream(down):
            down.wait_event(roll_done[q])
            h_rew[q].copy_(reward[q], non_blocking=True)
            h_done[q].copy_(done[q], non_blocking=True)
            h_agg[q].copy_(agg[q], non_blocking=True)
            d2h_done[q].record(down)

    for q in range(2):
        d2h_done[q].record(down)
    one(0)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(comp)
    up.wait_event(a)
    for i in range(steps):
        one(i)
    b.record(down)
    torch.cuda.synchronize()
    ms = a.elapsed_time(b)
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    h2d = N * (8 + 2 * K_ASSETS + 4)
    d2h = T * N * 5 + 64
    return {"value": N * T * world * steps / (ms / 1e3), "unit": "env-steps/s", "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": d2h, "steps": steps, "overlap": "H2D / D2H on their own streams, double-buffered"}


def extras(fin, torch, pol):
    """Secondary measurements printed inside the same JSON line (rank 0, N = 1 GPU):
    the exact configs[1] rollout (2048 envs, T = 30), the HBM-bound kernels against
    the measured HBM copy bandwidth, the crypto, ensemble and paper-net variants."""
    out = {}
    flush = L2Flush(torch)
    env = make_env(fin, 2048, 0)
    times, _ = time_rollouts(fin, torch, env, pol, 2048, 30, 10, 3, flush)
    out["configs1_2048envs_T30"] = 2048 * 30 / (statistics.mean(times) / 1e3)
    del env
    out["z1s_precompute"] = z1s_cost(fin, torch)
    out.update(hbm_kernels(fin, torch))
    out["crypto_c3"] = crypto_c3(fin, torch)
    out["ensembles"] = ensembles(fin, torch)
    out["paper_nets"] = paper_nets(fin, torch)
    out["market_prep"] = market_prep(fin, torch)
    out["consumer"] = consumer(fin, torch)
    return out


def z1s_cost(fin, torch):
    """The per-day shared layer-1 term z1s (1008 days x 270 x 256 float64 FMAs) is cached per env
    and recomputed only when the member list changes, so the headline's timed calls do not
    include it (its first call does).  A training loop that updates the weights before every
    rollout pays it each time: alternate two policies (every call recomputes) vs one policy."""
    from synth import policy as spol
    N, T = N_HEAD, T_HEAD
    env = make_env(fin, N, 0)
    pa = fin.fin_policy_create(fin.FIN_PPO_GAUSS, spol.kaiming_bf16(spol.STOCK_DIMS, 0))
    pb = fin.fin_policy_create(fin.FIN_PPO_GAUSS, spol.kaiming_bf16(spol.STOCK_DIMS, 1))
    z = lambda s, d: torch.zeros(s, dtype=d, device="cuda")  # noqa: E731
    tr = fin.make_traj(reward=z((T, N), torch.float32), done=z((T, N), torch.uint8), agg=z(8, torch.float64))
    nz = fin.make_noise(fin.FIN_NOISE_PHILOX, 3)

    def timed(pols):
        for q in pols[:2]:
            fin.fin_rollout(env, [q], T, nz, tr)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for q in pols:
            fin.fin_rollout(env, [q], T, nz, tr)
        b.record()
        torch.cuda.synchronize()
        return a.elapsed_time(b) / len(pols)

    same = timed([pa] * 6)
    alt = timed([pa, pb] * 3)
    return {"ms_per_rollout_same_policy": same, "ms_per_rollout_new_weights_each_call": alt,
            "z1s_ms": alt - same, "note": "excluded from the headline (cached); paid once per weight update"}


def consumer(fin, torch):
    """The consumer's first steps on the rollout's tensors (NEXT-4): GAE over the headline
    trajectory shape (65,536 envs x 256 steps; 17 B per env-step: reward f32 + done u8 +
    value f32 read, advantage + return f32 written), with and without batch normalisation,
    and the Eq. 5 KL term of three members over 65,536 states."""
    pk = peaks()
    N, T = N_HEAD, T_HEAD
    g = torch.Generator(device="cuda").manual_seed(4)
    rew = torch.randn((T, N), device="cuda", generator=g)
    val = torch.randn((T + 1, N), device="cuda", generator=g)
    done = torch.zeros((T, N), dtype=torch.uint8, device="cuda")
    done[29::30] = 1
    adv, ret = torch.empty_like(rew), torch.empty_like(rew)
    res = {}
    for norm in (False, True):
        for _ in range(3):
            fin.fin_gae(rew, val, done, adv, ret, normalise=norm)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(10):
            fin.fin_gae(rew, val, done, adv, ret, normalise=norm)
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / 10
        byts = T * N * 17 + N * 4 + (T * N * 8 if norm else 0)
        gbs = byts / (ms / 1e3) / 1e9
        res["gae" + ("_normalised" if norm else "")] = {
            "envs": N, "T": T, "ms": ms, "env_steps_per_s": N * T / (ms / 1e3), "bytes_per_launch": byts,
            "achieved_gbs": gbs, "frac": gbs / pk["hbm_gbs"]}
    out = torch.tanh(torch.randn((3, N, 30), device="cuda", generator=g))
    D = torch.zeros((3, 3), dtype=torch.float64, device="cuda")
    fin.fin_kl_diversity(out, D)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    fin.fin_kl_diversity(out, D)
    b.record()
    torch.cuda.synchronize()
    res["kl_diversity_3x65536x30"] = {"ms": a.elapsed_time(b)}
    res["ppo_step"] = ppo_step(fin, torch)
    res["ppo_iteration"] = ppo_iteration(fin, torch)
    res["actor_critic"] = {f"{kind}_B{B}": ac_update(fin, torch, kind, B) for kind in ("ddpg", "sac") for B in (64, 65536)}
    return res


def ppo_iteration(fin, torch, B=65536):
    """One producer -> consumer iteration at the headline size (NEXT-4): the fused rollout of 65,536
    envs x 256 steps logging the env-private observation entries and days; then on a minibatch of
    B random samples: gather the observations, the old policy's forward, the Philox noise, the
    Gaussian sample and its log-density, the PPO gradient, Adam, and installing the new weights."""
    import numpy as np
    from synth import policy as spol
    N, T = N_HEAD, T_HEAD
    env = make_env(fin, N, 0)
    layers = spol.kaiming_bf16(spol.STOCK_DIMS, 0)
    pol = fin.fin_policy_create(fin.FIN_PPO_GAUSS, layers)
    z = lambda s, d: torch.zeros(s, dtype=d, device="cuda")  # noqa: E731
    logs = dict(reward=z((T, N), torch.float32), done=z((T, N), torch.uint8), obs_private=z((T, N, 32), torch.int16),
                day=z((T, N), torch.int32))
    tr = fin.make_traj(**logs)
    seed = 5
    ev = lambda: (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))  # noqa: E731
    fin.fin_rollout(env, [pol], T, fin.make_noise(fin.FIN_NOISE_PHILOX, seed), tr)
    t_base = fin.fin_env_clock(env)
    a0, a1 = ev()
    a0.record()
    fin.fin_rollout(env, [pol], T, fin.make_noise(fin.FIN_NOISE_PHILOX, seed), tr)
    a1.record()
    g = torch.Generator(device="cuda").manual_seed(3)
    idx = torch.randint(0, T * N, (B,), device="cuda", generator=g, dtype=torch.int64)
    x, zo, hid = z((B, 301), torch.int16), z((B, 30), torch.float32), z((B, 2, 256), torch.int16)
    eps, a, lpo = z((B, 30), torch.float32), z((B, 30), torch.float32), z(B, torch.float32)
    adv = torch.randn(B, device="cuda", generator=g)
    w = [torch.from_numpy((W.astype(np.uint32) << 16).view(np.float32)).cuda() for W, _ in layers]
    bias = [z(W.shape[0], torch.float32) for W in w]
    grads = [(torch.empty_like(W), torch.empty(W.shape[0], device="cuda")) for W in w]
    opt = [(torch.zeros_like(p), torch.zeros_like(p)) for p in w + bias]
    stats = z(4, torch.float64)

    def learner():
        fin.fin_gather_observations(env, logs["obs_private"], logs["day"], idx, x)
        fin.fin_mlp_forward(pol, x, zo, hid)
        fin.fin_rollout_noise(env, seed, t_base, idx, eps)
        fin.fin_ppo_prepare(zo, eps, a, lpo)
        fin.fin_ppo_grad(x, hid, zo, a, lpo, adv, w[1], w[2], grads, stats)
        for p, gr, (mm, vv) in zip(w + bias, [q for q, _ in grads] + [q for _, q in grads], opt):
            fin.fin_adam_step(p, mm, vv, gr, 1, lr=1e-5)

    learner()
    torch.cuda.synchronize()
    b0, b1 = ev()
    b0.record()
    learner()
    b1.record()
    torch.cuda.synchronize()
    learner_ms = b0.elapsed_time(b1)
    fin.fin_policy_load(pol, w, bias)   # first call: builds the handle's gather table
    torch.cuda.synchronize()
    b0.record()
    fin.fin_policy_load(pol, w, bias)
    b1.record()
    torch.cuda.synchronize()
    return {"rollout_ms_with_obs_logs": a0.elapsed_time(a1), "minibatch": B, "learner_ms": learner_ms,
            "policy_load_ms": b0.elapsed_time(b1), "obs_log_bytes_per_env_step": 64 + 4,
            "note": "learner = gather + forward + noise + prepare + PPO gradient + Adam; policy_load gathers the "
                    "bf16 tcgen05 image on the device (stream-ordered)"}


def ac_update(fin, torch, kind: str, B: int):
    """One DDPG or SAC update (reading R-AC; learner.ddpg_update / sac_update) on B samples of the C1
    actor (301-256-256-30, tcgen05 forward) with 331-256-256-1 fp32 critics (two for SAC) and their
    targets: forwards, float64 heads, backwards, Adam, soft updates and the actor's fin_policy_load
    (a host repack that synchronises the stream).  B = 64 is the paper's batch size."""
    import numpy as np
    from paper_2501_10709_b200 import learner
    from synth import policy as spol
    sac = kind == "sac"
    layers = spol.kaiming_bf16(spol.STOCK_DIMS, 0)
    k = fin.FIN_SAC_SQUASH if sac else fin.FIN_DDPG_OU
    actor = learner.Actor(k, layers)
    g = torch.Generator(device="cuda").manual_seed(5)
    batch = dict(x=torch.randn((B, 301), device="cuda", generator=g).to(torch.bfloat16).view(torch.int16),
                 x_next=torch.randn((B, 301), device="cuda", generator=g).to(torch.bfloat16).view(torch.int16),
                 a=torch.tanh(torch.randn((B, 30), device="cuda", generator=g)),
                 reward=torch.randn(B, device="cuda", generator=g), done=torch.zeros(B, dtype=torch.uint8, device="cuda"))
    if sac:
        batch["eps"] = torch.randn((B, 30), device="cuda", generator=g)
        batch["eps_next"] = torch.randn((B, 30), device="cuda", generator=g)
        critics = [learner.DenseNet((331, 256, 256, 1), s) for s in (1, 2)]
        targs = [c.copy() for c in critics]
        step = lambda: learner.sac_update(actor, critics, targs, batch)
    else:
        actor_t = learner.Actor(k, layers)
        critic = learner.DenseNet((331, 256, 256, 1), 1)
        targ = critic.copy()
        step = lambda: learner.ddpg_update(actor, actor_t, critic, targ, batch)
    for _ in range(3):
        step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        step()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    return {"samples": B, "ms_per_update": ms, "samples_per_s": B / (ms / 1e3),
            "note": "critic layers and weight gradients on the tensor cores (bf16 hi/lo split), heads in float64; includes the actor's fin_policy_load (device gather)"}


def ppo_step(fin, torch, B=65536):
    """The policy-gradient step (Eq. 3-4, PPO surrogate; NEXT-4) on a minibatch of B samples of
    the C1 policy: the tcgen05 forward (fin_mlp_forward), fin_ppo_grad (float64 head, fp32 CUDA-core
    contractions) and one Adam step over the 150,304 parameters.  FLOPs: forward 2 B (301 256 +
    256 256 + 256 30), backward 2 B (30 256 + 256 256) for the propagated deltas and 2 B (30 256 +
    256 256 + 256 301) for the weight gradients; the contractions' bound is the fp32 CUDA-core
    peak 148 SMs x 128 lanes x 2 FLOP x 1.965 GHz = 74.4 TFLOP/s (alu)."""
    import numpy as np
    from synth import policy as spol
    layers = spol.kaiming_bf16(spol.STOCK_DIMS, 0)
    pol = fin.fin_policy_create(fin.FIN_PPO_GAUSS, layers)
    g = torch.Generator(device="cuda").manual_seed(9)
    x = torch.randn((B, 301), device="cuda", generator=g).to(torch.bfloat16).view(torch.int16)
    z = torch.empty((B, 30), dtype=torch.float32, device="cuda")
    hid = torch.empty((B, 2, 256), dtype=torch.int16, device="cuda")
    a = torch.randn((B, 30), device="cuda", generator=g) * 0.1
    logp_old = torch.zeros(B, device="cuda")
    adv = torch.randn(B, device="cuda", generator=g)
    ws = [torch.from_numpy((w.astype(np.uint32) << 16).view(np.float32)).cuda() for w, _ in layers]
    grads = [(torch.empty_like(w), torch.empty(w.shape[0], device="cuda")) for w in ws]
    stats = torch.empty(4, dtype=torch.float64, device="cuda")
    n = sum(w.numel() + w.shape[0] for w in ws)
    theta, m, v, gflat = (torch.zeros(n, device="cuda") for _ in range(4))

    def step():
        fin.fin_mlp_forward(pol, x, z, hid)
        fin.fin_ppo_grad(x, hid, z, a, logp_old, adv, ws[1], ws[2], grads, stats)
        fin.fin_adam_step(theta, m, v, gflat, 1)

    for _ in range(3):
        step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        fin.fin_ppo_grad(x, hid, z, a, logp_old, adv, ws[1], ws[2], grads, stats)
    e1.record()
    torch.cuda.synchronize()
    ms_grad = e0.elapsed_time(e1) / 5
    e0.record()
    for _ in range(5):
        step()
    e1.record()
    torch.cuda.synchronize()
    ms_step = e0.elapsed_time(e1) / 5
    flop_grad = 2 * B * (30 * 256 + 256 * 256) + 2 * B * (30 * 256 + 256 * 256 + 256 * 301)
    return {"samples": B, "ms_forward_grad_adam": ms_step, "ms_grad": ms_grad,
            "samples_per_s": B / (ms_step / 1e3), "grad_tflops": flop_grad / (ms_grad / 1e3) / 1e12,
            "grad_frac_of_fp32_simt_peak": flop_grad / (ms_grad / 1e3) / 1e12 / 74.4,  # (context: mixed TC / CUDA-core path)
            "note": "weight gradients and the K = 256 backpropagated product on the tensor cores (tc_gemm.cu: bf16 hi/lo split operands, fp32 accumulation); the K = 30 product and the forward on fp32 CUDA cores; grad_tflops counts the useful FLOPs"}


def market_prep(fin, torch):
    """The step before the rollout on the device (NEXT-3): fin_market_prepare at the C1
    shape (30 assets, 64 warm-up + 1,008 stored days, 8 indicator families, +-1% price-scale
    perturbation) and fin_crypto_market at the C3 length (480,000 steps x 144 f32)."""
    import numpy as np
    from synth import market
    res = {}
    m = market.stock_c1()
    x = np.stack([m.open_all, m.high_all, m.low_all, m.close_all, m.volume_all], axis=1).astype(np.float32)
    D, K = x.shape[0], x.shape[2]
    xd = torch.from_numpy(x).cuda()
    ind = list(range(8))
    mk = torch.zeros((D - market.WARMUP_DAYS, 10, K), dtype=torch.float32, device="cuda")
    raw = torch.zeros((8, K, D - market.WARMUP_DAYS), dtype=torch.float64, device="cuda")

    def ev(fn):
        fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        return a.elapsed_time(b)

    ms = ev(lambda: fin.fin_market_prepare(xd, market.WARMUP_DAYS, ind, mk, raw, magnitude=0.01, seed=7))
    res["stock_prepare_c1"] = {"assets": K, "days": D, "indicators": 8, "ms": ms}
    og = torch.zeros((D, 5, K), dtype=torch.float32, device="cuda")
    ms = ev(lambda: fin.fin_stock_market(D, K, 21, og))
    res["stock_generate_c1"] = {"assets": K, "days": D, "ms": ms, "note": "GBM close + OHLV (R-SGEN)"}
    steps = 480000
    rows = torch.zeros((steps + 1, 144), dtype=torch.float32, device="cuda")
    ms = ev(lambda: fin.fin_crypto_market(steps, 43, rows))
    res["crypto_market_c3"] = {"steps": steps, "ms": ms, "bytes_written": (steps + 1) * 144 * 4}
    return res


def paper_nets(fin, torch):
    """The paper's own network shapes (NEXT-3 / NEXT-2 variants): the stock PPO policy with
    hidden layers of 64 and 32 units on the headline workload (C1 env, 65,536 envs,
    T = 256, Philox noise; weights resident in shared memory), and the crypto Q-net with
    three 128-unit hidden layers on the C3 env (4,096 envs, 48,000 steps)."""
    from synth import market
    from synth import policy as spol
    res = {}
    flush = L2Flush(torch)
    N = N_HEAD
    env = make_env(fin, N, 0)
    pol = fin.fin_policy_create(fin.FIN_PPO_GAUSS, spol.kaiming_bf16(spol.STOCK_PAPER_DIMS, 0))
    times, _ = time_rollouts(fin, torch, env, pol, N, T_HEAD, 5, 3, flush)
    ms = statistics.mean(times)
    d = spol.STOCK_PAPER_DIMS
    res["stock_64_32"] = {"dims": list(d), "envs": N, "T": T_HEAD, "ms": ms, "env_steps_per_s": N * T_HEAD / (ms / 1e3),
                          "flop_per_env_step_executed": 2 * (64 * 32 + 32 * 64 + 32 * 32),
                          "flop_per_env_step_unfactored": 2 * sum(a * b for a, b in zip(d[:-1], d[1:])),
                          "note": "10 KB of weights resident in shared memory; env-side bound (trade, noise, obs)"}
    del env, pol
    z = lambda s, dt: torch.zeros(s, dtype=dt, device="cuda")  # noqa: E731
    N, T = 4096, 48000
    rows = market.crypto_market(T, seed=41)
    cfg = fin.env_config(task=fin.FIN_CRYPTO, num_envs=N, num_assets=1, num_indicators=0, num_rows=T + 1,
                         episode_len=T, reward_scale=1.0, cost_rate=0.0, epsilon=0.005, seed=43)
    pol = fin.fin_policy_create(fin.FIN_Q_ARGMAX, spol.kaiming_bf16(spol.CRYPTO_PAPER_DIMS, 4))
    nz = fin.make_noise(fin.FIN_NOISE_PHILOX, 43)
    fin.fin_rollout(fin.fin_env_create(cfg, rows), [pol], 1000, nz, fin.make_traj(reward=z((1000, N), torch.float32)))
    env = fin.fin_env_create(cfg, rows)
    tr = fin.make_traj(reward=z((T, N), torch.float32), done=z((T, N), torch.uint8))
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    fin.fin_rollout(env, [pol], T, nz, tr)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b)
    res["crypto_3x128"] = {"dims": list(spol.CRYPTO_PAPER_DIMS), "envs": N, "T": T, "ms": ms,
                           "env_steps_per_s": N * T / (ms / 1e3), "us_per_lockstep_step": 1e3 * ms / T}
    return res


def ensembles(fin, torch):
    """Ensemble rollouts (§5.2, §6.3-6.4): the C2 config (PPO + SAC + DDPG with OU,
    5-day test windows advancing on reset, uniform mean), the Sharpe-softmax weighted
    Ensemble-2 / -3 (5 / 10 members of each kind: 15 / 30 MLPs per env-step) at 16,384 envs,
    T = 30; and the crypto DQN / Double DQN / Dueling DQN vote at 4,096 envs."""
    from synth import market
    from synth import policy as spol
    res = {}
    flush = L2Flush(torch)
    z = lambda s, d: torch.zeros(s, dtype=d, device="cuda")  # noqa: E731
    m = market.stock_c1(rows=ROWS)
    kinds = [fin.FIN_PPO_GAUSS, fin.FIN_SAC_SQUASH, fin.FIN_DDPG_OU]
    for name, per_kind, N, T in (("c2_3_members", 1, 65536, 30), ("ensemble2_15_members", 5, 16384, 30),
                                 ("ensemble3_30_members", 10, 16384, 30)):
        M = 3 * per_kind
        cfg = fin.env_config(num_envs=N, num_assets=K_ASSETS, num_indicators=N_IND, num_rows=ROWS, episode_len=5,
                             window_stride=5, window_offset=35, num_windows=194, window_block=128,
                             advance_window_on_reset=1, seed=23)
        env = fin.fin_env_create(cfg, m.market)
        pols = [fin.fin_policy_create(kinds[j % 3], spol.kaiming_bf16(spol.STOCK_DIMS, 1 + j)) for j in range(M)]
        w = None if per_kind == 1 else [1.0 / M] * M
        tr = fin.make_traj(reward=z((T, N), torch.float32), done=z((T, N), torch.uint8), agg=z(8, torch.float64))
        nz = fin.make_noise(fin.FIN_NOISE_PHILOX, 33)
        for _ in range(2):
            fin.fin_rollout(env, pols, T, nz, tr, member_w=w)
        ts = []
        for _ in range(3):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fin.fin_rollout(env, pols, T, nz, tr, member_w=w)
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        ms = statistics.median(ts)
        res[name] = {"members": M, "envs": N, "T": T, "ms": ms, "env_steps_per_s": N * T / (ms / 1e3),
                     "mlp_evals_per_s": M * N * T / (ms / 1e3),
                     "combine": "uniform mean" if w is None else "weighted (member_w)"}
        del env, pols
    rows = market.crypto_market(4800, seed=41)
    N, T = 4096, 4800
    cfg = fin.env_config(task=fin.FIN_CRYPTO, num_envs=N, num_assets=1, num_indicators=0, num_rows=T + 1,
                         episode_len=T, reward_scale=1.0, cost_rate=0.0, epsilon=0.005, seed=43)
    qk = [fin.FIN_Q_ARGMAX, fin.FIN_Q_ARGMAX, fin.FIN_Q_DUELING]
    pols = []
    for j in range(3):
        dims = spol.CRYPTO_DIMS if qk[j] == fin.FIN_Q_ARGMAX else tuple(spol.CRYPTO_DIMS[:-1]) + (4,)
        pols.append(fin.fin_policy_create(qk[j], spol.kaiming_bf16(dims, 4 + j)))
    tr = fin.make_traj(reward=z((T, N), torch.float32), done=z((T, N), torch.uint8))
    nz = fin.make_noise(fin.FIN_NOISE_PHILOX, 43)
    fin.fin_rollout(fin.fin_env_create(cfg, rows), pols, 500, nz, fin.make_traj(reward=z((500, N), torch.float32)))
    env = fin.fin_env_create(cfg, rows)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    fin.fin_rollout(env, pols, T, nz, tr)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b)
    res["crypto_vote_3_members"] = {"members": 3, "envs": N, "T": T, "ms": ms, "env_steps_per_s": N * T / (ms / 1e3),
                                    "us_per_lockstep_step": 1e3 * ms / T}
    return res


def crypto_c3(fin, torch):
    """BASELINE configs[3] at full length: 4096 envs x 480,000 one-second steps (one
    episode), Q-net 103-128-128-3, epsilon-greedy 0.005 (Philox), in 10 calls of 48,000
    steps; latency-bound (all envs advance in lockstep)."""
    from synth import market
    from synth import policy as spol
    N, T, calls = 4096, 480000, 10
    rows = market.crypto_market(T, seed=41)
    cfg = fin.env_config(task=fin.FIN_CRYPTO, num_envs=N, num_assets=1, num_indicators=0, num_rows=T + 1,
                         episode_len=T, reward_scale=1.0, cost_rate=0.0, epsilon=0.005, seed=43)
    pol = fin.fin_policy_create(fin.FIN_Q_ARGMAX, spol.kaiming_bf16(spol.CRYPTO_DIMS, 4))
    Tc = T // calls
    z = lambda s, d: torch.zeros(s, dtype=d, device="cuda")  # noqa: E731
    rew, done, agg = z((Tc, N), torch.float32), z((Tc, N), torch.uint8), z(8, torch.float64)
    tr = fin.make_traj(reward=rew, done=done, agg=agg)
    nz = fin.make_noise(fin.FIN_NOISE_PHILOX, 43)
    warm = fin.fin_env_create(cfg, rows)
    for _ in range(3):
        fin.fin_rollout(warm, [pol], 1000, nz, fin.make_traj(reward=rew[:1000], done=done[:1000]))
    del warm
    env = fin.fin_env_create(cfg, rows)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(calls):
        fin.fin_rollout(env, [pol], Tc, nz, tr)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b)
    return {"envs": N, "steps": T, "ms": ms, "env_steps_per_s": N * T / (ms / 1e3),
            "us_per_lockstep_step": 1e3 * ms / T, "episodes": int(done.sum().item()),
            "note": "one 480,000-step episode per env (reading R27), latency-bound: 32 tiles of 128 envs"}


def hbm_kernels(fin, torch):
    """The HBM-bound kernels at working sets far above the 126 MB L2, timed as 10
    back-to-back launches between CUDA events (no flush needed): K1 fin_env_step
    (N = 2^22), K4 fin_rollout_actions (N = 2^20, T = 32), K6 fin_episode_metrics
    (T = 2048, N = 2^18).  achieved = algorithmic bytes / launch time."""
    import statistics as st
    pk = peaks()
    res = {}

    def b2b(fn, reps=10):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            fn()
        b.record()
        torch.cuda.synchronize()
        return a.elapsed_time(b) / reps

    def entry(name, kernel, units, bytes_, ms, note):
        gbs = bytes_ / (ms / 1e3) / 1e9
        res[name] = {"kernel": kernel, "env_steps": units, "ms": ms, "env_steps_per_s": units / (ms / 1e3),
                     "bytes_per_launch": bytes_, "achieved_gbs": gbs, "peak_gbs": pk["hbm_gbs"],
                     "frac": gbs / pk["hbm_gbs"], "frac_of_8tbs": gbs / 8000.0, "note": note}

    g = torch.Generator(device="cuda").manual_seed(5)
    z = lambda s, d: torch.zeros(s, dtype=d, device="cuda")  # noqa: E731
    N = 1 << 22
    env = make_env(fin, N, 0)
    acts = torch.randint(-100, 101, (N, K_ASSETS), device="cuda", generator=g, dtype=torch.int16)
    tr = fin.make_traj(reward=z(N, torch.float32), done=z(N, torch.uint8))
    ms = b2b(lambda: fin.fin_env_step(env, acts, tr))
    entry("step_kernel_hbm", "k_stock_step2 (K1, packed per-warp form)", N, STEP_BYTES_ALGO * N, ms,
          "SURVEY d.3's 209 B/env-step (the kernel moves 237 B: cached asset, window, holdings octet padding); "
          "steady state: "
          "the same seeded U{-100..100} actions every step, so the cash binds in most steps")
    res["step_kernel_hbm"]["moved_gbs"] = STEP_BYTES_MOVED * N / (ms / 1e3) / 1e9
    del env, acts, tr
    N, T = 1 << 20, 32
    env = make_env(fin, N, 0)
    acts = torch.randint(-100, 101, (T, N, K_ASSETS), device="cuda", generator=g, dtype=torch.int16)
    tr = fin.make_traj(reward=z((T, N), torch.float32), done=z((T, N), torch.uint8))
    ms = b2b(lambda: fin.fin_rollout_actions(env, acts, T, tr))
    state = 2 * (8 + 8 + 60 + 4 + 4 + 52)   # per env per call: cash, asset, holdings, clock, window, metrics
    entry("replay_kernel_hbm", "k_stock_replay2 (K4, packed per-warp form)", N * T, N * T * 65 + N * state, ms,
          "actions 60 + reward 4 + done 1 per env-step, state in/out once per call")
    del env, acts, tr
    T, N = 2048, 1 << 18
    # lockstep episodes of 30 steps, as the rollouts produce them (dones of a tile coincide)
    done = torch.zeros((T, N), dtype=torch.uint8, device="cuda")
    done[29::30] = 1
    eq = 1e6 * torch.exp(torch.cumsum(0.01 * torch.randn((T + 1, N), device="cuda", generator=g,
                                                         dtype=torch.float64), 0))
    epm, cnt = z((160, N, 3), torch.float64), z(N, torch.int32)
    ms = b2b(lambda: fin.fin_episode_metrics(eq, done, 1e6, ep_metrics=epm, ep_count=cnt))
    entry("metrics_kernel_hbm", "k_pass_a/b/c (K6)", N * T,
          T * N * 9 + N * 8 + int(cnt.sum().item()) * 24 + N * 4, ms,
          "equity f64 + done u8 per env-step read, episode rows written; lockstep 30-step episodes")
    return res


def run_reference(args):
    """The reference arm: the float64 oracle as it stands, on the host cores, each step a
    bounded sample of the headline workload."""
    rank, world, _ = dist_info()
    if rank != 0:
        return
    import multiprocessing as mp
    for v in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
        os.environ[v] = "1"
    cores = len(os.sched_getaffinity(0))
    n_envs, T = 512, 4    # per core and step: 2,048 env-steps (the MLP batched over 512 envs), ~0.3 s
    rates = []
    t0 = time.perf_counter()
    with mp.get_context("spawn").Pool(cores) as pool:   # one pool: its start-up is not a step
        for i in range(args.warmup + args.steps):
            ts = time.perf_counter()
            pool.map(_oracle_shard, [(n_envs, T, 128 * c) for c in range(cores)])
            wall_i = time.perf_counter() - ts
            if i >= args.warmup:
                rates.append(n_envs * T * cores / wall_i)
    wall = time.perf_counter() - t0
    sample = (f"{cores} shards x {n_envs} envs x {T} steps of the headline workload per step (float64 oracle "
              f"incl. the 301-256-256-30 MLP), one process pool for all steps")
    value = statistics.mean(rates)
    out = {"impl": "reference", "metric": METRIC, "value": value, "unit": "env-steps/s", "n_gpus": world,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * wall / (args.warmup + args.steps),
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": {"workload": WORKLOAD, "envs_per_gpu": N_HEAD, "horizon": T_HEAD, "episode_len": L_EP,
                      "note": "each step is a bounded sample of this workload on the host cores"},
           "cpu_baseline": {"value": value, "unit": "env-steps/s", "cores": cores, "kind": "oracle", "sample": sample},
           "e2e": {"value": value, "unit": "env-steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
           "gpu_launches": 0}
    print(json.dumps(out), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-extras", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    if args.impl == "ours":
        rc = self_launch(args)
        if rc is not None:
            sys.exit(rc)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
