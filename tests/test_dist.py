"""CPU tests of the N>1 path with the gloo backend (world_size 2): env sharding, the
per-rollout aggregate all-reduce and max-over-ranks timing.  Each rank runs the
float64 oracle on its shard (the GPU kernels are covered by the -m gpu suite), so
this checks that the sharded job reproduces the single-process result exactly."""
import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2501_10709_b200 import dist as fdist


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _agg_of(cfg, mk, acts):
    """FIN_AGG_* partials of an oracle replay (same definition as the kernels)."""
    from oracle import metrics as omet
    from oracle import stock as ostock
    out, _ = ostock.run_actions(cfg, mk, acts)
    a = np.zeros(8)
    a[6] = a[7] = math.inf
    for i in range(cfg.num_envs):
        curves, _ = omet.split_episodes(cfg.initial_cash, out["asset"][:, i], out["done"][:, i])
        for cv in curves:
            cum, sh, mdd = omet.episode_metrics(cv)
            a[0] += 1
            a[1] += cum
            if math.isfinite(sh):
                a[2] += sh
                a[3] += 1
            a[4] += mdd
            a[6] = min(a[6], mdd)
            a[7] = min(a[7], cum)
    a[5] = float(np.sum(out["reward"]))
    return a


def _worker(rank, world, port, n_global, result_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import stock as ostock
    from synth import inputs, market
    m = market.stock_c1(rows=90)
    acts = inputs.stock_actions(14, n_global, 30, seed=3)
    off, n = fdist.shard(n_global, rank, world)
    cfg = ostock.StockEnvConfig(num_envs=n, num_assets=30, num_indicators=8, num_rows=90, episode_len=6,
                                num_windows=16, window_block=4, env_offset=off)
    agg = torch.tensor(_agg_of(cfg, m.market, acts[:, off:off + n]), dtype=torch.float64)
    fdist.allreduce_agg(agg)
    t = fdist.max_over_ranks(float(rank + 1))
    if rank == 0:
        result_q.put((agg.numpy().tolist(), t))
    dist.destroy_process_group()


def test_shard_covers_every_env_once():
    for n in (1, 7, 64, 65536, 100003):
        for w in (1, 2, 3, 8):
            spans = [fdist.shard(n, r, w) for r in range(w)]
            assert spans[0][0] == 0 and sum(s[1] for s in spans) == n
            for (o0, n0), (o1, _) in zip(spans, spans[1:]):
                assert o0 + n0 == o1


@pytest.mark.timeout(300)
def test_gloo_world2_matches_single_process():
    from oracle import stock as ostock
    from synth import inputs, market
    n_global = 10
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n_global, q)) for r in range(2)]
    for p in procs:
        p.start()
    agg, tmax = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    m = market.stock_c1(rows=90)
    acts = inputs.stock_actions(14, n_global, 30, seed=3)
    cfg = ostock.StockEnvConfig(num_envs=n_global, num_assets=30, num_indicators=8, num_rows=90, episode_len=6,
                                num_windows=16, window_block=4)
    ref = _agg_of(cfg, m.market, acts)
    np.testing.assert_allclose(agg, ref, rtol=1e-12)
    assert tmax == 2.0
    s = fdist.summarize_agg(agg)
    assert s["episodes"] == ref[0]


def _ens_worker(rank, world, port, n_global, M, result_q):
    """Ensemble validation exchange: each rank validates every
    member on its env shard (here: member m = its own seeded action stream replayed by the
    oracle), all-reduces the [M][8] aggregate rows, and derives the softmax weights."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import policy as opol
    from oracle import stock as ostock
    from synth import inputs, market
    m = market.stock_c1(rows=90)
    off, n = fdist.shard(n_global, rank, world)
    cfg = ostock.StockEnvConfig(num_envs=n, num_assets=30, num_indicators=8, num_rows=90, episode_len=5,
                                num_windows=16, window_block=4, env_offset=off)
    aggs = torch.zeros((M, 8), dtype=torch.float64)
    for j in range(M):
        acts = inputs.stock_actions(10, n_global, 30, seed=20 + j)
        aggs[j] = torch.tensor(_agg_of(cfg, m.market, acts[:, off:off + n]), dtype=torch.float64)
    fdist.allreduce_aggs(aggs)
    sharpes = [float(a[2] / a[3]) if a[3] > 0 else math.nan for a in aggs]
    w = opol.softmax_weights(sharpes, -10.0, 0.5)
    if rank == 0:
        result_q.put((aggs.numpy().tolist(), w))
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_gloo_world2_ensemble_weights_match_single_process():
    from oracle import policy as opol
    from oracle import stock as ostock
    from synth import inputs, market
    n_global, M = 9, 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ens_worker, args=(r, 2, port, n_global, M, q)) for r in range(2)]
    for p in procs:
        p.start()
    aggs, w = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    m = market.stock_c1(rows=90)
    cfg = ostock.StockEnvConfig(num_envs=n_global, num_assets=30, num_indicators=8, num_rows=90, episode_len=5,
                                num_windows=16, window_block=4)
    ref = [_agg_of(cfg, m.market, inputs.stock_actions(10, n_global, 30, seed=20 + j)) for j in range(M)]
    np.testing.assert_allclose(aggs, ref, rtol=1e-12)
    sharpes = [a[2] / a[3] for a in ref]
    np.testing.assert_allclose(w, opol.softmax_weights(sharpes, -10.0, 0.5), rtol=1e-12)
    assert abs(sum(w) - 1.0) < 1e-12
