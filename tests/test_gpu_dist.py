"""The N > 1 path through libfinenv.so: two ranks (two processes, one process group)
each run their env shard of the fused rollout with env_offset = the global id of
their first env, and all-reduce the per-rank FIN_AGG_* partials with the product's
dist.allreduce_agg -- the job bench.py --gpus N runs, on one GPU with the gloo
backend (the kernels of the two ranks never wait on one another: each rank's rollout
is independent, only the host-side all-reduce joins them).

The sharded job must reproduce the single-process rollout of all envs: every per-env
output bitwise (window assignment and Philox streams are keyed by the global env id,
PAPER.md P:201), the aggregate's counts and minima bitwise, its float64
sums up to reassociation (the ranks' partial sums are added in a different order than
one process's tiles: rel 1e-12)."""
import os
import socket
import tempfile

import numpy as np
import pytest

from gpu_util import needs_gpu

pytestmark = [pytest.mark.gpu, needs_gpu]

N_GLOBAL, T, WORLD = 600, 40, 2    # 600 = 2 x 300: ragged tiles on both ranks, a reset at t = 30


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run(n, offset, allreduce):
    import torch

    from paper_2501_10709_b200 import dist as fdist
    from paper_2501_10709_b200 import fin
    from synth import market
    from synth import policy as spol
    m = market.stock_c1(rows=200)
    cfg = fin.env_config(num_envs=n, num_assets=30, num_indicators=8, num_rows=200, episode_len=30, window_stride=5,
                         num_windows=30, window_block=128, env_offset=offset, seed=23)
    env = fin.fin_env_create(cfg, m.market)
    pol = fin.fin_policy_create(fin.FIN_PPO_GAUSS, spol.kaiming_bf16(spol.STOCK_DIMS, 0))
    z = lambda s, d: torch.zeros(s, dtype=d, device="cuda")  # noqa: E731
    out = dict(reward=z((T, n), torch.float32), done=z((T, n), torch.uint8), actions=z((T, n, 30), torch.int16),
               cash=z((T, n), torch.float64), ep_metrics=z((2, n, 3), torch.float64), ep_count=z(n, torch.int32),
               agg=z(8, torch.float64))
    fin.fin_rollout(env, [pol], T, fin.make_noise(fin.FIN_NOISE_PHILOX, 1234), fin.make_traj(**out))
    if allreduce:
        torch.cuda.synchronize()
        fdist.allreduce_agg(out["agg"])
    torch.cuda.synchronize()
    assert fin.fin_env_check(env) == 0
    return {k: v.cpu().numpy() for k, v in out.items()}


def _worker(rank, world, port, path):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), GLOO_SOCKET_IFNAME="lo")
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2501_10709_b200 import dist as fdist
    off, n = fdist.shard(N_GLOBAL, rank, world)
    res = _run(n, off, allreduce=True)
    np.savez(os.path.join(path, f"rank{rank}.npz"), offset=off, **res)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(600)
def test_two_ranks_through_the_library_match_one_process():
    import torch.multiprocessing as mp
    with tempfile.TemporaryDirectory() as d:
        mp.start_processes(_worker, args=(WORLD, _free_port(), d), nprocs=WORLD, join=True, start_method="spawn")
        parts = [dict(np.load(os.path.join(d, f"rank{r}.npz"))) for r in range(WORLD)]
    one = _run(N_GLOBAL, 0, allreduce=False)
    assert [int(p["offset"]) for p in parts] == [0, N_GLOBAL // 2]
    for k in ("reward", "done", "actions", "cash", "ep_metrics"):
        both = np.concatenate([p[k] for p in parts], axis=1)
        assert np.array_equal(both.view(np.uint8), one[k].view(np.uint8)), k
    assert np.array_equal(np.concatenate([p["ep_count"] for p in parts]), one["ep_count"])
    assert int(one["done"].sum()) == N_GLOBAL          # one reset per env at t = 30
    for p in parts:                                     # the all-reduce gave every rank the same vector
        assert np.array_equal(p["agg"], parts[0]["agg"])
    agg = parts[0]["agg"]
    for j in (0, 3, 6, 7):                              # counts (exact integers) and minima: bitwise
        assert agg[j] == one["agg"][j], j
    np.testing.assert_allclose(agg[[1, 2, 4, 5]], one["agg"][[1, 2, 4, 5]], rtol=1e-12, atol=0)
