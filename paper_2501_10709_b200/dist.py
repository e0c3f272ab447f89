"""Multi-GPU plumbing for the env-sharded rollout.

Envs are independent, so rank r of a world of size
W owns a contiguous block of global env ids and creates its handle with
``env_offset`` = the global id of its first env; window assignment and Philox
streams are keyed by the global id, so every rank computes exactly what a single
GPU would for those envs.  The only collective is one all-reduce per rollout of the
per-rank FIN_AGG_* partials (entries [0, FIN_AGG_NSUM) summed, the rest min-reduced),
carried by torch.distributed (NCCL over NVLink on the GPU box, gloo in the CPU tests).
"""
from __future__ import annotations

FIN_AGG_NSUM = 6
FIN_AGG_LEN = 8


def shard(n_global: int, rank: int, world: int):
    """(env_offset, n_local) of ``rank``: contiguous blocks, the first n % W ranks one larger."""
    base, extra = divmod(n_global, world)
    n_local = base + (1 if rank < extra else 0)
    offset = rank * base + min(rank, extra)
    return offset, n_local


def allreduce_agg(agg, group=None):
    """In-place all-reduce of a FIN_AGG_LEN float64 tensor: SUM over [0, NSUM), MIN after."""
    import torch.distributed as dist
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size(group) == 1:
        return agg
    dist.all_reduce(agg[:FIN_AGG_NSUM], op=dist.ReduceOp.SUM, group=group)
    dist.all_reduce(agg[FIN_AGG_NSUM:], op=dist.ReduceOp.MIN, group=group)
    return agg


def allreduce_aggs(aggs, group=None):
    """In-place all-reduce of an [M][FIN_AGG_LEN] float64 tensor (one aggregate row per
    ensemble member, e.g. the validation statistics of fin_member_weights)."""
    import torch.distributed as dist
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size(group) == 1:
        return aggs
    sums = aggs[:, :FIN_AGG_NSUM].contiguous()
    mins = aggs[:, FIN_AGG_NSUM:].contiguous()
    dist.all_reduce(sums, op=dist.ReduceOp.SUM, group=group)
    dist.all_reduce(mins, op=dist.ReduceOp.MIN, group=group)
    aggs[:, :FIN_AGG_NSUM] = sums
    aggs[:, FIN_AGG_NSUM:] = mins
    return aggs


def max_over_ranks(value: float, device=None, group=None) -> float:
    """Max of a host float over all ranks (the timing rule: slowest rank)."""
    import torch
    import torch.distributed as dist
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size(group) == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


def summarize_agg(agg) -> dict:
    """Human-readable ensemble / metric summary of a reduced FIN_AGG_* vector."""
    a = [float(x) for x in agg]
    n = a[0]
    return {"episodes": n,
            "mean_cum_return": a[1] / n if n else float("nan"),
            "mean_sharpe": a[2] / a[3] if a[3] else float("nan"),
            "mean_mdd": a[4] / n if n else float("nan"),
            "sum_reward": a[5], "worst_mdd": a[6], "worst_cum_return": a[7]}
