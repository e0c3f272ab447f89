"""Ensemble workflow of PAPER.md §5.2 on top of the C ABI.

Stock (§5.2.1): after training, each member is validated on the 5-day
window that follows its 30-day training window; members with a low Sharpe ratio are
discarded and the rest weighted by a softmax of their Sharpe ratios; the ensemble then
trades the next 5-day window with the weighted average of the members' actions.
``validate_and_weight`` runs one deterministic validation rollout per member
(FIN_NOISE_NONE) writing that member's aggregate row, all-reduces the rows over the
ranks (the ensemble's one real cross-GPU exchange: every rank validated its own env
shard), and turns them into weights with ``fin_member_weights`` on the device.

Crypto (§5.2.2): the vote over DQN / Double DQN / Dueling DQN members runs
inside ``fin_rollout`` (members of kind FIN_Q_ARGMAX / FIN_Q_DUELING, member_w NULL).

Everything here is argument marshalling and sequencing; the arithmetic is in the
library's kernels.
"""
from __future__ import annotations

from . import dist as fdist
from . import fin


def validate_and_weight(env_val, members, T_val: int, threshold: float = 0.0, temperature: float = 1.0,
                        group=None, stream=None):
    """Returns (w f32 [M] on the device, sharpe f64 [M] on the device, aggs f64 [M][8]).

    env_val: a stock handle whose windows are the validation windows (e.g. window_offset
    = 30 after 30-day training windows, episode_len = 5, advance_window_on_reset).  It is
    reset before each member, so every member sees the same validation episodes.

    Every step -- the zeroing of ``aggs``, the rollouts, the all-reduce and the weights --
    is enqueued on ``stream`` (default: the current stream), so the collective reads the
    aggregate rows only after the rollouts that write them."""
    import contextlib

    import torch
    ctx = torch.cuda.stream(stream) if stream is not None else contextlib.nullcontext()
    with ctx:
        M = len(members)
        aggs = torch.zeros((M, fin.FIN_AGG_LEN), dtype=torch.float64, device="cuda")
        for m, pol in enumerate(members):
            fin.fin_env_reset(env_val)
            fin.fin_rollout(env_val, [pol], T_val, fin.make_noise(fin.FIN_NOISE_NONE), fin.make_traj(agg=aggs[m]))
        fdist.allreduce_aggs(aggs, group)
        w = torch.empty(M, dtype=torch.float32, device="cuda")
        sharpe = torch.empty(M, dtype=torch.float64, device="cuda")
        fin.fin_member_weights(aggs, w, sharpe, threshold, temperature)
    return w, sharpe, aggs


def weighted_rollout(env, members, w, T: int, noise=None, traj=None, stream=None):
    """Trade T steps with the weighted ensemble (fin_rollout's member_w is a host array:
    the M weights are read back once, outside the rollout; the read-back is ordered after
    the work of ``stream`` that produced them)."""
    import contextlib

    import torch
    ctx = torch.cuda.stream(stream) if stream is not None else contextlib.nullcontext()
    with ctx:
        wh = w.float().cpu().numpy()          # synchronises with the current (= given) stream
        return fin.fin_rollout(env, members, T, noise, traj, member_w=wh)
