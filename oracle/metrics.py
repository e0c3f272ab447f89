"""Episode metrics oracle (test infrastructure only).

PAPER.md §6.1 and Eq. 6; SPEC S:582-590, S:612-620;
readings R21-R23 of DESIGN.md:
  equity     v_0 (at reset), v_1 .. v_L (v' of each step)
  cumulative cum = v_L / v_0 - 1
  returns    r_t = v_t / v_{t-1} - 1
  Sharpe     sqrt(252) * mean(r) / std(r, ddof=1), r_f = 0; NaN if L < 2 or std = 0
  MDD        min_t (v_t / max_{s<=t} v_s - 1)  (<= 0)
Textbook two-pass mean / variance and a serial running-peak scan.
"""
from __future__ import annotations

import math


def returns(equity) -> list:
    return [equity[t] / equity[t - 1] - 1.0 for t in range(1, len(equity))]


def cumulative_return(equity) -> float:
    return equity[-1] / equity[0] - 1.0


def sharpe(equity, periods_per_year: float = 252.0, rf: float = 0.0) -> float:
    r = returns(equity)
    n = len(r)
    if n < 2:
        return math.nan
    mean = 0.0
    for x in r:
        mean = mean + x
    mean = mean / n
    ss = 0.0
    for x in r:
        ss = ss + (x - mean) * (x - mean)
    std = math.sqrt(ss / (n - 1))
    if std == 0.0:
        return math.nan
    return math.sqrt(periods_per_year) * (mean - rf) / std


def drawdown_curve(equity) -> list:
    peak = equity[0]
    out = []
    for v in equity:
        if v > peak:
            peak = v
        out.append(v / peak - 1.0)
    return out


def max_drawdown(equity) -> float:
    return min(drawdown_curve(equity))


def episode_metrics(equity, periods_per_year: float = 252.0):
    """(cum, sharpe, mdd) of one episode's equity curve [v_0 .. v_L]."""
    return (cumulative_return(equity), sharpe(equity, periods_per_year), max_drawdown(equity))


def split_episodes(v0, assets, dones):
    """Per-env episode equity curves from a transition log.

    ``v0``      equity at the start of the log (float)
    ``assets``  v' of each transition (list, length T)
    ``dones``   done flag of each transition
    Returns (completed_curves, open_curve).  After a done the next episode
    starts at ``v0_next`` = the reset equity, passed as the same ``v0``
    (initial cash) -- autoreset restores b = initial cash, h = 0.
    """
    curves = []
    cur = [v0]
    for v, d in zip(assets, dones):
        cur.append(v)
        if d:
            curves.append(cur)
            cur = [v0]
    return curves, cur
