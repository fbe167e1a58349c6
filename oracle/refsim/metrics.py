"""Restatement of tokensim.metrics (TEST ORACLE)."""
from __future__ import annotations

import math

from .pysum import pysum


def timely_weight(b: int, out_len: int, tau1: float = 0.10, tau2: float = 0.20) -> float:
    """metrics.py:93-108 effective_token_weight."""
    lo, hi = tau1 * out_len, tau2 * out_len
    if b < lo:
        return 1.0
    if b >= hi:
        return 0.0
    return (hi - b) / (hi - lo)


def effective_tps(records, total_time: float) -> float:
    """metrics.py:111-125 effective_throughput."""
    acc = 0.0
    for r in records:
        acc += pysum(timely_weight(b, r.output_len) for b in r.buffer_at_gen)
    return acc / total_time


def raw_tps(records, total_time: float) -> float:
    """metrics.py:128-132."""
    return sum(len(r.gen_times) for r in records) / total_time


def rank_pct(values, pct: float) -> float:
    """metrics.py:135-141 nearest_rank."""
    n = len(values)
    return values[min(n, math.floor(pct * n / 100.0) + 1) - 1]


def ttft(records) -> dict:
    """metrics.py:144-155 ttft_stats (absolute time, reference quirk 0(a))."""
    v = sorted(r.ttft for r in records)
    return {"mean": pysum(v) / len(v), "p50": rank_pct(v, 50.0), "p99": rank_pct(v, 99.0)}


def ttft_latency_p99(records) -> float:
    """P99 of gen_times[0] - arrival (the latency form SURVEY 0(a) asks for)."""
    return rank_pct(sorted(r.gen_times[0] - r.arrival for r in records), 99.0)
