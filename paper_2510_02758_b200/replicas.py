"""Request-sharded replicas (C3): one process per GPU, no data-path collective.

Requests are independent and every scheduling decision is per replica
(SURVEY.md 8e), so request i of the job goes to replica i mod N in arrival
order; each replica runs its own engine, policy, KV pool and host link.
Results are aggregated by concatenating records; the job's wall time is the
slowest replica's (max over ranks).  torch.distributed is used only for the
final gather of per-replica summaries (and the bench's max-over-ranks).
"""
from __future__ import annotations

from .workload import RequestSpec, Trace


def partition(trace: Trace, rank: int, world: int):
    """Replica ``rank``'s share: (local trace with dense ids, local->global id map)."""
    if not 0 <= rank < world:
        raise ValueError("rank out of range")
    mine = [r for i, r in enumerate(trace.requests) if i % world == rank]
    local = Trace(tuple(RequestSpec(k, r.arrival_time, r.prompt_len, r.output_len, r.consume_rate)
                        for k, r in enumerate(mine)), trace.seed)
    return local, [r.id for r in mine]


def scale_trace(trace: Trace, world: int) -> Trace:
    """C3 weak scaling: the burst scaled per GPU (world copies, interleaved in arrival order)."""
    reqs = []
    for r in trace.requests:
        for g in range(world):
            reqs.append((r.arrival_time, r, g))
    return Trace(tuple(RequestSpec(i, a, r.prompt_len, r.output_len, r.consume_rate)
                       for i, (a, r, _) in enumerate(reqs)), trace.seed)


def merge(summaries: list) -> dict:
    """Combine per-replica (records, total_time) into job-level metric inputs."""
    records = [rec for s in summaries for rec in s["records"]]
    return {"records": records, "total_time": max(s["total_time"] for s in summaries)}
