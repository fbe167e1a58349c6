"""Restatement of tokensim.kvstore and tokensim.costs (TEST ORACLE)."""
from __future__ import annotations

from dataclasses import dataclass, field


class ResidencyError(RuntimeError):
    """kvstore.py:31-32."""


@dataclass(frozen=True)
class Costs:
    """costs.py:14-42 CostModel."""

    prefill_per_token: float = 5e-4
    decode_base: float = 0.0225
    decode_per_request: float = 0.0025
    decode_per_ctx_token: float = 0.0
    h2d_bandwidth: float = 20000.0
    d2h_bandwidth: float = 20000.0
    schedule_tick_cost: float = 4e-4

    def bw(self, direction: str) -> float:
        if direction == "h2d":
            return self.h2d_bandwidth
        if direction == "d2h":
            return self.d2h_bandwidth
        raise ValueError(direction)


def iter_seconds(n: int, ctx: int, c: Costs) -> float:
    """costs.py:45-59 decode_iteration_time."""
    if n < 1 or ctx < 0:
        raise ValueError("bad decode shape")
    return c.decode_base + c.decode_per_request * n + c.decode_per_ctx_token * ctx


def move_seconds(n: int, direction: str, c: Costs) -> float:
    """costs.py:69-75 transfer_time."""
    if n < 0:
        raise ValueError("n_tokens must be >= 0")
    return 0.0 if n == 0 else n / c.bw(direction)


@dataclass
class Placement:
    """kvstore.py:35-59 KvResidency."""

    request_id: int
    total_kv: int = 0
    gpu_resident: int = 0
    cpu_synced: int = 0
    inflight_d2h: int = 0
    inflight_h2d: int = 0

    @property
    def resumable(self) -> bool:
        return self.cpu_synced + self.gpu_resident >= self.total_kv

    @property
    def unsynced(self) -> int:
        return max(0, self.total_kv - self.cpu_synced - self.inflight_d2h)


@dataclass(frozen=True)
class Xfer:
    """kvstore.py:62-70 Chunk."""

    owner: int
    tokens: int
    direction: str
    kind: str
    queued_at: float = 0.0


@dataclass
class QueueView:
    """kvstore.py:87-98 TransferQueueState."""

    d2h_queue: list = field(default_factory=list)
    h2d_queue: list = field(default_factory=list)
    measured_d2h_rate: float = 0.0
    measured_h2d_rate: float = 0.0

    def backlog(self, direction: str) -> int:
        acc = 0
        for c in (self.d2h_queue if direction == "d2h" else self.h2d_queue):
            acc = acc + c.tokens
        return acc


def pieces(n: int, size: int) -> tuple:
    """kvstore.py:101-109 split_chunks."""
    if n <= 0:
        return ()
    q, r = divmod(n, size)
    return tuple([size] * q + ([r] if r else []))


def writeback_plan(pending: dict, interval: float, c: Costs, buffers: dict) -> list:
    """kvstore.py:112-141 plan_write_chunk."""
    if interval <= 0:
        raise ValueError("est_compute_interval must be > 0")
    room = int(interval * c.d2h_bandwidth)
    plan = []
    for rid in sorted((r for r, n in pending.items() if n > 0), key=lambda r: (-buffers.get(r, 0), r)):
        if room <= 0:
            break
        t = min(pending[rid], room)
        plan.append((rid, t))
        room -= t
    return plan


def eviction(p: Placement):
    """kvstore.py:144-154 preempt -> (instant_release, residual_d2h)."""
    if p.gpu_resident <= 0:
        raise ResidencyError(f"request {p.request_id} has no GPU-resident tokens")
    return min(p.gpu_resident, p.cpu_synced), p.total_kv - p.cpu_synced


def reload(p: Placement, size: int):
    """kvstore.py:157-170 resume -> (h2d_tokens, chunks)."""
    if not p.resumable:
        raise ResidencyError(f"request {p.request_id} is not resumable; recompute instead")
    miss = p.total_kv - p.gpu_resident
    return miss, pieces(miss, size)


def io_estimate(p: Placement, q: QueueView, c: Costs) -> float:
    """kvstore.py:173-193 io_overhead_estimate."""
    d2h = q.measured_d2h_rate or c.d2h_bandwidth
    h2d = q.measured_h2d_rate or c.h2d_bandwidth
    res = max(0, p.total_kv - p.cpu_synced)
    ld = max(0, p.total_kv - p.gpu_resident)
    if p.gpu_resident >= p.total_kv:
        res = ld = 0
    return q.backlog("d2h") / d2h + res / d2h + q.backlog("h2d") / h2d + ld / h2d


def ema(prev: float, sample: float, f: float = 0.3) -> float:
    """kvstore.py:255-259 update_rate_ema."""
    return sample if prev <= 0 else prev + f * (sample - prev)
