"""Scheduling policies - the reference's ``tokensim.scheduler`` plug-in API.

``BufferAwarePolicy`` (CLI name ``tokenflow``) keeps the reference's
``Policy`` interface (scheduler.py:409-446): ``on_tick``, ``opportunistic``,
``iteration_batch`` plus ``exhaustion_action`` / ``uses_kv_hierarchy`` /
``interleave_prefill_chunks``.  Its decisions are computed on the GPU by the
batch-priority selector kernel (csrc/tf_select.cu): one launch per tick
scores every request by buffer occupancy and consumption rate, orders
victims / criticals / incoming requests and runs select_batch's local
search, bit-exact with the reference's float64 Python.  The FCFS, chunked
and QoE baselines are comparison policies only (out of scope
for kernels) and run on the host unchanged.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

from .metrics import QosConfig, token_weight

BUFFER_AWARE = "buffer_aware"
FCFS_FALLBACK = "fcfs_fallback"
LATENCY_BYPASS_S = 1.3


@dataclass(frozen=True)
class SchedulerConfig:
    schedule_interval: float = 1.0
    per_request_mem_estimate: float = 1024.0
    workingset_adjust_rate: float = 0.5
    buffer_safety_factor: float = 2.0
    penalty_weight: float = 0.5
    tau_schedule: float = 1.0
    critical_buffer_seconds: float = 1.0
    max_batch: int | None = None
    value_threshold_frac: float = 0.10
    value_decay_alpha: float = 0.01
    pacing_buffer_seconds: float = 3.0
    chunk_prefill_tokens: int = 256
    ema_factor: float = 0.3

    def __post_init__(self):
        if self.schedule_interval <= 0:
            raise ValueError("schedule_interval must be > 0")
        if not 0.0 <= self.workingset_adjust_rate <= 1.0:
            raise ValueError("workingset_adjust_rate must be in [0, 1]")
        if self.buffer_safety_factor < 1.0:
            raise ValueError("buffer_safety_factor must be >= 1")
        if self.per_request_mem_estimate <= 0:
            raise ValueError("per_request_mem_estimate must be > 0")

    def value_config(self) -> QosConfig:
        return QosConfig(buffer_threshold_frac=self.value_threshold_frac, decay_alpha=self.value_decay_alpha)


@dataclass(frozen=True)
class RequestPriorityView:
    request_id: int
    b_rem: int
    b_pred: float
    rate: float
    value: float
    t_prime: float
    t_overhead: float
    phi: float
    utility: float


# ----------------------------------------------------------------- pure functions
def buffer_penalty(b_rem: float, rate: float, schedule_interval: float) -> float:
    return math.exp(-max(b_rem, 0.0) / max(rate * schedule_interval, 1e-9))


def build_priority_view(request_id, b_rem, rate, output_len, t_prime, t_overhead, expected_tokens,
                        cfg: SchedulerConfig) -> RequestPriorityView:
    value = token_weight(b_rem, output_len, cfg.value_config())
    phi = buffer_penalty(b_rem, rate, cfg.schedule_interval)
    utility = value * max(t_prime - t_overhead, 0.0) - cfg.penalty_weight * phi
    b_pred = max(b_rem + expected_tokens - rate * (cfg.schedule_interval + t_overhead), 0.0)
    return RequestPriorityView(request_id, b_rem, b_pred, rate, value, t_prime, t_overhead, phi, utility)


def working_set_size(total_mem, per_request_estimate, n_running, cfg: SchedulerConfig) -> int:
    if per_request_estimate <= 0:
        raise ValueError("per_request_estimate must be > 0")
    if total_mem < per_request_estimate:
        raise ValueError("total_mem must cover at least one request")
    cap = int(total_mem // per_request_estimate)
    if n_running >= cap:
        return max(1, cap)
    w = int(math.floor(cap - cfg.workingset_adjust_rate * (cap - n_running) + 0.5))
    return max(1, min(w, cap))


def should_tick(now, last_tick, waiting_count, drain_times, cfg: SchedulerConfig) -> bool:
    if now - last_tick < cfg.schedule_interval:
        return False
    return waiting_count > 0 or any(d < cfg.critical_buffer_seconds for d in drain_times)


def admit(view, tau_evict, tau_load, tau_schedule, cfg: SchedulerConfig) -> bool:
    if view is None or view.b_rem is None:
        return True
    return view.b_rem >= cfg.buffer_safety_factor * view.rate * (tau_evict + tau_load + tau_schedule)


def check_schedulability(rates, gamma) -> str:
    return BUFFER_AWARE if sum(rates) <= gamma else FCFS_FALLBACK


def recompute_or_load(t_io: float, t_recompute: float) -> str:
    return "recompute" if t_io > t_recompute else "load"


def _greedy_key(v):
    return (-v.phi, -(v.value * v.t_prime), -v.rate, v.request_id)


def _fit(order, gpu_mem, max_batch, lengths) -> list:
    chosen, used = [], 0.0
    for v in order:
        if len(chosen) >= max_batch:
            break
        if used + lengths[v.request_id] <= gpu_mem:
            chosen.append(v.request_id)
            used += lengths[v.request_id]
    return chosen


def select_batch(candidates, gpu_mem, max_batch, lengths, selector=None) -> set:
    """Greedy + adjacent-swap local search (scheduler.py:230-269), on the GPU."""
    if max_batch < 0 or gpu_mem < 0:
        raise ValueError("budgets must be non-negative")
    from .selector import default_selector

    return (selector or default_selector()).select_batch(list(candidates), gpu_mem, max_batch, lengths)


def greedy_batch_utility(candidates, gpu_mem, max_batch, lengths) -> float:
    util = {v.request_id: v.utility for v in candidates}
    return sum(util[i] for i in _fit(sorted(candidates, key=_greedy_key), gpu_mem, max_batch, lengths))


@dataclass(frozen=True)
class PrefillItem:
    request_id: int
    tokens: int
    waited_s: float = 0.0
    buffer_critical: bool = False


def partition_prefill(pending, remaining_mem) -> list:
    if remaining_mem < 0:
        raise ValueError("remaining_mem must be >= 0")
    urgent = [p for p in pending if p.buffer_critical or p.waited_s > LATENCY_BYPASS_S]
    batches = [[p.request_id] for p in urgent if p.tokens <= remaining_mem]
    cur, used = [], 0.0
    for p in pending:
        if p in urgent or p.tokens > remaining_mem:
            continue
        if cur and used + p.tokens > remaining_mem:
            batches.append(cur)
            cur, used = [], 0.0
        cur.append(p.request_id)
        used += p.tokens
    if cur:
        batches.append(cur)
    return batches


# ------------------------------------------------------------- snapshot records
@dataclass
class MemberView:
    request_id: int
    arrival_time: float
    rate: float
    prompt_len: int
    output_len: int
    generated: int
    consumed: int
    ctx_tokens: int
    gpu_resident: int
    releasable_now: int
    running: bool
    pinned: bool
    busy_since_tick: float
    tau_evict: float
    tau_load: float
    t_io: float
    t_recompute: float
    last_iter_time: float | None

    @property
    def b_rem(self) -> int:
        return self.generated - self.consumed

    @property
    def drain_s(self) -> float:
        return self.b_rem / self.rate


@dataclass
class WaitingView:
    request_id: int
    arrival_time: float
    prompt_len: int
    output_len: int
    rate: float
    waited_s: float


@dataclass
class SystemSnapshot:
    now: float
    members: list
    waiting: list
    free_slots: int
    gpu_mem_free: float
    gpu_mem_total: float
    cpu_mem_total: float
    max_batch: int
    gamma: float
    prefill_s_per_token: float
    offload_enabled: bool
    h2d_blocked_tokens: int = 0


@dataclass
class RowsSnapshot:
    """A SystemSnapshot whose member view is built ON THE DEVICE:
    the engine ships its raw per-request counters (``rows``: tf_req_row, every
    request in id order) and the queue / rate globals; tf_policy_tick_rows
    derives the MemberView fields, compacts the members and runs the tick
    with no host round trip.  ``materialize`` is the host equivalent (for
    host-side policies and tests)."""

    now: float
    rows: object
    n_rows: int
    globals: object
    waiting: list
    free_slots: int
    gpu_mem_free: float
    gpu_mem_total: float
    cpu_mem_total: float
    max_batch: int
    gamma: float
    prefill_s_per_token: float
    offload_enabled: bool
    h2d_blocked_tokens: int = 0
    materialize: object = None


@dataclass
class TickDecision:
    mode: str
    preempt: list = field(default_factory=list)
    resume: list = field(default_factory=list)
    prefill_batches: list = field(default_factory=list)
    log: dict = field(default_factory=dict)


@dataclass
class OpportunisticDecision:
    resume: list = field(default_factory=list)
    prefill_batches: list = field(default_factory=list)


# ------------------------------------------------------------------- policies
class Policy:
    name = "abstract"
    interleave_prefill_chunks = False
    uses_kv_hierarchy = False
    exhaustion_action = "evict"

    def __init__(self, cfg: SchedulerConfig | None = None):
        self.cfg = cfg or SchedulerConfig()
        self.mode = BUFFER_AWARE

    def prefill_chunk_tokens(self):
        return None

    def on_tick(self, view: SystemSnapshot) -> TickDecision:
        raise NotImplementedError

    def opportunistic(self, view: SystemSnapshot) -> OpportunisticDecision:
        raise NotImplementedError

    def iteration_batch(self, running, contention: bool) -> list:
        return [rid for rid, _, _ in running]


class BufferAwarePolicy(Policy):
    """Two-step buffer-aware preemptive scheduler; decisions on the GPU selector."""

    name = "tokenflow"
    uses_kv_hierarchy = True
    exhaustion_action = "pace"

    def __init__(self, cfg: SchedulerConfig | None = None, selector=None):
        super().__init__(cfg)
        self._t_prime: dict = {}
        self.preemption_count = 0
        self.mode_changes: list = []
        self._selector = selector

    @property
    def selector(self):
        if self._selector is None:
            from .selector import default_selector

            self._selector = default_selector()
        return self._selector

    def set_mode(self, now, mode):
        if mode != self.mode:
            self.mode_changes.append((now, mode))
        self.mode = mode

    device_snapshot = True  # the engine may hand on_tick a RowsSnapshot

    def on_tick(self, view) -> TickDecision:
        if isinstance(view, RowsSnapshot):
            mode, pre, resume, adm, rc, batches = self.selector.tick_rows(view, self.cfg, self._t_prime, self.mode)
        else:
            mode, pre, resume, adm, rc, batches = self.selector.tick(view, self.cfg, self._t_prime, self.mode)
        self.set_mode(view.now, mode)
        self.preemption_count += len(pre)
        return TickDecision(mode=mode, preempt=pre, resume=resume, prefill_batches=batches,
                            log={"mode": mode, "admitted": adm, "preempted": list(pre),
                                 "resumed": [r for r, _ in resume], "recomputed": rc})

    def opportunistic(self, view: SystemSnapshot) -> OpportunisticDecision:
        if self.mode == FCFS_FALLBACK:
            return OpportunisticDecision()
        _, _, resume, _, _, batches = self.selector.fastpath(view, self.cfg, self.mode)
        return OpportunisticDecision(resume=resume, prefill_batches=batches)

    def iteration_batch(self, running, contention: bool) -> list:
        if not contention or self.mode == FCFS_FALLBACK:
            return [rid for rid, _, _ in running]
        return self.selector.iteration_batch(running, contention, self.mode, self.cfg.pacing_buffer_seconds)


class FcfsPolicy(Policy):
    """Comparison baseline: arrival order with worst-case reservation (scheduler.py:828-880)."""

    name = "fcfs"

    def opportunistic(self, view):
        out = OpportunisticDecision()
        slots = view.free_slots
        for m in sorted((m for m in view.members if not m.running and not m.pinned),
                        key=lambda m: (m.arrival_time, m.request_id)):
            if slots <= 0 or m.ctx_tokens > view.gpu_mem_free:
                break
            out.resume.append((m.request_id, "recompute"))
            slots -= 1
        held = sum(m.prompt_len + m.output_len for m in view.members)
        batch = []
        for w in view.waiting:
            need = w.prompt_len + w.output_len
            if slots <= 0 or held + need > view.gpu_mem_total:
                break
            batch.append(w.request_id)
            held += need
            slots -= 1
        if batch:
            out.prefill_batches = [batch]
        return out

    def on_tick(self, view):
        o = self.opportunistic(view)
        return TickDecision(mode=BUFFER_AWARE, resume=o.resume, prefill_batches=o.prefill_batches,
                            log={"mode": BUFFER_AWARE, "admitted": [r for b in o.prefill_batches for r in b],
                                 "preempted": [], "resumed": [r for r, _ in o.resume],
                                 "recomputed": [r for r, h in o.resume if h == "recompute"]})


class ChunkedFcfsPolicy(FcfsPolicy):
    name = "chunked"
    interleave_prefill_chunks = True

    def prefill_chunk_tokens(self):
        return self.cfg.chunk_prefill_tokens


class QoePolicy(Policy):
    """Comparison baseline: drain-time priority, recompute on resume (scheduler.py:893-993)."""

    name = "qoe"

    def __init__(self, cfg=None):
        super().__init__(cfg)
        self.preemption_count = 0

    def on_tick(self, view):
        dec = TickDecision(mode=BUFFER_AWARE)
        pool = [m for m in view.members if not m.pinned]
        ranked = sorted([(m.drain_s, m.request_id, 0, m) for m in pool] +
                        [(max(0.0, LATENCY_BYPASS_S - w.waited_s), w.request_id, 1, w) for w in view.waiting],
                        key=lambda t: (t[0], t[1]))
        pinned = [m for m in view.members if m.pinned]
        budget = view.max_batch - len(pinned)
        mem_cap = view.gpu_mem_total - sum(m.ctx_tokens for m in pinned)
        keep, adm, used_m, used = [], [], 0.0, 0.0
        for _, _, kind, obj in ranked:
            need = obj.ctx_tokens if kind == 0 else obj.prompt_len + 1
            if len(keep) + len(adm) >= budget:
                break
            if used + need > mem_cap:
                continue
            used += need
            if kind == 0:
                keep.append(obj)
                used_m += need
            else:
                adm.append(obj)
        ids = {m.request_id for m in keep}
        for m in pool:
            if m.running and m.request_id not in ids:
                dec.preempt.append(m.request_id)
                self.preemption_count += 1
        rc = [m.request_id for m in keep if not m.running]
        dec.resume = [(r, "recompute") for r in rc]
        if adm:
            dec.prefill_batches = partition_prefill(
                [PrefillItem(w.request_id, w.prompt_len + 1, w.waited_s) for w in adm], mem_cap - used_m)
        dec.log = {"mode": BUFFER_AWARE, "admitted": [w.request_id for w in adm], "preempted": dec.preempt,
                   "resumed": list(rc), "recomputed": list(rc)}
        return dec

    def opportunistic(self, view):
        out = OpportunisticDecision()
        slots, mem = view.free_slots, view.gpu_mem_free
        for m in sorted((m for m in view.members if not m.running and not m.pinned),
                        key=lambda m: (m.drain_s, m.request_id)):
            if slots <= 0 or m.ctx_tokens > mem:
                break
            out.resume.append((m.request_id, "recompute"))
            slots, mem = slots - 1, mem - m.ctx_tokens
        batch = []
        for w in view.waiting:
            need = w.prompt_len + 1
            if slots <= 0 or need > mem:
                break
            batch.append(w.request_id)
            slots, mem = slots - 1, mem - need
        if batch:
            out.prefill_batches = [batch]
        return out


POLICIES = {"tokenflow": BufferAwarePolicy, "fcfs": FcfsPolicy, "chunked": ChunkedFcfsPolicy, "qoe": QoePolicy}


def make_policy(name: str, cfg: SchedulerConfig | None = None) -> Policy:
    try:
        cls = POLICIES[name]
    except KeyError:
        raise ValueError(f"unknown policy {name!r}; expected one of {sorted(POLICIES)}") from None
    return cls(cfg)
