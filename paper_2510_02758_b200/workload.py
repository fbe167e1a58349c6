"""Request traces - the reference's ``tokensim.workload`` API (workload.py:52-290).

Synthetic traces use numpy's PCG64 streams seeded ``[stream, seed]`` exactly
as the reference does, so the same (config, seed) gives the same requests;
the frozen CSVs under tests/golden/traces/ pin that across numpy versions.
"""
from __future__ import annotations

import csv
from dataclasses import dataclass, field

import numpy as np

TRACE_HEADER = ["id", "arrival_s", "prompt_tokens", "output_tokens", "rate_tps"]
_ARRIVALS, _LENGTHS, _RATES = 0, 1, 2


class WorkloadError(ValueError):
    pass


class TraceParseError(ValueError):
    def __init__(self, message: str, line: int):
        super().__init__(f"line {line}: {message}")
        self.line = line


class TraceInvariantError(ValueError):
    def __init__(self, message: str, fieldname: str):
        super().__init__(message)
        self.field = fieldname


@dataclass(frozen=True)
class RequestSpec:
    id: int
    arrival_time: float
    prompt_len: int
    output_len: int
    consume_rate: float

    def validate(self) -> None:
        for ok, name, msg in ((self.arrival_time >= 0, "arrival_time", "< 0"), (self.prompt_len >= 1, "prompt_len", "< 1"),
                              (self.output_len >= 1, "output_len", "< 1"), (self.consume_rate > 0, "consume_rate", "<= 0")):
            if not ok:
                raise TraceInvariantError(f"request {self.id}: {name} {getattr(self, name)} {msg}", name)


@dataclass(frozen=True)
class Trace:
    requests: tuple
    seed: int | None = None

    def __post_init__(self):
        if sorted(r.id for r in self.requests) != list(range(len(self.requests))):
            raise TraceInvariantError("request ids must be unique and dense (0..n-1)", "id")
        prev = None
        for r in self.requests:
            r.validate()
            if prev is not None and r.arrival_time < prev:
                raise TraceInvariantError(f"arrival_time not sorted at request {r.id}", "arrival_time")
            prev = r.arrival_time

    def __len__(self):
        return len(self.requests)


@dataclass(frozen=True)
class WorkloadConfig:
    kind: str
    burst_size: int | None = None
    poisson_rate: float | None = None
    duration: float | None = None
    prompt_len_dist: tuple = (512.0, 128.0)
    output_len_dist: tuple = (1024.0, 256.0)
    rate_profile: dict = field(default_factory=lambda: {20.0: 1.0})
    path: str | None = None


def _lengths(rng, mean, std) -> int:
    if std == 0:
        return max(1, int(round(mean)))
    while True:
        v = int(round(rng.normal(mean, std)))
        if v >= 1:
            return v


def _bodies(cfg: WorkloadConfig, seed: int, n: int) -> list:
    lr = np.random.default_rng([_LENGTHS, seed])
    rr = np.random.default_rng([_RATES, seed])
    rates = sorted(cfg.rate_profile)
    w = np.asarray([cfg.rate_profile[r] for r in rates])
    out = []
    for _ in range(n):
        p = _lengths(lr, *cfg.prompt_len_dist)
        o = _lengths(lr, *cfg.output_len_dist)
        out.append((p, o, float(rr.choice(rates, p=w / w.sum()))))
    return out


def generate_burst(cfg: WorkloadConfig, seed: int) -> Trace:
    if cfg.kind != "burst" or not cfg.burst_size or cfg.burst_size < 1:
        raise WorkloadError("generate_burst needs kind='burst' and burst_size >= 1")
    return Trace(tuple(RequestSpec(i, 0.0, p, o, r) for i, (p, o, r) in enumerate(_bodies(cfg, seed, cfg.burst_size))),
                 seed)


def generate_poisson(cfg: WorkloadConfig, seed: int) -> Trace:
    if cfg.kind != "poisson" or not cfg.poisson_rate or not cfg.duration:
        raise WorkloadError("generate_poisson needs kind='poisson', poisson_rate and duration")
    ar = np.random.default_rng([_ARRIVALS, seed])
    t, times = 0.0, []
    while True:
        t += float(ar.exponential(1.0 / cfg.poisson_rate))
        if t > cfg.duration:
            break
        times.append(t)
    bodies = _bodies(cfg, seed, len(times))
    return Trace(tuple(RequestSpec(i, times[i], p, o, r) for i, (p, o, r) in enumerate(bodies)), seed)


def load_trace(path: str) -> Trace:
    rows = []
    with open(path, newline="", encoding="utf-8") as f:
        for lineno, row in enumerate(csv.reader(f), start=1):
            if not row or (len(row) == 1 and not row[0].strip()):
                continue
            if lineno == 1 and [c.strip() for c in row] == TRACE_HEADER:
                continue
            if len(row) != 5:
                raise TraceParseError(f"expected 5 fields, got {len(row)}", lineno)
            try:
                spec = RequestSpec(int(row[0]), float(row[1]), int(row[2]), int(row[3]), float(row[4]))
            except ValueError as exc:
                raise TraceParseError(str(exc), lineno) from exc
            spec.validate()
            rows.append(spec)
    rows.sort(key=lambda r: (r.arrival_time, r.id))
    return Trace(tuple(rows))


def write_trace(trace: Trace, path: str) -> None:
    with open(path, "w", newline="", encoding="utf-8") as f:
        w = csv.writer(f, lineterminator="\n")
        w.writerow(TRACE_HEADER)
        for r in trace.requests:
            w.writerow([r.id, r.arrival_time, r.prompt_len, r.output_len, r.consume_rate])
