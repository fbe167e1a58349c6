"""Report / wire formats of a serving run, byte-compatible with the reference.

Restates what the reference experiment runner writes per cell
(tokensim/cli.py:218-288, :354-385) so that a B200 run diffs against the
reference's own outputs column for column:

* ``report_<cell>.json``   ``cell_report``            (cli.py:218-234, :373-374)
* ``requests_<cell>.csv``  ``write_request_csv``      (cli.py:276-288)
* ``events_<cell>.jsonl``  ``SimResult.events_jsonl`` (engine.py:179-187)
* ``summary.csv/.txt``     ``emit_summary``           (cli.py:291-351)

plus one B200-only file, ``transfers_<cell>.csv``: the chunk_transfer_done
audit rows of the event log (engine.py:582-595) joined with what the data
plane measured for the same chunk (bytes moved, CUDA-event milliseconds,
GB/s), so a real-time run's virtual-clock rows carry their wall-clock
evidence.
"""
from __future__ import annotations

import csv
import json
from dataclasses import dataclass, replace
from pathlib import Path

from .engine import CHUNK_TRANSFER_DONE, CapacityError, DeadlockError, SimResult, run
from .metrics import (
    EffectiveThroughputConfig,
    QosConfig,
    effective_throughput,
    effective_token_weight,
    qos,
    raw_throughput,
    ttft_stats,
)
from .scheduler import make_policy


@dataclass(frozen=True)
class AblationSpec:
    """Memory-management ablation cell (tokensim/cli.py:50-59)."""

    name: str = "full"
    write_through: bool = True
    overlap: bool = True
    offload: bool = True


@dataclass
class CellResult:
    policy: str
    ablation: str
    seed: int
    report: dict
    result: SimResult | None
    error: str | None = None

    @property
    def cell_id(self) -> str:
        tag = f"_{self.ablation}" if self.ablation != "full" else ""
        return f"{self.policy}{tag}_s{self.seed}"


def cell_report(result: SimResult, qos_cfg: QosConfig | None = None,
                eff_cfg: EffectiveThroughputConfig | None = None) -> dict:
    """Per-cell metrics dict (tokensim/cli.py:218-234); ``seed`` is filled by the caller."""
    qos_cfg = qos_cfg or QosConfig()
    eff_cfg = eff_cfg or EffectiveThroughputConfig()
    st = ttft_stats(result.records)
    return {
        "policy": result.policy,
        "seed": None,
        "qos": round(qos(result.records, result.total_time, qos_cfg), 9),
        "effective_tps": round(effective_throughput(result.records, result.total_time, eff_cfg), 9),
        "raw_tps": round(raw_throughput(result.records, result.total_time), 9),
        "ttft_mean": round(st["mean"], 9),
        "ttft_p50": round(st["p50"], 9),
        "ttft_p99": round(st["p99"], 9),
        "total_rebuffer_s": round(sum(r.rebuffer_s for r in result.records), 9),
        "completion_time_s": round(result.total_time, 9),
        "preemptions": result.total_preemptions,
        "recomputes": result.total_recomputes,
    }


def report_json(report: dict) -> str:
    """The exact text of ``report_<cell>.json`` (cli.py:373-374)."""
    return json.dumps(report, sort_keys=True, indent=2) + "\n"


def write_request_csv(path, result: SimResult, eff_cfg: EffectiveThroughputConfig | None = None) -> None:
    """One row per generated token (tokensim/cli.py:276-288)."""
    eff_cfg = eff_cfg or EffectiveThroughputConfig()
    with Path(path).open("w", newline="", encoding="utf-8") as f:
        w = csv.writer(f, lineterminator="\n")
        w.writerow(["request_id", "token_index", "gen_time_s", "consume_time_s", "weight"])
        for rec in result.records:
            for j, (g, c, b) in enumerate(zip(rec.gen_times, rec.consume_times, rec.buffer_at_gen)):
                w.writerow([rec.request_id, j, f"{g:.9f}", f"{c:.9f}",
                            f"{effective_token_weight(b, rec.output_len, eff_cfg):.6f}"])


def write_transfer_audit(path, result: SimResult, dataplane=None, bytes_per_token: int | None = None) -> int:
    """B200 audit rows: each chunk_transfer_done of the event log (engine.py:582-595)
    plus, when a real-time data plane ran the chunk, the bytes it moved and the
    CUDA-event time of the copy.  Returns the number of rows."""
    log = dataplane.transfer_log() if dataplane is not None else []
    bpt = bytes_per_token if bytes_per_token is not None else (
        dataplane.pool.block_bytes // dataplane.pool.B if dataplane is not None else 0)
    # each channel is FIFO with one chunk in service (engine.py:736-779), so
    # per direction the launch order of the copies is the landing order
    measured = {"d2h": [x for x in log if x[0] == "d2h"], "h2d": [x for x in log if x[0] == "h2d"]}
    seen = {"d2h": 0, "h2d": 0}
    rows = [e.info for e in result.event_log if e.kind == CHUNK_TRANSFER_DONE]
    with Path(path).open("w", newline="", encoding="utf-8") as f:
        w = csv.writer(f, lineterminator="\n")
        w.writerow(["direction", "owner", "tokens", "kind", "queued_at", "started_at", "done_at",
                    "bytes", "device_ms", "gbs"])
        for r in rows:
            d, ms, gbs = r["direction"], "", ""
            i = seen[d]
            seen[d] += 1
            if i < len(measured[d]) and measured[d][i][1] == r["tokens"]:
                ms = f"{measured[d][i][2]:.6f}"
                if measured[d][i][2] > 0:
                    gbs = f"{r['tokens'] * bpt / (measured[d][i][2] / 1e3) / 1e9:.3f}"
            w.writerow([d, r["owner"], r["tokens"], r["kind"], f"{r['queued_at']:.9f}",
                        f"{r['started_at']:.9f}", f"{r['done_at']:.9f}", r["tokens"] * bpt, ms, gbs])
    return len(rows)


def run_cell(trace, policy_name: str, ablation: AblationSpec, seed: int, sched_cfg, cm, sim,
             qos_cfg=None, eff_cfg=None, dataplane_factory=None, policy_factory=make_policy) -> CellResult:
    """One (policy, ablation, seed) cell (tokensim/cli.py:237-273)."""
    sim = replace(sim, write_through=ablation.write_through, overlap=ablation.overlap,
                  offload=ablation.offload, seed=seed)
    policy = policy_factory(policy_name, sched_cfg)
    dp = dataplane_factory(trace, sim) if dataplane_factory else None
    try:
        result = run(trace, policy, cm, sim, dataplane=dp)
    except (DeadlockError, CapacityError) as exc:
        return CellResult(policy_name, ablation.name, seed, {}, None, f"{type(exc).__name__}: {exc}")
    rep = cell_report(result, qos_cfg, eff_cfg)
    rep["seed"] = seed
    rep["ablation"] = ablation.name
    return CellResult(policy_name, ablation.name, seed, rep, result)


def emit_summary(cells, out_dir) -> list:
    """summary.csv + summary.txt with deltas against FCFS of the same seed (tokensim/cli.py:291-351)."""
    out_dir = Path(out_dir)
    fcfs = {c.seed: c.report for c in cells if c.policy == "fcfs" and not c.error}
    rows = []
    for c in cells:
        row = {"cell": c.cell_id, "policy": c.policy, "ablation": c.ablation, "seed": c.seed}
        if c.error:
            row["error"] = c.error
            rows.append(row)
            continue
        row.update({k: v for k, v in c.report.items() if k not in ("policy", "seed", "ablation")})
        base = fcfs.get(c.seed)
        if base and c.policy != "fcfs":
            if base["ttft_p99"] > 0:
                row["ttft_p99_reduction_pct"] = round(100.0 * (1.0 - c.report["ttft_p99"] / base["ttft_p99"]), 6)
            if base["effective_tps"] > 0:
                row["eff_tps_gain_pct"] = round(
                    100.0 * (c.report["effective_tps"] / base["effective_tps"] - 1.0), 6)
        rows.append(row)
    header: list = []
    for row in rows:
        header.extend(k for k in row if k not in header)
    with (out_dir / "summary.csv").open("w", newline="", encoding="utf-8") as f:
        w = csv.DictWriter(f, fieldnames=header, lineterminator="\n")
        w.writeheader()
        w.writerows(rows)
    lines = []
    for row in rows:
        if "error" in row:
            lines.append(f"{row['cell']}: FAILED {row['error']}")
            continue
        parts = [f"{row['cell']:<28}"]
        parts += [f"{k}={row[k]:.3f}" for k in ("qos", "effective_tps", "raw_tps", "ttft_p99", "total_rebuffer_s",
                                                  "completion_time_s") if k in row]
        parts += [f"{k}={row[k]:+.1f}" for k in ("ttft_p99_reduction_pct", "eff_tps_gain_pct") if k in row]
        lines.append("  ".join(parts))
    (out_dir / "summary.txt").write_text("\n".join(lines) + "\n")
    return rows


def run_experiment(trace, policies, seeds, sched_cfg, cm, sim, out_dir, ablations=(AblationSpec(),),
                   qos_cfg=None, eff_cfg=None, emit_events=False, dataplane_factory=None,
                   policy_factory=make_policy) -> int:
    """The policy x seed x ablation matrix with every file the reference writes
    (tokensim/cli.py:354-385); returns 0, or 2 when a cell failed (EXIT_SIM).
    ``trace`` is a Trace or a callable seed -> Trace."""
    out_dir = Path(out_dir)
    out_dir.mkdir(parents=True, exist_ok=True)
    cells, failed = [], False
    for seed in seeds:
        tr = trace(seed) if callable(trace) else trace
        for pol in policies:
            for ab in ablations:
                if ab.name != "full" and pol != "tokenflow":
                    continue
                cell = run_cell(tr, pol, ab, seed, sched_cfg, cm, sim, qos_cfg, eff_cfg, dataplane_factory,
                                policy_factory)
                cells.append(cell)
                if cell.error:
                    failed = True
                    continue
                (out_dir / f"report_{cell.cell_id}.json").write_text(report_json(cell.report))
                write_request_csv(out_dir / f"requests_{cell.cell_id}.csv", cell.result, eff_cfg)
                if emit_events:
                    (out_dir / f"events_{cell.cell_id}.jsonl").write_text(cell.result.events_jsonl())
    emit_summary(cells, out_dir)
    return 2 if failed else 0
