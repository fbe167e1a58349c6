"""Generate the golden fixtures under tests/golden/ from the reference simulator.

Runs ONLY in the build container (it imports ``tokensim`` from
/root/reference/pkg/src, which does not exist on the GPU box).  Everything it
writes is committed, so the GPU-side tests never need the reference.

What it records (all produced by the unmodified reference code):

* traces/*.csv            frozen request traces (``tokensim.workload.write_trace``)
* runs/<name>.json        per-run event hash, decision log, chunk-transfer rows
                          (or their hash for large runs), metrics
* ticks/<name>.json       (snapshot, policy state) -> decision pairs captured
                          around ``BufferAwarePolicy.on_tick`` /
                          ``opportunistic`` / ``iteration_batch`` calls
* select_batch.json       select_batch instances + reference answers

Usage:  PYTHONDONTWRITEBYTECODE=1 python tools/make_golden.py [--only NAME]
"""
from __future__ import annotations

import argparse
import dataclasses
import gzip
import hashlib
import json
import os
import random
import sys
from pathlib import Path

REF_SRC = "/root/reference/pkg/src"
sys.path.insert(0, REF_SRC)
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from tokensim import scheduler as ref_sched  # noqa: E402
from tokensim.cli import parse_config, preset_path  # noqa: E402
from tokensim.costs import CostModel  # noqa: E402
from tokensim.engine import SimConfig, run  # noqa: E402
from tokensim.metrics import (  # noqa: E402
    EffectiveThroughputConfig,
    QosConfig,
    effective_throughput,
    qos,
    raw_throughput,
    ttft_stats,
)
from tokensim.scheduler import SchedulerConfig, make_policy  # noqa: E402
from tokensim.workload import (  # noqa: E402
    RequestSpec,
    Trace,
    WorkloadConfig,
    generate_burst,
    generate_poisson,
    load_trace,
    write_trace,
)

from paper_2510_02758_b200 import configs  # noqa: E402

OUT = Path(__file__).resolve().parents[1] / "tests" / "golden"


def _dump(path: Path, obj) -> None:
    """Write gzipped compact JSON (mtime pinned so reruns are byte-identical)."""
    path = path.with_suffix(path.suffix + ".gz")
    path.parent.mkdir(parents=True, exist_ok=True)
    data = (json.dumps(obj, separators=(",", ":"), sort_keys=True) + "\n").encode()
    with open(path, "wb") as raw, gzip.GzipFile(fileobj=raw, mode="wb", mtime=0, filename="") as f:
        f.write(data)


def _sha(rows) -> str:
    h = hashlib.sha256()
    for r in rows:
        h.update(json.dumps(r, separators=(",", ":"), sort_keys=True).encode())
        h.update(b"\n")
    return h.hexdigest()


# --------------------------------------------------------------------------
# traces


def build_traces() -> dict[str, Trace]:
    traces = {}
    c1 = configs.C1
    traces["c1_burst32_s7"] = generate_burst(
        WorkloadConfig(
            kind="burst",
            burst_size=c1.n_requests,
            prompt_len_dist=c1.prompt_len_dist,
            output_len_dist=c1.output_len_dist,
            rate_profile=dict(c1.rate_profile),
        ),
        c1.seed,
    )
    c2 = configs.C2
    wl = WorkloadConfig(
        kind="poisson",
        poisson_rate=c2.poisson_rate,
        duration=c2.duration,
        prompt_len_dist=c2.prompt_len_dist,
        output_len_dist=c2.output_len_dist,
        rate_profile=dict(c2.rate_profile),
    )
    full = generate_poisson(wl, c2.seed)
    traces["c2_poisson256_s1"] = Trace(requests=full.requests[: c2.n_requests])
    traces["c2_burst256_s1"] = Trace(
        requests=tuple(
            RequestSpec(r.id, 0.0, r.prompt_len, r.output_len, r.consume_rate)
            for r in full.requests[: c2.n_requests]
        )
    )
    traces["figure7"] = load_trace(str(Path(REF_SRC) / "tokensim/presets/figure7_trace.csv"))
    # table2 seeds and the two desk-scale presets
    cfg, _ = parse_config(preset_path("table2"))
    for s in cfg.seeds:
        traces[f"table2_s{s}"] = generate_burst(cfg.workload, s)
    cfg, _ = parse_config(preset_path("burst-4090b"))
    traces["burst4090b_s1"] = generate_burst(cfg.workload, 1)
    cfg, _ = parse_config(preset_path("poisson-h200c"))
    traces["poissonh200c_s1"] = generate_poisson(cfg.workload, 1)
    for name, tr in traces.items():
        write_trace(tr, str(OUT / "traces" / f"{name}.csv"))
    return traces


# --------------------------------------------------------------------------
# recording policy wrapper


def _member_dict(m) -> dict:
    return dataclasses.asdict(m)


def snapshot_dict(view) -> dict:
    d = dataclasses.asdict(view)
    return d


def _decision_dict(dec) -> dict:
    return {
        "mode": dec.mode,
        "preempt": list(dec.preempt),
        "resume": [[rid, how] for rid, how in dec.resume],
        "prefill_batches": [list(b) for b in dec.prefill_batches],
        "log": dec.log,
    }


class Recorder:
    """Wraps a reference policy instance and records its calls."""

    def __init__(self, policy, keep_every: int = 1, cap: int = 400, iter_cap: int = 2000):
        self.p = policy
        self.ticks: list[dict] = []
        self.opps: list[dict] = []
        self.iters: list[dict] = []
        self._n_tick = 0
        self._n_opp = 0
        self._n_iter = 0
        self.keep_every = keep_every
        self.cap = cap
        self.iter_cap = iter_cap
        orig_tick = policy.on_tick
        orig_opp = policy.opportunistic
        orig_iter = policy.iteration_batch

        def on_tick(view):
            tprime = dict(getattr(policy, "_t_prime", {}))
            mode_before = policy.mode
            dec = orig_tick(view)
            self._n_tick += 1
            if len(self.ticks) < cap and (self._n_tick - 1) % keep_every == 0:
                self.ticks.append(
                    {
                        "view": snapshot_dict(view),
                        "t_prime": [[k, v] for k, v in sorted(tprime.items())],
                        "mode_before": mode_before,
                        "decision": _decision_dict(dec),
                        "t_prime_after": [
                            [k, v] for k, v in sorted(getattr(policy, "_t_prime", {}).items())
                        ],
                    }
                )
            return dec

        def opportunistic(view):
            mode_before = policy.mode
            dec = orig_opp(view)
            self._n_opp += 1
            if len(self.opps) < cap and (self._n_opp - 1) % keep_every == 0:
                self.opps.append(
                    {
                        "view": snapshot_dict(view),
                        "mode_before": mode_before,
                        "decision": {
                            "resume": [[r, h] for r, h in dec.resume],
                            "prefill_batches": [list(b) for b in dec.prefill_batches],
                        },
                    }
                )
            return dec

        def iteration_batch(running, contention):
            out = orig_iter(running, contention)
            self._n_iter += 1
            if len(self.iters) < iter_cap and (self._n_iter - 1) % max(1, keep_every) == 0:
                self.iters.append(
                    {
                        "running": [list(t) for t in running],
                        "contention": contention,
                        "mode": policy.mode,
                        "out": list(out),
                    }
                )
            return out

        policy.on_tick = on_tick
        policy.opportunistic = opportunistic
        policy.iteration_batch = iteration_batch


# --------------------------------------------------------------------------
# runs


def _chunk_rows(res) -> list[list]:
    rows = []
    for ev in res.event_log:
        if ev.kind == "chunk_transfer_done":
            i = ev.info
            rows.append(
                [i["direction"], i["owner"], i["tokens"], i["kind"], i["queued_at"], i["started_at"], i["done_at"]]
            )
    return rows


def _record_rows(res) -> list[list]:
    return [
        [
            r.request_id,
            r.ttft,
            r.gen_times,
            r.buffer_at_gen,
            r.consume_times,
            r.rebuffer_s,
            r.gen_done_time,
            r.done_time,
            r.preemptions,
            r.resumes,
            r.recomputes,
        ]
        for r in res.records
    ]


def run_and_record(name, trace_name, trace, policy_name, sched_cfg, cm, sim, full_rows: bool, rec_kw=None):
    policy = make_policy(policy_name, sched_cfg)
    rec = Recorder(policy, **(rec_kw or {}))
    res = run(trace, policy, cm, sim)
    stats = ttft_stats(res.records)
    lat = sorted(r.gen_times[0] - r.arrival for r in res.records)
    chunks = _chunk_rows(res)
    records = _record_rows(res)
    out = {
        "name": name,
        "trace": trace_name,
        "policy": policy_name,
        "sched": dataclasses.asdict(sched_cfg),
        "cm": dataclasses.asdict(cm),
        "sim": dataclasses.asdict(sim),
        "event_hash": res.event_hash(),
        "n_events": len(res.event_log),
        "total_time": res.total_time,
        "total_preemptions": res.total_preemptions,
        "total_recomputes": res.total_recomputes,
        "mode_changes": [[t, m] for t, m in res.mode_changes],
        "decision_log": res.decision_log,
        "chunk_hash": _sha(chunks),
        "n_chunks": len(chunks),
        "record_hash": _sha(records),
        "metrics": {
            "effective_tps": effective_throughput(res.records, res.total_time, EffectiveThroughputConfig()),
            "raw_tps": raw_throughput(res.records, res.total_time),
            "qos": qos(res.records, res.total_time, QosConfig()),
            "ttft_mean": stats["mean"],
            "ttft_p50": stats["p50"],
            "ttft_p99": stats["p99"],
            "ttft_latency_p99": lat[min(len(lat), int(99 * len(lat) / 100.0) + 1) - 1],
            "total_rebuffer_s": sum(r.rebuffer_s for r in res.records),
        },
    }
    if full_rows:
        out["chunks"] = chunks
        if name.startswith(("figure7", "c1_")):
            out["events"] = [[ev.time, ev.kind, ev.subject] for ev in res.event_log]
            out["records"] = records
    _dump(OUT / "runs" / f"{name}.json", out)
    if rec.ticks or rec.opps or rec.iters:
        _dump(
            OUT / "ticks" / f"{name}.json",
            {
                "name": name,
                "sched": dataclasses.asdict(sched_cfg),
                "policy": policy_name,
                "ticks": rec.ticks,
                "opportunistic": rec.opps,
                "iteration_batch": rec.iters,
            },
        )
    print(f"{name}: hash {out['event_hash'][:12]} events {out['n_events']} chunks {len(chunks)} "
          f"ticks {len(rec.ticks)} pre {res.total_preemptions}")
    return out


def build_runs(traces, only=None):
    jobs = []
    # figure7 preset
    cfg, cm = parse_config(preset_path("figure7"))
    jobs.append(("figure7_tokenflow", "figure7", "tokenflow", cfg.scheduler, cm, cfg.sim, True, None))
    # C1 oracle config, all four policies
    c1 = configs.C1
    for pol in ("tokenflow", "fcfs", "chunked", "qoe"):
        jobs.append((f"c1_{pol}", "c1_burst32_s7", pol, c1.sched_cfg(SchedulerConfig), c1.cost_model(CostModel),
                     c1.sim_cfg(SimConfig), True, None))
    # C1 ablations
    for abl, kw in (("no_overlap", dict(overlap=False)), ("no_write_through", dict(write_through=False)),
                    ("no_offload", dict(write_through=False, overlap=False, offload=False))):
        sim = dataclasses.replace(c1.sim_cfg(SimConfig), **kw)
        jobs.append((f"c1_tokenflow_{abl}", "c1_burst32_s7", "tokenflow", c1.sched_cfg(SchedulerConfig),
                     c1.cost_model(CostModel), sim, True, None))
    # table2: 5 seeds x 4 ablations
    cfg, cm = parse_config(preset_path("table2"))
    for s in cfg.seeds:
        for ab in cfg.ablations:
            sim = dataclasses.replace(cfg.sim, write_through=ab.write_through, overlap=ab.overlap,
                                      offload=ab.offload, seed=s)
            jobs.append((f"table2_s{s}_{ab.name}", f"table2_s{s}", "tokenflow", cfg.scheduler, cm, sim, s == 3,
                         None if s == 3 else dict(cap=0, iter_cap=0)))
    # desk-scale presets (large: hashes only, sampled ticks)
    cfg, cm = parse_config(preset_path("burst-4090b"))
    for pol in ("tokenflow", "fcfs", "qoe"):
        jobs.append((f"burst4090b_{pol}", "burst4090b_s1", pol, cfg.scheduler, cm,
                     dataclasses.replace(cfg.sim, seed=1, debug_checks=False), False,
                     dict(keep_every=3, cap=60, iter_cap=300)))
    cfg, cm = parse_config(preset_path("poisson-h200c"))
    jobs.append(("poissonh200c_tokenflow", "poissonh200c_s1", "tokenflow", cfg.scheduler, cm,
                 dataclasses.replace(cfg.sim, seed=1, debug_checks=False), False,
                 dict(keep_every=2, cap=60, iter_cap=300)))
    # C2 token analog (Llama3-8B-shaped 256-request trace; virtual-time replay config)
    c2 = configs.C2
    for tn in ("c2_poisson256_s1", "c2_burst256_s1"):
        jobs.append((f"{tn}_tokenflow", tn, "tokenflow", c2.sched_cfg(SchedulerConfig), c2.cost_model(CostModel),
                     dataclasses.replace(c2.sim_cfg(SimConfig), debug_checks=False), False,
                     dict(keep_every=3, cap=40, iter_cap=300)))
    for job in jobs:
        if only and only not in job[0]:
            continue
        name, tn, pol, sc, cm, sim, full_rows, rk = job
        run_and_record(name, tn, traces[tn], pol, sc, cm, sim, full_rows, rk)


# --------------------------------------------------------------------------
# select_batch instances (test_acceptance.py:93-152 generator, plus n=256)


def build_select_batch():
    rng = random.Random(20240809)
    cfg = SchedulerConfig()
    cases = []

    def make(n, lo_len, hi_len):
        views = []
        lengths = {}
        for i in range(n):
            b_rem = rng.randint(0, 400)
            rate = rng.choice([15.0, 20.0, 25.0, 30.0])
            value = rng.random()
            t_prime = rng.random() * 1.5
            t_overhead = rng.random() * 0.4
            phi = ref_sched.buffer_penalty(b_rem, rate, cfg.schedule_interval)
            utility = value * max(t_prime - t_overhead, 0.0) - cfg.penalty_weight * phi
            views.append(ref_sched.RequestPriorityView(i, b_rem, 0.0, rate, value, t_prime, t_overhead, phi, utility))
            lengths[i] = rng.randint(lo_len, hi_len)
        return views, lengths

    for _ in range(1000):
        n = rng.randint(2, 8)
        views, lengths = make(n, 100, 800)
        mem = int(sum(lengths.values()) * rng.uniform(0.25, 0.65))
        batch = rng.randint(1, max(1, n - 1))
        cases.append((views, lengths, mem, batch))
    for n in (16, 32, 64, 128, 256, 256, 256, 512):
        views, lengths = make(n, 100, 3000)
        mem = int(sum(lengths.values()) * rng.uniform(0.2, 0.5))
        batch = rng.randint(max(1, n // 4), max(1, n // 2))
        cases.append((views, lengths, mem, batch))
    out = []
    for views, lengths, mem, batch in cases:
        chosen = ref_sched.select_batch(views, mem, batch, lengths)
        greedy = ref_sched.greedy_batch_utility(views, mem, batch, lengths)
        out.append(
            {
                "views": [dataclasses.asdict(v) for v in views],
                "lengths": [[k, v] for k, v in lengths.items()],
                "mem": mem,
                "batch": batch,
                "chosen": sorted(chosen),
                "greedy_utility": greedy,
            }
        )
    _dump(OUT / "select_batch.json", {"cases": out})
    print(f"select_batch: {len(out)} cases")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default=None)
    args = ap.parse_args()
    traces = build_traces()
    if not args.only or args.only == "select":
        build_select_batch()
    if args.only != "select":
        build_runs(traces, args.only)


if __name__ == "__main__":
    main()
