"""The CPU oracle is pinned to the reference's own outputs (golden fixtures
made by tools/make_golden.py from the unmodified tokensim) and to the
reference's known-answer tests (tests/test_kvstore.py, test_scheduler.py)."""
import math
import random

import pytest
from conftest import golden_names, load_golden, pool_blocks, trace_path

from oracle.dataplane import CpuDataPlane
from oracle.refsim import planner as P
from oracle.refsim.metrics import effective_tps, raw_tps, ttft, ttft_latency_p99
from oracle.refsim.policy import Knobs, Prio, build_policy, choose_batch, greedy_utility, starvation
from oracle.refsim.pysum import pysum
from oracle.refsim.sim import SimKnobs, simulate
from oracle.refsim.traces import read_trace

FAST = [n for n in golden_names("runs") if not n.startswith(("c2_", "burst4090b", "poissonh200c"))]
LARGE = [n for n in golden_names("runs") if n not in FAST]


def _run(name, dp=False):
    g = load_golden("runs", name)
    reqs = read_trace(trace_path(g["trace"]))
    sim = SimKnobs(**g["sim"])
    plane = None
    if dp:
        plane = CpuDataPlane(reqs, pool_blocks(g["sim"], len(reqs)), 16384, 2, 2, 64)
    out = simulate(reqs, build_policy(g["policy"], Knobs(**g["sched"])), P.Costs(**g["cm"]), sim, dp=plane)
    return g, out, plane


@pytest.mark.parametrize("name", FAST)
def test_oracle_reproduces_reference_run(name):
    g, out, _ = _run(name)
    assert out.event_hash() == g["event_hash"]
    assert out.decisions == g["decision_log"]
    assert out.total_preemptions == g["total_preemptions"]
    assert out.total_recomputes == g["total_recomputes"]
    if "chunks" in g:
        assert out.chunk_rows() == g["chunks"]
    m = g["metrics"]
    assert effective_tps(out.records, out.total_time) == m["effective_tps"]
    assert raw_tps(out.records, out.total_time) == m["raw_tps"]
    assert ttft(out.records)["p99"] == m["ttft_p99"]
    assert ttft(out.records)["mean"] == m["ttft_mean"]
    assert ttft_latency_p99(out.records) == m["ttft_latency_p99"]


@pytest.mark.slow
@pytest.mark.parametrize("name", LARGE)
def test_oracle_reproduces_large_reference_run(name):
    g, out, _ = _run(name)
    assert out.event_hash() == g["event_hash"]
    assert out.decisions == g["decision_log"]


@pytest.mark.parametrize("name", ["figure7_tokenflow", "c1_tokenflow", "c1_tokenflow_no_overlap", "c1_qoe",
                                  "table2_s3_full", "table2_s3_no_offload"])
def test_cpu_dataplane_follows_reference_counts(name):
    """The token-range restatement stays consistent with the reference's
    counters at every event (audit inside the data plane) and never reads a
    non-resident or never-written position."""
    g, out, plane = _run(name, dp=True)
    assert out.event_hash() == g["event_hash"]
    assert plane.peak_blocks <= pool_blocks(g["sim"], len(out.records))


def test_select_batch_golden_cases():
    import gzip
    import json

    from conftest import GOLDEN

    cases = json.load(gzip.open(GOLDEN / "select_batch.json.gz"))["cases"]
    for c in cases:
        views = [Prio(**v) for v in c["views"]]
        lengths = {k: v for k, v in c["lengths"]}
        assert sorted(choose_batch(views, c["mem"], c["batch"], lengths)) == c["chosen"]
        assert greedy_utility(views, c["mem"], c["batch"], lengths) == c["greedy_utility"]


def test_select_batch_feasible_and_not_worse_than_greedy():
    """tests/test_acceptance.py:93-152 generator (seed 20240809)."""
    rng = random.Random(20240809)
    k = Knobs()
    for _ in range(300):
        n = rng.randint(2, 8)
        views, lengths = [], {}
        for i in range(n):
            b, r = rng.randint(0, 400), rng.choice([15.0, 20.0, 25.0, 30.0])
            v, tp, to = rng.random(), rng.random() * 1.5, rng.random() * 0.4
            phi = starvation(b, r, k.schedule_interval)
            views.append(Prio(i, b, 0.0, r, v, tp, to, phi, v * max(tp - to, 0.0) - k.penalty_weight * phi))
            lengths[i] = rng.randint(100, 800)
        mem = int(sum(lengths.values()) * rng.uniform(0.25, 0.65))
        cap = rng.randint(1, max(1, n - 1))
        ch = choose_batch(views, mem, cap, lengths)
        assert len(ch) <= cap and sum(lengths[i] for i in ch) <= mem
        assert pysum(v.utility for v in views if v.request_id in ch) >= greedy_utility(views, mem, cap, lengths) - 1e-12


class TestPlannerKnownAnswers:
    """Known answers of tests/test_kvstore.py:24-186."""

    CM = P.Costs(h2d_bandwidth=100000, d2h_bandwidth=100000)

    def test_write_plan_priority(self):
        assert P.writeback_plan({1: 3000, 2: 4000}, 0.05, self.CM, {1: 50, 2: 200}) == [(2, 4000), (1, 1000)]
        assert P.writeback_plan({2: 10, 1: 10}, 1.0, self.CM, {1: 5, 2: 5}) == [(1, 10), (2, 10)]
        with pytest.raises(ValueError):
            P.writeback_plan({1: 10}, 0.0, self.CM, {1: 1})

    def test_preempt_resume(self):
        assert P.eviction(P.Placement(0, 4000, 4000, 3500)) == (3500, 500)
        assert P.eviction(P.Placement(0, 4000, 4000, 0)) == (0, 4000)
        with pytest.raises(P.ResidencyError):
            P.eviction(P.Placement(0, 100, 0, 100))
        assert P.reload(P.Placement(0, 4000, 0, 4000), 512) == (4000, (512,) * 7 + (416,))
        with pytest.raises(P.ResidencyError):
            P.reload(P.Placement(0, 4000, 0, 1000), 512)

    def test_io_estimate(self):
        assert P.io_estimate(P.Placement(0, 4000, 0, 3500), P.QueueView(), self.CM) == pytest.approx(0.045)
        q = P.QueueView(h2d_queue=[P.Xfer(9, 10000, "h2d", "load")])
        assert P.io_estimate(P.Placement(0, 4000, 0, 4000), q, self.CM) == pytest.approx(0.14)
        assert P.io_estimate(P.Placement(0, 4000, 4000, 4000), P.QueueView(), self.CM) == 0.0

    def test_split_chunks_partition(self):
        for n in range(0, 3000, 37):
            for c in (1, 7, 128, 512):
                s = P.pieces(n, c)
                assert sum(s) == n and all(0 < x <= c for x in s) and all(x == c for x in s[:-1])


def test_pysum_matches_builtin_sum():
    rng = random.Random(5)
    for _ in range(20000):
        xs = [rng.choice([rng.random(), -rng.random() * 1e3, 1e16, -1e16, rng.gauss(0, 1)])
              for _ in range(rng.randint(0, 10))]
        a, b = sum(xs), pysum(xs)
        assert a == b and math.copysign(1, a) == math.copysign(1, b)


def test_realtime_b200_ticks_match_oracle():
    """Every on_tick decision the GPU selector took during a real-time C2 bench
    run on a B200 (member view built on the device; recorded by
    ``bench.py --dump-ticks``) equals the oracle restatement's decision on the
    same snapshot and policy state - parity in the measured regime, not only on
    the reference's own recorded ticks."""
    import gzip
    import json
    from dataclasses import asdict

    from conftest import GOLDEN

    from oracle.refsim.policy import Knobs, TokenFlowPolicy, snapshot_from_dict
    from paper_2510_02758_b200 import configs
    from paper_2510_02758_b200.scheduler import SchedulerConfig

    d = json.load(gzip.open(GOLDEN / "realtime" / "c2_burst_b200_ticks.json.gz"))
    knobs = Knobs(**asdict(configs.C2.sched_cfg(SchedulerConfig)))
    assert len(d["ticks"]) > 100
    for t in d["ticks"]:
        pol = TokenFlowPolicy(knobs)
        pol._t_prime = {int(k): v for k, v in t["t_prime"]}
        pol.mode = t["mode_before"]
        want = pol.on_tick(snapshot_from_dict(t["snapshot"]))
        assert (want.mode, list(want.preempt), [list(r) for r in want.resume],
                [list(b) for b in want.prefill_batches]) == \
            (t["mode"], t["preempt"], [list(r) for r in t["resume"]], t["prefill_batches"])
        assert sorted((int(k), v) for k, v in pol._t_prime.items()) == [(int(k), v) for k, v in t["t_prime_after"]]
