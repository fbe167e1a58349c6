"""Host-side logic of the product (no GPU): the runtime's event semantics,
the reference-API planner/scheduler/metrics/workload mirrors, and the C-ABI
library's exports."""
import ctypes as C
import math
import random
import re

import pytest
from conftest import ROOT, golden_names, load_golden, trace_path

from paper_2510_02758_b200 import kvstore, metrics, scheduler, workload
from paper_2510_02758_b200.costs import CostModel, decode_iteration_time, transfer_time
from paper_2510_02758_b200.engine import CapacityError, Engine, SimConfig

FAST = [n for n in golden_names("runs") if not n.startswith(("c2_", "burst4090b", "poissonh200c"))]


def _oracle_policy(g):
    from oracle.refsim.policy import Knobs, build_policy

    return build_policy(g["policy"], Knobs(**g["sched"]))


@pytest.mark.parametrize("name", FAST)
def test_runtime_event_semantics_match_reference(name):
    """The product runtime (driven here by the oracle's policy restatement,
    no data plane) reproduces the reference's event hash, decisions and
    chunk rows - its event loop is a faithful drop-in."""
    g = load_golden("runs", name)
    tr = workload.load_trace(trace_path(g["trace"]))
    res = Engine(tr, _oracle_policy(g), CostModel(**g["cm"]), SimConfig(**g["sim"])).run()
    assert res.event_hash() == g["event_hash"]
    assert res.decision_log == g["decision_log"]
    if "chunks" in g:
        assert res.chunk_rows() == g["chunks"]
    m = g["metrics"]
    eff = metrics.effective_throughput(res.records, res.total_time, metrics.EffectiveThroughputConfig())
    assert eff == m["effective_tps"]
    assert metrics.ttft_stats(res.records)["p99"] == m["ttft_p99"]
    assert metrics.ttft_latency_stats(res.records)["p99"] == m["ttft_latency_p99"]


def test_runtime_records_match_reference_c1():
    g = load_golden("runs", "c1_tokenflow")
    tr = workload.load_trace(trace_path(g["trace"]))
    res = Engine(tr, _oracle_policy(g), CostModel(**g["cm"]), SimConfig(**g["sim"])).run()
    rows = [[r.request_id, r.ttft, r.gen_times, r.buffer_at_gen, r.consume_times, r.rebuffer_s, r.gen_done_time,
             r.done_time, r.preemptions, r.resumes, r.recomputes] for r in res.records]
    assert rows == g["records"]


def test_capacity_error():
    tr = workload.Trace((workload.RequestSpec(0, 0.0, 100, 100, 20.0),))
    with pytest.raises(CapacityError):
        Engine(tr, "fcfs", CostModel(), SimConfig(gpu_mem_tokens=150, max_batch=2))


def test_frozen_traces_regenerate():
    """The product's generators reproduce the reference's frozen traces."""
    from paper_2510_02758_b200 import configs

    c1 = configs.C1
    tr = workload.generate_burst(workload.WorkloadConfig(kind="burst", burst_size=32, prompt_len_dist=c1.prompt_len_dist,
                                                         output_len_dist=c1.output_len_dist,
                                                         rate_profile=dict(c1.rate_profile)), 7)
    assert tr.requests == workload.load_trace(trace_path("c1_burst32_s7")).requests
    c2 = configs.C2
    full = workload.generate_poisson(workload.WorkloadConfig(kind="poisson", poisson_rate=10.0, duration=30.0,
                                                             prompt_len_dist=c2.prompt_len_dist,
                                                             output_len_dist=c2.output_len_dist,
                                                             rate_profile=dict(c2.rate_profile)), 1)
    assert full.requests[:256] == workload.load_trace(trace_path("c2_poisson256_s1")).requests


class TestPlannerApi:
    CM = CostModel(h2d_bandwidth=100000, d2h_bandwidth=100000)

    def test_known_answers(self):
        assert kvstore.plan_write_chunk({1: 3000, 2: 4000}, 0.05, self.CM, {1: 50, 2: 200}) == [(2, 4000), (1, 1000)]
        assert kvstore.preempt(kvstore.KvResidency(0, 4000, 4000, 3500)) == kvstore.EvictionPlan(0, 3500, 500)
        assert kvstore.resume(kvstore.KvResidency(0, 4000, 0, 4000)).chunks == (512,) * 7 + (416,)
        with pytest.raises(kvstore.ResidencyError):
            kvstore.resume(kvstore.KvResidency(0, 4000, 0, 1000))
        r = kvstore.KvResidency(0, 4000, 0, 3500)
        assert kvstore.io_overhead_estimate(r, kvstore.TransferQueueState(), self.CM) == pytest.approx(0.045)

    def test_overlap_timeline(self):
        ev = [kvstore.EvictionPlan(0, 3500, 500)]
        ld = [kvstore.LoadPlan(1, 2000, (2000,))]
        tq = kvstore.TransferQueueState()
        assert kvstore.overlap_timeline(ev, ld, tq, self.CM, 10000)[1] == pytest.approx(0.02)
        assert kvstore.overlap_timeline(ev, ld, tq, self.CM, 10000, overlap=False)[1] == pytest.approx(0.025)
        ev = [kvstore.EvictionPlan(0, 0, 500)]
        ld = [kvstore.LoadPlan(1, 400, (400,))]
        assert kvstore.overlap_timeline(ev, ld, tq, self.CM, 0)[1] == pytest.approx(0.009)
        with pytest.raises(MemoryError):
            kvstore.overlap_timeline([], ld, tq, self.CM, 0)

    def test_costs(self):
        cm = CostModel(decode_base=0.02, decode_per_request=0.005)
        assert decode_iteration_time(2, 100, cm) == pytest.approx(0.03)
        assert transfer_time(0, "d2h", cm) == 0.0
        with pytest.raises(ValueError):
            decode_iteration_time(0, 0, cm)


class TestSchedulerApi:
    CFG = scheduler.SchedulerConfig()

    def test_working_set(self):
        assert scheduler.working_set_size(1000, 250, 10, self.CFG) == 4
        with pytest.raises(ValueError):
            scheduler.working_set_size(100, 250, 0, self.CFG)

    def test_admit_and_restore(self):
        v = scheduler.build_priority_view(0, 100, 20.0, 500, 1.0, 0.0, 0.0, self.CFG)
        assert scheduler.admit(v, 0.5, 0.5, 1.0, self.CFG)
        assert scheduler.recompute_or_load(1.0, 1.0) == "load"
        assert scheduler.recompute_or_load(2.0, 1.0) == "recompute"

    def test_partition(self):
        items = [scheduler.PrefillItem(0, 100), scheduler.PrefillItem(1, 100, waited_s=2.0),
                 scheduler.PrefillItem(2, 150), scheduler.PrefillItem(3, 500)]
        assert scheduler.partition_prefill(items, 260) == [[1], [0, 2]]

    def test_registry(self):
        assert set(scheduler.POLICIES) == {"tokenflow", "fcfs", "chunked", "qoe"}
        with pytest.raises(ValueError):
            scheduler.make_policy("nope")


def test_metric_known_answers():
    cfg = metrics.EffectiveThroughputConfig()
    assert metrics.effective_token_weight(5, 100, cfg) == 1.0
    assert metrics.effective_token_weight(15, 100, cfg) == pytest.approx(0.5)
    assert metrics.effective_token_weight(20, 100, cfg) == 0.0
    assert metrics.nearest_rank([1.0, 2.0, 3.0], 99.0) == 3.0
    assert metrics.replay_rebuffer(0.0, [0.0, 0.05, 0.5], 20.0) == pytest.approx(0.4)
    # QosConfig validates like tokensim/metrics.py:25-31
    for bad in ({"buffer_threshold_frac": 0.0}, {"buffer_threshold_frac": 1.0}, {"decay_alpha": 0.0},
                {"ttft_penalty_weight": -1.0}, {"rebuffer_penalty_weight": -0.5}):
        with pytest.raises(metrics.MetricError):
            metrics.QosConfig(**bad)
    with pytest.raises(metrics.MetricError):
        scheduler.SchedulerConfig(value_threshold_frac=1.5).value_config()


def test_library_exports_every_header_symbol():
    from paper_2510_02758_b200 import _lib

    hdr = (ROOT / "include" / "tokenflow_b200.h").read_text()
    declared = set(re.findall(r"^\s*(?:const char\*|void\*|int64_t|int|double)\s+(tf_\w+)\s*\(", hdr, re.M))
    assert declared, "no declarations parsed"
    assert declared == set(_lib.SIGNATURES)
    for name in declared:
        assert getattr(_lib.lib, name) is not None


def test_library_host_entry_points():
    """Calls that need no GPU: glibc-exact exp, allocator, argument checks."""
    from paper_2510_02758_b200._lib import check, lib

    rng = random.Random(3)
    for _ in range(50000):
        x = -rng.random() * 900.0
        assert lib.tf_host_glibc_exp(x) == math.exp(x)
    h = C.c_int64()
    check(lib.tf_pool_init(C.c_void_p(256), 8, None, 0, 2, 16, 2, 64, 0, C.byref(h)))
    ids = (C.c_int32 * 3)()
    check(lib.tf_blocks_alloc(h, 0, 3, ids))
    assert list(ids) == [0, 1, 2]
    check(lib.tf_blocks_free(h, 0, ids, 3))
    again = (C.c_int32 * 1)()
    check(lib.tf_blocks_alloc(h, 0, 1, again))
    assert again[0] == 2  # LIFO: the last freed block is handed out first
    # double free below capacity, a duplicate inside one list and an
    # out-of-range id are all rejected without changing the allocator
    n_free = lib.tf_blocks_free_count(h, 0)
    with pytest.raises(ValueError, match="double free"):
        check(lib.tf_blocks_free(h, 0, (C.c_int32 * 1)(0), 1))
    with pytest.raises(ValueError, match="double free"):
        check(lib.tf_blocks_free(h, 0, (C.c_int32 * 2)(2, 2), 2))
    with pytest.raises(ValueError, match="out of range"):
        check(lib.tf_blocks_free(h, 0, (C.c_int32 * 2)(2, 99), 2))
    assert lib.tf_blocks_free_count(h, 0) == n_free
    check(lib.tf_blocks_free(h, 0, again, 1))  # block 2 is still allocated: a valid free
    assert lib.tf_blocks_free_count(h, 0) == n_free + 1
    with pytest.raises(MemoryError):
        check(lib.tf_blocks_alloc(h, 0, 99, (C.c_int32 * 99)()))
    with pytest.raises(ValueError):
        check(lib.tf_pool_init(C.c_void_p(256), 8, None, 0, 2, 16, 2, 60, 0, C.byref(h)))
    check(lib.tf_pool_destroy(h))


def test_bench_helpers():
    """bench.py's roofline traffic (scaled from the committed ncu capture) and
    TTFT summary (nearest-rank P99 over first-token latencies)."""
    import types

    import bench

    t, src = bench._ncu_traffic(400e6)
    assert src and "ncu" in src and 1.0 <= t / 400e6 <= 1.1
    recs = [types.SimpleNamespace(gen_times=[float(i) + 1.0], arrival=0.0) for i in range(100)]
    s = bench._ttft_summary(recs, 100, 1, False)
    v = [float(i) + 1.0 for i in range(100)]
    assert s["complete"] and s["requests"] == 100
    assert s["p99_s"] == metrics.nearest_rank(v, 99.0) and s["p50_s"] == metrics.nearest_rank(v, 50.0)
    assert bench._ttft_summary([], 5, 1, False) is None


def test_prefill_graph_layout():
    """Host-side layout of a captured prefill graph: real sequences first,
    zero-length unused slots, the padding sequence on the scratch row; every
    token's row / position, the cu_seqlens and the last-token indices."""
    import numpy as np

    from paper_2510_02758_b200.model import PagedDecoder

    T, NS, scratch = 64, 4, 99
    meta, last = PagedDecoder.prefill_layout([7, 3], [10, 5], T, NS, scratch)
    rows, pos, cu = meta[:T], meta[T:2 * T], meta[2 * T:]
    assert cu.tolist() == [0, 10, 15, 15, 15, 64]
    assert last.tolist() == [9, 14, 0, 0]
    assert (rows[:10] == 7).all() and (rows[10:15] == 3).all() and (rows[15:] == scratch).all()
    assert pos[:10].tolist() == list(range(10)) and pos[10:15].tolist() == list(range(5))
    assert pos[15:].tolist() == list(range(T - 15))
    # exactly full: the padding sequence is empty
    meta, last = PagedDecoder.prefill_layout([1, 2, 3, 4], [16, 16, 16, 16], T, NS, scratch)
    assert meta[2 * T:].tolist() == [0, 16, 32, 48, 64, 64] and last.tolist() == [15, 31, 47, 63]
    with pytest.raises(ValueError):
        PagedDecoder.prefill_layout([1, 2, 3, 4, 5], [1] * 5, T, NS, scratch)
    with pytest.raises(ValueError):
        PagedDecoder.prefill_layout([1], [65], T, NS, scratch)
    b = PagedDecoder._prefill_bucket_sizes(4700, 128)
    assert b[:8] == [128 * i for i in range(1, 9)] and b[-1] == 4700 and b == sorted(set(b))
    assert all(y - x <= 512 for x, y in zip(b, b[1:]))
    assert np.all(np.diff(b) > 0)
