"""GPU selector parity: every tick / fast-path / pacing decision the
reference made (golden fixtures) is reproduced bit for bit by the
single-CTA selector kernel, and random snapshots agree with the oracle."""
import gzip
import json
import random

import pytest
from conftest import GOLDEN, golden_names, load_golden

from oracle.refsim.policy import Knobs, Prio, TokenFlowPolicy, choose_batch, snapshot_from_dict, starvation

pytestmark = pytest.mark.gpu

TICK_FILES = golden_names("ticks")


@pytest.fixture(scope="module")
def sel(cuda):
    from paper_2510_02758_b200.selector import GpuSelector

    return GpuSelector()


def _cfg(d):
    from paper_2510_02758_b200.scheduler import SchedulerConfig

    return SchedulerConfig(**d)


@pytest.mark.parametrize("name", TICK_FILES)
def test_ticks_match_reference(sel, name):
    g = load_golden("ticks", name)
    if g["policy"] != "tokenflow":
        pytest.skip("baseline policy (host-side)")
    cfg = _cfg(g["sched"])
    for t in g["ticks"]:
        snap = snapshot_from_dict(t["view"])
        tp = {k: v for k, v in t["t_prime"]}
        mode, pre, resume, adm, rc, batches = sel.tick(snap, cfg, tp, t["mode_before"])
        d = t["decision"]
        assert mode == d["mode"]
        assert pre == d["preempt"]
        assert [[r, h] for r, h in resume] == d["resume"]
        assert batches == d["prefill_batches"]
        assert adm == d["log"]["admitted"] and rc == d["log"]["recomputed"]
        assert sorted(tp.items()) == sorted((k, v) for k, v in t["t_prime_after"])
    for o in g["opportunistic"]:
        snap = snapshot_from_dict(o["view"])
        if o["mode_before"] == "fcfs_fallback":
            continue
        _, _, resume, _, _, batches = sel.fastpath(snap, cfg, o["mode_before"])
        assert [[r, h] for r, h in resume] == o["decision"]["resume"]
        assert batches == o["decision"]["prefill_batches"]
    for it in g["iteration_batch"]:
        running = [tuple(x) for x in it["running"]]
        if not it["contention"] or it["mode"] == "fcfs_fallback":
            continue
        assert sel.iteration_batch(running, it["contention"], it["mode"], cfg.pacing_buffer_seconds) == it["out"]


def test_select_batch_golden(sel):
    cases = json.load(gzip.open(GOLDEN / "select_batch.json.gz"))["cases"]
    for c in cases:
        views = [Prio(**v) for v in c["views"]]
        lengths = {k: v for k, v in c["lengths"]}
        assert sorted(sel.select_batch(views, c["mem"], c["batch"], lengths)) == c["chosen"]


def test_random_snapshots_match_oracle(sel):
    """Fuzz: perturbed golden snapshots (buffers, near-tie drains, rates,
    memory) decided by the kernel and by the oracle restatement."""
    rng = random.Random(11)
    g = load_golden("ticks", "c1_tokenflow")
    cfg_d = g["sched"]
    cfg = _cfg(cfg_d)
    base = [t["view"] for t in g["ticks"]] + [t["view"] for t in load_golden("ticks", "table2_s3_full")["ticks"]]
    n = 0
    for _ in range(300):
        v = json.loads(json.dumps(rng.choice(base)))
        for m in v["members"]:
            if rng.random() < 0.5:
                m["consumed"] = max(0, m["generated"] - rng.randint(0, 60))
            if rng.random() < 0.2:
                m["rate"] = rng.choice([15.0, 20.0, 25.0, 30.0])
            if rng.random() < 0.2:
                m["running"], m["pinned"] = rng.choice([(True, False), (False, False), (False, True)])
        v["gpu_mem_free"] = rng.randint(-200, 1500)
        v["free_slots"] = rng.randint(-1, 4)
        v["gamma"] = rng.choice([v["gamma"], 1e9, 10.0])
        snap = snapshot_from_dict(v)
        pol = TokenFlowPolicy(Knobs(**cfg_d))
        tp = {m["request_id"]: rng.random() for m in v["members"] if rng.random() < 0.7}
        pol._t_prime = dict(tp)
        want = pol.on_tick(snap)
        tp2 = dict(tp)
        mode, pre, resume, adm, rc, batches = sel.tick(snapshot_from_dict(v), cfg, tp2, "buffer_aware")
        assert (mode, pre, resume, batches) == (want.mode, want.preempt, want.resume, want.prefill_batches)
        assert tp2 == pol._t_prime
        n += 1
    assert n == 300


def test_select_batch_large_random(sel):
    rng = random.Random(7)
    k = Knobs()
    for n in (32, 128, 256, 512):
        views, lengths = [], {}
        for i in range(n):
            b, r = rng.randint(0, 400), rng.choice([15.0, 20.0, 25.0, 30.0])
            v, tp, to = rng.random(), rng.random() * 1.5, rng.random() * 0.4
            phi = starvation(b, r, k.schedule_interval)
            views.append(Prio(i, b, 0.0, r, v, tp, to, phi, v * max(tp - to, 0.0) - k.penalty_weight * phi))
            lengths[i] = rng.randint(100, 3000)
        mem = int(sum(lengths.values()) * 0.3)
        assert sel.select_batch(views, mem, n // 3, lengths) == choose_batch(views, mem, n // 3, lengths)


@pytest.mark.parametrize("name", ["c1_tokenflow", "table2_s3_full", "c2_burst256_s1_tokenflow"])
def test_device_snapshot_builder_matches_reference(sel, name):
    """with the member view built on the device from the raw
    request counters (tf_policy_tick_rows), the runtime reproduces the
    reference's event hash and decision log - same as the host-built view."""
    from conftest import trace_path

    from paper_2510_02758_b200.costs import CostModel
    from paper_2510_02758_b200.engine import Engine, SimConfig
    from paper_2510_02758_b200.scheduler import SchedulerConfig, make_policy
    from paper_2510_02758_b200.workload import load_trace

    g = load_golden("runs", name)
    tr = load_trace(trace_path(g["trace"]))
    hashes = []
    for device in (True, False):
        eng = Engine(tr, make_policy(g["policy"], SchedulerConfig(**g["sched"])), CostModel(**g["cm"]),
                     SimConfig(**g["sim"]))
        eng.device_snapshot = device
        res = eng.run()
        assert res.decision_log == g["decision_log"], f"device_snapshot={device}"
        hashes.append(res.event_hash())
    assert hashes[0] == hashes[1] == g["event_hash"]
