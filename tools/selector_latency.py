"""Batch-priority selector latency (SURVEY 8(d) `select_topk` row).

GPU: microseconds per call of the C-ABI selector entry points at N members
  * tf_policy_tick        on_tick from a host-built member view
  * tf_policy_tick_rows   on_tick with the member view built on the device
  * tf_policy_fastpath    opportunistic fast-path resumes
  * tf_iteration_batch    per-dispatch pacing filter over N running requests
  * tf_select_batch       select_batch over N priority views
  each end to end (pack -> H2D -> one single-CTA launch -> D2H -> unpack,
  host wall clock) and on the device (CUDA events on the selector's stream
  around the same call), next to the empty-kernel launch floor
  (tf_launch_floor, same two clocks).
CPU: the same snapshots through the oracle restatement of the reference's
  on_tick / select_batch (tokensim/scheduler.py:513-736, :230-269) on one host
  core - called ONLY from bench.py's cpu_baseline leg.

Snapshots: the C2 burst tick with the most members (tests/golden/ticks,
recorded from the unmodified reference), its members tiled with fresh request
ids (and perturbed buffers) to N = 32 / 128 / 256 / 1024.
"""
from __future__ import annotations

import copy
import gzip
import json
import random
import statistics
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
NS = (32, 128, 256, 1024)


def snapshot_dicts(ns=NS, seed=0):
    g = json.load(gzip.open(ROOT / "tests" / "golden" / "ticks" / "c2_burst256_s1_tokenflow.json.gz"))
    base = max((t["view"] for t in g["ticks"]), key=lambda v: len(v["members"]))
    rng = random.Random(seed)
    out = {}
    for n in ns:
        v = copy.deepcopy(base)
        mem = []
        for i in range(n):
            m = dict(base["members"][i % len(base["members"])])
            m["request_id"] = i
            m["consumed"] = max(0, m["generated"] - rng.randint(0, 200))
            mem.append(m)
        v["members"] = mem
        v["waiting"] = [dict(w, request_id=n + j) for j, w in enumerate(base["waiting"][:64])]
        out[n] = v
    return out, g["sched"]


def _product_snapshot(v):
    from paper_2510_02758_b200.scheduler import MemberView, SystemSnapshot, WaitingView

    return SystemSnapshot(v["now"], [MemberView(**m) for m in v["members"]], [WaitingView(**w) for w in v["waiting"]],
                          v["free_slots"], v["gpu_mem_free"], v["gpu_mem_total"], v["cpu_mem_total"], v["max_batch"],
                          v["gamma"], v["prefill_s_per_token"], v["offload_enabled"], v["h2d_blocked_tokens"])


def _rows_snapshot(v):
    """The same members as raw request counters (device-built view)."""
    from paper_2510_02758_b200 import _lib
    from paper_2510_02758_b200.scheduler import RowsSnapshot, WaitingView

    n = len(v["members"])
    rows = (_lib.TfReqRow * max(1, n))()
    for i, m in enumerate(v["members"]):
        r = rows[i]
        r.request_id, r.prompt_len, r.output_len = m["request_id"], m["prompt_len"], m["output_len"]
        r.status = _lib.STATUS_CODES["running" if m["running"] else "preempted"]
        r.generated, r.consumed, r.total_kv, r.gpu_resident = m["generated"], m["consumed"], m["ctx_tokens"], \
            m["gpu_resident"]
        r.cpu_synced, r.inflight_d2h = m["releasable_now"], 0
        r.arrival_time, r.rate, r.busy_since_tick = m["arrival_time"], m["rate"], m["busy_since_tick"]
        r.last_iter_time = m["last_iter_time"] or 0.0
    g = _lib.TfSnapGlobals()
    g.q_d2h_tokens, g.q_h2d_tokens, g.d2h_rate, g.h2d_rate = 0, 0, 4.0e5, 4.0e5
    g.prefill_s_per_token = v["prefill_s_per_token"]
    return RowsSnapshot(v["now"], rows, n, g, [WaitingView(**w) for w in v["waiting"]], v["free_slots"],
                        v["gpu_mem_free"], v["gpu_mem_total"], v["cpu_mem_total"], v["max_batch"], v["gamma"],
                        v["prefill_s_per_token"], v["offload_enabled"], v["h2d_blocked_tokens"])


def _prio_views(n, seed=7):
    from paper_2510_02758_b200.scheduler import RequestPriorityView

    rng = random.Random(seed)
    views, lengths = [], {}
    for i in range(n):
        b, r = rng.randint(0, 400), rng.choice([15.0, 20.0, 25.0, 30.0])
        v, tp, to = rng.random(), rng.random() * 1.5, rng.random() * 0.4
        phi = 2.718281828 ** (-b / (r * 0.5))
        views.append(RequestPriorityView(i, b, 0.0, r, v, tp, to, phi, v * max(tp - to, 0.0) - 0.1 * phi))
        lengths[i] = rng.randint(100, 3000)
    return views, lengths


def _time(fn, stream, reps):
    import torch

    fn()
    fn()
    host, dev = [], []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        t0 = time.perf_counter()
        fn()
        host.append((time.perf_counter() - t0) * 1e6)
        e1.record(stream)
        e1.synchronize()
        dev.append(e0.elapsed_time(e1) * 1e3)
    return {"e2e_us": round(statistics.median(host), 1), "device_us": round(statistics.median(dev), 1)}


def gpu_selector_latency(ns=NS, reps=30):
    import ctypes as C

    import torch

    from paper_2510_02758_b200 import _lib
    from paper_2510_02758_b200.scheduler import SchedulerConfig
    from paper_2510_02758_b200.selector import GpuSelector

    snaps, sched = snapshot_dicts(ns)
    cfg = SchedulerConfig(**sched)
    sel = GpuSelector()
    st = sel.stream
    out = {"launch_floor": _time(lambda: (_lib.check(_lib.lib.tf_launch_floor(C.c_void_p(st.cuda_stream))),
                                          st.synchronize()), st, reps)}
    for n in ns:
        v = snaps[n]
        snap, rows = _product_snapshot(v), _rows_snapshot(v)
        running = [(m["request_id"], m["generated"] - m["consumed"], m["rate"]) for m in v["members"]]
        views, lengths = _prio_views(n)
        row = {
            "tick": _time(lambda: sel.tick(snap, cfg, {}, "buffer_aware"), st, reps),
            "tick_rows": _time(lambda: sel.tick_rows(rows, cfg, {}, "buffer_aware"), st, reps),
            "fastpath": _time(lambda: sel.fastpath(snap, cfg, "buffer_aware"), st, reps),
            "iteration_batch": _time(lambda: sel.iteration_batch(running, True, "buffer_aware",
                                                                 cfg.pacing_buffer_seconds), st, reps),
            "select_batch": _time(lambda: sel.select_batch(views, int(sum(lengths.values()) * 0.3), n // 3,
                                                           lengths), st, reps),
        }
        out[str(n)] = row
    torch.cuda.synchronize()
    return out


def cpu_selector_latency(ns=NS, reps=5):
    """Oracle restatement of the reference policy on one core (cpu_baseline leg only)."""
    from oracle.refsim.policy import Knobs, Prio, TokenFlowPolicy, choose_batch, snapshot_from_dict

    snaps, sched = snapshot_dicts(ns)
    out = {}
    for n in ns:
        v = snaps[n]
        ts = []
        for _ in range(reps):
            pol = TokenFlowPolicy(Knobs(**sched))
            snap = snapshot_from_dict(v)
            t0 = time.perf_counter()
            pol.on_tick(snap)
            ts.append((time.perf_counter() - t0) * 1e6)
        views, lengths = _prio_views(n)
        pv = [Prio(x.request_id, x.b_rem, x.b_pred, x.rate, x.value, x.t_prime, x.t_overhead, x.phi, x.utility)
              for x in views]
        tb = []
        for _ in range(max(1, reps // 2)):
            t0 = time.perf_counter()
            choose_batch(pv, int(sum(lengths.values()) * 0.3), n // 3, lengths)
            tb.append((time.perf_counter() - t0) * 1e6)
        out[str(n)] = {"on_tick_us": round(statistics.median(ts), 1), "select_batch_us": round(statistics.median(tb), 1)}
    return out
