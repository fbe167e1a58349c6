"""Benchmark: effective tok/s (+ P99 TTFT, KV swap GB/s) of the B200 TokenFlow
hot path on C2 (Llama3-8B bf16 random-init, the 256-request C2 population
arriving as a burst at t=0, KV swap to pinned host), 1 GPU per process.

python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                [--config c2|c4] [--arrivals burst|poisson] [--full-run]

A *step* is one decode iteration of the real-time serving loop
(realtime.RealtimeEngine): the GPU selector's pacing / tick decisions (member
view built on the device), the Llama3-8B forward (captured CUDA graph: fused
RMSNorm / rope+append / paged attention / SwiGLU around cuBLAS GEMMs) and the
write-through / evict / load chunks the engine issues meanwhile on the two
high-priority copy streams.  W warm-up steps from t=0, then EXACTLY K timed
steps (default 1000: the admission / preemption / swap-heavy phase of the
burst).

value  = effective tokens (tokensim.metrics weights, tau1/tau2 = 10%/20% of
         the output length) generated in the K steps / device time of every
         GPU job (decode steps and the prefills between them) in the window
         (CUDA events on the compute stream), max over ranks; weights and KV
         resident in HBM.
e2e    = the same tokens / host wall-clock span of the K steps through the
         public API (engine loop), including every step's host<->device
         traffic (step inputs, sampled ids, load / write-through / evict
         chunks: h2d_bytes_per_step / d2h_bytes_per_step).
ttft   = after the window the loop keeps serving until every request of the
         burst has its first token: complete nearest-rank P99 TTFT.
roofline / swap.hidden_under_decode are measured right after the window on
the running batch; gpu_launches are counted by the library.  The working set
(16 GB weights + ~20 GiB KV) exceeds the 126 MB L2 (no flush needed).
Multi-GPU: request i -> replica i mod N (C3, weak scaling); --config c4 runs
Qwen2.5-32B tensor-parallel over the launched ranks (strong scaling).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))
METRIC = "effective tok/s & P99 TTFT under burst; KV swap GB/s vs PCIe Gen5 roofline"
PCIE_GEN5_GBS = 63.0  # x16, 32 GT/s, 128b/130b, per direction


def _peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return d.get("hbm_gbs", 6650.0), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    FIELDS = "clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown," \
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap"

    def __init__(self, index=0):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                vals = [v.strip() for v in out.stdout.strip().split(",")]
                if len(vals) == 6:
                    self.samples.append(vals)
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=6)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def _dist():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def _max_over_ranks(x: float, world: int, device) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def _sum_over_ranks(x: float, world: int, device) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def _trace_for_rank(rank, world, arrivals="burst"):
    from paper_2510_02758_b200 import replicas
    from paper_2510_02758_b200.workload import load_trace

    name = "c2_burst256_s1" if arrivals == "burst" else "c2_poisson256_s1"
    tr = load_trace(str(ROOT / "tests" / "golden" / "traces" / f"{name}.csv"))
    if world == 1:
        return tr
    # C3: the burst scaled per GPU (256 requests per replica), request i -> GPU i mod N
    return replicas.partition(replicas.scale_trace(tr, world), rank, world)[0]


def run_ours(args):
    import torch

    from paper_2510_02758_b200 import configs
    from paper_2510_02758_b200.costs import CostModel
    from paper_2510_02758_b200.dataplane import GpuDataPlane, KvPool
    from paper_2510_02758_b200.engine import SimConfig
    from paper_2510_02758_b200.metrics import ttft_latency_stats
    from paper_2510_02758_b200.model import PagedDecoder
    from paper_2510_02758_b200.realtime import RealtimeEngine
    from paper_2510_02758_b200.scheduler import BufferAwarePolicy, SchedulerConfig

    world, rank, local = _dist()
    # (debug: TF_BENCH_ONE_GPU=1 runs every rank on cuda:0 with a gloo group,
    # to exercise the multi-rank code path on a one-GPU box)
    one_gpu = os.environ.get("TF_BENCH_ONE_GPU") == "1"
    if one_gpu:
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    tp_mode = args.config == "c4"
    tp = lockstep = None
    if world > 1:
        import torch.distributed as dist

        if one_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    if tp_mode:
        # C4: one model over all ranks (TP = world), NCCL all-reduces on the
        # data path, completion/clock consensus over a CPU group on the control path
        from paper_2510_02758_b200.tp import Lockstep, TpGroup

        tp = TpGroup(rank, world)
        if world > 1:
            import torch.distributed as dist

            lockstep = Lockstep(dist.new_group(backend="gloo"))
        c2 = configs.c4(world)
        tr = _trace_for_rank(0, 1, args.arrivals)
        if world > 1 and args.graphs:
            args.graphs = 0  # eager decode under TP: NCCL all-reduces are not captured in graphs
    else:
        c2 = configs.C2
        tr = _trace_for_rank(rank, world, args.arrivals)
    shape = c2.model
    tp_size = world if tp_mode else 1
    n_blocks = math.ceil(c2.gpu_mem_tokens / 16) + 4 * len(tr.requests) + c2.max_batch + 1
    pool = KvPool(n_blocks, args.host_blocks, shape.n_layers, shape.n_kv_heads // tp_size, shape.head_dim,
                  device=dev)
    model = PagedDecoder(shape, device=dev, seed=0 if tp_mode else rank, tp=tp)
    dp = GpuDataPlane(tr.requests, pool, mode="realtime", kv_source="model", model=model,
                      n_q_heads=shape.n_q_heads // tp_size, engine=args.swap_engine)
    if args.fused_wt:
        dp.enable_fused_write_through()
    if args.profile_hooks:
        from paper_2510_02758_b200.dataplane import profile_hooks

        profile_hooks(dp)
    if args.graphs:
        dp.enable_scratch()
        model.enable_graphs(dp)
    policy = BufferAwarePolicy(c2.sched_cfg(SchedulerConfig))
    tick_dump = []
    if args.dump_ticks:
        import dataclasses

        lo_t, hi_t = (float(x) for x in args.dump_window.split(","))
        orig_tick = policy.on_tick

        def on_tick(view):
            tp_before, mode_before = dict(policy._t_prime), policy.mode
            dec = orig_tick(view)
            if lo_t <= view.now <= hi_t:
                # a device-built snapshot (RowsSnapshot) is dumped as its host
                # equivalent, so the shadow check also verifies the builder
                view = view.materialize() if getattr(view, "materialize", None) else view
                snap = {k: getattr(view, k) for k in ("now", "free_slots", "gpu_mem_free", "gpu_mem_total",
                                                      "cpu_mem_total", "max_batch", "gamma", "prefill_s_per_token",
                                                      "offload_enabled", "h2d_blocked_tokens")}
                snap["members"] = [dataclasses.asdict(m) for m in view.members]
                snap["waiting"] = [dataclasses.asdict(w) for w in view.waiting]
                tick_dump.append({"snapshot": snap, "t_prime": sorted(tp_before.items()), "mode_before": mode_before,
                                  "t_prime_after": sorted(policy._t_prime.items()),
                                  "mode": dec.mode, "preempt": list(dec.preempt),
                                  "resume": [list(r) for r in dec.resume],
                                  "prefill_batches": [list(b) for b in dec.prefill_batches]})
            return dec

        policy.on_tick = on_tick
    sim = c2.sim_cfg(SimConfig, debug_checks=False)
    cm = c2.cost_model(CostModel)

    t_start = time.perf_counter()
    state = {"phase": "warm", "timed": [], "wall0": None, "wall1": None}

    def window_probes(eng, timed):
        """Right at the end of the timed window (device idle, live batch intact):
        the roofline of the dominant kernel (paged attention re-launched on the
        running batch, all layers, CUDA events) and transfer hidden under the
        captured decode of that batch."""
        torch.cuda.synchronize()
        hbm, peak_kind = _peaks()
        # the decode batch at the window's end: every running request (what the
        # next step would read), capped at max_batch
        live = sorted(r for r in eng.running if eng.state[r].status == "running")[: c2.max_batch]
        if not live:
            return
        per = model.measure_attention(dp, live, [eng.state[r].kv.total_kv - 1 for r in live])
        avg_ms = sum(ms for _, ms in per) / len(per)
        avg_bytes = sum(b for b, _ in per) / len(per)
        ach = avg_bytes / (avg_ms / 1e3) / 1e9
        G = shape.n_q_heads // shape.n_kv_heads
        kname = {"1": "paged_attn_kernel (v1)", "2": "paged_attn_tma_kernel (v2)",
                 "3": f"paged_attn_mma_kernel<{G}> (v3) + combine"}.get(
            os.environ.get("TF_ATTN_IMPL", "3")[:1], f"paged_attn_stream_kernel<{G}> (v4 stream-K, tensor cores)")
        traffic, tsrc = _ncu_traffic(avg_bytes)
        state["roof"] = {"bound": "hbm", "kernel": kname, "achieved": round(ach, 1),
                         "peak": hbm, "peak_kind": peak_kind, "unit": "GB/s", "frac": round(ach / hbm, 4),
                         "traffic": traffic, "traffic_source": tsrc,
                         "launches": len(per), "avg_ms": round(avg_ms, 4), "batch": len(live),
                         "algorithmic_bytes_per_launch": round(avg_bytes),
                         "note": f"bytes = sum(ctx) x {pool.H * pool.D * 4} B (K+V, {pool.H} kv heads x {pool.D} x "
                                 "bf16) + q/out + table entries per layer; re-launched right after the window on "
                                 "the running batch"}
        if args.graphs:
            xf = dp.transfer_log()[state["ev0"]:state["ev1"]]
            per_step = lambda k: math.ceil(sum(n for d, n, _ in xf if d == k) / 16 / len(timed))  # noqa: E731
            hid_w = measure_hidden(model, dp, eng, live, per_step("d2h"), per_step("h2d"))
            # blocks per direction that keep a ~55 GB/s link busy for one decode step
            sat = max(1, int(55e9 * (hid_w["t_decode_ms"] if hid_w else 7.0) / 1e3 / dp.pool.block_bytes))
            hid_s = measure_hidden(model, dp, eng, live, sat, sat)
            state["hidden"] = {"window_volume": hid_w, "link_saturating": hid_s,
                               "note": "hidden = 1 - (T_both - T_decode)/T_swap; decode = the captured forward of "
                                       "the live batch; swaps on copy engines, own streams"}

    def on_step(rec, eng):
        n = len(eng.steps)
        if args.verbose and n % 100 == 0:
            print(f"[bench] step {n} t={eng.now:.2f}s batch={rec['batch']} dur={rec['dur'] * 1e3:.2f}ms "
                  f"pre={eng.total_preemptions} rc={eng.total_recomputes} running={len(eng.running)} "
                  f"waiting={len(eng.waiting)} d2h={dp.stats['d2h_tokens']} h2d={dp.stats['h2d_tokens']} "
                  f"wall={time.perf_counter() - t_start:.1f}s", file=sys.stderr, flush=True)
        if state["phase"] == "warm":
            if n >= args.warmup:
                state["phase"] = "timed"
                state["wall0"] = time.perf_counter()
                state["ev0"] = len(dp._events)
                state["pre0"], state["rc0"] = eng.total_preemptions, eng.total_recomputes
                state["launch0"] = model.launch_count()
                torch.cuda.nvtx.range_push("bench_timed")  # ncu --nvtx --nvtx-include bench_timed/
            return
        if state["phase"] == "timed":
            state["timed"].append(dict(rec))
            if len(state["timed"]) >= args.steps:
                state["wall1"] = time.perf_counter()
                state["ev1"] = len(dp._events)
                state["pre1"], state["rc1"] = eng.total_preemptions, eng.total_recomputes
                state["launch1"] = model.launch_count()
                state["phase"] = "done"
                torch.cuda.nvtx.range_pop()
                t_p = time.perf_counter()
                window_probes(eng, state["timed"])
                if args.full_run or args.ttft:
                    # the probes' pause is not serving time: shift the real-time clock back
                    eng.shift_clock(time.perf_counter() - t_p)
                    state["phase"] = "ttft" if not args.full_run else "rest"
                else:
                    eng._stop = True
            return
        if state["phase"] == "ttft" and all(st.record.gen_times for st in eng.state.values()):
            state["ttft_done_at"] = eng.now
            eng._stop = True

    eng = RealtimeEngine(tr, policy, cm, sim, dp, skip_idle=True, on_step=on_step, lockstep=lockstep,
                         max_wall_s=args.max_wall if args.full_run else None)
    if args.watchdog:
        _start_watchdog(eng, dp, args.watchdog)
    if world > 1:
        import torch.distributed as dist

        dist.barrier()
    torch.cuda.synchronize()
    sampler = ClockSampler(local)
    with sampler:
        res = eng.run()
    torch.cuda.synchronize()
    if state["phase"] not in ("done", "ttft", "rest"):
        raise RuntimeError(f"bench ended in phase {state['phase']} after {len(eng.steps)} steps")
    timed = state["timed"]
    # device time of the window: every GPU job (decode iterations and the
    # prefill / recompute jobs interleaved with them) that ran inside it
    t_lo, t_hi = timed[0]["start"], timed[-1]["end"]
    win_jobs = [j for j in eng.jobs if t_lo <= j[1] and j[2] <= t_hi]
    dev_s = sum(j[3] for j in win_jobs)
    prefill_s = sum(j[3] for j in win_jobs if j[0] == "prefill")
    eff = sum(s["effective"] for s in timed)
    toks = sum(s["tokens"] for s in timed)
    wall = state["wall1"] - state["wall0"]
    dev_s = _max_over_ranks(dev_s, world, dev)
    wall = _max_over_ranks(wall, world, dev)
    if not tp_mode:  # replicas: every rank generated its own tokens
        eff = _sum_over_ranks(eff, world, dev)
        toks = _sum_over_ranks(toks, world, dev)
    # swap traffic of the window (bytes per token = all layers' K and V of this rank's shard)
    bpt = shape.kv_bytes_per_token // tp_size
    xfers = dp.transfer_log()[state["ev0"]:state["ev1"]]
    d2h_tok = sum(n for k, n, _ in xfers if k == "d2h")
    h2d_tok = sum(n for k, n, _ in xfers if k == "h2d")
    d2h_ms = sum(ms for k, _, ms in xfers if k == "d2h")
    h2d_ms = sum(ms for k, _, ms in xfers if k == "h2d")
    if world > 1 and not tp_mode:  # C3: every replica's own link, rates over all replicas' chunks
        d2h_tok, h2d_tok = int(_sum_over_ranks(d2h_tok, world, dev)), int(_sum_over_ranks(h2d_tok, world, dev))
        d2h_ms, h2d_ms = _sum_over_ranks(d2h_ms, world, dev), _sum_over_ranks(h2d_ms, world, dev)
    swap = {"d2h_tokens": d2h_tok, "h2d_tokens": h2d_tok, "chunks": len(xfers),
            "engine": {0: "SM kernel", 1: "copy-engine batch", 2: "auto (CE whole blocks + SM partial)"}[
                args.swap_engine],
            "d2h_gbs": (d2h_tok * bpt / (d2h_ms / 1e3) / 1e9) if d2h_ms else None,
            "h2d_gbs": (h2d_tok * bpt / (h2d_ms / 1e3) / 1e9) if h2d_ms else None,
            "pcie_gen5_gbs": PCIE_GEN5_GBS,
            "preemptions": state["pre1"] - state["pre0"], "recomputes": state["rc1"] - state["rc0"]}
    for k in ("d2h", "h2d"):
        if swap[f"{k}_gbs"]:
            swap[f"{k}_frac_pcie"] = swap[f"{k}_gbs"] / PCIE_GEN5_GBS
    roof = state.get("roof")
    if state.get("hidden"):
        swap["hidden_under_decode"] = state["hidden"]
    ttft = [r for r in res.records if r.gen_times]
    out = {
        "metric": METRIC,
        "value": eff / dev_s if dev_s > 0 else None,
        "unit": "effective tok/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": dev_s / len(timed) * 1e3,
        "decode_ms_per_step": sum(s["dur"] for s in timed) / len(timed) * 1e3,
        "prefill_device_s_in_window": round(prefill_s, 4),
        "higher_is_better": True,
        "scaling": "strong" if tp_mode else "weak",
        "vs_baseline": None,
        "dtype": "bf16",
        "data": f"synthetic (random-init {shape.name} weights, seeded prompt token ids, frozen C2 trace)",
        "config": {"workload": (f"C4: Qwen2.5-32B bf16 random-init, tensor-parallel TP={world} (NCCL all-reduce "
                                f"after o_proj / down_proj), 256-request {args.arrivals} (C2 population), KV ledger "
                                "163,840 tokens (40 GiB over the TP ranks) + pinned host tier per rank, block 16, "
                                "max_batch 128") if tp_mode else
                               (f"C2: Llama3-8B bf16 random-init, 1xB200 per replica, 256-request {args.arrivals} "
                                "(bodies of the first 256 arrivals of the lambda=10/s 30 s trace, seed 1), KV pool "
                                "163,840 tokens (20 GiB) + pinned host tier, block 16, max_batch 128"),
                   "model": shape.name, "global_batch": max(s["batch"] for s in timed),
                   "mean_batch": round(statistics.mean(s["batch"] for s in timed), 1),
                   "seq_len": None, "parallelism": f"tp{world}" if tp_mode else f"replicas x{world}",
                   "arrivals": args.arrivals,
                   "l2": "working set (weights + KV, tens of GB) >> 126 MB L2; no flush needed",
                   "timed_region": f"decode iterations [{args.warmup}, {args.warmup + args.steps}) from t=0 "
                                   "of the real-time loop (measured clock, idle gaps skipped)",
                   "cuda_graphs": bool(args.graphs), "fused_write_through": bool(args.fused_wt)},
        "raw_tok_s": toks / dev_s if dev_s > 0 else None,
        "e2e": {"value": eff / wall if wall > 0 else None, "unit": "effective tok/s",
                "h2d_bytes_per_step": int((h2d_tok * bpt + sum(s["batch"] for s in timed) * 24) / len(timed)),
                "d2h_bytes_per_step": int((d2h_tok * bpt + sum(s["batch"] for s in timed) * 8) / len(timed))},
        "swap": swap,
        "roofline": roof,
        "clocks": sampler.summary(),
        "gpu_launches": None,
        "first_tokens_in_window": len(ttft),
        "ttft": _ttft_summary(ttft, len(res.records), world, tp_mode),
    }
    # this library's kernel launches inside the window, counted: every C-ABI
    # launch increments a counter in the .so, and each graph replay adds the
    # number of the library's kernels captured in that graph
    out["gpu_launches"] = int(state["launch1"] - state["launch0"])
    if args.full_run:
        from paper_2510_02758_b200.metrics import EffectiveThroughputConfig, effective_throughput

        done = [r for r in res.records if r.gen_times]
        out["full_run"] = {"truncated": eng.truncated, "requests_with_first_token": len(done),
                           "ttft_latency": ttft_latency_stats(done) if done else None,
                           "total_time_s": res.total_time, "wall_s": eng.wall_s,
                           "preemptions": res.total_preemptions, "recomputes": res.total_recomputes}
        if not eng.truncated:
            out["full_run"]["effective_tok_s"] = effective_throughput(res.records, res.total_time,
                                                                      EffectiveThroughputConfig())
    if args.profile_hooks:
        out["host_hook_ms"] = {k: {"calls": c, "avg_ms": round(t / c * 1e3, 4), "total_s": round(t, 3)}
                               for k, (c, t) in dp.hook_time.items() if c}
        for k, (c, t, ntok) in model.host_s.items():
            out["host_hook_ms"][f"model.{k}"] = {"calls": c, "avg_ms": round(t / c * 1e3, 4), "total_s": round(t, 3),
                                                 "avg_tokens": round(ntok / c, 1)}
    if args.dump_ticks:
        import gzip

        with gzip.open(args.dump_ticks, "wt") as f:
            json.dump({"ticks": tick_dump, "decision_log": res.decision_log}, f)
    if rank == 0 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(args, timed, quick=True)
    if rank == 0:
        print(json.dumps(out))
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()
    return out


def _ttft_summary(recs, n_records, world, tp_mode):
    """TTFT latency stats (first token - arrival, nearest-rank P99,
    tokensim/metrics.py:144-155) over ALL replicas' requests (C3: gathered)."""
    from paper_2510_02758_b200.metrics import nearest_rank

    lat = [r.gen_times[0] - r.arrival for r in recs]
    total = n_records
    if world > 1 and not tp_mode:
        import torch.distributed as dist

        parts = [None] * world
        dist.all_gather_object(parts, (lat, n_records))
        lat = [x for p in parts for x in p[0]]
        total = sum(p[1] for p in parts)
    if not lat:
        return None
    v = sorted(lat)
    return {"p99_s": round(nearest_rank(v, 99.0), 4), "p50_s": round(nearest_rank(v, 50.0), 4),
            "mean_s": round(sum(v) / len(v), 4), "requests": len(v), "of": total, "complete": len(v) == total,
            "note": "TTFT latency = first token - arrival (nearest-rank P99, tokensim/metrics.py:144-155)" + (
                ", real-time serving continued after the window until every request had its first token"
                if len(v) == total else ", requests that had their first token by the end of the run")}


def _ncu_traffic(alg_bytes):
    """DRAM bytes per launch for the attention kernel: the DRAM-traffic /
    algorithmic-bytes ratio of the committed ncu --set full capture of the
    same kernel (profiles/r1_attn_ncu_v3_v4.json) at the closest launch size,
    applied to this launch's algorithmic bytes."""
    p = ROOT / "profiles" / "r1_attn_ncu_v3_v4.json"
    impl = os.environ.get("TF_ATTN_IMPL", "3")[:1]
    want = "stream" if impl == "4" else "mma"
    try:
        caps = [k for k in json.loads(p.read_text())["kernels"] if want in k["kernel"]]
    except (OSError, ValueError, KeyError):
        return None, None
    if not caps:
        return None, None
    k = min(caps, key=lambda c: abs(math.log(c["algorithmic_bytes"] / alg_bytes)))
    return int(k["traffic_over_algorithmic"] * alg_bytes), (
        f"ncu --set full capture {k['capture']}: dram read+write / algorithmic = {k['traffic_over_algorithmic']}")


def _start_watchdog(eng, dp, period):
    """Debug aid: dump the engine's state (and every thread's stack) every
    ``period`` seconds to stderr."""
    import collections
    import faulthandler

    def loop():
        while True:
            time.sleep(period)
            st = collections.Counter(s.status for s in eng.state.values())
            print(f"[watchdog] now={eng.now:.3f} steps={len(eng.steps)} live={eng.live} status={dict(st)} "
                  f"gpu={eng._gpu[0] if eng._gpu else None} lanes={[k for k, v in eng._lanes.items() if v]} "
                  f"d2hq={len(eng.d2h.queue)} h2dq={len(eng.h2d.queue)} h2d_head="
                  f"{eng.h2d.queue[0].tokens if eng.h2d.queue else None} mem_used={eng.mem_used} "
                  f"committed={eng.mem_committed} free={eng._mem_free()} heap={len(eng._heap)} "
                  f"heap0={eng._heap[0][:2] if eng._heap else None} skipped={eng.skipped_s:.2f} "
                  f"pre={eng.total_preemptions} prefillq={len(eng.prefill_queue)} "
                  f"gpu_free_blocks={dp.pool.free_count(0)} host_free={dp.pool.free_count(1)} "
                  f"rates d2h={eng.measured_d2h:.0f} h2d={eng.measured_h2d:.0f} tok/s "
                  f"prefill={eng._prefill_s_per_token():.3e} s/tok rc={eng.total_recomputes}",
                  file=sys.stderr, flush=True)
            faulthandler.dump_traceback(file=sys.stderr, all_threads=True)

    threading.Thread(target=loop, daemon=True).start()


def measure_hidden(model, dp, eng, rids, blocks_out, blocks_in, steps=24):
    """Transfer hidden under decode: the real decode step (the
    captured Llama3-8B forward of the live batch) S times alone, the swap
    traffic alone (``blocks_out`` 2 MiB blocks gathered to pinned host on the
    evict stream + ``blocks_in`` scattered from it on the load stream, per
    step, copy engines), and both concurrently.
    hidden = 1 - (T_both - T_decode) / T_swap.  Runs after the timed window on
    free pool / host blocks (no live KV is touched)."""
    import ctypes as C

    import torch

    from paper_2510_02758_b200 import _lib

    pool = dp.pool
    nb = max(blocks_out, blocks_in)
    if nb == 0 or pool.free_count(_lib.TIER_GPU) < nb or pool.free_count(_lib.TIER_HOST) < 2 * nb:
        return None
    g = pool.alloc(_lib.TIER_GPU, nb)
    h = pool.alloc(_lib.TIER_HOST, 2 * nb)
    segs_out = dp._seg_array([(g[i], h[i], 0, 16) for i in range(blocks_out)])
    segs_in = dp._seg_array([(g[i], h[nb + i], 0, 16) for i in range(blocks_in)])
    pos = [eng.state[r].kv.total_kv - 1 for r in rids]
    st = dp.s_compute

    def decode():
        with torch.cuda.stream(st):
            model._decode_graph(dp, rids, pos, st)

    def swaps():
        if blocks_out:
            _lib.check(_lib.lib.tf_kv_gather_d2h(pool.handle, segs_out, blocks_out, 0, pool.L, _lib.ENGINE_CE,
                                                 C.c_void_p(dp.s_evict.cuda_stream)))
        if blocks_in:
            _lib.check(_lib.lib.tf_kv_scatter_h2d(pool.handle, segs_in, blocks_in, 0, pool.L, _lib.ENGINE_CE,
                                                  C.c_void_p(dp.s_load.cuda_stream)))

    def run(fns):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(steps):
            for f in fns:
                f()
        torch.cuda.synchronize()
        return (time.perf_counter() - t0) / steps

    for f in (decode, swaps):  # warm-up
        f()
    # alternate the three measurements over several rounds and take medians:
    # a small swap volume makes the difference T_both - T_decode tiny, so
    # drift between separate runs would otherwise dominate it
    rounds = {"dec": [], "swp": [], "both": []}
    for _ in range(5):
        rounds["dec"].append(run([decode]))
        rounds["both"].append(run([decode, swaps]))
        rounds["swp"].append(run([swaps]))
    t_dec, t_swp, t_both = (statistics.median(rounds[k]) for k in ("dec", "swp", "both"))
    pool.free(_lib.TIER_GPU, g)
    pool.free(_lib.TIER_HOST, h)
    return {"blocks_out_per_step": blocks_out, "blocks_in_per_step": blocks_in, "batch": len(rids),
            "t_decode_ms": round(t_dec * 1e3, 3), "t_swap_ms": round(t_swp * 1e3, 3),
            "t_both_ms": round(t_both * 1e3, 3),
            "swap_gbs": round((blocks_out + blocks_in) * pool.block_bytes / t_swp / 1e9, 2),
            "hidden_frac": round(min(1.0, 1.0 - max(0.0, t_both - t_dec) / t_swp), 4),
            "method": "median of 5 alternating rounds of 24 steps each (decode alone / both / swaps alone)"}


def cpu_baseline(args, timed, quick=False):
    """The oracle's CPU restatement of one decode step of the same batch shape."""
    from oracle.cpu_baseline import time_cpu_step

    b = max(1, int(statistics.median([s["batch"] for s in timed])) if timed else 32)
    return time_cpu_step(batch=b, ctx=2600, threads=os.cpu_count() or 1, seconds=args.cpu_seconds)


def run_reference(args):
    world, rank, _ = _dist()
    if rank != 0:
        return None
    from oracle.cpu_baseline import time_cpu_step

    cb = time_cpu_step(batch=args.ref_batch, ctx=2600, threads=os.cpu_count() or 1, seconds=args.cpu_seconds)
    out = {"metric": METRIC, "value": cb["value"], "unit": cb["unit"], "n_gpus": world, "steps": args.steps,
           "warmup": args.warmup, "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
           "data": "synthetic", "impl": "reference",
           "config": {"workload": "C2: Llama3-8B bf16 random-init, 256-request burst (the same population and "
                                  "metric as the ours arm); the reference's CPU path = the oracle restatement of one "
                                  "decode step of the C2 batch on the host cores (tokensim itself has no tensors)",
                      "model": "llama3-8b", "parallelism": "host CPU"},
           "cpu_baseline": cb, "e2e": {"value": cb["value"], "unit": cb["unit"], "h2d_bytes_per_step": 0,
                                       "d2h_bytes_per_step": 0}}
    print(json.dumps(out))
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    # pinned host tier: 16384 x 2 MiB = 32 GiB covers the timed window; a
    # full run of the burst peaks near 22K blocks (replay of the same trace)
    ap.add_argument("--host-blocks", type=int, default=int(os.environ.get("TF_HOST_BLOCKS", 0)))
    ap.add_argument("--swap-engine", type=int, default=2, help="0 SM kernel, 1 copy engines, 2 auto (whole "
                    "blocks on copy engines, partial blocks on the SM kernel)")
    ap.add_argument("--arrivals", default="burst", choices=["burst", "poisson"])
    ap.add_argument("--config", default="c2", choices=["c2", "c4"], help="c2: Llama3-8B replicas (C2/C3, default); "
                    "c4: Qwen2.5-32B tensor-parallel over the launched ranks")
    ap.add_argument("--graphs", type=int, default=1)
    ap.add_argument("--fused-wt", type=int, default=0, help="1: mirror KV to the host inside the prefill/decode "
                    "epilogue (SURVEY 8f #1) instead of the reference's write-through chunks.  Off by default: it "
                    "makes every preemption an instant full release, which tips the reference policy into "
                    "preempt/recompute churn on the C2 burst (DESIGN.md section 7)")
    ap.add_argument("--full-run", action="store_true")
    ap.add_argument("--ttft", type=int, default=-1, help="after the window keep serving until every request has "
                    "its first token (complete P99 TTFT of the burst); default on for c2, off for c4")
    ap.add_argument("--max-wall", type=float, default=600.0, help="--full-run: stop (truncated) after this many "
                    "seconds of wall time")
    ap.add_argument("--cpu-seconds", type=float, default=20.0)
    ap.add_argument("--ref-batch", type=int, default=64)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--verbose", action="store_true")
    ap.add_argument("--watchdog", type=float, default=0.0, help="debug: dump engine state every N seconds")
    ap.add_argument("--profile-hooks", action="store_true", help="debug: host time per data-plane hook")
    ap.add_argument("--dump-ticks", default=None, help="debug: gzip JSON of the policy's snapshots + decisions")
    ap.add_argument("--dump-window", default="0,1e9", help="debug: virtual-time window of --dump-ticks")
    args = ap.parse_args()
    if args.ttft < 0:
        args.ttft = 1 if args.config == "c2" else 0
    if args.host_blocks <= 0:
        # a full run / the TTFT continuation of the burst peaks near 22K blocks
        args.host_blocks = 26000 if (args.full_run or args.ttft) else 16384
        # never pin more than ~60% of the host's available RAM across the
        # node's ranks (one pinned host tier per GPU replica)
        try:
            avail_kb = next(int(line.split()[1]) for line in open("/proc/meminfo") if line.startswith("MemAvailable"))
            world = max(1, int(os.environ.get("LOCAL_WORLD_SIZE", os.environ.get("WORLD_SIZE", "1"))))
            blk = (4 << 20) // world if args.config == "c4" else (2 << 20)  # pinned bytes per host block
            cap = int(avail_kb * 1024 * 0.6 / world / blk)
            args.host_blocks = max(1024, min(args.host_blocks, cap))
        except (OSError, StopIteration, ValueError):
            pass
    if args.warmup < 3:
        raise SystemExit("--warmup must be >= 3")
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
