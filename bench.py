"""Benchmark: effective tok/s (+ P99 TTFT, KV swap GB/s) of the B200 TokenFlow
hot path on C2 (Llama3-8B bf16 random-init, the 256-request C2 population
arriving as a burst at t=0, KV swap to pinned host), 1 GPU per process.

python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                [--config c2|c4] [--arrivals burst|poisson] [--full-run]

A *step* is one schedule interval of the real-time serving loop
(realtime.RealtimeEngine; 0.5 s of serving clock, `--step-unit tick`, the
default): one selector tick (the GPU selector's member view and decisions)
and everything the engine runs until the next one - the decode iterations
(Llama3-8B forward from a captured CUDA graph: fused RMSNorm / rope+append /
paged attention / SwiGLU around cuBLAS GEMMs), the prefills / recomputes the
tick admitted, and the write-through / evict / load chunks on the two
high-priority copy streams.  W warm-up intervals from t=0, then EXACTLY K
timed intervals (default K=20, W=5: serving clock [2.5, 12.5) s of the burst,
the admission / preemption / swap phase).  `--step-unit iter` times decode
iterations instead (the round-1 definition): a 20-iteration window from t=0
sits on the burst's first rotation tick (t = 2.0 s, 53 preemptions + 53
admissions) on some boxes and not on others, so its value is bimodal
(~22.5K vs ~3K, profiles/r2_bench20_windows.json).

value  = effective tokens (tokensim.metrics weights, tau1/tau2 = 10%/20% of
         the output length) generated in the K steps / device time of every
         GPU job (decode iterations and the prefills between them) in the window
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
    from paper_2510_02758_b200 import model as model_mod
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
            if args.tp_data == "peer" and not one_gpu:
                # (the one-GPU dry run keeps the gloo data path: its ranks are
                # processes time-slicing one device, so a peer barrier would wait
                # a scheduling slice per all-reduce; tests/test_ar_gpu.py covers
                # the peer kernel across processes on one GPU)
                # data path: each rank's o_proj / down_proj partial goes into its
                # registered buffer, one kernel reads the peers' over NVLink and
                # fuses residual + RMSNorm (csrc/tf_ar.cu); handles over gloo
                from paper_2510_02758_b200.tp import PeerAllReduce

                tp.ar = PeerAllReduce.from_group(rank, world, 8192 * configs.c4(world).model.hidden * 2,
                                                 group=lockstep.group, device=dev)
        c2 = configs.c4(world)
        tr = _trace_for_rank(0, 1, args.arrivals)
        if world > 1 and args.graphs and one_gpu:
            # the one-GPU dry run shares one device between the ranks' processes
            # (time-sliced contexts): run it eager.  On a real C4 run the decode
            # forward WITH its all-reduces (peer kernel or NCCL) is captured per
            # bucket like the TP=1 one
            args.graphs = 0
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
        if tp is not None and getattr(tp, "ar", None) is not None:
            # the capture warm-up runs the peer all-reduce eagerly: start it together
            import torch.distributed as dist

            dist.barrier(group=lockstep.group)
        model.enable_graphs(dp)
    if args.policy == "fcfs":  # the paper's comparison baseline on the same data plane
        from paper_2510_02758_b200.scheduler import FcfsPolicy

        policy = FcfsPolicy(c2.sched_cfg(SchedulerConfig))
    else:
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
    tick_s = policy.cfg.schedule_interval
    t_warm, t_end = args.warmup * tick_s, (args.warmup + args.steps) * tick_s  # --step-unit tick

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
        plan = "graph" if args.graphs else "exact"
        per = model.measure_attention(dp, live, [eng.state[r].kv.total_kv - 1 for r in live], plan=plan,
                                      graph_reps=5)
        ev_ms = sum(ms for _, ms in per) / len(per)
        avg_bytes = sum(b for b, _ in per) / len(per)
        # headline: the launches as the decode graphs run them (all layers back
        # to back inside one CUDA graph, one event pair around 5 replays);
        # beside it the same launches each bracketed by its own event pair
        avg_ms = model.attn_graph_ms or ev_ms
        ach = avg_bytes / (avg_ms / 1e3) / 1e9
        traffic, tsrc = _ncu_traffic(avg_bytes)
        state["roof"] = {"bound": "hbm", "kernel": _attn_kernel_name(shape, len(live), bool(args.graphs)),
                         "achieved": round(ach, 1), "peak": hbm, "peak_kind": peak_kind, "unit": "GB/s",
                         "frac": round(ach / hbm, 4), "traffic": traffic, "traffic_source": tsrc,
                         "launches": len(per), "avg_ms": round(avg_ms, 4), "batch": len(live), "plan": plan,
                         "timing": "CUDA graph of the 32 layers' launches, 5 replays, one event pair",
                         "avg_ms_per_launch_events": round(ev_ms, 4),
                         "frac_per_launch_events": round(avg_bytes / (ev_ms / 1e3) / 1e9 / hbm, 4),
                         "algorithmic_bytes_per_launch": round(avg_bytes),
                         "note": f"bytes = sum(ctx) x {pool.H * pool.D * 4} B (K+V, {pool.H} kv heads x {pool.D} x "
                                 "bf16) + q/out + table entries per layer (real rows only); re-launched right after "
                                 "the window on the running batch with the plan the decode graphs replay (batch "
                                 "padded to its bucket with scratch rows, max_ctx = the pool maximum)"}
        if args.graphs:
            hid_m = measure_hidden_mix(model, dp, eng, live, state["ev0"], state["ev1"], len(timed),
                                       args.swap_engine)
            # blocks per direction that keep the duplex link (~45 GB/s each way
            # when both run) busy for ~80% of one decode step: the transfer CAN
            # then be hidden completely, so the fraction measures overlap quality
            t_dec = hid_m["t_decode_ms"] if hid_m else 7.0
            sat = max(1, int(0.8 * 45e9 * t_dec / 1e3 / dp.pool.block_bytes))
            hid_s = measure_hidden(model, dp, eng, live, sat, sat)
            state["hidden"] = {"window_mix": hid_m, "link_saturating": hid_s,
                               "note": "hidden = 1 - (T_both - T_decode)/T_swap; decode = the captured forward of "
                                       "the live batch; window_mix replays the window's own chunks (segment shapes, "
                                       "engine, order) scaled to ~50% of a decode step; link_saturating moves whole "
                                       "blocks both ways sized to ~80% of a decode step (the window's own volume, "
                                       "~0.1-0.3 ms of copies per step, is below the step-to-step noise of "
                                       "T_decode)"}
        if not args.no_selector:
            sys.path.insert(0, str(ROOT / "tools"))
            from selector_latency import gpu_selector_latency

            state["selector_gpu"] = gpu_selector_latency()

    def on_step(rec, eng):
        n = len(eng.steps)
        if args.verbose and n % 100 == 0:
            print(f"[bench] step {n} t={eng.now:.2f}s batch={rec['batch']} dur={rec['dur'] * 1e3:.2f}ms "
                  f"pre={eng.total_preemptions} rc={eng.total_recomputes} running={len(eng.running)} "
                  f"waiting={len(eng.waiting)} d2h={dp.stats['d2h_tokens']} h2d={dp.stats['h2d_tokens']} "
                  f"wall={time.perf_counter() - t_start:.1f}s", file=sys.stderr, flush=True)
        if state["phase"] == "warm":
            # iter: W decode iterations from t=0; tick: the decode iteration
            # that reaches the W-th schedule tick (t = W x interval) closes the
            # warm-up, so the timed steps start at the tick
            if (n >= args.warmup) if args.step_unit == "iter" else (rec["end"] >= t_warm):
                state["phase"] = "timed"
                state["wall0"] = time.perf_counter()
                state["ev0"] = len(dp._events)
                state["pre0"], state["rc0"] = eng.total_preemptions, eng.total_recomputes
                state["launch0"] = model.launch_count()
                torch.cuda.nvtx.range_push("bench_timed")  # ncu --nvtx --nvtx-include bench_timed/
            return
        if state["phase"] == "timed":
            state["timed"].append(dict(rec))
            if (len(state["timed"]) >= args.steps) if args.step_unit == "iter" else (rec["end"] >= t_end):
                state["wall1"] = time.perf_counter()
                state["ev1"] = len(dp._events)
                state["pre1"], state["rc1"] = eng.total_preemptions, eng.total_recomputes
                state["launch1"] = model.launch_count()
                state["phase"] = "done"
                state["h2d_launch_at_end"] = dp.stats["h2d_launches"]
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
        if state["phase"] in ("ttft", "rest") and args.swap_steps > 0:
            # swap-phase sub-window: the next --swap-steps decode steps after the
            # first load (h2d chunk) issued once the main window ended - so even
            # a short main window from t=0 (decode + write-through only) comes
            # with measured evict / load traffic from the same run
            sw = state.setdefault("sw", {"phase": "wait"})
            if sw["phase"] == "wait" and dp.stats["h2d_launches"] > state["h2d_launch_at_end"]:
                sw.update(phase="on", ev0=len(dp._events), pre0=eng.total_preemptions, rc0=eng.total_recomputes,
                          steps=[], wall0=time.perf_counter())
            elif sw["phase"] == "on":
                sw["steps"].append(dict(rec))
                if len(sw["steps"]) >= args.swap_steps:
                    sw.update(phase="done", ev1=len(dp._events), pre1=eng.total_preemptions,
                              rc1=eng.total_recomputes, wall1=time.perf_counter())
                    if args.graphs:
                        t_p = time.perf_counter()
                        torch.cuda.synchronize()
                        live = sorted(r for r in eng.running if eng.state[r].status == "running")[: c2.max_batch]
                        if live:
                            sw["hidden"] = measure_hidden_mix(model, dp, eng, live, sw["ev0"], sw["ev1"],
                                                              len(sw["steps"]), args.swap_engine)
                        eng.shift_clock(time.perf_counter() - t_p)
        if state["phase"] == "ttft" and all(st.record.gen_times for st in eng.state.values()):
            sw = state.get("sw", {"phase": "done"})
            if sw["phase"] == "done" or args.swap_steps <= 0 or (sw["phase"] == "wait" and not eng.h2d.queue):
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
    if tp is not None and getattr(tp, "ar", None) is not None and tp.ar.status() != 0:
        raise RuntimeError("peer all-reduce: a barrier wait timed out (a rank fell > 10 s behind)")
    if state["phase"] not in ("done", "ttft", "rest"):
        raise RuntimeError(f"bench ended in phase {state['phase']} after {len(eng.steps)} steps")
    timed = state["timed"]
    n_steps = len(timed) if args.step_unit == "iter" else args.steps
    bpt = shape.kv_bytes_per_token // tp_size  # swap bytes per token: all layers' K and V of this rank's shard
    local = _window_stats(eng, dp, timed, state["ev0"], state["ev1"], bpt)
    local.update(ttft_lat=[r.gen_times[0] - r.arrival for r in res.records if r.gen_times],
                 n_records=len(res.records), preemptions=state["pre1"] - state["pre0"],
                 recomputes=state["rc1"] - state["rc0"], wall=state["wall1"] - state["wall0"])
    red_dev = torch.device("cpu") if (world > 1 and one_gpu) else dev
    agg = _aggregate(local, world, tp_mode, red_dev)
    sw = state.get("sw")
    sw_out = None
    if sw and sw.get("steps"):
        sl = _window_stats(eng, dp, sw["steps"], sw["ev0"], sw.get("ev1", len(dp._events)), bpt)
        sl.update(ttft_lat=[], n_records=0, preemptions=sw.get("pre1", eng.total_preemptions) - sw["pre0"],
                  recomputes=sw.get("rc1", eng.total_recomputes) - sw["rc0"],
                  wall=sw.get("wall1", time.perf_counter()) - sw["wall0"])
        sa = _aggregate(sl, 1, tp_mode, red_dev)  # rank-local (each replica's own window)
        sw_out = {"steps": len(sw["steps"]), "complete": sw["phase"] == "done",
                  "value": sa["value"], "e2e_value": sa["e2e"], "swap": _swap_block(sa, args.swap_engine),
                  "preemptions": sl["preemptions"], "recomputes": sl["recomputes"],
                  "hidden_under_decode": sw.get("hidden"),
                  "note": f"the {args.swap_steps} decode steps after the first load (h2d chunk) issued once the main "
                          "window ended (rank 0's replica); value = effective tokens / device time, e2e = / host wall"}
    swap = _swap_block(agg, args.swap_engine)
    swap.update(preemptions=local["preemptions"], recomputes=local["recomputes"])
    if state.get("hidden"):
        swap["hidden_under_decode"] = state["hidden"]
    out = {
        "metric": METRIC,
        "value": agg["value"],
        "unit": "effective tok/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "step_unit": "schedule interval" if args.step_unit == "tick" else "decode iteration",
        "ms_per_step": agg["dev_s"] / n_steps * 1e3,
        "decode_iterations": len(timed),
        "decode_ms_per_iter": sum(st_["dur"] for st_ in timed) / len(timed) * 1e3,
        "prefill_device_s_in_window": round(local["prefill_s"], 4),
        "higher_is_better": True,
        "scaling": "strong" if tp_mode else "weak",
        "vs_baseline": None,
        "dtype": "bf16",
        "data": f"synthetic (random-init {shape.name} weights, seeded prompt token ids, frozen C2 trace)",
        "config": {"workload": (f"C4: Qwen2.5-32B bf16 random-init, tensor-parallel TP={world} ("
                                + ("peer-memory all-reduce fused with residual + RMSNorm" if args.tp_data == "peer"
                                   else "NCCL all-reduce") +
                                f" after o_proj / down_proj), 256-request {args.arrivals} (C2 population), KV ledger "
                                "163,840 tokens (40 GiB over the TP ranks) + pinned host tier per rank, block 16, "
                                "max_batch 128") if tp_mode else
                               (f"C2: Llama3-8B bf16 random-init, 1xB200 per replica, 256-request {args.arrivals} "
                                "(bodies of the first 256 arrivals of the lambda=10/s 30 s trace, seed 1), KV pool "
                                "163,840 tokens (20 GiB) + pinned host tier, block 16, max_batch 128"),
                   "model": shape.name, "global_batch": max(st_["batch"] for st_ in timed),
                   "mean_batch": round(statistics.mean(st_["batch"] for st_ in timed), 1),
                   "seq_len": None, "parallelism": f"tp{world}" if tp_mode else f"replicas x{world}",
                   "policy": policy.name, "arrivals": args.arrivals,
                   "l2": "working set (weights + KV, tens of GB) >> 126 MB L2; no flush needed",
                   "timed_region": (f"decode iterations [{args.warmup}, {args.warmup + args.steps}) from t=0 "
                                    "of the real-time loop (measured clock, idle gaps skipped)")
                   if args.step_unit == "iter" else
                   (f"schedule intervals [{args.warmup}, {args.warmup + args.steps}) of {tick_s:g} s from t=0 of "
                    f"the real-time loop = serving clock [{t_warm:g}, {t_end:g}) s (measured clock, idle gaps "
                    "skipped): every tick, decode iteration, prefill / recompute and swap chunk in between"),
                   "cuda_graphs": bool(args.graphs),
                   "prompt_graphs": bool(args.graphs) and model_mod._PROMPT_GRAPHS, "fused_write_through": bool(args.fused_wt)},
        "raw_tok_s": agg["raw"],
        "e2e": {"value": agg["e2e"], "unit": "effective tok/s",
                "h2d_bytes_per_step": int((agg["h2d_tok"] * bpt + local["batch_sum"] * 24) / n_steps),
                "d2h_bytes_per_step": int((agg["d2h_tok"] * bpt + local["batch_sum"] * 8) / n_steps)},
        "swap": swap,
        "swap_window": sw_out,
        "roofline": state.get("roof"),
        "clocks": sampler.summary(),
        "gpu_launches": int(state["launch1"] - state["launch0"]),
        "first_tokens_in_window": len(local["ttft_lat"]),
        "window_clock": _window_clock(eng, timed),
        "ttft": agg["ttft"],
    }
    # gpu_launches: this library's kernel launches inside the window, counted:
    # every C-ABI launch increments a counter in the .so, and each graph replay
    # adds the number of the library's kernels captured in that graph
    if state.get("selector_gpu"):
        out["selector"] = {"gpu": state["selector_gpu"],
                           "note": "us per call at N members: e2e = host wall (pack, H2D, one single-CTA launch, "
                                   "D2H, unpack), device = CUDA events around the call on the selector's stream; "
                                   "launch_floor = an empty kernel (tf_launch_floor); the CPU reference (oracle "
                                   "restatement of tokensim on_tick / select_batch, 1 core) is in cpu_baseline"}
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
        if out.get("selector") and out["cpu_baseline"].get("selector_cpu"):
            out["selector"]["cpu_oracle_1core"] = out["cpu_baseline"]["selector_cpu"]
    if rank == 0:
        print(json.dumps(out))
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()
    return out


def _window_clock(eng, steps):
    """Where the window sits on the serving clock: its first / last decode
    iteration, the run's first decode iteration, and the schedule ticks from
    t=0 to one interval past the window (how many fired; the ones that moved
    requests, with their preempt / admit / resume counts) - a window that
    holds a rotation tick's preemptions and readmission prefills shows it."""
    t_lo, t_hi = steps[0]["start"], steps[-1]["end"]
    fired, moved = 0, []
    for e in eng.decision_log:
        if e["time"] > t_hi + eng.policy.cfg.schedule_interval:
            break
        fired += 1
        n = {k: len(e.get(k) or ()) for k in ("preempted", "admitted", "resumed", "recomputed")}
        if any(n.values()):
            moved.append({"t": round(e["time"], 4), "mode": e.get("mode"), **n})
    return {"start_s": round(t_lo, 4), "end_s": round(t_hi, 4),
            "first_decode_s": round(eng.steps[0]["start"], 4) if eng.steps else None,
            "schedule_interval_s": eng.policy.cfg.schedule_interval, "ticks_fired": fired,
            "ticks_that_moved_requests": moved[:40]}


def _window_stats(eng, dp, steps, ev0, ev1, bpt):
    """This rank's numbers for a window of decode steps: device time of every
    GPU job inside it (decode iterations and the prefills between them),
    effective / raw tokens, and the window's swap chunks (tokens, CUDA-event ms)."""
    t_lo, t_hi = steps[0]["start"], steps[-1]["end"]
    win_jobs = [j for j in eng.jobs if t_lo <= j[1] and j[2] <= t_hi]
    xf = dp.transfer_log()[ev0:ev1]
    return {"dev_s": sum(j[3] for j in win_jobs), "prefill_s": sum(j[3] for j in win_jobs if j[0] == "prefill"),
            "eff": sum(st_["effective"] for st_ in steps), "toks": sum(st_["tokens"] for st_ in steps),
            "batch_sum": sum(st_["batch"] for st_ in steps),
            "d2h_tok": sum(n for k, n, _ in xf if k == "d2h"), "h2d_tok": sum(n for k, n, _ in xf if k == "h2d"),
            "d2h_ms": sum(ms for k, _, ms in xf if k == "d2h"), "h2d_ms": sum(ms for k, _, ms in xf if k == "h2d"),
            "chunks": len(xf), "bpt": bpt}


def _aggregate(local, world, tp_mode, device):
    """Whole-job numbers from every rank's window stats.  Replicas (C2/C3):
    tokens and swap traffic are summed (each replica serves its own requests
    over its own link), device time and wall time are the max over ranks, and
    TTFT latencies are gathered from every rank.  Tensor parallel (C4): every
    rank serves the same tokens in lockstep, so rank 0's counts stand and the
    times are still the max over ranks."""
    dev_s = _max_over_ranks(local["dev_s"], world, device)
    wall = _max_over_ranks(local["wall"], world, device)
    eff, toks = local["eff"], local["toks"]
    d2h_tok, h2d_tok, d2h_ms, h2d_ms = local["d2h_tok"], local["h2d_tok"], local["d2h_ms"], local["h2d_ms"]
    if not tp_mode:
        eff, toks = _sum_over_ranks(eff, world, device), _sum_over_ranks(toks, world, device)
        if world > 1:
            d2h_tok, h2d_tok = int(_sum_over_ranks(d2h_tok, world, device)), int(_sum_over_ranks(h2d_tok, world, device))
            d2h_ms, h2d_ms = _sum_over_ranks(d2h_ms, world, device), _sum_over_ranks(h2d_ms, world, device)
    bpt = local["bpt"]
    return {"dev_s": dev_s, "wall": wall, "eff": eff, "toks": toks,
            "value": eff / dev_s if dev_s > 0 else None, "raw": toks / dev_s if dev_s > 0 else None,
            "e2e": eff / wall if wall > 0 else None,
            "d2h_tok": d2h_tok, "h2d_tok": h2d_tok, "chunks": local["chunks"],
            "d2h_gbs": (d2h_tok * bpt / (d2h_ms / 1e3) / 1e9) if d2h_ms else None,
            "h2d_gbs": (h2d_tok * bpt / (h2d_ms / 1e3) / 1e9) if h2d_ms else None,
            "ttft": _ttft_summary_lat(local["ttft_lat"], local["n_records"], world, tp_mode)}


def _swap_block(agg, engine):
    sw = {"d2h_tokens": agg["d2h_tok"], "h2d_tokens": agg["h2d_tok"], "chunks": agg["chunks"],
          "engine": "SM kernel" if engine == 0 else
                    "copy engines (whole blocks as merged 1-D runs, partial blocks as 2-D copies, two copy queues)",
          "d2h_gbs": agg["d2h_gbs"], "h2d_gbs": agg["h2d_gbs"], "pcie_gen5_gbs": PCIE_GEN5_GBS}
    for k in ("d2h", "h2d"):
        if sw[f"{k}_gbs"]:
            sw[f"{k}_frac_pcie"] = sw[f"{k}_gbs"] / PCIE_GEN5_GBS
    return sw


def _attn_kernel_name(shape, batch, graphs):
    """The decode-attention implementation the library picks for this launch
    (tf_paged_decode_attn_impl default: v3 at every batch)."""
    G = shape.n_q_heads // shape.n_kv_heads
    env = os.environ.get("TF_ATTN_IMPL", "")[:1]
    impl = int(env) if env in ("1", "2", "3", "4", "5") else 0
    if impl == 0:
        impl = 3
    return {1: "paged_attn_kernel (v1, CUDA cores)", 2: "paged_attn_tma_kernel (v2, bulk copy)",
            3: f"paged_attn_mma_kernel<{G}> (v3, split-KV cp.async + mma.sync, in-kernel split merge)",
            4: f"paged_attn_stream_kernel<{G}> (v4 stream-K)",
            5: f"paged_attn_tma5_kernel<{G}> (v5, TMA tensor loads + stream-K)"}[impl]


def _ttft_summary_lat(lat, n_records, world, tp_mode):
    """TTFT latency stats (first token - arrival, nearest-rank P99,
    tokensim/metrics.py:144-155) over ALL replicas' requests (C3: gathered)."""
    from paper_2510_02758_b200.metrics import nearest_rank

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


def _ttft_summary(recs, n_records, world, tp_mode):
    return _ttft_summary_lat([r.gen_times[0] - r.arrival for r in recs], n_records, world, tp_mode)


def _ncu_traffic(alg_bytes):
    """DRAM bytes per launch for the attention kernel: the DRAM-traffic /
    algorithmic-bytes ratio of the committed ncu --set full capture of the
    same kernel (profiles/r2_attn_ncu_live.json, r1_attn_ncu_v3_v4.json) at the closest launch size,
    applied to this launch's algorithmic bytes."""
    impl = os.environ.get("TF_ATTN_IMPL", "3")[:1]
    want = "stream" if impl == "4" else "mma"
    caps = []
    for name in ("r2_attn_ncu_live.json", "r1_attn_ncu_v3_v4.json"):
        try:
            caps += [k for k in json.loads((ROOT / "profiles" / name).read_text())["kernels"] if want in k["kernel"]]
        except (OSError, ValueError, KeyError):
            pass
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


def measure_hidden(model, dp, eng, rids, blocks_out, blocks_in, steps=48, rounds=7):
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
    samples = {"dec": [], "swp": [], "both": []}
    for _ in range(rounds):
        samples["dec"].append(run([decode]))
        samples["both"].append(run([decode, swaps]))
        samples["swp"].append(run([swaps]))
    t_dec, t_swp, t_both = (statistics.median(samples[k]) for k in ("dec", "swp", "both"))
    pool.free(_lib.TIER_GPU, g)
    pool.free(_lib.TIER_HOST, h)
    return {"blocks_out_per_step": blocks_out, "blocks_in_per_step": blocks_in, "batch": len(rids),
            "t_decode_ms": round(t_dec * 1e3, 3), "t_swap_ms": round(t_swp * 1e3, 3),
            "t_both_ms": round(t_both * 1e3, 3),
            "swap_gbs": round((blocks_out + blocks_in) * pool.block_bytes / t_swp / 1e9, 2),
            "hidden_frac": round(min(1.0, 1.0 - max(0.0, t_both - t_dec) / t_swp), 4),
            "method": f"median of {rounds} alternating rounds of {steps} steps each (decode alone / both / swaps "
                      "alone)"}


def measure_hidden_mix(model, dp, eng, rids, ev0, ev1, nsteps, engine, steps=48, rounds=7):
    """Transfer hidden under decode for the window's OWN swap mix: the chunks
    the engine issued in the window (their segment shapes, one call per chunk,
    the serving engine), spread at the window's per-step density over
    ``steps`` decode steps of the captured forward of the live batch, alone /
    with the swaps / swaps alone.  Scratch blocks stand in for the live ones
    (same shapes, no live KV touched)."""
    import ctypes as C

    import torch

    from paper_2510_02758_b200 import _lib

    chunks = [(dp._events[i][0], dp._seglog[i]) for i in range(ev0, min(ev1, len(dp._seglog)))]
    if not chunks or nsteps <= 0:
        return None
    per_step = len(chunks) / nsteps
    take = chunks[: max(1, round(per_step * steps))]
    nseg = max(len(sg) for _, sg in take)
    pool = dp.pool
    k = min(64, nseg * 4)
    if pool.free_count(_lib.TIER_GPU) < k or pool.free_count(_lib.TIER_HOST) < k:
        return None
    g = pool.alloc(_lib.TIER_GPU, k)
    h = pool.alloc(_lib.TIER_HOST, k)
    calls, j = [[] for _ in range(steps)], 0
    for i, (kind, sg) in enumerate(take):
        arr = dp._seg_array([(g[(j + t) % k], h[(j + t) % k], s0, n) for t, (s0, n) in enumerate(sg)])
        j += len(sg)
        calls[min(steps - 1, int(i / per_step))].append((kind, arr, len(sg)))
    pos = [eng.state[r].kv.total_kv - 1 for r in rids]
    st = dp.s_compute

    def decode():
        with torch.cuda.stream(st):
            model._decode_graph(dp, rids, pos, st)

    scale = {"x": 1}

    def swaps(si):
        for _ in range(scale["x"]):
            for kind, arr, n in calls[si]:
                fn = _lib.lib.tf_kv_gather_d2h if kind == "d2h" else _lib.lib.tf_kv_scatter_h2d
                stream = dp.s_evict if kind == "d2h" else dp.s_load
                _lib.check(fn(pool.handle, arr, n, 0, pool.L, engine, C.c_void_p(stream.cuda_stream)))

    def run(dec, swp):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for si in range(steps):
            if dec:
                decode()
            if swp:
                swaps(si)
        torch.cuda.synchronize()
        return (time.perf_counter() - t0) / steps

    decode()
    swaps(0)
    # The window's own density is ~0.1-0.3 ms of copies per ~6 ms step - the
    # size of the step-to-step noise of T_decode, which would dominate
    # T_both - T_decode.  The same chunk mix (shapes, engine, order) is
    # therefore replayed `scale` times per step, scaled to ~50% of the decode
    # step (still fully hideable); the unscaled density is reported beside it.
    base_swp, base_dec = run(False, True), run(True, False)
    scale["x"] = max(1, min(64, round(0.5 * base_dec / max(base_swp, 1e-6))))
    samples = {"dec": [], "swp": [], "both": []}
    for _ in range(rounds):
        samples["dec"].append(run(True, False))
        samples["both"].append(run(True, True))
        samples["swp"].append(run(False, True))
    t_dec, t_swp, t_both = (statistics.median(samples[x]) for x in ("dec", "swp", "both"))
    pool.free(_lib.TIER_GPU, g)
    pool.free(_lib.TIER_HOST, h)
    toks = sum(n for _, sg in take for _, n in sg)
    return {"chunks_per_step": round(per_step, 2), "tokens_per_step": round(toks / steps, 1), "batch": len(rids),
            "replay_scale": scale["x"], "t_swap_unscaled_ms": round(base_swp * 1e3, 3),
            "t_decode_ms": round(t_dec * 1e3, 3), "t_swap_ms": round(t_swp * 1e3, 3),
            "t_both_ms": round(t_both * 1e3, 3),
            "hidden_frac": round(min(1.0, 1.0 - max(0.0, t_both - t_dec) / t_swp), 4) if t_swp > 0 else None,
            "method": f"the window's chunks (segment shapes, engine, order) replayed at replay_scale x its per-step "
                      f"density (~50% of a decode step); median of {rounds} alternating rounds of {steps} steps "
                      "(decode alone / both / swaps alone)"}


def cpu_baseline(args, timed, quick=False):
    """CPU baseline (reported beside the GPU numbers),
    all of it the oracle's restatement of the reference on the host:
    one C2 decode step of the window's median batch (all host cores), the
    reference simulator on the same C2 burst (1 core, per-call on_tick /
    plan_write_chunk / _snapshot), the policy's on_tick / select_batch at the
    selector's N, and the host's CPU model / NUMA layout."""
    from oracle.cpu_baseline import host_info, time_cpu_gather, time_cpu_step, time_reference_sim

    b = max(1, int(statistics.median([s["batch"] for s in timed])) if timed else 128)
    out = time_cpu_step(batch=b, ctx=2600, threads=os.cpu_count() or 1, seconds=args.cpu_seconds)
    out["reference_sim"] = time_reference_sim("c2_burst256_s1_tokenflow")
    out["host"] = host_info()
    out["kv_gather_cpu"] = time_cpu_gather(threads=os.cpu_count() or 1)
    if not args.no_selector:
        sys.path.insert(0, str(ROOT / "tools"))
        from selector_latency import cpu_selector_latency

        out["selector_cpu"] = cpu_selector_latency()
    return out


def run_reference(args):
    world, rank, _ = _dist()
    if rank != 0:
        return None
    from oracle.cpu_baseline import host_info, time_cpu_gather, time_cpu_step, time_reference_sim

    cb = time_cpu_step(batch=args.ref_batch, ctx=2600, threads=os.cpu_count() or 1, seconds=args.cpu_seconds)
    cb["reference_sim"] = time_reference_sim("c2_burst256_s1_tokenflow")
    cb["host"] = host_info()
    out = {"metric": METRIC, "value": cb["value"], "unit": cb["unit"], "n_gpus": max(world, args.gpus),
           "steps": args.steps, "warmup": args.warmup, "higher_is_better": True, "scaling": "weak",
           "vs_baseline": None, "dtype": "bf16", "data": "synthetic", "impl": "reference",
           "config": {"workload": "C2: Llama3-8B bf16 random-init, 256-request burst (the same population and "
                                  "metric as the ours arm); the reference's CPU path = the oracle restatement of one "
                                  f"decode step at B={args.ref_batch} (the median decode batch of the ours arm's "
                                  "default window, 20 schedule intervals of the burst) on the host cores (tokensim "
                                  "itself has no tensors)",
                      "model": "llama3-8b", "parallelism": "host CPU", "global_batch": args.ref_batch},
           "cpu_baseline": cb, "e2e": {"value": cb["value"], "unit": cb["unit"], "h2d_bytes_per_step": 0,
                                       "d2h_bytes_per_step": 0}}
    print(json.dumps(out))
    return out


def run_dry(args):
    """--dry-run: the multi-rank plumbing without a GPU (gloo on the CPU):
    every rank fabricates deterministic window stats, and the SAME aggregation
    and reporting path as a real run turns them into the line (CPU tests of
    --gpus N self-launch and the C3 aggregation)."""
    import torch

    world, rank, _ = _dist()
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("gloo")
    tp_mode = args.config == "c4"
    local = {"dev_s": 1.0 + 0.25 * rank, "prefill_s": 0.0, "eff": 100.0 * (rank + 1), "toks": 120.0 * (rank + 1),
             "batch_sum": 10, "d2h_tok": 1000 * (rank + 1), "h2d_tok": 500, "d2h_ms": 10.0, "h2d_ms": 5.0,
             "chunks": 7, "bpt": 131072, "ttft_lat": [float(rank) + i / 10 for i in range(10)], "n_records": 10,
             "wall": 2.0 + rank}
    agg = _aggregate(local, world, tp_mode, torch.device("cpu"))
    out = {"metric": METRIC, "value": agg["value"], "unit": "effective tok/s", "n_gpus": world,
           "steps": args.steps, "warmup": args.warmup, "higher_is_better": True,
           "scaling": "strong" if tp_mode else "weak", "data": "dry-run (no GPU work; fabricated per-rank stats)",
           "config": {"parallelism": f"tp{world}" if tp_mode else f"replicas x{world}"},
           "e2e": {"value": agg["e2e"]}, "swap": _swap_block(agg, args.swap_engine), "ttft": agg["ttft"]}
    if rank == 0:
        print(json.dumps(out))
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()
    return out


def _free_port() -> int:
    import socket

    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def _self_launch(args) -> bool:
    """``--gpus N`` without a launcher: re-run this script under
    torch.distributed.run with one rank per GPU (127.0.0.1 rendezvous); rank 0
    prints the single aggregated line.  Under torchrun (WORLD_SIZE set) the
    ranks are already there."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ or args.impl == "reference":
        return False
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", str(Path(__file__).resolve()), *sys.argv[1:]]
    rc = subprocess.call(cmd)
    raise SystemExit(rc)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--step-unit", default="tick", choices=["tick", "iter"],
                    help="tick (default): a step is one schedule interval of the serving loop (0.5 s of serving "
                         "clock: one selector tick and every decode iteration, prefill and swap chunk until the "
                         "next); iter: one decode iteration (round-1 definition)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    # pinned host tier: 16384 x 2 MiB = 32 GiB covers the timed window; a
    # full run of the burst peaks near 22K blocks (replay of the same trace)
    ap.add_argument("--host-blocks", type=int, default=int(os.environ.get("TF_HOST_BLOCKS", 0)))
    ap.add_argument("--swap-engine", type=int, default=2, help="0 SM kernel; 1, 2 or 3 copy engines (whole blocks as "
                    "merged 1-D runs, each partial block one 2-D copy, alternated over two copy queues)")
    ap.add_argument("--arrivals", default="burst", choices=["burst", "poisson"])
    ap.add_argument("--config", default="c2", choices=["c2", "c4"], help="c2: Llama3-8B replicas (C2/C3, default); "
                    "c4: Qwen2.5-32B tensor-parallel over the launched ranks")
    ap.add_argument("--graphs", type=int, default=1)
    ap.add_argument("--tp-data", default="peer", choices=["peer", "nccl"],
                    help="c4 data path: peer-memory all-reduce fused with residual + RMSNorm (default) or NCCL")
    ap.add_argument("--fused-wt", type=int, default=0, help="1: mirror KV to the host inside the prefill/decode "
                    "epilogue (SURVEY 8f #1) instead of the reference's write-through chunks.  Off by default: it "
                    "makes every preemption an instant full release, which tips the reference policy into "
                    "preempt/recompute churn on the C2 burst (DESIGN.md section 7)")
    ap.add_argument("--full-run", action="store_true")
    ap.add_argument("--ttft", type=int, default=-1, help="after the window keep serving until every request has "
                    "its first token (complete P99 TTFT of the burst); default on for c2, off for c4")
    ap.add_argument("--max-wall", type=float, default=600.0, help="--full-run: stop (truncated) after this many "
                    "seconds of wall time")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--ref-batch", type=int, default=80, help="reference arm: the decode batch of the timed "
                    "window (median 78-81 over the default 20 schedule intervals of the C2 burst)")
    ap.add_argument("--policy", default="tokenflow", choices=["tokenflow", "fcfs"], help="fcfs: the paper's "
                    "comparison baseline (tokensim/scheduler.py:828-880) on the same B200 data plane")
    ap.add_argument("--swap-steps", type=int, default=200, help="swap-phase sub-window: decode steps after the first "
                    "load issued once the main window ended (0: off)")
    ap.add_argument("--no-selector", action="store_true", help="skip the selector latency block")
    ap.add_argument("--dry-run", action="store_true", help="multi-rank plumbing only (no GPU work; CPU tests)")
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
    _self_launch(args)
    if args.dry_run:
        run_dry(args)
    elif args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
