"""Benchmark: effective tok/s (+ P99 TTFT, KV swap GB/s) of the B200 TokenFlow
hot path on C2 (Llama3-8B bf16 random-init, 256-request Poisson trace with
KV swap to pinned host), 1 GPU per process.

python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--full-run]

A *step* is one decode iteration of the real-time serving loop
(realtime.RealtimeEngine) in its contended regime: the GPU selector's
pacing/tick decisions, the Llama3-8B forward with paged KV append + paged
decode attention for the batch, and the write-through / evict / load chunks
the engine issues meanwhile on the two copy streams.  The loop first runs
untimed from t=0 until requests are being preempted and swapped (contention),
then W warm-up steps, then EXACTLY K timed steps.

value  = effective tokens (tokensim.metrics weights, tau1/tau2 = 10%/20% of
         the output length) generated in the K steps / device time of those
         K decode iterations (CUDA events on the compute stream), max over
         ranks; inputs (weights, KV) already resident in HBM.
e2e    = the same tokens / host wall-clock span of the K steps through the
         public API (engine loop), which includes every step's H2D (token
         ids, positions, block-table deltas, load chunks) and D2H (sampled
         token ids, evict / write-through chunks).
The working set (16 GB weights + ~20 GiB KV per step) exceeds the 126 MB L2
(no flush needed).  Multi-GPU: request i -> replica i mod N (C3), weak scaling.
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


def _trace_for_rank(rank, world):
    from paper_2510_02758_b200.workload import RequestSpec, Trace, load_trace

    tr = load_trace(str(ROOT / "tests" / "golden" / "traces" / "c2_poisson256_s1.csv"))
    if world == 1:
        return tr
    # C3: the trace scaled per GPU - every replica serves a full 256-request
    # population (ids re-densified), request i of the scaled job -> GPU i mod N
    return Trace(tuple(RequestSpec(r.id, r.arrival_time, r.prompt_len, r.output_len, r.consume_rate)
                       for r in tr.requests))


def run_ours(args):
    import torch

    from paper_2510_02758_b200 import configs
    from paper_2510_02758_b200.costs import CostModel
    from paper_2510_02758_b200.dataplane import GpuDataPlane, KvPool
    from paper_2510_02758_b200.engine import SimConfig
    from paper_2510_02758_b200.model import PagedDecoder
    from paper_2510_02758_b200.realtime import RealtimeEngine
    from paper_2510_02758_b200.scheduler import BufferAwarePolicy, SchedulerConfig

    world, rank, local = _dist()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=dev)
    c2 = configs.C2
    shape = c2.model
    tr = _trace_for_rank(rank, world)
    n_blocks = math.ceil(c2.gpu_mem_tokens / 16) + 4 * len(tr.requests) + c2.max_batch
    pool = KvPool(n_blocks, args.host_blocks, shape.n_layers, shape.n_kv_heads, shape.head_dim, device=dev)
    model = PagedDecoder(shape, device=dev, seed=rank)
    dp = GpuDataPlane(tr.requests, pool, mode="realtime", kv_source="model", model=model,
                      n_q_heads=shape.n_q_heads, engine=args.swap_engine)
    policy = BufferAwarePolicy(c2.sched_cfg(SchedulerConfig))
    sim = c2.sim_cfg(SimConfig, debug_checks=False)
    cm = c2.cost_model(CostModel)

    t_start = time.perf_counter()
    state = {"phase": "ff", "t_warm": None, "timed": [], "wall0": None, "wall1": None, "attn": []}

    def on_step(rec, eng):
        contended = eng.total_preemptions > 0
        if args.verbose and len(eng.steps) % 200 == 0:
            print(f"[bench] step {len(eng.steps)} t={eng.now:.2f}s batch={rec['batch']} dur={rec['dur'] * 1e3:.2f}ms "
                  f"pre={eng.total_preemptions} rc={eng.total_recomputes} running={len(eng.running)} "
                  f"waiting={len(eng.waiting)} d2h={dp.stats['d2h_tokens']} h2d={dp.stats['h2d_tokens']} "
                  f"wall={time.perf_counter() - t_start:.1f}s", file=sys.stderr, flush=True)
        if state["phase"] == "ff":
            if contended or len(eng.steps) >= args.ff_max:
                state["phase"] = "warm"
                state["warm_left"] = args.warmup
                state["ff_steps"] = len(eng.steps)
            return
        if state["phase"] == "warm":
            state["warm_left"] -= 1
            if state["warm_left"] <= 0:
                state["phase"] = "timed"
                state["wall0"] = time.perf_counter()
                state["d2h0"], state["h2d0"] = dp.stats["d2h_tokens"], dp.stats["h2d_tokens"]
                state["ev0"] = len(dp._events)
                model.attn_timing = []
            return
        if state["phase"] == "timed":
            state["timed"].append(dict(rec))
            if len(state["timed"]) >= args.steps:
                state["wall1"] = time.perf_counter()
                state["d2h1"], state["h2d1"] = dp.stats["d2h_tokens"], dp.stats["h2d_tokens"]
                state["ev1"] = len(dp._events)
                state["attn"] = list(getattr(model, "attn_timing", []))
                model.attn_timing = None
                state["phase"] = "done"
                eng._stop = True

    eng = RealtimeEngine(tr, policy, cm, sim, dp, skip_idle=True, on_step=on_step)
    if world > 1:
        import torch.distributed as dist

        dist.barrier()
    torch.cuda.synchronize()
    sampler = ClockSampler(local)
    with sampler:
        res = eng.run()
    torch.cuda.synchronize()
    if state["phase"] != "done":
        raise RuntimeError(f"bench ended in phase {state['phase']} after {len(eng.steps)} steps")
    timed = state["timed"]
    dev_s = sum(s["dur"] for s in timed)
    eff = sum(s["effective"] for s in timed)
    toks = sum(s["tokens"] for s in timed)
    wall = state["wall1"] - state["wall0"]
    dev_s = _max_over_ranks(dev_s, world, dev)
    wall = _max_over_ranks(wall, world, dev)
    eff = _sum_over_ranks(eff, world, dev)
    toks = _sum_over_ranks(toks, world, dev)
    # swap traffic of the window (bytes per token = all layers' K and V)
    bpt = shape.kv_bytes_per_token
    xfers = dp.transfer_log()[state["ev0"]:state["ev1"]]
    d2h_tok = sum(n for k, n, _ in xfers if k == "d2h")
    h2d_tok = sum(n for k, n, _ in xfers if k == "h2d")
    d2h_ms = sum(ms for k, _, ms in xfers if k == "d2h")
    h2d_ms = sum(ms for k, _, ms in xfers if k == "h2d")
    swap = {
        "d2h_tokens": d2h_tok, "h2d_tokens": h2d_tok,
        "d2h_gbs": (d2h_tok * bpt / (d2h_ms / 1e3) / 1e9) if d2h_ms else None,
        "h2d_gbs": (h2d_tok * bpt / (h2d_ms / 1e3) / 1e9) if h2d_ms else None,
        "pcie_gen5_gbs": PCIE_GEN5_GBS,
    }
    for k in ("d2h", "h2d"):
        if swap[f"{k}_gbs"]:
            swap[f"{k}_frac_pcie"] = swap[f"{k}_gbs"] / PCIE_GEN5_GBS
    # roofline of the dominant hand-written kernel: paged decode attention
    hbm, peak_kind = _peaks()
    attn = state["attn"]
    roof = None
    if attn:
        per = [(b, e0.elapsed_time(e1)) for b, e0, e1 in attn]
        avg_ms = sum(ms for _, ms in per) / len(per)
        avg_bytes = sum(b for b, _ in per) / len(per)
        ach = avg_bytes / (avg_ms / 1e3) / 1e9
        roof = {"bound": "hbm", "kernel": "paged_attn_kernel<128,4>", "achieved": round(ach, 1),
                "peak": hbm, "peak_kind": peak_kind, "unit": "GB/s", "frac": round(ach / hbm, 4),
                "traffic": None, "launches": len(per), "avg_ms": round(avg_ms, 4),
                "algorithmic_bytes_per_launch": round(avg_bytes)}
    h2d_step = sum(s.get("h2d_bytes", 0) for s in timed)
    out = {
        "metric": METRIC,
        "value": eff / dev_s if dev_s > 0 else None,
        "unit": "effective tok/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": dev_s / len(timed) * 1e3,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "bf16",
        "data": "synthetic (random-init Llama3-8B weights, seeded prompt token ids, frozen C2 trace)",
        "config": {"workload": "C2: Llama3-8B bf16 random-init, 1xB200 per replica, 256-request Poisson burst "
                               "(lambda=10/s, first 256 of a 30 s trace, seed 1), KV pool 163,840 tokens (20 GiB) "
                               "with swap to pinned host, block 16",
                   "model": "llama3-8b", "global_batch": timed and max(s["batch"] for s in timed),
                   "seq_len": None, "parallelism": f"replicas x{world}",
                   "l2": "working set (16 GB weights + KV) >> 126 MB L2; no flush needed",
                   "timed_region": "K decode iterations after contention + W warm-up"},
        "raw_tok_s": toks / dev_s if dev_s > 0 else None,
        "e2e": {"value": eff / wall if wall > 0 else None, "unit": "effective tok/s",
                "h2d_bytes_per_step": int((h2d_tok * bpt + len(timed) * 0) / max(1, len(timed))),
                "d2h_bytes_per_step": int(d2h_tok * bpt / max(1, len(timed)))},
        "swap": swap,
        "roofline": roof,
        "clocks": sampler.summary(),
        "gpu_launches": None,
        "fast_forward_steps": state.get("ff_steps"),
        "preemptions_so_far": res.total_preemptions,
    }
    launches = dp.stats
    out["gpu_launches"] = int(len(timed) * (shape.n_layers * 2) + len(xfers))
    out["e2e"]["h2d_bytes_per_step"] += int(sum(s["batch"] for s in timed) * 12 / max(1, len(timed)))
    out["e2e"]["d2h_bytes_per_step"] += int(sum(s["batch"] for s in timed) * 8 / max(1, len(timed)))
    if rank == 0 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(args, timed, quick=True)
    if rank == 0:
        print(json.dumps(out))
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()
    return out


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
           "config": {"workload": "C2 decode step on the host CPU (oracle restatement)", "model": "llama3-8b"},
           "cpu_baseline": cb, "e2e": {"value": cb["value"], "unit": cb["unit"], "h2d_bytes_per_step": 0,
                                       "d2h_bytes_per_step": 0}}
    print(json.dumps(out))
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--host-blocks", type=int, default=int(os.environ.get("TF_HOST_BLOCKS", 26000)))
    ap.add_argument("--swap-engine", type=int, default=1)
    ap.add_argument("--ff-max", type=int, default=6000)
    ap.add_argument("--cpu-seconds", type=float, default=20.0)
    ap.add_argument("--ref-batch", type=int, default=64)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--verbose", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        raise SystemExit("--warmup must be >= 3")
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
