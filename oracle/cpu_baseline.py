"""CPU baseline / reference arm (TEST INFRASTRUCTURE; timed, never shipped).

Times the oracle's CPU restatement of one C2 decode step on the host cores:
  * Llama3-8B layer forward for B tokens (torch CPU, bf16 GEMMs, all threads)
  * fp32 GQA decode attention over each member's KV (ctx tokens)
  * KV gather of one step's swap traffic (numpy fancy-index copy)
  * the buffer-aware tick decision (oracle.refsim.policy) on a C2 snapshot
A bounded sample: L_SAMPLE of the 32 layers are executed and the per-layer
cost is scaled to 32 layers (every layer does identical work); the sample
description says so.  When the host cannot keep up with its readers every
token is generated into an empty buffer, so its effective weight is 1 and
effective tok/s = B / step time.
"""
from __future__ import annotations

import gzip
import json
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
L_SAMPLE = 2


def _tick_seconds(reps=3) -> float:
    from oracle.refsim.policy import Knobs, TokenFlowPolicy, snapshot_from_dict

    g = json.load(gzip.open(ROOT / "tests" / "golden" / "ticks" / "c2_burst256_s1_tokenflow.json.gz"))
    views = [t["view"] for t in g["ticks"]][:reps]
    t0 = time.perf_counter()
    for v in views:
        pol = TokenFlowPolicy(Knobs(**g["sched"]))
        pol.on_tick(snapshot_from_dict(v))
    return (time.perf_counter() - t0) / len(views)


def time_reference_sim(name: str = "c1_tokenflow") -> dict:
    """the reference simulator (oracle restatement,
    strictly sequential: 1 core) on a frozen golden run, with the per-call
    cost of its hot-path functions measured inside that run: on_tick
    (tokensim/scheduler.py:513-736), plan_write_chunk (tokensim/kvstore.py:
    112-141, writeback_plan here) and _snapshot (tokensim/engine.py:993-1061).
    The event hash is checked against the golden run (same work as the reference)."""
    import oracle.refsim.sim as simmod
    from oracle.refsim.planner import Costs
    from oracle.refsim.policy import Knobs, build_policy
    from oracle.refsim.sim import SimKnobs
    from oracle.refsim.traces import read_trace

    g = json.load(gzip.open(ROOT / "tests" / "golden" / "runs" / f"{name}.json.gz"))
    reqs = read_trace(str(ROOT / "tests" / "golden" / "traces" / f"{g['trace']}.csv"))
    acc = {"on_tick": [0, 0.0], "plan_write_chunk": [0, 0.0], "snapshot": [0, 0.0]}

    def timed(key, fn):
        def w(*a, **k):
            t0 = time.perf_counter()
            try:
                return fn(*a, **k)
            finally:
                acc[key][0] += 1
                acc[key][1] += time.perf_counter() - t0
        return w

    pol = build_policy(g["policy"], Knobs(**g["sched"]))
    pol.on_tick = timed("on_tick", pol.on_tick)
    orig_wb, orig_snap = simmod.writeback_plan, simmod.Sim.snapshot
    simmod.writeback_plan = timed("plan_write_chunk", orig_wb)
    simmod.Sim.snapshot = timed("snapshot", orig_snap)
    try:
        t0 = time.perf_counter()
        out = simmod.Sim(reqs, pol, Costs(**g["cm"]), SimKnobs(**g["sim"])).run()
        wall = time.perf_counter() - t0
    finally:
        simmod.writeback_plan, simmod.Sim.snapshot = orig_wb, orig_snap
    return {"run": name, "requests": len(reqs), "wall_s": round(wall, 4), "cores": 1,
            "event_hash_ok": out.event_hash() == g["event_hash"],
            "per_call_us": {k: round(v[1] / v[0] * 1e6, 2) for k, v in acc.items() if v[0]},
            "calls": {k: v[0] for k, v in acc.items()}}


def host_info() -> dict:
    """CPU model, core count and NUMA layout of the host."""
    import os

    info = {"nproc": os.cpu_count()}
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                info["cpu_model"] = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    nodes = []
    base = Path("/sys/devices/system/node")
    for d in sorted(base.glob("node[0-9]*")) if base.exists() else []:
        try:
            nodes.append({"node": d.name, "cpus": (d / "cpulist").read_text().strip()})
        except OSError:
            pass
    info["numa_nodes"] = nodes
    return info


def time_cpu_step(batch: int = 64, ctx: int = 2600, threads: int = 16, seconds: float = 20.0,
                  swap_tokens_per_step: int = 64) -> dict:
    from paper_2510_02758_b200.configs import LLAMA3_8B as S

    torch.set_num_threads(threads)
    d, hq, hkv, hd, ffn = S.hidden, S.n_q_heads, S.n_kv_heads, S.head_dim, S.ffn
    bf = torch.bfloat16
    gen = torch.Generator().manual_seed(0)

    def w(*sh):  # random-init N(0, 0.02) like the GPU arm's weights
        return (torch.randn(*sh, generator=gen) * 0.02).to(bf)

    layers = [{k: w(*sh) for k, sh in (("wqkv", (d, (hq + 2 * hkv) * hd)), ("wo", (hq * hd, d)),
                                       ("wgu", (d, 2 * ffn)), ("wd", (ffn, d)))}
              for _ in range(L_SAMPLE)]
    lm = w(d, S.vocab)
    kv = [torch.randn(batch, 2, hkv, ctx, hd, dtype=torch.float32) for _ in range(L_SAMPLE)]
    x0 = torch.randn(batch, d, dtype=bf)

    def layer_pass(li):
        L = layers[li]
        x = x0
        qkv = (x @ L["wqkv"]).float().view(batch, hq + 2 * hkv, hd)
        q = qkv[:, :hq]
        k = kv[li][:, 0]
        v = kv[li][:, 1]
        qg = q.view(batch, hkv, hq // hkv, hd)
        s = torch.einsum("bkgd,bktd->bkgt", qg, k) / hd ** 0.5
        a = torch.einsum("bkgt,bktd->bkgd", torch.softmax(s, -1), v).reshape(batch, hq * hd).to(bf)
        x = x + a @ L["wo"]
        gu = x @ L["wgu"]
        g, u = gu.chunk(2, -1)
        return x + (torch.nn.functional.silu(g) * u) @ L["wd"]

    # warm-up, then sample
    layer_pass(0)
    per_layer, n = [], 0
    t_end = time.perf_counter() + seconds * 0.7
    while time.perf_counter() < t_end or n < 2:
        t0 = time.perf_counter()
        layer_pass(n % L_SAMPLE)
        per_layer.append(time.perf_counter() - t0)
        n += 1
    t0 = time.perf_counter()
    (x0 @ lm).argmax(-1)
    t_lm = time.perf_counter() - t0
    # swap: gather one step's chunk bytes (128 KiB per token) from a pool
    pool = np.zeros((256, 2 * 1024 * 1024 // 2), np.uint16)
    idx = np.random.default_rng(0).permutation(256)[: max(1, swap_tokens_per_step // 16)]
    t0 = time.perf_counter()
    for _ in range(3):
        pool[idx].copy()
    t_swap = (time.perf_counter() - t0) / 3
    t_tick = _tick_seconds()
    ticks_per_step = 0.5 / 0.0075  # one tick per 0.5 s of schedule interval at ~7.5 ms steps
    step = float(np.median(per_layer)) * S.n_layers + t_lm + t_swap + t_tick / ticks_per_step
    return {"value": batch / step, "unit": "effective tok/s", "cores": threads, "kind": "port",
            "step_s": step, "per_layer_s": float(np.median(per_layer)), "lm_head_s": t_lm, "tick_s": t_tick,
            "sample": f"{n} single-layer passes of a B={batch}, ctx={ctx} Llama3-8B decode step (bf16 GEMMs + fp32 "
                      f"GQA attention) scaled x{S.n_layers} layers + lm_head + one step's swap gather + 1/"
                      f"{ticks_per_step:.0f} of an on_tick (oracle restatement); torch CPU, {threads} threads"}


def time_cpu_gather(blocks: int = 256, pool_blocks: int = 512, threads: int = 16, reps: int = 5) -> dict:
    """The unpinned byte path on the host: gather ``blocks``
    random 2 MiB Llama3-8B KV blocks (all layers) out of a ``pool_blocks``
    host-resident pool into a staging buffer and scatter them back - the
    CPU restatement of tf_kv_gather_d2h / tf_kv_scatter_h2d on whole blocks,
    torch index_select / index_copy_ on ``threads`` threads.  Bounded: a 1 GiB
    pool, 512 MiB moved per direction per rep."""
    torch.set_num_threads(threads)
    elems = 32 * 2 * 8 * 16 * 128  # bf16 elements per block (2 MiB)
    pool = torch.empty(pool_blocks, elems, dtype=torch.int16).random_()
    stage = torch.empty(blocks, elems, dtype=torch.int16)
    ids = torch.randperm(pool_blocks, generator=torch.Generator().manual_seed(0))[:blocks]
    torch.index_select(pool, 0, ids, out=stage)  # warm-up (page faults)
    t0 = time.perf_counter()
    for _ in range(reps):
        torch.index_select(pool, 0, ids, out=stage)
    t_g = (time.perf_counter() - t0) / reps
    t0 = time.perf_counter()
    for _ in range(reps):
        pool.index_copy_(0, ids, stage)
    t_s = (time.perf_counter() - t0) / reps
    nbytes = blocks * elems * 2
    return {"gather_gbs": round(nbytes / t_g / 1e9, 2), "scatter_gbs": round(nbytes / t_s / 1e9, 2),
            "blocks": blocks, "block_bytes": elems * 2, "threads": threads,
            "sample": f"{blocks} random 2 MiB blocks of a {pool_blocks}-block host pool, {reps} reps per direction"}
