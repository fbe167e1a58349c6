"""Paged decode attention micro-benchmark (Llama3-8B layer shapes).

python tools/attn_bench.py [--impl 3] [--out gpurun_out/attn_bench.json]

For a set of (batch, context distribution, planned max_ctx) cases: one layer's
paged attention over a random block permutation of a C2-sized pool, timed
with CUDA events on the launching stream (median of 20 launches after
warm-up) -> GB/s of algorithmic bytes (K+V of every context token + q/out +
table entries) and the fraction of the measured HBM peak.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import statistics
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_2510_02758_b200 import _lib  # noqa: E402
from paper_2510_02758_b200.dataplane import KvPool  # noqa: E402


def peak():
    p = ROOT / "MEASURED_PEAKS.json"
    return json.loads(p.read_text()).get("hbm_gbs", 6650.0) if p.exists() else 6650.0


LAYOUT = "random"


def run_case(pool, B, ctxs, plan_ctx, hq=32, reps=20, stream=None):
    dev = pool.device
    H, D = pool.H, pool.D
    nlb = (max(plan_ctx, max(ctxs)) + 15) // 16
    rng = np.random.default_rng(B * 7 + len(ctxs))
    need = [(c + 15) // 16 for c in ctxs]
    if LAYOUT == "contig":  # every request's blocks consecutive (TLB / DRAM-page locality probe)
        perm = np.arange(sum(need), dtype=np.int32)
    else:
        perm = rng.permutation(pool.n_blocks)[: sum(need)].astype(np.int32)
    tab = np.zeros((B, nlb), np.int32)
    o = 0
    for i, n in enumerate(need):  # distinct blocks for every context block (no L2 reuse)
        tab[i, :n] = perm[o:o + n]
        o += n
    table = torch.from_numpy(tab).to(dev)
    rows = torch.arange(B, dtype=torch.int32, device=dev)
    ctx = torch.tensor(ctxs, dtype=torch.int32, device=dev)
    q = (torch.randn(B, hq, D, device=dev) * 0.5).to(torch.bfloat16)
    out = torch.empty_like(q)
    ws_n = max(1, int(_lib.lib.tf_paged_decode_attn_workspace(pool.handle, B, plan_ctx, hq)))
    ws = torch.zeros(ws_n, dtype=torch.uint8, device=dev)
    st = stream or torch.cuda.current_stream()

    def launch(layer):
        _lib.check(_lib.lib.tf_paged_decode_attn(pool.handle, C.c_void_p(q.data_ptr()), C.c_void_p(table.data_ptr()),
                                                 nlb, C.c_void_p(rows.data_ptr()), C.c_void_p(ctx.data_ptr()), B,
                                                 plan_ctx, layer, hq, 0.0884, C.c_void_p(out.data_ptr()),
                                                 C.c_void_p(ws.data_ptr()), ws_n, C.c_void_p(st.cuda_stream)))

    for i in range(5):
        launch(i % pool.L)
    times = []
    for i in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        launch(i % pool.L)
        e1.record(st)
        times.append((e0, e1))
    torch.cuda.synchronize()
    ms = statistics.median(a.elapsed_time(b) for a, b in times)
    abytes = sum(ctxs) * 2 * H * D * 2 + 2 * B * hq * D * 2 + sum((c + 15) // 16 for c in ctxs) * 4
    return ms, abytes


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="gpurun_out/attn_bench.json")
    ap.add_argument("--only", default=None, help="B:ctx:plan, e.g. 64:ragged500-3000:exact (one case, for ncu)")
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--batches", default="32,64,96,128")
    ap.add_argument("--plans", default="exact,pool")
    ap.add_argument("--impls", default="0,3,5", help="comma list of implementations (tf_paged_decode_attn_impl)")
    ap.add_argument("--layout", default="random", choices=["random", "contig"])
    ap.add_argument("--pool-blocks", type=int, default=22000)
    ap.add_argument("--orders", default="asis", help="comma list: asis (random order), desc (longest context "
                    "first = LPT order of the CTAs)")
    args = ap.parse_args()
    global LAYOUT
    LAYOUT = args.layout
    dev = torch.device("cuda")
    pool = KvPool(args.pool_blocks, 1, 32, 8, 128, device=dev)
    pool.gpu.view(torch.bfloat16).normal_(0, 1)
    pk = peak()
    rng = np.random.default_rng(0)
    cases = []
    for B in [int(x) for x in args.batches.split(",")]:
        for name, ctxs in (("uniform2600", [2600] * B),
                           ("ragged500-3000", list(rng.integers(500, 3000, B))),
                           ("short736", list(rng.integers(600, 870, B))),
                           ("c2live560", list(rng.integers(200, 920, B)))):
            for plan in args.plans.split(","):
                if args.only and args.only != f"{B}:{name}:{plan}":
                    continue
                plan_ctx = max(ctxs) if plan == "exact" else 4096
                for order in args.orders.split(","):
                    cc = sorted(ctxs, reverse=True) if order == "desc" else ctxs
                    for impl in [int(x) for x in args.impls.split(",")]:
                        _lib.lib.tf_paged_decode_attn_impl(impl)
                        ms, ab = run_case(pool, B, [int(c) for c in cc], plan_ctx, reps=args.reps)
                        gbs = ab / (ms / 1e3) / 1e9
                        row = {"impl": impl, "B": B, "ctx": name, "plan": plan, "order": order,
                               "us": round(ms * 1e3, 2), "MB": round(ab / 1e6, 1), "gbs": round(gbs, 1),
                               "frac": round(gbs / pk, 4)}
                        cases.append(row)
                        print(json.dumps(row), flush=True)
    Path(args.out).parent.mkdir(parents=True, exist_ok=True)
    Path(args.out).write_text(json.dumps({"peak_gbs": pk, "cases": cases}, indent=1))


if __name__ == "__main__":
    main()
