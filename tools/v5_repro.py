"""Find the v5 attention launch whose bounded wait expires in the full-size C2
replay (tiny shapes: 2 layers, 2 kv heads, head_dim 64, 4 q heads) and dump
its inputs for an offline reproduction.

python tools/v5_repro.py [--out gpurun_out/v5_repro.json] [--max-s 600]

Runs the reference-time replay (engine.Engine + GpuDataPlane, synthetic KV /
q) with TF_ATTN_IMPL=5; after every decode step's attention the workspace's
diagnostic words (bytes [8, 64)) are read; at the first expired wait the
batch (rows, contexts, max_ctx), the workspace size and the diagnostics are
written out and the run stops.  Then the same launch is repeated in
isolation to see whether it stalls again.
"""
import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

from conftest import load_golden, pool_blocks, trace_path  # noqa: E402

from paper_2510_02758_b200 import _lib  # noqa: E402
from paper_2510_02758_b200.costs import CostModel  # noqa: E402
from paper_2510_02758_b200.dataplane import GpuDataPlane, KvPool  # noqa: E402
from paper_2510_02758_b200.engine import Engine, SimConfig  # noqa: E402
from paper_2510_02758_b200.scheduler import SchedulerConfig, make_policy  # noqa: E402
from paper_2510_02758_b200.workload import load_trace  # noqa: E402


class Found(Exception):
    pass


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--run", default="c2_burst256_s1_tokenflow")
    ap.add_argument("--out", default="gpurun_out/v5_repro.json")
    ap.add_argument("--max-s", type=float, default=600)
    ap.add_argument("--tee", action="store_true", help="run under the GPU test harness (CPU data plane in lockstep)")
    args = ap.parse_args()
    _lib.lib.tf_paged_decode_attn_impl(5)
    dev = torch.device("cuda")
    g = load_golden("runs", args.run)
    tr = load_trace(trace_path(g["trace"]))
    nb = pool_blocks(g["sim"], len(tr.requests))
    nh = g["sim"]["cpu_mem_tokens"] // 16 + len(tr.requests)
    pool = KvPool(nb, nh, n_layers=2, kv_heads=2, head_dim=64, device=dev)
    dp = GpuDataPlane(tr.requests, pool, mode="replay", attention="all", n_q_heads=4)
    plane = dp
    if args.tee:
        from test_dataplane_gpu import Tee

        from oracle.dataplane import CpuDataPlane

        plane = Tee(dp, CpuDataPlane(tr.requests, nb, nh, 2, 2, 64), check_every=10 ** 9)
    eng = Engine(tr, make_policy(g["policy"], SchedulerConfig(**g["sched"])), CostModel(**g["cm"]),
                 SimConfig(**g["sim"]), dataplane=plane)
    orig = dp._synthetic_attention
    t0 = time.time()
    state = {"launches": 0}

    def attn(batch, e):
        orig(batch, e)
        state["launches"] += 1
        if not args.tee:
            torch.cuda.synchronize()
        elif state["launches"] % 50:
            return  # under the harness: check every 50th step (keep its timing)
        torch.cuda.synchronize()
        diag = dp._attn_ws[8:64].view(torch.int32).cpu().numpy()
        if diag[0] > 0 or time.time() - t0 > args.max_s:
            pos = [e.state[r].kv.total_kv for r in batch]
            rec = {"expired_waits": int(diag[0]), "first": diag[2:10].tolist(),
                   "fields": ["kind(1 tma,2 merge)", "lid", "warp", "B", "sid", "seen", "want", "iter"],
                   "B": len(batch), "rows": list(map(int, batch)), "ctx": [p + 1 for p in pos],
                   "max_ctx": max(pos) + 1, "ws_bytes": int(dp._attn_ws.numel()), "launch_index": state["launches"],
                   "elapsed_s": time.time() - t0, "timeout": diag[0] == 0}
            state["rec"] = rec
            raise Found()

    dp._synthetic_attention = attn
    try:
        eng.run()
        print(json.dumps({"completed": True, "launches": state["launches"], "elapsed_s": time.time() - t0}))
        return
    except Found:
        pass
    rec = state["rec"]
    # the same launch in isolation, fresh workspace, every layer
    B, ctx = rec["B"], rec["ctx"]
    rows = torch.tensor(rec["rows"], dtype=torch.int32, device=dev)
    ctxd = torch.tensor(ctx, dtype=torch.int32, device=dev)
    q = torch.randn(B, 4, 64, device=dev).to(torch.bfloat16)
    out = torch.empty_like(q)
    ws_n = int(_lib.lib.tf_paged_decode_attn_workspace(pool.handle, B, rec["max_ctx"], 4))
    iso = []
    for fresh in (True, False):
        ws = torch.zeros(max(1, ws_n), dtype=torch.uint8, device=dev) if fresh else dp._attn_ws
        import ctypes as C

        for layer in range(2):
            _lib.check(_lib.lib.tf_paged_decode_attn(
                pool.handle, C.c_void_p(q.data_ptr()), C.c_void_p(dp.table.data_ptr()), dp.nlb,
                C.c_void_p(rows.data_ptr()), C.c_void_p(ctxd.data_ptr()), B, rec["max_ctx"], layer, 4, 0.125,
                C.c_void_p(out.data_ptr()), C.c_void_p(ws.data_ptr()), ws.numel(), None))
        torch.cuda.synchronize()
        d = ws[8:64].view(torch.int32).cpu().numpy()
        ctr = ws[256:256 + 1024 * 2 * 4].view(torch.int32).cpu().numpy()
        iso.append({"fresh_workspace": fresh, "expired_waits": int(d[0]), "first": d[2:10].tolist(),
                    "nonzero_counters": np.nonzero(ctr)[0][:20].tolist()})
    rec["isolated"] = iso
    rec["ticket"] = int(dp._attn_ws[:8].view(torch.int64).item())
    print(json.dumps(rec))
    Path(args.out).parent.mkdir(exist_ok=True)
    Path(args.out).write_text(json.dumps(rec, indent=1))


if __name__ == "__main__":
    main()
