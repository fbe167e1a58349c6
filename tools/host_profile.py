"""Host time of one decode dispatch, piece by piece (Llama3-8B C2 shapes,
B=128): dataplane.decode_start bookkeeping, the decode graph's staging, the
zero-copy input copy, the graph replay launch, the sampled-id readback launch.

python tools/host_profile.py [--batch 128] [--reps 200]
"""
import argparse
import ctypes as C
import json
import sys
import time
import types
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_2510_02758_b200 import _lib, configs  # noqa: E402
from paper_2510_02758_b200.dataplane import GpuDataPlane, KvPool  # noqa: E402
from paper_2510_02758_b200.model import PagedDecoder  # noqa: E402
from paper_2510_02758_b200.workload import RequestSpec  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=128)
    ap.add_argument("--ctx", type=int, default=600)
    ap.add_argument("--reps", type=int, default=200)
    args = ap.parse_args()
    dev = torch.device("cuda")
    S = configs.LLAMA3_8B
    B, ctx = args.batch, args.ctx
    reqs = [RequestSpec(i, 0.0, ctx, 4000, 20.0) for i in range(B)]
    nlb = (ctx + 4000 + 2 + 15) // 16
    pool = KvPool(B * ((ctx + args.reps + 32) // 16 + 2) + 64, 8, S.n_layers, S.n_kv_heads, S.head_dim, device=dev)
    model = PagedDecoder(S, device=dev)
    dp = GpuDataPlane(reqs, pool, mode="realtime", kv_source="model", model=model, n_q_heads=S.n_q_heads)
    dp.enable_scratch()
    model.enable_graphs(dp, buckets=(B,), prefill_buckets=0)
    state = {r: types.SimpleNamespace(kv=types.SimpleNamespace(total_kv=ctx)) for r in range(B)}
    eng = types.SimpleNamespace(state=state, debug_checks=False)
    from paper_2510_02758_b200.dataplane import LIVE
    for r in range(B):
        dp.flags[r, :ctx] = LIVE
        dp._reconcile(r, range(0, (ctx - 1) // 16 + 1))
        model.pending[r] = 1
    torch.cuda.synchronize()
    batch = tuple(range(B))
    st = dp.s_compute
    t = {"decode_start_total": 0.0, "dp_bookkeeping": 0.0, "model_decode": 0.0, "stage_write": 0.0,
         "copy_small": 0.0, "replay": 0.0}
    for i in range(args.reps):
        for r in range(B):
            state[r].kv.total_kv = ctx + i
        t0 = time.perf_counter()
        dp.decode_start(batch, eng)
        t1 = time.perf_counter()
        st.synchronize()
        dp.decode_done(batch, batch)
        t["decode_start_total"] += t1 - t0
    # pieces of the model side, in isolation
    g, io, stage, out, _ = model._graphs[B]
    rids, pos = list(range(B)), [ctx] * B
    for _ in range(args.reps):
        t0 = time.perf_counter()
        sn = stage.numpy()
        sn[0, :B] = [model.pending[r] for r in rids]
        sn[1, :B] = rids
        sn[2, :B] = pos
        t1 = time.perf_counter()
        _lib.check(_lib.lib.tf_copy_small(C.c_void_p(io.data_ptr()), C.c_void_p(stage.data_ptr()),
                                          io.numel() * io.element_size(), C.c_void_p(st.cuda_stream)))
        t2 = time.perf_counter()
        with torch.cuda.stream(st):
            g.replay()
        t3 = time.perf_counter()
        st.synchronize()
        t["stage_write"] += t1 - t0
        t["copy_small"] += t2 - t1
        t["replay"] += t3 - t2
    res = {k: round(v / args.reps * 1e6, 1) for k, v in t.items()}
    res["unit"] = "us per call"
    print(json.dumps(res))


if __name__ == "__main__":
    main()
