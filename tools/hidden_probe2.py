"""Where does a decode step lose time when swaps run beside it?

Llama3-8B decode graph of B requests at ctx tokens (synthetic KV), timed over
24-step rounds (medians of 5 alternating rounds) in four decode variants x
three swap loads:

  decode variants
    full     : model._decode_graph (host staging -> zero-copy tf_copy_small of
               the step inputs over PCIe -> graph replay) + the sampled-id
               readback (tf_copy_small to pinned host), as the serving loop does
    replay   : graph replay only (inputs already in HBM, no readback)
  swap loads (copy engines, partial-block 2-D copies like the window mix)
    none / d2h / h2d / both, at `--tokens` tokens per step per direction

python tools/hidden_probe2.py [--batch 128] [--ctx 600] [--tokens 40] [--engine 3]
"""
import argparse
import ctypes as C
import json
import statistics
import sys
import time
import types
from pathlib import Path

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
    ap.add_argument("--tokens", type=int, default=40, help="swap tokens per step per direction")
    ap.add_argument("--seg", type=int, default=8, help="slots per partial-block segment (16 = whole blocks)")
    ap.add_argument("--engine", type=int, default=3)
    ap.add_argument("--steps", type=int, default=24)
    ap.add_argument("--out", default="gpurun_out/hidden_probe2.json")
    args = ap.parse_args()
    dev = torch.device("cuda")
    S = configs.LLAMA3_8B
    B, ctx = args.batch, args.ctx
    reqs = [RequestSpec(i, 0.0, ctx, 64, 20.0) for i in range(B)]
    nlb = (ctx + 64 + 2 + 15) // 16
    nseg = max(1, args.tokens // args.seg)
    pool = KvPool(B * nlb + 2 * nseg + 8, 2 * nseg + 8, S.n_layers, S.n_kv_heads, S.head_dim, device=dev)
    model = PagedDecoder(S, device=dev)
    dp = GpuDataPlane(reqs, pool, mode="realtime", kv_source="model", model=model, n_q_heads=S.n_q_heads)
    dp.enable_scratch()
    ids = pool.alloc(0, B * nlb)
    dp.table[:B, :nlb] = torch.tensor(ids, dtype=torch.int32, device=dev).view(B, nlb)
    torch.cuda.synchronize()
    model.enable_graphs(dp, buckets=(B,), prefill_buckets=0)
    for r in range(B):
        model.pending[r] = 1
    rids = list(range(B))
    pos = [ctx - 1] * B
    st = dp.s_compute
    g_blocks = pool.alloc(0, 2 * nseg)
    h_blocks = pool.alloc(1, 2 * nseg)
    segs_out = dp._seg_array([(g_blocks[i], h_blocks[i], 0, args.seg) for i in range(nseg)])
    segs_in = dp._seg_array([(g_blocks[nseg + i], h_blocks[nseg + i], 0, args.seg) for i in range(nseg)])
    g, io, stage, out, _ = model._graphs[B]
    host_ids = model._dec_out[:B]

    def dec_full():
        with torch.cuda.stream(st):
            nxt = model._decode_graph(dp, rids, pos, st).contiguous()
            _lib.check(_lib.lib.tf_copy_small(C.c_void_p(host_ids.data_ptr()), C.c_void_p(nxt.data_ptr()),
                                              host_ids.numel() * 8, C.c_void_p(st.cuda_stream)))

    def dec_replay():
        with torch.cuda.stream(st):
            g.replay()

    def swp(d2h, h2d):
        def f():
            if d2h:
                _lib.check(_lib.lib.tf_kv_gather_d2h(pool.handle, segs_out, nseg, 0, pool.L, args.engine,
                                                     C.c_void_p(dp.s_evict.cuda_stream)))
            if h2d:
                _lib.check(_lib.lib.tf_kv_scatter_h2d(pool.handle, segs_in, nseg, 0, pool.L, args.engine,
                                                      C.c_void_p(dp.s_load.cuda_stream)))
        return f

    loads = {"none": None, "d2h": swp(True, False), "h2d": swp(False, True), "both": swp(True, True)}
    decs = {"full": dec_full, "replay": dec_replay}

    def run(dec, sw):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            if dec:
                dec()
            if sw:
                sw()
        torch.cuda.synchronize()
        return (time.perf_counter() - t0) / args.steps * 1e3

    for d in decs.values():
        d()
    for s in loads.values():
        if s:
            s()
    res = {k: [] for k in [f"{d}+{s}" for d in decs for s in loads] + [f"swap_{s}" for s in loads if s != "none"]}
    for _ in range(5):
        for d, df in decs.items():
            for s, sf in loads.items():
                res[f"{d}+{s}"].append(run(df, sf))
        for s, sf in loads.items():
            if sf:
                res[f"swap_{s}"].append(run(None, sf))
    med = {k: round(statistics.median(v), 4) for k, v in res.items()}
    summary = {}
    for d in decs:
        for s in ("d2h", "h2d", "both"):
            t_dec, t_both, t_sw = med[f"{d}+none"], med[f"{d}+{s}"], med[f"swap_{s}"]
            summary[f"{d}/{s}"] = {"slowdown_us": round((t_both - t_dec) * 1e3, 1),
                                   "hidden": round(1 - max(0.0, t_both - t_dec) / t_sw, 4)}
    outj = {"args": vars(args), "ms_per_step": med, "summary": summary}
    print(json.dumps(outj, indent=1))
    Path(args.out).parent.mkdir(exist_ok=True)
    Path(args.out).write_text(json.dumps(outj, indent=1))


if __name__ == "__main__":
    main()
