"""A steady-state C2 decode step for profilers (ncu launch lists / --set full).

Builds the Llama3-8B model and a KV pool holding B requests of ctx tokens
(synthetic KV), then runs N decode steps through the same code the engine
uses (model._decode_rows: fused rope+append, paged attention, cuBLAS GEMMs)
with one step's worth of swap traffic (write-through gather + load scatter)
on the copy streams.  Prints per-step CUDA-event times.

python tools/step_profile.py [--batch 64] [--ctx 2600] [--steps 5] [--swap-blocks 64] [--engine 0]
"""
import argparse
import ctypes as C
import sys
import types
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2510_02758_b200 import _lib, configs  # noqa: E402
from paper_2510_02758_b200.dataplane import KvPool  # noqa: E402
from paper_2510_02758_b200.model import PagedDecoder  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=64)
    ap.add_argument("--ctx", type=int, default=2600)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--swap-blocks", type=int, default=64)
    ap.add_argument("--engine", type=int, default=0)
    ap.add_argument("--attn-only", action="store_true")
    args = ap.parse_args()
    dev = torch.device("cuda")
    S = configs.LLAMA3_8B
    B, ctx = args.batch, args.ctx
    nlb = (ctx + 64) // 16 + 1
    nb = B * nlb + args.swap_blocks + 8
    pool = KvPool(nb, max(1, args.swap_blocks), S.n_layers, S.n_kv_heads, S.head_dim, device=dev)
    table = torch.arange(B * nlb, dtype=torch.int32, device=dev).view(B, nlb)
    spans = (_lib.TfSpan * B)()
    for b in range(B):
        spans[b].row, spans[b].rid, spans[b].pos_begin, spans[b].pos_end = b, b, 0, ctx
    _lib.check(_lib.lib.tf_kv_fill_synthetic(pool.handle, C.c_void_p(table.data_ptr()), nlb, spans, B, 0, None))
    model = PagedDecoder(S, device=dev) if not args.attn_only else None
    dp = types.SimpleNamespace(pool=pool, table=table, nlb=nlb, stats={"attn_launches": 0})
    sc, sd, sh = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
    g = np.arange(B * nlb, B * nlb + args.swap_blocks)
    segs = (_lib.TfSeg * max(1, args.swap_blocks))()
    for i, blk in enumerate(g):
        segs[i].gpu_block, segs[i].host_block, segs[i].slot_begin, segs[i].n_slots = int(blk), i, 0, 16
    torch.cuda.synchronize()
    for step in range(args.steps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(sc)
        if args.swap_blocks:
            _lib.check(_lib.lib.tf_kv_gather_d2h(pool.handle, segs, args.swap_blocks, 0, S.n_layers, args.engine,
                                                 C.c_void_p(sd.cuda_stream)))
            _lib.check(_lib.lib.tf_kv_scatter_h2d(pool.handle, segs, args.swap_blocks, 0, S.n_layers, args.engine,
                                                  C.c_void_p(sh.cuda_stream)))
        with torch.cuda.stream(sc):
            if model is not None:
                toks = torch.randint(0, S.vocab, (B,), device=dev)
                model._decode_rows(dp, list(range(B)), toks, [ctx - 1] * B, sc)
        e1.record(sc)
        torch.cuda.synchronize()
        print(f"step {step}: {e0.elapsed_time(e1):.3f} ms (B={B}, ctx={ctx})", flush=True)


if __name__ == "__main__":
    main()
