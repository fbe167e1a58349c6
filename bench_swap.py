"""C5: KV swap bandwidth sweep + transfer-hidden-under-decode measurement.

python bench_swap.py [--max-blocks 65536] [--engines 0,1] [--out gpurun_out/swap_sweep.json]

Llama3-8B block format (2 MiB per block = 16 tokens x 32 layers x K,V x 8
heads x 128 x bf16).  For block counts 1, 2, 4, ..., max: a random
permutation of pool block ids (seed 0) is gathered to (d2h) / scattered from
(h2d) pinned host blocks, either all 32 layers per launch or one layer per
launch (per-layer chunking), with the SM zero-copy kernel (engine 0) and the
copy-engine path (engine 1: one cudaMemcpyAsync per maximal contiguous run; engine 3: + one 2-D copy per partial block); plus both directions concurrently on two
streams.  GB/s are reported against PCIe Gen5 x16 (63.0 GB/s per direction)
and against the box's measured contiguous pinned cudaMemcpyAsync peak.

--overlap: decode attention over a C2-sized batch alone, swaps alone, and
both concurrently -> hidden = 1 - (T_both - T_decode) / T_swap.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

from paper_2510_02758_b200 import _lib  # noqa: E402
from paper_2510_02758_b200.dataplane import KvPool  # noqa: E402

PCIE = 63.0


def segs_for(gblocks, hblocks):
    arr = (_lib.TfSeg * len(gblocks))()
    for i, (g, h) in enumerate(zip(gblocks, hblocks)):
        arr[i].gpu_block, arr[i].host_block, arr[i].slot_begin, arr[i].n_slots = int(g), int(h), 0, 16
    return arr


def timed(fn, stream, reps=3):
    fn()
    stream.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(reps):
        fn()
    e1.record(stream)
    e1.synchronize()
    return e0.elapsed_time(e1) / 1e3 / reps


def memcpy_peak(pool, stream):
    n = min(pool.n_host_blocks, 512) * pool.block_bytes // 2
    g, h = pool.gpu[:n], pool.host[:n]
    def cp(dst, src):
        with torch.cuda.stream(stream):
            dst.copy_(src, non_blocking=True)
    d2h = timed(lambda: cp(h, g), stream)
    h2d = timed(lambda: cp(g, h), stream)
    return n * 2 / d2h / 1e9, n * 2 / h2d / 1e9


def sweep(args):
    dev = torch.device("cuda")
    L, H, D = 32, 8, 128
    pool = KvPool(args.max_blocks, args.host_blocks, L, H, D, device=dev)
    pool.gpu.zero_()
    bb = pool.block_bytes
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    peak_d2h, peak_h2d = memcpy_peak(pool, s1)
    rng = np.random.default_rng(0)
    perm = rng.permutation(args.max_blocks)
    rows = []
    n = 1
    while n <= args.max_blocks:
        g = perm[:n]
        h = np.arange(n) % args.host_blocks
        segs = segs_for(g, h)
        for eng in args.engines:
            for per_layer in (False, True):
                ranges = [(l, l + 1) for l in range(L)] if per_layer else [(0, L)]

                def d2h(st=s1):
                    for l0, l1 in ranges:
                        _lib.check(_lib.lib.tf_kv_gather_d2h(pool.handle, segs, n, l0, l1, eng,
                                                             C.c_void_p(st.cuda_stream)))

                def h2d(st=s1):
                    for l0, l1 in ranges:
                        _lib.check(_lib.lib.tf_kv_scatter_h2d(pool.handle, segs, n, l0, l1, eng,
                                                              C.c_void_p(st.cuda_stream)))

                reps = 3 if n >= 64 else 10
                td = timed(d2h, s1, reps)
                th = timed(h2d, s1, reps)
                # both directions concurrently (full duplex)
                t0 = time.perf_counter()
                torch.cuda.synchronize()
                e0 = torch.cuda.Event(enable_timing=True)
                e0.record(s1)
                s2.wait_event(e0)
                for _ in range(reps):
                    d2h(s1)
                    h2d(s2)
                e1, e2 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e1.record(s1)
                e2.record(s2)
                torch.cuda.synchronize()
                tb = max(e0.elapsed_time(e1), e0.elapsed_time(e2)) / 1e3 / reps
                del t0
                nbytes = n * bb
                rows.append({"blocks": n, "engine": {0: "sm", 1: "ce", 2: "auto", 3: "ce2d"}[eng], "per_layer": per_layer,
                             "bytes": nbytes, "d2h_gbs": nbytes / td / 1e9, "h2d_gbs": nbytes / th / 1e9,
                             "duplex_gbs": 2 * nbytes / tb / 1e9,
                             "d2h_frac_pcie": nbytes / td / 1e9 / PCIE, "h2d_frac_pcie": nbytes / th / 1e9 / PCIE,
                             "d2h_frac_memcpy": nbytes / td / 1e9 / peak_d2h,
                             "h2d_frac_memcpy": nbytes / th / 1e9 / peak_h2d})
                print(json.dumps(rows[-1]), flush=True)
        n *= 2
    # bit-exact round trip at the largest size, SM engine
    k = min(args.max_blocks, args.host_blocks, 4096)
    g = perm[:k]
    pool.gpu.view(args.max_blocks, -1)[torch.from_numpy(g).to(dev)] = torch.randint(
        -30000, 30000, (k, pool.block_elems), dtype=torch.int16, device=dev)
    ref = pool.gpu.view(args.max_blocks, -1)[torch.from_numpy(g).to(dev)].clone()
    torch.cuda.synchronize()  # fills above ran on the default stream
    segs = segs_for(g, np.arange(k))
    _lib.check(_lib.lib.tf_kv_gather_d2h(pool.handle, segs, k, 0, L, 0, C.c_void_p(s1.cuda_stream)))
    s1.synchronize()
    pool.gpu.view(args.max_blocks, -1)[torch.from_numpy(g).to(dev)] = 0
    torch.cuda.synchronize()
    _lib.check(_lib.lib.tf_kv_scatter_h2d(pool.handle, segs, k, 0, L, 0, C.c_void_p(s1.cuda_stream)))
    s1.synchronize()
    ok = torch.equal(pool.gpu.view(args.max_blocks, -1)[torch.from_numpy(g).to(dev)], ref)
    out = {"pcie_gen5_gbs": PCIE, "memcpy_peak_d2h_gbs": peak_d2h, "memcpy_peak_h2d_gbs": peak_h2d,
           "roundtrip_bit_exact_blocks": k if ok else -1, "rows": rows}
    if args.overlap:
        out["overlap"] = overlap(pool, args)
    out["wt_chunks"] = wt_chunks(pool, args)
    Path(args.out).parent.mkdir(parents=True, exist_ok=True)
    Path(args.out).write_text(json.dumps(out, indent=1))
    print(json.dumps({k: v for k, v in out.items() if k != "rows"}))
    pool.close()


def wt_chunks(pool, args):
    """Write-through-shaped chunks: n tokens starting at slot 5 of a block
    (unaligned, as the reference's write-through pointer is), gathered to the
    host with each engine; per-chunk CUDA-event time -> algorithmic GB/s
    (tokens x 128 KiB / time)."""
    dev = pool.device
    st = torch.cuda.Stream(priority=-1)
    bpt = pool.block_bytes // pool.B
    rows = []
    for n in (8, 16, 32, 64, 128, 256, 512):
        segs = []
        pos, first = 5, 5
        blk = 0
        left = n
        while left > 0:
            k = min(left, 16 - pos % 16)
            segs.append((blk, blk, pos % 16, k))
            left -= k
            pos += k
            blk += 1
        arr = (_lib.TfSeg * len(segs))()
        for i, (g, h, s0, k) in enumerate(segs):
            arr[i].gpu_block, arr[i].host_block, arr[i].slot_begin, arr[i].n_slots = g, h, s0, k
        for eng in (0, 1, 2, 3):
            for d in ("d2h", "h2d"):
                fn = _lib.lib.tf_kv_gather_d2h if d == "d2h" else _lib.lib.tf_kv_scatter_h2d

                def go(fn=fn, eng=eng):
                    _lib.check(fn(pool.handle, arr, len(segs), 0, pool.L, eng, C.c_void_p(st.cuda_stream)))
                t = timed(go, st, reps=20)
                rows.append({"tokens": n, "dir": d, "engine": {0: "sm", 1: "ce", 2: "auto", 3: "ce2d"}[eng],
                             "segments": len(segs), "us": round(t * 1e6, 2), "gbs": round(n * bpt / t / 1e9, 2)})
                print(json.dumps(rows[-1]), flush=True)
    del first, dev
    return rows


def overlap(pool, args):
    """Decode attention (B=64, ctx 2600, 32 layers) alone / swaps alone / both."""
    dev = pool.device
    B, ctx, L, HQ = 64, 2600, 32, 32
    nblk = (ctx + 15) // 16
    table = torch.arange(B * nblk, dtype=torch.int32, device=dev).view(B, nblk) % (pool.n_blocks // 2)
    rows = torch.arange(B, dtype=torch.int32, device=dev)
    ctxs = torch.full((B,), ctx, dtype=torch.int32, device=dev)
    q = torch.randn(B, HQ, 128, device=dev).to(torch.bfloat16)
    out = torch.empty_like(q)
    ws_n = max(1, int(_lib.lib.tf_paged_decode_attn_workspace(pool.handle, B, ctx, HQ)))
    ws = torch.zeros(ws_n, dtype=torch.uint8, device=dev)
    sc, sd, sh = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
    res = {}
    for eng in args.engines:
        def decode():
            for layer in range(L):
                _lib.check(_lib.lib.tf_paged_decode_attn(pool.handle, C.c_void_p(q.data_ptr()),
                                                         C.c_void_p(table.data_ptr()), nblk,
                                                         C.c_void_p(rows.data_ptr()), C.c_void_p(ctxs.data_ptr()),
                                                         B, ctx, layer, HQ, 0.088, C.c_void_p(out.data_ptr()),
                                                         C.c_void_p(ws.data_ptr()), ws_n,
                                                         C.c_void_p(sc.cuda_stream)))

        def swaps():
            _lib.check(_lib.lib.tf_kv_gather_d2h(pool.handle, segs, nbk, 0, 32, eng, C.c_void_p(sd.cuda_stream)))
            _lib.check(_lib.lib.tf_kv_scatter_h2d(pool.handle, segs, nbk, 0, 32, eng, C.c_void_p(sh.cuda_stream)))

        def run(fns, reps=5):
            for f in fns:
                f()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for _ in range(reps):
                for f in fns:
                    f()
            torch.cuda.synchronize()
            return (time.perf_counter() - t0) / reps

        t_dec = run([decode])
        # swap traffic sized to ~80% of one decode (at ~45 GB/s per direction
        # when both run): 100% hiding is then possible, so the fraction
        # measures overlap quality, not the ratio of the two volumes.
        # NB blocks out (write-through + evict) and NB in (loads), 2 MiB each
        nbk = args.overlap_blocks or max(1, int(0.8 * t_dec * 45e9 / pool.block_bytes))
        nbk = min(nbk, pool.n_blocks // 2, pool.n_host_blocks)
        g = np.arange(pool.n_blocks // 2, pool.n_blocks // 2 + nbk)
        segs = segs_for(g, np.arange(nbk) % pool.n_host_blocks)
        t_swp = run([swaps])
        t_both = run([decode, swaps])
        hidden = 1.0 - max(0.0, t_both - t_dec) / t_swp
        res[{0: "sm", 1: "ce", 2: "auto", 3: "ce2d"}[eng]] = {"blocks_each_way": nbk,
                                           "t_decode_ms": t_dec * 1e3, "t_swap_ms": t_swp * 1e3,
                                           "t_both_ms": t_both * 1e3, "hidden_frac": hidden,
                                           "note": "hidden = 1 - (T_both - T_decode)/T_swap; decode = 32 layers of "
                                                   "paged attention B=64 ctx=2600; swap = NB x 2 MiB out + NB x 2 MiB in, concurrent"}
        print(json.dumps(res), flush=True)
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--max-blocks", type=int, default=65536)
    ap.add_argument("--host-blocks", type=int, default=8192)
    ap.add_argument("--engines", default="0,1")
    ap.add_argument("--overlap", action="store_true")
    ap.add_argument("--overlap-blocks", type=int, default=0, help="0: sized to ~80%% of the decode time")
    ap.add_argument("--out", default="gpurun_out/swap_sweep.json")
    ap.add_argument("--wt-only", action="store_true", help="only the write-through-shaped chunk sizes")
    args = ap.parse_args()
    args.engines = [int(x) for x in args.engines.split(",")]
    if args.wt_only:
        pool = KvPool(64, 64, 32, 8, 128, device=torch.device("cuda"))
        rows = wt_chunks(pool, args)
        Path(args.out).parent.mkdir(parents=True, exist_ok=True)
        Path(args.out).write_text(json.dumps({"wt_chunks": rows}, indent=1))
        return
    sweep(args)


if __name__ == "__main__":
    main()
