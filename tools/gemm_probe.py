"""Decode-step projection GEMMs on B200: cuBLAS addmm (residual fused in the
epilogue, the current path) vs plain mm at the C2 decode shapes, CUDA-graph
replayed (how the decode step runs them).

python tools/gemm_probe.py [--out gpurun_out/gemm_probe.json]
"""
import argparse
import json
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def time_graph(fn, reps=200):
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(3):
            fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(10):
            fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):  # replay on the stream the events are recorded on
        e0.record(s)
        for _ in range(reps // 10):
            g.replay()
        e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3  # us


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="gpurun_out/gemm_probe.json")
    ap.add_argument("--blas", default="default", choices=["default", "cublas", "cublaslt"])
    ap.add_argument("--ms", default="32,64,96,128", help="comma list of GEMM row counts (decode batch buckets)")
    args = ap.parse_args()
    if args.blas != "default":
        torch.backends.cuda.preferred_blas_library(args.blas)
    dev = torch.device("cuda")
    bf = torch.bfloat16
    rows = []
    # Llama3-8B: wqkv 4096x6144, wo 4096x4096, wgu 4096x28672, wd 14336x4096
    for M in (int(m) for m in args.ms.split(",")):
        for name, K, N in (("wqkv", 4096, 6144), ("wo", 4096, 4096), ("wgu", 4096, 28672), ("wd", 14336, 4096)):
            # distinct weight copies so consecutive launches do not hit L2
            ws = [torch.randn(K, N, device=dev, dtype=bf) * 0.02 for _ in range(4)]
            a = torch.randn(M, K, device=dev, dtype=bf)
            x = torch.randn(M, N, device=dev, dtype=bf)
            out = torch.empty(M, N, device=dev, dtype=bf)
            it = {"i": 0}

            def mm():
                it["i"] = (it["i"] + 1) % 4
                torch.mm(a, ws[it["i"]], out=out)

            def addmm():
                it["i"] = (it["i"] + 1) % 4
                torch.addmm(x, a, ws[it["i"]], out=out)

            t_mm, t_add = time_graph(mm), time_graph(addmm)
            wbytes = K * N * 2
            rows.append({"blas": args.blas, "M": M, "gemm": name, "K": K, "N": N, "mm_us": round(t_mm, 2), "addmm_us": round(t_add, 2),
                         "mm_gbs": round(wbytes / t_mm / 1e3, 1), "addmm_gbs": round(wbytes / t_add / 1e3, 1)})
            print(json.dumps(rows[-1]), flush=True)
            del ws
    Path(args.out).parent.mkdir(exist_ok=True)
    Path(args.out).write_text(json.dumps(rows, indent=1))


if __name__ == "__main__":
    main()
