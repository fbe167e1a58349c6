"""Does splitting the gate/up GEMM along N change cuBLAS's kernel choice at
decode batch sizes?  Times (CUDA graph, 50 launches, 4 weight copies so no L2
reuse) wgu [4096 x 28672] as one GEMM vs 2 x N=14336 vs 4 x N=7168, and wqkv at
M rows vs padded to 128 rows.

python tools/gemm_split_probe.py > gpurun_out/gemm_split.json
"""
import json

import torch


def time_graph(fn, reps=50):
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(3):
            fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(reps):
            fn()
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / (5 * reps) * 1e3


def main():
    dev, bf = torch.device("cuda"), torch.bfloat16
    rows = []
    for M in (64, 80, 96, 112, 128):
        a = torch.randn(128, 4096, device=dev, dtype=bf)
        for parts in (1, 2, 4):
            n = 28672 // parts
            ws = [[torch.randn(4096, n, device=dev, dtype=bf) * 0.02 for _ in range(parts)] for _ in range(4)]
            outs = [torch.empty(M, n, device=dev, dtype=bf) for _ in range(parts)]
            it = {"i": 0}

            def f():
                it["i"] = (it["i"] + 1) % 4
                for w, o in zip(ws[it["i"]], outs):
                    torch.mm(a[:M], w, out=o)

            rows.append({"gemm": "wgu", "M": M, "parts": parts, "us": round(time_graph(f), 2)})
            print(json.dumps(rows[-1]), flush=True)
            del ws
        for Mg in sorted({M, 128}):
            ws = [torch.randn(4096, 6144, device=dev, dtype=bf) * 0.02 for _ in range(4)]
            o = torch.empty(Mg, 6144, device=dev, dtype=bf)
            it = {"i": 0}

            def f():
                it["i"] = (it["i"] + 1) % 4
                torch.mm(a[:Mg], ws[it["i"]], out=o)

            rows.append({"gemm": "wqkv", "M": M, "M_gemm": Mg, "us": round(time_graph(f), 2)})
            print(json.dumps(rows[-1]), flush=True)
            del ws
    print(json.dumps(rows))


if __name__ == "__main__":
    main()
