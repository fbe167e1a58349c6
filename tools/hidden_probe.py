"""Which copy direction costs the decode step time?  Llama3-8B decode graph of
B requests at ctx tokens (synthetic KV) alone, and concurrently with copy-
engine swaps of N blocks per step: d2h only, h2d only, both (bench.py's
measure_hidden method: medians of alternating rounds).

python tools/hidden_probe.py [--batch 128] [--ctx 1500] [--blocks 130]
"""
import argparse
import json
import sys
import types
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402
from paper_2510_02758_b200 import configs  # noqa: E402
from paper_2510_02758_b200.dataplane import GpuDataPlane, KvPool  # noqa: E402
from paper_2510_02758_b200.model import PagedDecoder  # noqa: E402
from paper_2510_02758_b200.workload import RequestSpec  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=128)
    ap.add_argument("--ctx", type=int, default=1500)
    ap.add_argument("--blocks", type=int, default=130)
    args = ap.parse_args()
    dev = torch.device("cuda")
    S = configs.LLAMA3_8B
    B, ctx = args.batch, args.ctx
    reqs = [RequestSpec(i, 0.0, ctx, 64, 20.0) for i in range(B)]
    nlb = (ctx + 64 + 2 + 15) // 16
    pool = KvPool(B * nlb + 2 * args.blocks + 8, 2 * args.blocks + 8, S.n_layers, S.n_kv_heads, S.head_dim,
                  device=dev)
    model = PagedDecoder(S, device=dev)
    dp = GpuDataPlane(reqs, pool, mode="realtime", kv_source="model", model=model, n_q_heads=S.n_q_heads)
    dp.enable_scratch()
    ids = pool.alloc(0, B * nlb)
    dp.table[:B, :nlb] = torch.tensor(ids, dtype=torch.int32, device=dev).view(B, nlb)
    torch.cuda.synchronize()
    model.enable_graphs(dp, buckets=(B,), prefill_buckets=0)
    for r in range(B):
        model.pending[r] = 1
    eng = types.SimpleNamespace(state={r: types.SimpleNamespace(kv=types.SimpleNamespace(total_kv=ctx))
                                       for r in range(B)})
    rids = list(range(B))
    out = {}
    for name, (o, i) in {"d2h": (args.blocks, 0), "h2d": (0, args.blocks), "both": (args.blocks, args.blocks)}.items():
        out[name] = bench.measure_hidden(model, dp, eng, rids, o, i)
        print(name, json.dumps(out[name]), flush=True)
    Path("gpurun_out").mkdir(exist_ok=True)
    Path("gpurun_out/hidden_probe.json").write_text(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
