"""Single-process reproduction of one C3 replica's start-up (rank R of N):
trace shard, pool, model, graph capture - for compute-sanitizer."""
import math
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
from paper_2510_02758_b200 import configs  # noqa: E402
from paper_2510_02758_b200.dataplane import GpuDataPlane, KvPool  # noqa: E402
from paper_2510_02758_b200.model import PagedDecoder  # noqa: E402

rank, world = int(sys.argv[1]), int(sys.argv[2])
tr = bench._trace_for_rank(rank, world, "burst")
c2 = configs.C2
shape = c2.model
print("requests", len(tr.requests), "ids", min(r.id for r in tr.requests), max(r.id for r in tr.requests),
      "max_len", max(r.prompt_len + r.output_len for r in tr.requests), flush=True)
dev = torch.device("cuda", 0)
n_blocks = math.ceil(c2.gpu_mem_tokens / 16) + 4 * len(tr.requests) + c2.max_batch + 1
pool = KvPool(n_blocks, 1024, shape.n_layers, shape.n_kv_heads, shape.head_dim, device=dev)
model = PagedDecoder(shape, device=dev, seed=rank)
dp = GpuDataPlane(tr.requests, pool, mode="realtime", kv_source="model", model=model, n_q_heads=shape.n_q_heads,
                  engine=2)
dp.enable_scratch()
print("scratch row", dp.scratch_row, "block", dp.scratch_block, "nlb", dp.nlb, flush=True)
model.enable_graphs(dp)
torch.cuda.synchronize()
print("ok", flush=True)
