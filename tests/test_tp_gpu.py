"""C4 tensor-parallel sharding on ONE GPU: the TP=2 model (two shards driven by
two threads, their all-reduce done through shared memory on the same device)
writes the same paged KV and computes the same tokens as the TP=1 model -
i.e. a TP model is the TP=1 model partitioned (model.PagedDecoder(tp=...)).
The NCCL transport itself is torch.distributed's; only the partitioning and
the residual-on-rank-0 all-reduce placement are under test."""
import threading

import pytest

pytestmark = pytest.mark.gpu


class ThreadTp:
    """TpGroup stand-in: ranks are threads on one device; all_reduce sums the
    ranks' tensors in rank order (every rank computes the same sum)."""

    def __init__(self, rank, size, shared):
        self.rank, self.size, self.sh = rank, size, shared

    def all_reduce(self, x):
        import torch

        torch.cuda.current_stream().synchronize()
        self.sh["buf"][self.rank] = x
        self.sh["bar"].wait()
        acc = self.sh["buf"][0].float()
        for r in range(1, self.size):
            acc = acc + self.sh["buf"][r].float()
        torch.cuda.current_stream().synchronize()
        self.sh["bar"].wait()
        x.copy_(acc.to(x.dtype))
        torch.cuda.current_stream().synchronize()
        return x


def _setup(cuda, shape, tp, n_req, nlb):
    import torch

    from paper_2510_02758_b200.dataplane import GpuDataPlane, KvPool
    from paper_2510_02758_b200.model import PagedDecoder
    from paper_2510_02758_b200.workload import RequestSpec

    size = tp.size if tp else 1
    reqs = [RequestSpec(i, 0.0, 40 + 7 * i, 50, 20.0) for i in range(n_req)]
    pool = KvPool(n_req * nlb + 2, 1, shape.n_layers, shape.n_kv_heads // size, shape.head_dim, device=cuda)
    pool.gpu.zero_()
    model = PagedDecoder(shape, device=cuda, seed=3, tp=tp)
    dp = GpuDataPlane(reqs, pool, mode="realtime", kv_source="model", model=model,
                      n_q_heads=shape.n_q_heads // size)
    dp.table[:n_req, :nlb] = torch.arange(n_req * nlb, dtype=torch.int32, device=cuda).view(n_req, nlb)
    torch.cuda.synchronize()  # default-stream setup before the data plane's non-blocking streams
    return model, dp, pool


@pytest.mark.parametrize("qkv_bias", [False, True])
def test_tp2_equals_tp1(cuda, qkv_bias):
    import dataclasses

    import torch

    from paper_2510_02758_b200 import configs

    shape = dataclasses.replace(configs.TINY, qkv_bias=qkv_bias)
    n_req, nlb = 4, 5
    seqs = [(i, torch.randint(0, shape.vocab, (30 + 9 * i,), generator=torch.Generator().manual_seed(i)), 0)
            for i in range(n_req)]
    m1, dp1, pool1 = _setup(cuda, shape, None, n_req, nlb)
    m1.keep_logits = True
    with torch.cuda.stream(dp1.s_compute):
        tok1 = m1._prefill_batch(dp1, seqs, dp1.s_compute)
    torch.cuda.synchronize()

    shared = {"buf": [None, None], "bar": threading.Barrier(2)}
    outs = [None, None]
    shards = [_setup(cuda, shape, ThreadTp(r, 2, shared), n_req, nlb) for r in range(2)]

    def run(r):
        m, dp, _ = shards[r]
        m.keep_logits = True
        with torch.cuda.stream(dp.s_compute):
            outs[r] = m._prefill_batch(dp, seqs, dp.s_compute)
        dp.s_compute.synchronize()

    th = [threading.Thread(target=run, args=(r,)) for r in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    torch.cuda.synchronize()
    assert torch.equal(outs[0], outs[1]), "TP ranks disagree on the sampled tokens"
    # logits: the TP=2 sum of two bf16 partial projections vs one fp32-accumulated
    # GEMM -> per sequence max|l_tp - l_1| <= 2e-2 * max|l_1| (+ bf16 floor)
    l1 = m1.last_logits.float()
    for r in range(2):
        lr = shards[r][0].last_logits.float()
        assert torch.equal(lr, shards[0][0].last_logits.float()), "TP ranks disagree on the logits"
        err = (lr - l1).abs().amax(dim=-1)
        tol = 2e-2 * l1.abs().amax(dim=-1) + 2.0 ** -8
        assert bool((err <= tol).all()), f"TP=2 logits off by {err.tolist()} (tol {tol.tolist()})"
    # greedy tokens agree wherever the TP=1 top-2 margin exceeds that tolerance
    top2 = l1.topk(2, dim=-1).values
    clear = (top2[:, 0] - top2[:, 1]) > 2 * tol
    assert torch.equal(outs[0][clear], tok1[clear])
    # KV: shard r's pool holds kv head r of the TP=1 pool, layer by layer
    v1 = pool1.gpu_view().view(torch.bfloat16).float()
    for r in range(2):
        vr = shards[r][2].gpu_view().view(torch.bfloat16).float()
        ref = v1[:, :, :, r:r + 1]
        used = n_req * nlb
        err = (vr[:used] - ref[:used]).abs().max().item()
        assert err <= 2e-2 * max(1.0, ref[:used].abs().max().item()), f"rank {r} KV differs by {err}"
        # layer 0 K/V do not depend on any all-reduce: equal up to GEMM blocking
        e0 = (vr[:used, 0] - ref[:used, 0]).abs().max().item()
        assert e0 <= 1e-2 * max(1.0, ref[:used, 0].abs().max().item())


def test_prefill_varlen_matches_per_sequence_sdpa(cuda):
    """The batched prefill (one varlen flash-attention call per layer over all
    sequences) writes the same paged KV and picks the same next tokens as a
    per-sequence causal torch SDPA reference."""
    import torch
    import torch.nn.functional as F

    from paper_2510_02758_b200 import configs
    from paper_2510_02758_b200 import model as model_mod

    def ref_varlen(q, k, v, cu, cu_k, max_q, max_k, window_size=(-1, 0)):
        outs = []
        c = cu.tolist()
        for a, b in zip(c[:-1], c[1:]):
            qi, ki, vi = (t[a:b].transpose(0, 1)[None].float() for t in (q, k, v))
            outs.append(F.scaled_dot_product_attention(qi, ki, vi, is_causal=True)[0].transpose(0, 1).to(q.dtype))
        return torch.cat(outs)

    shape = configs.TINY
    n_req, nlb = 4, 5
    seqs = [(i, torch.randint(0, shape.vocab, (20 + 13 * i,), generator=torch.Generator().manual_seed(i)), 0)
            for i in range(n_req)]
    m1, dp1, pool1 = _setup(cuda, shape, None, n_req, nlb)
    m1.keep_logits = True
    with torch.cuda.stream(dp1.s_compute):
        tok_b = m1._prefill_batch(dp1, seqs, dp1.s_compute)
    torch.cuda.synchronize()
    m2, dp2, pool2 = _setup(cuda, shape, None, n_req, nlb)
    m2.keep_logits = True
    orig = model_mod.varlen_attn
    model_mod.varlen_attn = ref_varlen
    try:
        with torch.cuda.stream(dp2.s_compute):
            tok_r = m2._prefill_batch(dp2, seqs, dp2.s_compute)
        torch.cuda.synchronize()
    finally:
        model_mod.varlen_attn = orig
    lb, lr = m1.last_logits.float(), m2.last_logits.float()
    err = (lb - lr).abs().amax(dim=-1)
    tol = 2e-2 * lr.abs().amax(dim=-1) + 2.0 ** -8
    assert bool((err <= tol).all()), f"varlen prefill logits off by {err.tolist()} (tol {tol.tolist()})"
    top2 = lr.topk(2, dim=-1).values
    clear = (top2[:, 0] - top2[:, 1]) > 2 * tol
    assert torch.equal(tok_b[clear], tok_r[clear])
    used = n_req * nlb
    a = pool1.gpu_view()[:used].view(torch.bfloat16).float()
    b = pool2.gpu_view()[:used].view(torch.bfloat16).float()
    assert (a - b).abs().max().item() <= 2e-2 * max(1.0, b.abs().max().item())


def test_recompute_prefill_graph_matches_eager(cuda):
    """A recompute prefill replayed from its token-bucket CUDA graph (padded
    tail to the scratch row) writes the same paged KV as the eager prefill."""
    import torch

    from paper_2510_02758_b200 import configs
    from paper_2510_02758_b200.dataplane import GpuDataPlane, KvPool
    from paper_2510_02758_b200.model import PagedDecoder
    from paper_2510_02758_b200.workload import RequestSpec

    shape = configs.TINY
    reqs = [RequestSpec(i, 0.0, 60, 60, 20.0) for i in range(2)]
    nlb = 8
    outs = []
    for use_graph in (False, True):
        pool = KvPool(2 * nlb + 4, 1, shape.n_layers, shape.n_kv_heads, shape.head_dim, device=cuda)
        pool.gpu.zero_()
        model = PagedDecoder(shape, device=cuda, seed=5)
        dp = GpuDataPlane(reqs, pool, mode="realtime", kv_source="model", model=model, n_q_heads=shape.n_q_heads)
        dp.enable_scratch()  # takes a block from the allocator before the manual mapping below
        sb = dp.scratch_block
        free = [b for b in range(pool.n_blocks) if b != sb]
        dp.table[:2, :nlb] = torch.tensor(free[: 2 * nlb], dtype=torch.int32, device=cuda).view(2, nlb)
        torch.cuda.synchronize()  # default-stream setup before the compute stream
        toks = torch.randint(0, shape.vocab, (77,), generator=torch.Generator().manual_seed(3))
        st = dp.s_compute
        if use_graph:
            model.enable_graphs(dp, buckets=(8,), prefill_buckets=32)
            with torch.cuda.stream(st):
                model._recompute_graph(dp, 1, toks, st)
        else:
            with torch.cuda.stream(st):
                model._prefill_batch(dp, [(1, toks, 0)], st)
        torch.cuda.synchronize()
        blocks = dp.table[1, : (77 + 15) // 16].long()
        v = pool.gpu_view()[blocks].view(torch.bfloat16).float()
        outs.append(v.reshape(v.shape[0], shape.n_layers, 2, shape.n_kv_heads, 16, shape.head_dim))
    a, b = outs
    # positions 0..76 (the last block is partial)
    a = a.permute(0, 4, 1, 2, 3, 5).reshape(-1, shape.n_layers, 2, shape.n_kv_heads, shape.head_dim)[:77]
    b = b.permute(0, 4, 1, 2, 3, 5).reshape(-1, shape.n_layers, 2, shape.n_kv_heads, shape.head_dim)[:77]
    # padding changes the GEMM shapes (and so cuBLAS blocking): equal to bf16 noise
    assert (a - b).abs().max().item() <= 2e-2 * max(1.0, a.abs().max().item())


def test_prompt_prefill_graph_matches_eager(cuda):
    """A multi-request prompt prefill replayed from its token-bucket CUDA graph
    (real sequences, zero-length unused slots, a padding sequence on the
    scratch row) writes the same paged KV as the eager varlen prefill and
    picks the same first tokens wherever the eager logits are not a near tie."""
    import torch

    from paper_2510_02758_b200 import configs
    from paper_2510_02758_b200.dataplane import GpuDataPlane, KvPool
    from paper_2510_02758_b200.model import PagedDecoder
    from paper_2510_02758_b200.workload import RequestSpec

    shape = configs.TINY
    n_req, nlb = 3, 8
    reqs = [RequestSpec(i, 0.0, 90, 30, 20.0) for i in range(n_req)]
    g = torch.Generator().manual_seed(11)
    seqs = [(i, torch.randint(0, shape.vocab, (n,), generator=g), 0) for i, n in enumerate((37, 60, 5))]
    res = []
    for use_graph in (False, True):
        pool = KvPool(n_req * nlb + 4, 1, shape.n_layers, shape.n_kv_heads, shape.head_dim, device=cuda)
        pool.gpu.zero_()
        model = PagedDecoder(shape, device=cuda, seed=5)
        dp = GpuDataPlane(reqs, pool, mode="realtime", kv_source="model", model=model, n_q_heads=shape.n_q_heads)
        dp.enable_scratch()
        free = [b for b in range(pool.n_blocks) if b != dp.scratch_block]
        dp.table[:n_req, :nlb] = torch.tensor(free[: n_req * nlb], dtype=torch.int32, device=cuda).view(n_req, nlb)
        torch.cuda.synchronize()  # default-stream setup before the compute stream
        st = dp.s_compute
        if use_graph:
            model.enable_graphs(dp, buckets=(8,), prefill_buckets=32)
            assert model._prefill_fits_graph(seqs)
            with torch.cuda.stream(st):
                tok = model._prefill_graph(dp, seqs, st).clone()
        else:
            model.keep_logits = True
            with torch.cuda.stream(st):
                tok = model._prefill_batch(dp, seqs, st)
            logits = model.last_logits.float()
        torch.cuda.synchronize()
        kv = []
        for rid, t, _ in seqs:
            n = t.numel()
            blocks = dp.table[rid, : (n + 15) // 16].long()
            v = pool.gpu_view()[blocks].view(torch.bfloat16).float()
            v = v.permute(0, 4, 1, 2, 3, 5).reshape(-1, shape.n_layers, 2, shape.n_kv_heads, shape.head_dim)[:n]
            kv.append(v)
        res.append((tok, kv))
    (t_e, kv_e), (t_g, kv_g) = res
    for a, b in zip(kv_e, kv_g):
        assert (a - b).abs().max().item() <= 2e-2 * max(1.0, a.abs().max().item())
    top2 = logits.topk(2, dim=-1).values
    clear = (top2[:, 0] - top2[:, 1]) > 2e-2 * logits.abs().amax(-1) * 2
    assert torch.equal(t_e[clear], t_g[clear])


def _tp2_worker(rank, port, out):
    import os

    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    # both ranks share cuda:0 here, so the data-path all-reduce runs over gloo
    # (NCCL needs one device per rank); the kernels and engine are the product's
    dist.init_process_group("gloo", rank=rank, world_size=2)
    from conftest import load_golden, pool_blocks, trace_path

    from paper_2510_02758_b200 import configs
    from paper_2510_02758_b200.costs import CostModel
    from paper_2510_02758_b200.dataplane import GpuDataPlane, KvPool
    from paper_2510_02758_b200.engine import SimConfig
    from paper_2510_02758_b200.model import PagedDecoder
    from paper_2510_02758_b200.realtime import RealtimeEngine
    from paper_2510_02758_b200.scheduler import SchedulerConfig, make_policy
    from paper_2510_02758_b200.tp import Lockstep, TpGroup
    from paper_2510_02758_b200.workload import load_trace

    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    g = load_golden("runs", "c1_tokenflow")
    tr = load_trace(trace_path(g["trace"]))
    shape = configs.TINY
    pool = KvPool(pool_blocks(g["sim"], len(tr.requests)), 4096, shape.n_layers, shape.n_kv_heads // 2,
                  shape.head_dim, device=dev)
    model = PagedDecoder(shape, device=dev, seed=0, tp=TpGroup(rank, 2))
    dp = GpuDataPlane(tr.requests, pool, mode="realtime", kv_source="model", model=model,
                      n_q_heads=shape.n_q_heads // 2, engine=2)
    ls = Lockstep(dist.new_group(backend="gloo"))
    eng = RealtimeEngine(tr, make_policy("tokenflow", SchedulerConfig(**g["sched"])), CostModel(**g["cm"]),
                         SimConfig(**g["sim"]), dp, skip_idle=True, lockstep=ls)
    res = eng.run()
    eng._final_invariants(res.records)
    same = ls.same(res.event_hash())
    hist = {r: list(v) for r, v in model.history.items()}
    parts = [None, None]
    dist.all_gather_object(parts, {"hash": res.event_hash(), "same": same, "pre": res.total_preemptions,
                                   "h2d": dp.stats["h2d_tokens"], "hist": hist})
    if rank == 0:
        out.put(parts)
    dist.barrier()
    dist.destroy_process_group()


def test_tp2_lockstep_serving_on_one_gpu(cuda):
    """C4 end to end with TP=2 (two processes sharing one B200): sharded model,
    per-rank KV pools and swaps, lockstep real-time engines, GPU selector.
    Both ranks must take the identical event sequence and emit the same tokens."""
    import socket

    import torch.multiprocessing as mp

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_tp2_worker, args=(r, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    a, b = q.get(timeout=900)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert a["same"] and b["same"] and a["hash"] == b["hash"]
    assert a["pre"] > 0 and a["h2d"] > 0
    assert a["hist"] == b["hist"], "TP ranks emitted different tokens"
