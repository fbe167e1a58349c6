"""N>1 path on CPU: two gloo ranks each serve their request shard (i mod N)
with their own engine; the gathered job covers every request exactly once
and the job metrics use the slowest replica's time.  The scheduling logic is
the oracle restatement here (the GPU selector is covered by -m gpu tests)."""
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp
from conftest import load_golden, trace_path

from paper_2510_02758_b200 import metrics, replicas, workload


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle.refsim.policy import Knobs, build_policy
    from paper_2510_02758_b200.costs import CostModel
    from paper_2510_02758_b200.engine import Engine, SimConfig

    g = load_golden("runs", "c1_tokenflow")
    full = workload.load_trace(trace_path(g["trace"]))
    scaled = replicas.scale_trace(full, world)
    local, gids = replicas.partition(scaled, rank, world)
    res = Engine(local, build_policy("tokenflow", Knobs(**g["sched"])), CostModel(**g["cm"]),
                 SimConfig(**g["sim"])).run()
    summary = {"rank": rank, "gids": gids, "records": res.records, "total_time": res.total_time,
               "hash": res.event_hash()}
    gathered = [None] * world
    dist.all_gather_object(gathered, summary)
    if rank == 0:
        out.put(gathered)
    dist.barrier()
    dist.destroy_process_group()


def test_two_replicas_gloo():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    gathered = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    g = load_golden("runs", "c1_tokenflow")
    full = workload.load_trace(trace_path(g["trace"]))
    gids = sorted(i for s in gathered for i in s["gids"])
    assert gids == list(range(world * len(full.requests)))
    # weak scaling: each replica serves exactly the C1 burst -> reference behaviour per replica
    for s in gathered:
        assert s["hash"] == g["event_hash"]
    job = replicas.merge(gathered)
    eff = metrics.effective_throughput(job["records"], job["total_time"], metrics.EffectiveThroughputConfig())
    assert eff == pytest.approx(world * g["metrics"]["effective_tps"])


def test_partition_round_robin():
    tr = workload.load_trace(trace_path("c2_poisson256_s1"))
    seen = []
    for r in range(4):
        local, gids = replicas.partition(tr, r, 4)
        assert [x.id for x in local.requests] == list(range(len(local.requests)))
        assert all(g % 4 == r for g in gids)
        seen += gids
    assert sorted(seen) == list(range(256))
    with pytest.raises(ValueError):
        replicas.partition(tr, 4, 4)
