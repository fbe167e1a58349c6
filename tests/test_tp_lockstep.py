"""C4 control path on CPU: two gloo ranks run the real-time engine on the same
trace with DIFFERENT per-rank device timings (a timed stand-in data plane
whose job durations carry rank-specific jitter).  With ``Lockstep`` the
ranks agree completions and clock every loop iteration, so both take the
identical event sequence, decisions and chunk rows; without it the same
jitter drives them apart.  Decisions come from the oracle's policy
restatement here (the GPU selector's bit-exactness is a -m gpu test)."""
import os
import random
import socket
import time

import torch.distributed as dist
import torch.multiprocessing as mp
from conftest import load_golden, trace_path


class FakeEvent:
    def __init__(self, t_done):
        self.t = t_done

    def query(self):
        return time.perf_counter() >= self.t

    def synchronize(self):
        while not self.query():
            time.sleep(max(0.0, self.t - time.perf_counter()))

    def elapsed_time(self, other):
        return (other.t - self.t) * 1e3


class TimedPlane:
    """Three in-order lanes (compute / d2h / h2d) whose jobs take a
    deterministic cost x a rank-specific random factor of wall time."""

    mode = "realtime"
    fused_wt = False

    def __init__(self, rank, jitter):
        self.rng = random.Random(1000 + rank)
        self.jitter = jitter
        self.busy = {"c": 0.0, "d2h": 0.0, "h2d": 0.0}
        self.stats = {}

    def _run(self, lane, cost):
        cost *= 1.0 + self.jitter * (2 * self.rng.random() - 1)
        start = max(time.perf_counter(), self.busy[lane])
        self.busy[lane] = start + cost
        return FakeEvent(start), FakeEvent(self.busy[lane])

    def record_event(self):
        return FakeEvent(max(time.perf_counter(), self.busy["c"]))  # the compute lane's current tail

    def fill_start(self, job, eng):
        self._run("c", 2e-3 + 2e-6 * sum(job.reserve.values()))

    def decode_start(self, batch, eng):
        self._run("c", 1e-3 + 1e-4 * len(batch))

    def d2h_start(self, ch, eng):
        return self._run("d2h", 2e-4 + 4e-6 * ch.tokens)

    def h2d_start(self, ch, eng):
        return self._run("h2d", 2e-4 + 4e-6 * ch.tokens)

    def synchronize(self):
        FakeEvent(max(self.busy.values())).synchronize()

    def fill_done(self, rid): pass
    def decode_done(self, batch, made): pass
    def d2h_done(self, ch, alive): pass
    def release_prefix(self, rid, n): pass
    def cancel_evicts(self, rid): pass
    def drop_gpu(self, rid): pass
    def drop_host(self, rid): pass
    def finish(self, rid): pass
    def audit(self, eng): pass


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, lockstep, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle.refsim.policy import Knobs, build_policy
    from paper_2510_02758_b200 import workload
    from paper_2510_02758_b200.costs import CostModel
    from paper_2510_02758_b200.engine import SimConfig
    from paper_2510_02758_b200.realtime import RealtimeEngine
    from paper_2510_02758_b200.tp import Lockstep

    g = load_golden("runs", "c1_tokenflow")
    tr = workload.load_trace(trace_path(g["trace"]))
    ls = Lockstep() if lockstep else None
    eng = RealtimeEngine(tr, build_policy("tokenflow", Knobs(**g["sched"])), CostModel(**g["cm"]),
                         SimConfig(**{**g["sim"], "debug_checks": False}), TimedPlane(rank, 0.6),
                         skip_idle=True, lockstep=ls)
    res = eng.run()
    same = ls.same(res.event_hash()) if ls else None
    summary = {"rank": rank, "hash": res.event_hash(), "decisions": res.decision_log, "chunks": res.chunk_rows(),
               "pre": res.total_preemptions, "same": same, "calls": ls.calls if ls else 0,
               "steps": len(eng.steps)}
    gathered = [None] * world
    dist.all_gather_object(gathered, summary)
    if rank == 0:
        out.put(gathered)
    dist.barrier()
    dist.destroy_process_group()


def _run(lockstep):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, lockstep, q)) for r in range(world)]
    for p in procs:
        p.start()
    gathered = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    return gathered


def test_lockstep_ranks_take_identical_decisions():
    a, b = _run(lockstep=True)
    assert a["steps"] > 100 and a["pre"] > 0, "the run must exercise preemption / swap"
    assert a["same"] and b["same"]
    assert a["hash"] == b["hash"]
    assert a["decisions"] == b["decisions"]
    assert a["chunks"] == b["chunks"]
    assert a["calls"] == b["calls"] > 0


def test_without_lockstep_jitter_diverges():
    a, b = _run(lockstep=False)
    assert a["hash"] != b["hash"]


def test_tp_shards_partition_the_tp1_weights():
    """Every TP shard's weights are exact slices of the TP=1 weights (q/k/v
    heads, o_proj rows, gate/up columns, down_proj rows; Qwen2 qkv bias)."""
    import dataclasses

    import torch

    from paper_2510_02758_b200 import configs, model, tp

    s = dataclasses.replace(configs.TINY, qkv_bias=True)
    hq, hkv, hd, ffn = s.n_q_heads, s.n_kv_heads, s.head_dim, s.ffn
    full = model.PagedDecoder(s, device="cpu", seed=3)
    for size in (2,):
        for r in range(size):
            m = model.PagedDecoder(s, device="cpu", seed=3, tp=tp.TpGroup(r, size))
            q, k, f = hq // size, hkv // size, ffn // size
            for L, F in zip(m.layers, full.layers):
                cols = list(range(r * q * hd, (r + 1) * q * hd)) + \
                    list(range((hq + r * k) * hd, (hq + (r + 1) * k) * hd)) + \
                    list(range((hq + hkv + r * k) * hd, (hq + hkv + (r + 1) * k) * hd))
                assert torch.equal(L["wqkv"], F["wqkv"][:, cols])
                assert torch.equal(L["bqkv"], F["bqkv"][cols])
                assert torch.equal(L["wo"], F["wo"][r * q * hd:(r + 1) * q * hd])
                gu = list(range(r * f, (r + 1) * f)) + list(range(ffn + r * f, ffn + (r + 1) * f))
                assert torch.equal(L["wgu"], F["wgu"][:, gu])
                assert torch.equal(L["wd"], F["wd"][r * f:(r + 1) * f])
            assert torch.equal(m.embed, full.embed) and torch.equal(m.lm_head, full.lm_head)
