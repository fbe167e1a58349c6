"""Real-time serving loop on the GPU with a real (tiny, random-init) decoder:
overlapped compute / evict / load streams, measured durations, GPU selector.
Decisions follow measured timings here, so the checks are the reference's
invariants (conservation, causality, no token loss, ledger) rather than the
event hash."""
import pytest
from conftest import load_golden, pool_blocks, trace_path

pytestmark = pytest.mark.gpu


def _run(cuda, name="c1_tokenflow", engine=0, max_steps=None):
    from paper_2510_02758_b200 import configs
    from paper_2510_02758_b200.costs import CostModel
    from paper_2510_02758_b200.dataplane import GpuDataPlane, KvPool
    from paper_2510_02758_b200.engine import SimConfig
    from paper_2510_02758_b200.model import PagedDecoder
    from paper_2510_02758_b200.realtime import RealtimeEngine
    from paper_2510_02758_b200.scheduler import SchedulerConfig, make_policy
    from paper_2510_02758_b200.workload import load_trace

    g = load_golden("runs", name)
    tr = load_trace(trace_path(g["trace"]))
    shape = configs.TINY
    pool = KvPool(pool_blocks(g["sim"], len(tr.requests)), 4096, shape.n_layers, shape.n_kv_heads, shape.head_dim,
                  device=cuda)
    model = PagedDecoder(shape, device=cuda)
    dp = GpuDataPlane(tr.requests, pool, mode="realtime", kv_source="model", model=model,
                      n_q_heads=shape.n_q_heads, engine=engine)
    eng = RealtimeEngine(tr, make_policy(g["policy"], SchedulerConfig(**g["sched"])), CostModel(**g["cm"]),
                         SimConfig(**g["sim"]), dp, skip_idle=True, max_steps=max_steps)
    res = eng.run()
    return g, eng, res, dp, model


@pytest.mark.parametrize("engine", [0, 1])
def test_realtime_c1_completes_with_invariants(cuda, engine):
    g, eng, res, dp, model = _run(cuda, engine=engine)
    eng._final_invariants(res.records)
    assert all(len(r.gen_times) == r.output_len for r in res.records)
    assert res.total_preemptions > 0 and dp.stats["h2d_tokens"] > 0 and dp.stats["d2h_tokens"] > 0
    # every generated token id came out of the model's paged forward
    for rid, hist in model.history.items():
        assert len(hist) == res.records[rid].output_len
    assert eng.mem_used == 0 and eng.mem_committed == 0
