"""Wire / report formats: the files the product writes for a
serving run are byte-identical to what the reference experiment runner
writes for the same cell (fixtures: tools/make_golden_wire.py, made by the
unmodified tokensim.cli.run_experiment)."""
import hashlib
from pathlib import Path

import pytest
from conftest import load_golden, trace_path

from paper_2510_02758_b200 import report
from paper_2510_02758_b200.costs import CostModel
from paper_2510_02758_b200.engine import SimConfig
from paper_2510_02758_b200.scheduler import SchedulerConfig, make_policy
from paper_2510_02758_b200.workload import load_trace


def _oracle_policy_factory(name, cfg):
    """tokenflow decisions from the oracle restatement (no GPU here); the
    baseline policies are the product's own host policies."""
    if name != "tokenflow":
        return make_policy(name, cfg)
    from dataclasses import asdict

    from oracle.refsim.policy import Knobs, build_policy

    return build_policy(name, Knobs(**asdict(cfg)))


def _check(g, out: Path, events=True):
    for cell, want in g["cells"].items():
        assert (out / f"report_{cell}.json").read_text() == want["report"], cell
        req = (out / f"requests_{cell}.csv").read_bytes()
        assert hashlib.sha256(req).hexdigest() == want["requests_sha256"], cell
        if events:
            ev = (out / f"events_{cell}.jsonl").read_bytes()
            assert hashlib.sha256(ev).hexdigest() == want["events_sha256"], cell
    assert (out / "summary.csv").read_text() == g["summary_csv"]
    assert (out / "summary.txt").read_text() == g["summary_txt"]


def _experiment(g, out, policy_factory, dataplane_factory=None):
    ab = [report.AblationSpec(**a) for a in g["ablations"]]
    rc = report.run_experiment(load_trace(trace_path(g["trace"])), g["policies"], g["seeds"],
                               SchedulerConfig(**g["sched"]), CostModel(**g["cm"]), SimConfig(**g["sim"]), out,
                               ablations=ab, emit_events=True, policy_factory=policy_factory,
                               dataplane_factory=dataplane_factory)
    assert rc == g["rc"]


@pytest.mark.parametrize("name", ["figure7", "c1"])
def test_wire_formats_match_reference(name, tmp_path):
    g = load_golden("wire", name)
    _experiment(g, tmp_path, _oracle_policy_factory)
    _check(g, tmp_path)


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["figure7", "c1"])
def test_wire_formats_gpu_selector_and_dataplane(name, tmp_path):
    """Same files with the GPU selector deciding and the GPU data plane
    moving real KV (replay mode: the run is on the reference's virtual clock),
    plus the B200 transfer audit rows."""
    import math

    from paper_2510_02758_b200.dataplane import GpuDataPlane, KvPool

    g = load_golden("wire", name)
    planes = []

    def dp_factory(tr, sim):
        nb = math.ceil(sim.gpu_mem_tokens / 16) + 4 * len(tr.requests) + sim.max_batch
        pool = KvPool(nb, 4096, n_layers=2, kv_heads=2, head_dim=64, device="cuda:0")
        dp = GpuDataPlane(tr.requests, pool, mode="replay", n_q_heads=4)
        planes.append(dp)
        return dp

    _experiment(g, tmp_path, make_policy, dp_factory)
    _check(g, tmp_path)
    # B200 audit: every chunk row of the event log joined with the copy the
    # data plane launched for it (same direction order, same token count)
    cell = report.run_cell(load_trace(trace_path(g["trace"])), "tokenflow", report.AblationSpec(), g["seeds"][0],
                           SchedulerConfig(**g["sched"]), CostModel(**g["cm"]), SimConfig(**g["sim"]),
                           dataplane_factory=dp_factory)
    n = report.write_transfer_audit(tmp_path / "transfers.csv", cell.result, planes[-1])
    rows = (tmp_path / "transfers.csv").read_text().splitlines()[1:]
    assert n == len(rows) == len(cell.result.chunk_rows()) > 0
    assert all(r.split(",")[8] for r in rows), "a chunk row without a measured copy"
