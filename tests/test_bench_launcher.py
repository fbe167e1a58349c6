"""bench.py --gpus N (no launcher): self-launches N ranks over a 127.0.0.1
rendezvous and prints ONE aggregated line - exercised on the CPU with the
gloo dry run, which sends fabricated per-rank window stats through the same
aggregation as a real run (replicas sum tokens and swap traffic,
take the max device / wall time, gather every replica's TTFTs; TP counts
rank 0's tokens once)."""
import json
import subprocess
import sys

import pytest
from conftest import ROOT


def _run(*extra):
    res = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--dry-run", "--steps", "5", "--warmup", "3",
                          *extra], capture_output=True, text=True, timeout=240, cwd=str(ROOT))
    assert res.returncode == 0, res.stderr[-3000:]
    lines = [ln for ln in res.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, res.stdout
    return json.loads(lines[0])


@pytest.mark.parametrize("n", [2, 3])
def test_gpus_n_self_launch_aggregates_replicas(n):
    out = _run("--gpus", str(n))
    assert out["n_gpus"] == n and out["config"]["parallelism"] == f"replicas x{n}"
    eff = sum(100.0 * (r + 1) for r in range(n))
    dev_s = 1.0 + 0.25 * (n - 1)
    assert out["value"] == pytest.approx(eff / dev_s)
    assert out["e2e"]["value"] == pytest.approx(eff / (2.0 + n - 1))
    assert out["swap"]["d2h_tokens"] == sum(1000 * (r + 1) for r in range(n))
    assert out["ttft"]["requests"] == 10 * n and out["ttft"]["of"] == 10 * n
    assert out["ttft"]["p99_s"] == pytest.approx(max(float(r) + 0.9 for r in range(n)))


def test_tensor_parallel_counts_tokens_once():
    out = _run("--gpus", "2", "--config", "c4")
    assert out["scaling"] == "strong" and out["config"]["parallelism"] == "tp2"
    assert out["value"] == pytest.approx(100.0 / 1.25)  # rank 0's tokens / max device time


def test_single_process_line():
    out = _run()
    assert out["n_gpus"] == 1 and out["value"] == pytest.approx(100.0)
