"""Golden wire-format fixtures: the reference experiment runner's output files.

Runs the UNMODIFIED reference experiment runner (``tokensim.cli.run_experiment``,
/root/reference/pkg/src/tokensim/cli.py:354-385) on frozen traces and records
what it writes per cell (cli.py:218-288):

* ``report_<cell>.json``   verbatim text (small)
* ``requests_<cell>.csv``  sha256 + row count + first rows
* ``events_<cell>.jsonl``  sha256 + line count (``SimResult.events_jsonl``)
* ``summary.csv`` / ``summary.txt`` verbatim

into tests/golden/wire/<experiment>.json.gz.  Build container only (imports
the reference); the GPU box reads only the committed fixture.

Usage:  PYTHONDONTWRITEBYTECODE=1 python tools/make_golden_wire.py
"""
from __future__ import annotations

import gzip
import hashlib
import json
import sys
import tempfile
from pathlib import Path

REF_SRC = "/root/reference/pkg/src"
sys.path.insert(0, REF_SRC)
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from tokensim.cli import AblationSpec, ExperimentConfig, parse_config, preset_path, run_experiment  # noqa: E402
from tokensim.costs import CostModel  # noqa: E402
from tokensim.engine import SimConfig  # noqa: E402
from tokensim.metrics import EffectiveThroughputConfig, QosConfig  # noqa: E402
from tokensim.scheduler import SchedulerConfig  # noqa: E402
from tokensim.workload import WorkloadConfig  # noqa: E402

from paper_2510_02758_b200 import configs  # noqa: E402

OUT = ROOT / "tests" / "golden" / "wire"
TRACES = ROOT / "tests" / "golden" / "traces"


def _sha(p: Path) -> str:
    return hashlib.sha256(p.read_bytes()).hexdigest()


def capture(name: str, cfg: ExperimentConfig, cm: CostModel, trace_csv: str) -> None:
    with tempfile.TemporaryDirectory() as td:
        cfg.output_dir = td
        cfg.emit_events = True
        rc = run_experiment(cfg, cm)
        d = Path(td)
        cells = {}
        for rp in sorted(d.glob("report_*.json")):
            cell = rp.stem[len("report_"):]
            req = d / f"requests_{cell}.csv"
            ev = d / f"events_{cell}.jsonl"
            lines = req.read_text().splitlines()
            cells[cell] = {
                "report": rp.read_text(),
                "requests_sha256": _sha(req),
                "requests_rows": len(lines) - 1,
                "requests_head": "\n".join(lines[:6]),
                "events_sha256": _sha(ev),
                "events_lines": len(ev.read_text().splitlines()),
            }
        out = {
            "name": name,
            "trace": trace_csv[: -len(".csv")],
            "rc": rc,
            "policies": cfg.policies,
            "ablations": [a.__dict__ for a in cfg.ablations],
            "seeds": cfg.seeds,
            "sim": cfg.sim.__dict__,
            "sched": cfg.scheduler.__dict__,
            "cm": cm.__dict__,
            "cells": cells,
            "summary_csv": (d / "summary.csv").read_text(),
            "summary_txt": (d / "summary.txt").read_text(),
        }
    OUT.mkdir(parents=True, exist_ok=True)
    data = (json.dumps(out, sort_keys=True, separators=(",", ":")) + "\n").encode()
    with gzip.GzipFile(OUT / f"{name}.json.gz", "wb", mtime=0) as f:
        f.write(data)
    print(f"{name}: rc {rc}, cells {sorted(cells)}")


def main():
    # figure7 preset, replayed from the frozen copy of its trace
    cfg, cm = parse_config(preset_path("figure7"))
    cfg.workload = WorkloadConfig(kind="file", path=str(TRACES / "figure7.csv"))
    capture("figure7", cfg, cm, "figure7.csv")
    # C1 oracle config: four policies + the three memory-management ablations
    c1 = configs.C1
    cfg = ExperimentConfig(
        workload=WorkloadConfig(kind="file", path=str(TRACES / "c1_burst32_s7.csv")),
        sim=c1.sim_cfg(SimConfig),
        scheduler=c1.sched_cfg(SchedulerConfig),
        policies=["tokenflow", "fcfs", "chunked", "qoe"],
        qos=QosConfig(),
        eff=EffectiveThroughputConfig(),
        seeds=[7],
        ablations=[AblationSpec(), AblationSpec("no_overlap", overlap=False),
                   AblationSpec("no_write_through", write_through=False),
                   AblationSpec("no_offload", write_through=False, overlap=False, offload=False)],
    )
    capture("c1", cfg, c1.cost_model(CostModel), "c1_burst32_s7.csv")


if __name__ == "__main__":
    main()
