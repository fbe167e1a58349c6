"""Offline parity of the GPU selector's REAL-TIME decisions: replay every tick
dumped by ``bench.py --dump-ticks`` (snapshot, policy state before, GPU
decision) through the oracle's restatement of BufferAwarePolicy.on_tick
(oracle/refsim/policy.py) and report mismatches.  CPU only.

python tools/shadow_check.py gpurun_out/ticks.json.gz
"""
import gzip
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle.refsim.policy import Knobs, TokenFlowPolicy, snapshot_from_dict  # noqa: E402
from paper_2510_02758_b200 import configs  # noqa: E402
from paper_2510_02758_b200.scheduler import SchedulerConfig  # noqa: E402


def main():
    d = json.load(gzip.open(sys.argv[1]))
    from dataclasses import asdict

    knobs = Knobs(**asdict(configs.C2.sched_cfg(SchedulerConfig)))
    bad = 0
    for i, t in enumerate(d["ticks"]):
        pol = TokenFlowPolicy(knobs)
        pol._t_prime = {int(k): v for k, v in t.get("t_prime", [])}
        pol.mode = t.get("mode_before", "buffer_aware")
        want = pol.on_tick(snapshot_from_dict(t["snapshot"]))
        got = (t["mode"], t["preempt"], [list(r) for r in t["resume"]], t["prefill_batches"])
        exp = (want.mode, list(want.preempt), [list(r) for r in want.resume], [list(b) for b in want.prefill_batches])
        tp_ok = sorted((int(k), v) for k, v in pol._t_prime.items()) == [(int(k), v) for k, v in t.get("t_prime_after", [])]
        if got != exp or not tp_ok:
            bad += 1
            if bad <= 3:
                print(f"tick {i} t={t['snapshot']['now']:.3f}: GPU {got[0]} pre={got[1]} res={got[2]} pf={got[3]}")
                print(f"      oracle {exp[0]} pre={exp[1]} res={exp[2]} pf={exp[3]} t_prime_ok={tp_ok}")
    print(f"{len(d['ticks'])} ticks, {bad} mismatches")


if __name__ == "__main__":
    main()
