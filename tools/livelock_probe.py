"""Serve the C2 burst in real time with a TIMED STAND-IN data plane (no model,
no KV; job durations from B200-calibrated formulas) and a chosen policy
implementation: ``gpu`` (BufferAwarePolicy -> the CUDA selector) or
``oracle`` (the CPU restatement).  Separates policy-implementation effects
from data-plane effects in the real-time serving loop.

python tools/livelock_probe.py gpu|oracle [--fused 0|1] [--max-wall 300]
"""
import argparse
import collections
import json
import sys
import time
from dataclasses import asdict
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

from test_tp_lockstep import TimedPlane  # noqa: E402

from paper_2510_02758_b200 import configs  # noqa: E402
from paper_2510_02758_b200.costs import CostModel  # noqa: E402
from paper_2510_02758_b200.engine import SimConfig  # noqa: E402
from paper_2510_02758_b200.realtime import RealtimeEngine  # noqa: E402
from paper_2510_02758_b200.scheduler import BufferAwarePolicy, SchedulerConfig  # noqa: E402
from paper_2510_02758_b200.workload import load_trace  # noqa: E402


def _spin(ms):
    if ms > 0:
        t = time.perf_counter() + ms / 1e3
        while time.perf_counter() < t:
            pass


class B200Plane(TimedPlane):
    def __init__(self, fused, host_ms=(0.0, 0.0, 0.0)):
        super().__init__(0, 0.0)
        self.fused_wt = fused
        self.host_decode, self.host_copy, self.host_fill = host_ms

    def host_frontier(self, rid, cs, total):
        return total

    def fill_start(self, job, eng):
        self._run("c", 1e-3 + 1.76e-5 * job.process_tokens)
        _spin(self.host_fill)

    def decode_start(self, batch, eng):
        self._run("c", 1.5e-3 + 1.5e-5 * len(batch) + 1.2e-8 * sum(eng.state[r].kv.total_kv for r in batch))
        _spin(self.host_decode)

    def d2h_start(self, ch, eng):
        ev = self._run("d2h", 1e-5 + ch.tokens / 420000)
        _spin(self.host_copy)
        return ev

    def h2d_start(self, ch, eng):
        ev = self._run("h2d", 1e-5 + ch.tokens / 420000)
        _spin(self.host_copy)
        return ev


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("policy", choices=["gpu", "oracle"])
    ap.add_argument("--fused", type=int, default=0)
    ap.add_argument("--max-wall", type=float, default=300)
    ap.add_argument("--arrivals", default="burst")
    ap.add_argument("--host-ms", default="0,0,0", help="host time spent per decode / copy / prefill launch (ms)")
    args = ap.parse_args()
    c2 = configs.C2
    name = "c2_burst256_s1" if args.arrivals == "burst" else "c2_poisson256_s1"
    tr = load_trace(str(ROOT / "tests" / "golden" / "traces" / f"{name}.csv"))
    scfg = c2.sched_cfg(SchedulerConfig)
    if args.policy == "gpu":
        pol = BufferAwarePolicy(scfg)
    else:
        from oracle.refsim.policy import Knobs, build_policy

        pol = build_policy("tokenflow", Knobs(**asdict(scfg)))
    eng = RealtimeEngine(tr, pol, c2.cost_model(CostModel), c2.sim_cfg(SimConfig, debug_checks=False),
                         B200Plane(bool(args.fused), tuple(float(x) for x in args.host_ms.split(","))), skip_idle=True, max_wall_s=args.max_wall)
    t0 = time.time()
    res = eng.run()
    inv = "ok"
    if not eng.truncated:
        try:
            eng._final_invariants(res.records)
        except Exception as e:  # noqa: BLE001
            inv = f"{type(e).__name__}: {e}"
    st = collections.Counter(s.status for s in eng.state.values())
    print(json.dumps({"policy": args.policy, "fused": args.fused, "truncated": eng.truncated,
                      "total_time": res.total_time, "preemptions": res.total_preemptions,
                      "recomputes": res.total_recomputes, "steps": len(eng.steps), "wall": time.time() - t0,
                      "status": dict(st), "event_hash": res.event_hash()[:16], "invariants": inv}))


if __name__ == "__main__":
    main()
