"""The reference simulator (oracle/refsim, the restatement pinned to the
reference's golden runs) on the C2 burst with the TokenFlow and FCFS
policies: virtual time, the reference cost model.  The CPU-side comparison
point for bench.py --policy fcfs on the B200 data plane.

python tools/refsim_policies.py > profiles/r2_refsim_c2_burst_tokenflow_vs_fcfs.json
"""
import gzip
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import oracle.refsim.sim as simmod  # noqa: E402
from oracle.refsim import metrics as M  # noqa: E402
from oracle.refsim.planner import Costs  # noqa: E402
from oracle.refsim.policy import Knobs, build_policy  # noqa: E402
from oracle.refsim.sim import SimKnobs  # noqa: E402
from oracle.refsim.traces import read_trace  # noqa: E402


def main():
    g = json.load(gzip.open(ROOT / "tests/golden/runs/c2_burst256_s1_tokenflow.json.gz"))
    reqs = read_trace(str(ROOT / "tests/golden/traces" / f"{g['trace']}.csv"))
    runs = {}
    for name in ("tokenflow", "fcfs"):
        out = simmod.Sim(reqs, build_policy(name, Knobs(**g["sched"])), Costs(**g["cm"]), SimKnobs(**g["sim"])).run()
        runs[name] = {"effective_tps": round(M.effective_tps(out.records, out.total_time), 1),
                      "raw_tps": round(M.raw_tps(out.records, out.total_time), 1),
                      "ttft_latency_p99_s": round(M.ttft_latency_p99(out.records), 2),
                      "total_time_s": round(out.total_time, 1), "preemptions": out.total_preemptions}
        if name == "tokenflow":
            runs[name]["event_hash_matches_golden"] = out.event_hash() == g["event_hash"]
    print(json.dumps({"note": "reference simulator (oracle/refsim) on the C2 burst, TokenFlow vs FCFS, virtual time "
                              "with the reference cost model (tools/refsim_policies.py)", "runs": runs}, indent=1))


if __name__ == "__main__":
    main()
