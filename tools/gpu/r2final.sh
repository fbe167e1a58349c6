# round 2 final validation: full GPU suite, smoke, the driver command (interval steps), the round-1 iteration window,
# the ncu launch list of the driver command, reference arm
T=${1:-r2final}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 --timeout_method thread --durations 5 > gpurun_out/${T}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest.log
grep -E "FAILED|ERROR|Timeout|passed|failed|rc=" gpurun_out/${T}_pytest.log | tail -n 8
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_smoke.log
tail -n 2 gpurun_out/${T}_smoke.log
t0=$(date +%s); timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/${T}_bench20.json 2> gpurun_out/${T}_bench20.err; echo "rc=$? wall=$(( $(date +%s) - t0 ))s" >> gpurun_out/${T}_bench20.err
t0=$(date +%s); timeout 900 python bench.py --step-unit iter --steps 20 --warmup 5 --no-cpu-baseline --no-selector > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; echo "rc=$? wall=$(( $(date +%s) - t0 ))s" >> gpurun_out/${T}_bench.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --nvtx --nvtx-include bench_timed/ -c 1100 --csv --log-file gpurun_out/${T}_launches.csv python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-selector --ttft 0 --swap-steps 0 > gpurun_out/${T}_ncu_bench.json 2> gpurun_out/${T}_ncu_bench.err; echo "ncu rc=$?"
t0=$(date +%s); timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${T}_ref.json 2> gpurun_out/${T}_ref.err; echo "rc=$? wall=$(( $(date +%s) - t0 ))s" >> gpurun_out/${T}_ref.err
tail -n 1 gpurun_out/${T}_bench20.err gpurun_out/${T}_bench.err gpurun_out/${T}_ref.err
TAG=$T python - <<'PY'
import json, os
t = os.environ["TAG"]
for f in (f"gpurun_out/{t}_bench20.json", f"gpurun_out/{t}_bench.json"):
    try:
        d = json.load(open(f))
    except Exception as e:
        print(f, "unreadable", e); continue
    h = d["swap"].get("hidden_under_decode") or {}
    r = d.get("roofline") or {}
    print(f, {k: d.get(k) for k in ("value", "ms_per_step", "gpu_launches")}, "e2e", d["e2e"]["value"],
          "ttft", d["ttft"]["p99_s"], "unit", d.get("step_unit"), "iters", d.get("decode_iterations"), "pre", d["swap"].get("preemptions"), "roof", r.get("frac"), r.get("frac_per_launch_events"),
          "d2h", d["swap"].get("d2h_gbs"), "h2d", d["swap"].get("h2d_gbs"),
          "hidden", {k: (v or {}).get("hidden_frac") for k, v in h.items() if isinstance(v, dict)},
          "mean_batch", d["config"]["mean_batch"], "clocks", d.get("clocks"))
print(open(f"gpurun_out/{t}_ref.json").read()[:700])
PY
