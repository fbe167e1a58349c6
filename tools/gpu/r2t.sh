# round 2, call t: final validation - full GPU suite, smoke, driver-shaped + default bench lines
T=${1:-r2t}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 --timeout_method thread --durations 5 > gpurun_out/${T}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest.log
grep -E "FAILED|ERROR|Timeout|passed|failed|rc=" gpurun_out/${T}_pytest.log | tail -n 8
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_smoke.log
tail -n 2 gpurun_out/${T}_smoke.log
t0=$(date +%s); timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/${T}_bench20.json 2> gpurun_out/${T}_bench20.err; echo "rc=$? wall=$(( $(date +%s) - t0 ))s" >> gpurun_out/${T}_bench20.err
t0=$(date +%s); timeout 900 python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; echo "rc=$? wall=$(( $(date +%s) - t0 ))s" >> gpurun_out/${T}_bench.err
t0=$(date +%s); timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${T}_ref.json 2> gpurun_out/${T}_ref.err; echo "rc=$? wall=$(( $(date +%s) - t0 ))s" >> gpurun_out/${T}_ref.err
tail -n 1 gpurun_out/${T}_bench20.err gpurun_out/${T}_bench.err gpurun_out/${T}_ref.err
python - <<'PY'
import json
for f in ("gpurun_out/r2t_bench20.json", "gpurun_out/r2t_bench.json"):
    try:
        d = json.load(open(f))
    except Exception as e:
        print(f, "unreadable", e); continue
    h = d["swap"].get("hidden_under_decode") or {}
    print(f, {k: d.get(k) for k in ("value", "ms_per_step", "gpu_launches")}, "e2e", d["e2e"]["value"], "ttft", d["ttft"]["p99_s"],
          "roof", (d.get("roofline") or {}).get("frac"), "d2h", d["swap"].get("d2h_gbs"), "h2d", d["swap"].get("h2d_gbs"),
          "hidden", {k: (v or {}).get("hidden_frac") for k, v in h.items() if isinstance(v, dict)},
          "mean_batch", d["config"]["mean_batch"], "clocks", d.get("clocks"))
print(open("gpurun_out/r2t_ref.json").read()[:600])
PY
