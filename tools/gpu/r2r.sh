# round 2, call r: prefill graphs + host staging - tests, hook profile, bench lines
T=${1:-r2r}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_tp_gpu.py tests/test_realtime_gpu.py tests/test_model_gpu.py tests/test_dataplane_gpu.py -m gpu -q --timeout 400 --timeout_method thread > gpurun_out/${T}_tests.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_tests.log
tail -n 4 gpurun_out/${T}_tests.log
timeout 700 python bench.py --steps 200 --warmup 10 --no-cpu-baseline --no-selector --ttft 0 --swap-steps 0 --profile-hooks > gpurun_out/${T}_hooks.json 2> gpurun_out/${T}_hooks.err; echo "hooks rc=$?"
python -c "
import json;d=json.load(open('gpurun_out/${T}_hooks.json'));print(d['value'],d['e2e']['value'],d['ms_per_step']);h=d['host_hook_ms']
for k,v in sorted(h.items(),key=lambda x:-x[1]['total_s'])[:6]: print(k,v)"
t0=$(date +%s); timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/${T}_bench20.json 2> gpurun_out/${T}_bench20.err; echo "rc=$? wall=$(( $(date +%s) - t0 ))s" >> gpurun_out/${T}_bench20.err
t0=$(date +%s); timeout 900 python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; echo "rc=$? wall=$(( $(date +%s) - t0 ))s" >> gpurun_out/${T}_bench.err
tail -n 1 gpurun_out/${T}_bench20.err gpurun_out/${T}_bench.err
python - <<'PY'
import json
for f in ("gpurun_out/r2r_bench20.json", "gpurun_out/r2r_bench.json"):
    try:
        d = json.load(open(f))
    except Exception as e:
        print(f, "unreadable", e); continue
    h = d["swap"].get("hidden_under_decode") or {}
    print(f, {k: d.get(k) for k in ("value", "ms_per_step")}, "e2e", d["e2e"]["value"], "ttft", d["ttft"]["p99_s"],
          "roof", (d.get("roofline") or {}).get("frac"), "d2h", d["swap"].get("d2h_gbs"), "h2d", d["swap"].get("h2d_gbs"),
          "hidden", {k: (v or {}).get("hidden_frac") for k, v in h.items() if isinstance(v, dict)},
          "mean_batch", d["config"]["mean_batch"], "prefill_s", d.get("prefill_device_s_in_window"))
PY
