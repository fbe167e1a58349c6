# round 2, call m: bench lines with the per-token rope kernel + scaled window-mix hidden probe; ncu launch list
T=${1:-r2m}
mkdir -p gpurun_out
t0=$(date +%s); timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/${T}_bench20.json 2> gpurun_out/${T}_bench20.err; echo "rc=$? wall=$(( $(date +%s) - t0 ))s" >> gpurun_out/${T}_bench20.err
t0=$(date +%s); timeout 900 python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; echo "rc=$? wall=$(( $(date +%s) - t0 ))s" >> gpurun_out/${T}_bench.err
tail -n 1 gpurun_out/${T}_bench20.err gpurun_out/${T}_bench.err
python - <<'PY'
import json
for f in ("gpurun_out/r2m_bench20.json", "gpurun_out/r2m_bench.json"):
    try:
        d = json.load(open(f))
    except Exception as e:
        print(f, "unreadable", e); continue
    h = d["swap"].get("hidden_under_decode") or {}
    print(f, {k: d.get(k) for k in ("value", "ms_per_step")}, "e2e", d["e2e"]["value"], "ttft", d["ttft"]["p99_s"],
          "roof", (d.get("roofline") or {}).get("frac"), "d2h", d["swap"].get("d2h_gbs"), "h2d", d["swap"].get("h2d_gbs"),
          "hidden", {k: (v or {}).get("hidden_frac") for k, v in h.items() if isinstance(v, dict)},
          "mean_batch", d["config"]["mean_batch"])
PY
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --nvtx --nvtx-include "bench_timed/" -c 1100 --csv \
  --log-file gpurun_out/${T}_launches_bench.csv python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-selector --ttft 0 --swap-steps 0 \
  > gpurun_out/${T}_ncu_bench.log 2>&1; echo "ncu_rc=$?"
