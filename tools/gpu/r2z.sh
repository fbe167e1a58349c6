# round 2, call z: fused write-through line, C5 sweep to 64K blocks on the final copy-engine path
T=${1:-r2z}
mkdir -p gpurun_out
t0=$(date +%s); timeout 900 python bench.py --fused-wt 1 --no-cpu-baseline --no-selector > gpurun_out/${T}_fusedwt.json 2> gpurun_out/${T}_fusedwt.err; echo "fused rc=$? wall=$(( $(date +%s) - t0 ))s"
python - <<'PY'
import json
d = json.load(open("gpurun_out/r2z_fusedwt.json"))
h = d["swap"].get("hidden_under_decode") or {}
print({k: d.get(k) for k in ("value", "ms_per_step")}, "e2e", d["e2e"]["value"], "ttft", d["ttft"]["p99_s"],
      "d2h", d["swap"].get("d2h_gbs"), "h2d", d["swap"].get("h2d_gbs"), "pre", d["swap"].get("preemptions"),
      "hidden", {k: (v or {}).get("hidden_frac") for k, v in h.items() if isinstance(v, dict)}, "mean_batch", d["config"]["mean_batch"])
PY
t0=$(date +%s); timeout 2400 python bench_swap.py --max-blocks 65536 --host-blocks 16384 --engines 0,3 --overlap --out gpurun_out/${T}_swap64k.json > gpurun_out/${T}_swap64k.log 2>&1; echo "sweep rc=$? wall=$(( $(date +%s) - t0 ))s"
python -c "
import json;d=json.load(open('gpurun_out/${T}_swap64k.json'))
for r in d['rows']:
    if not r['per_layer'] and r['blocks'] in (1,16,256,4096,16384,65536): print(r['blocks'],r['engine'],round(r['d2h_gbs'],1),round(r['h2d_gbs'],1),round(r['duplex_gbs'],1))
print(json.dumps(d.get('overlap')))"
