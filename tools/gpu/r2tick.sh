# interval-step bench (the new default) three times on one box
T=${1:-r2tick}
mkdir -p gpurun_out
for i in 1 2 3; do
  t0=$(date +%s); timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/${T}_$i.json 2> gpurun_out/${T}_$i.err; echo "rc=$? wall=$(( $(date +%s) - t0 ))s" >> gpurun_out/${T}_$i.err
  tail -n 1 gpurun_out/${T}_$i.err
  python -c "
import json;d=json.load(open('gpurun_out/${T}_$i.json'));w=d['window_clock'];s=d['swap'];r=d['roofline'] or {}
print(round(d['value']), round(d['e2e']['value']), round(d['ms_per_step'],1), d['decode_iterations'], round(d['decode_ms_per_iter'],2), d['prefill_device_s_in_window'], d['config']['mean_batch'], 'pre', s['preemptions'], 'rc', s['recomputes'], 'd2h', s['d2h_gbs'], 'h2d', s['h2d_gbs'], 'h2d_tok', s['h2d_tokens'], 'roof', r.get('frac'), r.get('batch'), 'ttft', d['ttft']['p99_s'], 'launch', d['gpu_launches'], 'ticks', w['ticks_fired'], len(w['ticks_that_moved_requests']), w['start_s'], w['end_s'], 'hidden', {k:(v or {}).get('hidden_frac') for k,v in (s.get('hidden_under_decode') or {}).items() if isinstance(v,dict)})"
done
