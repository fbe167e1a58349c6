# interval-step bench with eager prompt prefills (TF_PROMPT_GRAPHS=0), twice
T=${1:-r2tickpg}
mkdir -p gpurun_out
for i in 1 2; do
  TF_PROMPT_GRAPHS=0 timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-selector > gpurun_out/${T}_$i.json 2> gpurun_out/${T}_$i.err
  python -c "
import json;d=json.load(open('gpurun_out/${T}_$i.json'));s=d['swap']
print(d['config']['prompt_graphs'], round(d['value']), round(d['e2e']['value']), round(d['ms_per_step'],1), d['decode_iterations'], d['prefill_device_s_in_window'], d['config']['mean_batch'], 'pre', s['preemptions'], 'rc', s['recomputes'], 'h2d', s['h2d_gbs'], 'ttft', d['ttft']['p99_s'])"
done
