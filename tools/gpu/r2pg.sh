T=${1:-r2pg}
mkdir -p gpurun_out
for pg in 1 0; do
  for i in 1 2; do
    TF_PROMPT_GRAPHS=$pg timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-selector > gpurun_out/${T}_b20_${pg}_$i.json 2>/dev/null
    python -c "
import json;d=json.load(open('gpurun_out/${T}_b20_${pg}_$i.json'));print('pg=$pg b20', round(d['value']), round(d['e2e']['value']), d['prefill_device_s_in_window'], d['ttft']['p99_s'])"
  done
done
TF_PROMPT_GRAPHS=1 timeout 900 python bench.py --full-run --arrivals burst --no-cpu-baseline --no-selector --max-wall 800 > gpurun_out/${T}_full1.json 2>/dev/null
python -c "
import json;d=json.load(open('gpurun_out/${T}_full1.json'));f=d['full_run'];print('pg=1 full', round(f.get('effective_tok_s',0)), round(f['ttft_latency']['p99'],1), f['preemptions'], f['recomputes'])"
