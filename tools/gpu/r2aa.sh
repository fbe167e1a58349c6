T=${1:-r2aa}
mkdir -p gpurun_out
timeout 700 python -m pytest tests/test_realtime_gpu.py tests/test_tp_gpu.py -m gpu -q --timeout 400 --timeout_method thread 2>&1 | tail -2
for i in 1 2; do
  timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-selector > gpurun_out/${T}_b20_$i.json 2>/dev/null
  python -c "
import json;d=json.load(open('gpurun_out/${T}_b20_$i.json'));print('b20', round(d['value']), round(d['e2e']['value']), round(d['e2e']['value']/d['value'],4), d['ttft']['p99_s'])"
done
timeout 900 python bench.py --full-run --arrivals burst --no-cpu-baseline --no-selector --max-wall 800 > gpurun_out/${T}_full.json 2>/dev/null
python -c "
import json;d=json.load(open('gpurun_out/${T}_full.json'));f=d['full_run'];print('full', round(f.get('effective_tok_s',0)), round(f['ttft_latency']['p99'],1), f['preemptions'], f['recomputes'])"
