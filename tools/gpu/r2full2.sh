T=${1:-r2full2}
mkdir -p gpurun_out
for i in 1 2; do
  timeout 900 python bench.py --full-run --arrivals burst --no-cpu-baseline --no-selector --max-wall 800 > gpurun_out/${T}_$i.json 2> gpurun_out/${T}_$i.err
  python -c "
import json;d=json.load(open('gpurun_out/${T}_$i.json'));f=d['full_run'];print('$i', round(f.get('effective_tok_s',0)), round(f['ttft_latency']['p99'],1), f['preemptions'], f['recomputes'])"
done
