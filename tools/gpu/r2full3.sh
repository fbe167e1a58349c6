T=${1:-r2full3}
mkdir -p gpurun_out
for pg in 0 0; do
  TF_PROMPT_GRAPHS=$pg timeout 900 python bench.py --full-run --arrivals burst --no-cpu-baseline --no-selector --max-wall 800 > gpurun_out/${T}_$pg.json 2> gpurun_out/${T}_$pg.err
  python -c "
import json;d=json.load(open('gpurun_out/${T}_$pg.json'));f=d['full_run'];print('prompt_graphs=$pg', round(f.get('effective_tok_s',0)), round(f['ttft_latency']['p99'],1), f['preemptions'], f['recomputes'])"
done
