T=${1:-r2ab}
mkdir -p gpurun_out
for g in 0 1 0 1; do
  TF_GROW_BATCH=$g timeout 600 python bench.py --no-cpu-baseline --no-selector --ttft 0 --swap-steps 0 > gpurun_out/${T}_g$g.json 2>/dev/null
  python -c "
import json;d=json.load(open('gpurun_out/${T}_g$g.json'));s=d['swap']
print('grow_batch=$g', round(d['value']), round(d['e2e']['value']), 'd2h', round(s['d2h_gbs'],1), 'h2d', round(s['h2d_gbs'],1), 'h2d_tok', s['h2d_tokens'], 'chunks', s['chunks'], 'mb', d['config']['mean_batch'])"
done
