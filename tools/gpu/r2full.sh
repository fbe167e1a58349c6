T=${1:-r2full}
mkdir -p gpurun_out
for arr in burst poisson; do
  t0=$(date +%s); timeout 1500 python bench.py --full-run --arrivals $arr --no-cpu-baseline --no-selector --max-wall 1200 > gpurun_out/${T}_$arr.json 2> gpurun_out/${T}_$arr.err; echo "$arr rc=$? wall=$(( $(date +%s) - t0 ))s"
  python -c "
import json;d=json.load(open('gpurun_out/${T}_$arr.json'));print('$arr', json.dumps(d.get('full_run')))"
done
