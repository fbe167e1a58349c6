# host split planner waves with the in-kernel merge (TF_ATTN_WAVES), and S=2 vs S=3 at B=128
T=${1:-r2q}
mkdir -p gpurun_out
for w in 2 3 4; do
  for st in 2 3; do
    TF_ATTN_WAVES=$w TF_ATTN_STAGES=$st timeout 300 python tools/attn_bench.py --batches 64,128 --plans pool --impls 0 --out gpurun_out/${T}_w${w}_s${st}.json > /dev/null 2>&1
    echo "waves=$w stages=$st"; python -c "
import json
for c in json.load(open('gpurun_out/${T}_w${w}_s${st}.json'))['cases']: print(' ',c['B'],c['ctx'],c['us'],c['frac'])"
  done
done
