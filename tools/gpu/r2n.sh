# round 2, call n: v3 transposed inner loop - parity tests under TF_ATTN_TR=1, sweep TR 0 vs 1
T=${1:-r2n}
mkdir -p gpurun_out
TF_ATTN_TR=1 timeout 600 python -m pytest tests/test_kernels_gpu.py tests/test_model_gpu.py -m gpu -q -k "paged_attention or decode_step" --timeout 300 > gpurun_out/${T}_tests.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_tests.log
tail -n 4 gpurun_out/${T}_tests.log
for tr in 0 1; do
  TF_ATTN_TR=$tr timeout 600 python tools/attn_bench.py --batches 32,64,96,128 --plans pool --impls 0 --out gpurun_out/${T}_tr$tr.json > gpurun_out/${T}_tr$tr.log 2>&1
  echo "tr=$tr"; python -c "
import json
for c in json.load(open('gpurun_out/${T}_tr$tr.json'))['cases']: print(c['B'],c['ctx'],c['us'],c['frac'])"
done
