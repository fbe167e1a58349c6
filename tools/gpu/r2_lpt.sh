# attention: LPT (longest-context-first) CTA order vs random order, v3 (2 / 3 stages) and v5
T=${1:-r2lpt}
mkdir -p gpurun_out
timeout 600 python tools/attn_bench.py --batches 64,128 --plans pool --impls 3,5 --orders asis,desc --out gpurun_out/${T}_s3.json > gpurun_out/${T}_s3.log 2>&1
TF_ATTN_STAGES=2 timeout 600 python tools/attn_bench.py --batches 64,128 --plans pool --impls 3 --orders asis,desc --out gpurun_out/${T}_s2.json > gpurun_out/${T}_s2.log 2>&1
timeout 600 python -m pytest tests/test_ar_gpu.py -q -x > gpurun_out/${T}_ar.log 2>&1; tail -3 gpurun_out/${T}_ar.log
grep -h '"c2live560"\|short736' gpurun_out/${T}_s3.log gpurun_out/${T}_s2.log
