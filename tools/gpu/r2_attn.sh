# round-2 attention: kernel parity tests + v3/v5 micro-benchmark (tag = $1)
T=${1:-r2attn}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_kernels_gpu.py -m gpu -q -x > gpurun_out/${T}_kernels.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_kernels.log
timeout 600 python tools/attn_bench.py --impls 3,5 --plans exact,pool --out gpurun_out/${T}_attn_bench.json > gpurun_out/${T}_attn_bench.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_attn_bench.log
tail -5 gpurun_out/${T}_kernels.log; cat gpurun_out/${T}_attn_bench.log
