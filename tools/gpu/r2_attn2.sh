# attention v5 iteration: parity tests, bench v3 / v5 / v5 without L2 prefetch, ncu of v5 (tag = $1)
T=${1:-r2attn}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_kernels_gpu.py -m gpu -q -x -k attention > gpurun_out/${T}_kernels.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_kernels.log
timeout 600 python tools/attn_bench.py --impls 3,5 --plans pool --out gpurun_out/${T}_attn_bench.json > gpurun_out/${T}_attn_bench.log 2>&1
TF_ATTN5_NOPF=1 timeout 600 python tools/attn_bench.py --impls 5 --plans pool --out gpurun_out/${T}_attn_bench_nopf.json > gpurun_out/${T}_attn_bench_nopf.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:paged_attn --launch-skip 5 --launch-count 1 \
    -o gpurun_out/${T}_v5 -f python tools/attn_bench.py --only 128:c2live560:exact --impls 5 --reps 3 --out gpurun_out/${T}_tmp.json > gpurun_out/${T}_ncu.log 2>&1
tail -3 gpurun_out/${T}_kernels.log; paste -d' ' <(cut -c1-120 gpurun_out/${T}_attn_bench.log) ; cat gpurun_out/${T}_attn_bench_nopf.log
