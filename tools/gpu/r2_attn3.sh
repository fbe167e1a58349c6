# attention: parity tests, v3/v5 bench, per-kernel launch durations under ncu (tag = $1)
T=${1:-r2attn}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_kernels_gpu.py -m gpu -q -x -k attention > gpurun_out/${T}_kernels.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_kernels.log
timeout 600 python tools/attn_bench.py --impls 3,5 --plans pool --batches 32,64,128 --out gpurun_out/${T}_attn_bench.json > gpurun_out/${T}_attn_bench.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:"paged_attn|attn5|combine" --csv \
   --log-file gpurun_out/${T}_launches.csv python tools/attn_bench.py --only 128:c2live560:pool --impls 3,5 --reps 3 --out gpurun_out/${T}_tmp.json > /dev/null 2>&1
tail -3 gpurun_out/${T}_kernels.log; grep -v "uniform\|ragged" gpurun_out/${T}_attn_bench.log
