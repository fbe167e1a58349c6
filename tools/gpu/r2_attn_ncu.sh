# ncu --set full of the attention kernels on the C2 live shape (tag = $1, impls = $2)
T=${1:-r2ncu}
mkdir -p gpurun_out
for impl in ${2:-5 3}; do
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:paged_attn --launch-skip 5 --launch-count 1 \
    -o gpurun_out/${T}_v${impl} -f python tools/attn_bench.py --only 128:c2live560:exact --impls $impl --reps 3 \
    --out gpurun_out/${T}_tmp.json > gpurun_out/${T}_v${impl}.log 2>&1
  echo "impl $impl rc=$?" >> gpurun_out/${T}_v${impl}.log
done
timeout 600 python -m pytest tests/test_kernels_gpu.py -m gpu -q -x -k attention > gpurun_out/${T}_kernels.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_kernels.log
tail -3 gpurun_out/${T}_kernels.log
