mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu26.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu26.log
timeout 300 python bench_swap.py --wt-only --out gpurun_out/wt26.json > gpurun_out/wt26.log 2>&1
for i in 1 2; do t0=$(date +%s); timeout 900 python bench.py > gpurun_out/bench26_$i.json 2> gpurun_out/bench26_$i.err; echo "rc=$? wall=$(( $(date +%s) - t0 ))s" >> gpurun_out/bench26_$i.err; done
tail -n 3 gpurun_out/pytest_gpu26.log
