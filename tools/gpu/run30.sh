mkdir -p gpurun_out
for i in 1 2; do timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu30_$i.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu30_$i.log; done
tail -n 2 gpurun_out/pytest_gpu30_1.log gpurun_out/pytest_gpu30_2.log
