mkdir -p gpurun_out
timeout 900 python -m pytest -q -p no:randomly "tests/test_realtime_gpu.py" "tests/test_report.py" -m gpu > gpurun_out/r29a.log 2>&1; echo "rc=$?" >> gpurun_out/r29a.log
timeout 1500 compute-sanitizer --tool memcheck --print-limit 5 python -m pytest -q -x "tests/test_realtime_gpu.py::test_realtime_c1_completes_with_invariants[2-True-False]" -m gpu > gpurun_out/r29b.log 2>&1; echo "rc=$?" >> gpurun_out/r29b.log
echo done
