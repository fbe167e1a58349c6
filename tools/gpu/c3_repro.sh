mkdir -p gpurun_out
timeout 300 python tools/c3_repro.py 1 2 > gpurun_out/c3_repro.log 2>&1; echo "rc=$?" >> gpurun_out/c3_repro.log
timeout 300 python tools/c3_repro.py 0 1 > gpurun_out/c3_repro0.log 2>&1; echo "rc=$?" >> gpurun_out/c3_repro0.log
tail -n 4 gpurun_out/c3_repro.log gpurun_out/c3_repro0.log
