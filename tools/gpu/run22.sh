mkdir -p gpurun_out
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --nvtx --nvtx-include "bench_timed/" -c 2500 --csv --log-file gpurun_out/launches22.csv \
  python bench.py --steps 20 --warmup 5 --no-cpu-baseline --ttft 0 > gpurun_out/ncu22.log 2>&1
echo done
