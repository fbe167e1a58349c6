mkdir -p gpurun_out
timeout 900 python -m cProfile -o gpurun_out/bench23.prof bench.py --no-cpu-baseline --ttft 0 > gpurun_out/bench23.json 2> gpurun_out/bench23.err
echo done
