mkdir -p gpurun_out
timeout 700 python bench.py --verbose --profile-hooks --no-cpu-baseline > gpurun_out/bench10.json 2> gpurun_out/bench10.err; echo "rc=$?" >> gpurun_out/bench10.err
timeout 400 python bench.py --full-run --no-cpu-baseline --verbose --max-wall 200 --profile-hooks > gpurun_out/full10.json 2> gpurun_out/full10.err
echo done
