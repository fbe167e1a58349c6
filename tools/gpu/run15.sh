mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu15.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu15.log
timeout 700 python bench.py --verbose --profile-hooks > gpurun_out/bench15.json 2> gpurun_out/bench15.err; echo "rc=$?" >> gpurun_out/bench15.err
timeout 500 python bench.py --full-run --no-cpu-baseline --verbose --max-wall 300 --profile-hooks > gpurun_out/full15.json 2> gpurun_out/full15.err
tail -n 3 gpurun_out/pytest_gpu15.log
