mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu14.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu14.log
timeout 700 python bench.py --verbose --profile-hooks > gpurun_out/bench14.json 2> gpurun_out/bench14.err; echo "rc=$?" >> gpurun_out/bench14.err
for st in 2 3; do TF_ATTN_STAGES=$st timeout 200 python tools/attn_bench.py --plans exact --out gpurun_out/attn_stages$st.json > /dev/null 2>&1; done
tail -n 3 gpurun_out/pytest_gpu14.log
