# round 2, call f: fixed host-tier byte test, v5 stall reproduction, ncu (bench window launch list + attention
# full captures at the live shapes), C5 sweep with the two-queue copy engines, driver-shaped bench line
T=${1:-r2f}
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_realtime_gpu.py tests/test_kernels_gpu.py -m gpu -q --timeout 300 --timeout_method thread > gpurun_out/${T}_tests.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_tests.log
tail -n 4 gpurun_out/${T}_tests.log
timeout 900 python tools/v5_repro.py --out gpurun_out/${T}_v5repro.json --max-s 400 > gpurun_out/${T}_v5repro.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_v5repro.log
tail -c 2500 gpurun_out/${T}_v5repro.log
t0=$(date +%s); timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/${T}_bench20.json 2> gpurun_out/${T}_bench20.err; echo "rc=$? wall=$(( $(date +%s) - t0 ))s" >> gpurun_out/${T}_bench20.err
tail -n 1 gpurun_out/${T}_bench20.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --nvtx --nvtx-include "bench_timed/" -c 4000 --csv \
  --log-file gpurun_out/${T}_launches_bench.csv python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-selector --ttft 0 \
  > gpurun_out/${T}_ncu_bench.log 2>&1; echo "ncu_rc=$?"
for case in 128:c2live560:pool 64:c2live560:pool; do
  tag=$(echo $case | cut -d: -f1,2 | tr ':' '_')
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:paged_attn -c 1 \
    -o gpurun_out/${T}_attn_v3_${tag} -f python tools/attn_bench.py --only $case --impls 0 --reps 1 --out /tmp/x.json \
    > gpurun_out/${T}_ncu_attn_${tag}.log 2>&1; echo "ncu_attn_rc=$?"
done
timeout 1200 python bench_swap.py --max-blocks 4096 --host-blocks 4096 --engines 0,3 --overlap --out gpurun_out/${T}_swap.json > gpurun_out/${T}_swap.log 2>&1; echo "swap_rc=$?"
python -c "import json;d=json.load(open('gpurun_out/${T}_swap.json'));print(json.dumps(d.get('overlap')))"
