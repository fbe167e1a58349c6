# round 2, call e: whole GPU suite + smoke with v3 default, v5 stall reproduction, whole-block hidden probe, bench
T=${1:-r2e}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${T}_smi.txt
timeout 1500 python -m pytest tests -m gpu -v --timeout 600 --timeout_method thread --durations 15 > gpurun_out/${T}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest.log
grep -E "FAILED|ERROR|Timeout|passed|failed|rc=" gpurun_out/${T}_pytest.log | tail -n 15
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_smoke.log
tail -n 2 gpurun_out/${T}_smoke.log
timeout 900 python tools/v5_repro.py --out gpurun_out/${T}_v5repro.json --max-s 400 > gpurun_out/${T}_v5repro.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_v5repro.log
tail -c 3000 gpurun_out/${T}_v5repro.log
timeout 600 python tools/hidden_probe2.py --batch 128 --ctx 600 --tokens 320 --seg 16 --out gpurun_out/${T}_hp2_blocks.json > gpurun_out/${T}_hp2_blocks.log 2>&1
python -c "import json;d=json.load(open('gpurun_out/${T}_hp2_blocks.json'));print(json.dumps(d['summary']));print(json.dumps(d['ms_per_step']))"
t0=$(date +%s); timeout 900 python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; echo "rc=$? wall=$(( $(date +%s) - t0 ))s" >> gpurun_out/${T}_bench.err
tail -n 2 gpurun_out/${T}_bench.err; head -c 1500 gpurun_out/${T}_bench.json
