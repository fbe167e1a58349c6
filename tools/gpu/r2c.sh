# round 2, call c: whole GPU suite (per-test timeout) + decode-slowdown attribution under swaps
T=${1:-r2c}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -v --timeout 600 --durations 15 > gpurun_out/${T}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest.log
grep -E "FAILED|ERROR|passed|failed|rc=" gpurun_out/${T}_pytest.log | tail -n 15
timeout 600 python tools/hidden_probe2.py --batch 128 --ctx 600 --tokens 40 --seg 8 --out gpurun_out/${T}_hp2.json > gpurun_out/${T}_hp2.log 2>&1
tail -n 40 gpurun_out/${T}_hp2.log
