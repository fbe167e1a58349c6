# QKV row padding: GPU numerics + interval-window bench A/B (padding on / off alternating)
T=${1:-r2qkv}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_model_gpu.py tests/test_tp_gpu.py tests/test_realtime_gpu.py tests/test_dataplane_gpu.py -m gpu -q --timeout 600 --timeout_method thread 2>&1 | tail -n 3
for i in 1 2; do
  for q in 128 0; do
    TF_QKV_ROWS=$q timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-selector > gpurun_out/${T}_${q}_$i.json 2>/dev/null
    python -c "
import json;d=json.load(open('gpurun_out/${T}_${q}_$i.json'))
print('qkv_rows=$q', round(d['value']), round(d['e2e']['value']), d['decode_iterations'], round(d['decode_ms_per_iter'],3), d['config']['mean_batch'], d['prefill_device_s_in_window'])"
  done
done
