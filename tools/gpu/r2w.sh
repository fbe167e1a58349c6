T=${1:-r2w}
mkdir -p gpurun_out
for i in 1 2 3 4 5 6 7 8; do
  timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-selector --ttft 0 > gpurun_out/${T}_$i.json 2>/dev/null
  python -c "
import json;d=json.load(open('gpurun_out/${T}_$i.json'));w=d['window_clock'];print(round(d['value']), d['prefill_device_s_in_window'], w['first_decode_s'], w['start_s'], w['end_s'], w['ticks'])"
done
