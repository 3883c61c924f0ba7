timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "luma_tma or forward_vehicle or pack_input" > gpurun_out/e17_t.log 2>&1; tail -2 gpurun_out/e17_t.log
timeout 600 python -m pytest tests/test_gpu_operating_point.py -x -q -k "operating_point" > gpurun_out/e17_t2.log 2>&1; tail -2 gpurun_out/e17_t2.log
timeout 300 python bench.py --config modes --steps 10 --warmup 3 > gpurun_out/e17_modes.jsonl 2>/dev/null; python -c "
import json
for l in open('gpurun_out/e17_modes.jsonl'):
    l=l.strip()
    if l.startswith('{'):
        d=json.loads(l); print(round(d['value']/1e6,2), d.get('stage_ms_per_step'), d['config'].get('mode', d['config'].get('input')))
"
