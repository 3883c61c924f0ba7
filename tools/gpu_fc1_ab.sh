timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_operating_point.py -q -x -k "dense or forward_vehicle or operating" 2>&1 | tail -1
for i in 1 2; do timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --check 0 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); s=d['stage_ms_per_step']
print('bench %.3f M img/s fc1 %.3f ms/step' % (d['value']/1e6, s['layer2']))"; done
timeout 300 python bench.py --config modes --steps 10 --warmup 3 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print(d['config']['workload'][-5:], round(d['value']/1e6,2), d['stage_ms']['layer2'])"
