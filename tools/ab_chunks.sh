for rep in 1 2; do for c in ${CHUNKS:-8192 16384 32768 65536}; do
echo -n "chunk $c: "; timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --check 0 --chunk $c 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); s=d['stage_ms_per_step']
print('%.2f M img/s  step %.3f ms  conv1 %.3f conv2 %.3f fc1 %.3f' % (d['value']/1e6, d['ms_per_step'], s['layer0'], s['layer1'], s['layer2']))"
done; done
