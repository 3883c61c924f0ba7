# bench.py A/B of option settings on one box: bash tools/ab_bench.sh "opts1" "opts2" ...  (opts: "k=v k=v", "" = defaults)
for rep in 1 2; do
for o in "$@"; do
  args=""; for kv in $o; do args="$args --opt $kv"; done
  echo -n "[$o] "; timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --check 0 $args 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); s=d['stage_ms_per_step']
print('%.2f M img/s  step %.3f ms  conv1 %.3f conv2 %.3f fc1 %.3f ms/step  clocks %s' % (d['value']/1e6, d['ms_per_step'], s['layer0'], s['layer1'], s['layer2'], d['clocks']))"
done
done
