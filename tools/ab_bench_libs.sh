# bench.py A/B of library variants (variants/<v>.so) on one box: bash tools/ab_bench_libs.sh v1 v2 ...
cp paper_1808_00209_b200/libbnn.so /tmp/libbnn_keep.so
for rep in 1 2; do
for v in "$@"; do
  cp variants/$v.so paper_1808_00209_b200/libbnn.so
  echo -n "[$v] "; timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --check 0 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); s=d['stage_ms_per_step']
print('%.2f M img/s  step %.3f ms  conv1 %.3f conv2 %.3f fc1 %.3f ms/step  clocks %s' % (d['value']/1e6, d['ms_per_step'], s['layer0'], s['layer1'], s['layer2'], d['clocks']['sm_mhz']))"
done
done
cp /tmp/libbnn_keep.so paper_1808_00209_b200/libbnn.so
