# all bench configs on one box: bash tools/gpu_configs.sh TAG
T=${1:-x}
for c in latency modes cifar sweep; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/cfg_${T}_$c.jsonl 2> gpurun_out/cfg_${T}_$c.err
  echo "$c rc=$?"; tail -c 400 gpurun_out/cfg_${T}_$c.jsonl
done
