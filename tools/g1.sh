T=${1:-g1}
timeout 600 python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; echo "bench rc=$?"; tail -c 600 gpurun_out/${T}_bench.err
for c in latency modes cifar sweep alg1; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/${T}_cfg_$c.jsonl 2> gpurun_out/${T}_cfg_$c.err; echo "$c rc=$?"; tail -c 300 gpurun_out/${T}_cfg_$c.err
done
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${T}_ref.json 2>&1; echo "ref rc=$?"
