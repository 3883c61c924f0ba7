# round-end evidence on one box: bash tools/gpu_final.sh TAG   (everything lands in gpurun_out/TAG_*)
T=${1:-final}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/${T}_smi.txt 2>&1
timeout 60 tools/probes/acc_probe > gpurun_out/${T}_acc_probe.txt 2>&1
timeout 60 tools/probes/issue_probe > gpurun_out/${T}_issue_probe.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/${T}_pytest.log 2>&1; tail -n 1 gpurun_out/${T}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/${T}_smoke.log 2>&1; tail -n 1 gpurun_out/${T}_smoke.log
timeout 300 python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; tail -c 200 gpurun_out/${T}_bench.json
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${T}_ref.json 2> gpurun_out/${T}_ref.err; tail -c 200 gpurun_out/${T}_ref.json
for c in latency modes cifar sweep alg1; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/${T}_cfg_$c.jsonl 2> gpurun_out/${T}_cfg_$c.err; echo "$c rc=$?"
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${T}_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e > gpurun_out/${T}_launches.log 2>&1; echo "launches rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"^(conv1_fp4_pool|conv_tc4_pool3|dense_tc4_kernel)" -c 3 -o /tmp/${T}_full python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/${T}_full.log 2>&1; echo "full rc=$?"
ncu -i /tmp/${T}_full.ncu-rep --page raw --csv > gpurun_out/${T}_full_raw.csv 2>&1
python tools/ncu_summary.py /tmp/${T}_full.ncu-rep 65536 gpurun_out/${T}_ncu > gpurun_out/${T}_ncu_summary.log 2>&1; cp profiles/ncu_traffic.json gpurun_out/${T}_ncu_traffic.json
