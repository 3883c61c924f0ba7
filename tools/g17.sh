T=${1:-g17}
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/${T}_pytest.log 2>&1; tail -n 2 gpurun_out/${T}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; tail -n 1 gpurun_out/${T}_smoke.log
timeout 600 python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; echo "bench rc=$?"; python tools/bench_summary.py gpurun_out/${T}_bench.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${T}_launches.csv python bench.py --steps 2 --warmup 1 --total-batch 65536 --no-cpu --no-e2e --check 0 > gpurun_out/${T}_launches.log 2>&1; echo "launches rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"conv1_fp4_pool|conv_tc4_pool|dense_tc4_kernel" -c 3 -o gpurun_out/${T}_full python bench.py --steps 1 --warmup 1 --total-batch 32768 --no-cpu --no-e2e --check 0 > gpurun_out/${T}_full.log 2>&1; echo "full rc=$?"
