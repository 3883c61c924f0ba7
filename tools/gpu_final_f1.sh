# post-f1 refresh of the evidence that depends on the batch-1 path: bash tools/gpu_final_f1.sh TAG
T=${1:-f1}
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/${T}_pytest.log 2>&1; tail -n 1 gpurun_out/${T}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/${T}_smoke.log 2>&1; tail -n 1 gpurun_out/${T}_smoke.log
timeout 600 python bench.py --config latency --steps 10 --warmup 3 > gpurun_out/${T}_cfg_latency.jsonl 2> gpurun_out/${T}_cfg_latency.err; tail -c 400 gpurun_out/${T}_cfg_latency.jsonl
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/${T}_bench_quick.json 2>/dev/null; tail -c 150 gpurun_out/${T}_bench_quick.json
