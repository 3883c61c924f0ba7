T=${1:-g2}
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/${T}_pytest.log 2>&1; tail -n 3 gpurun_out/${T}_pytest.log
timeout 600 python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; echo "bench rc=$?"; tail -c 600 gpurun_out/${T}_bench.err; tail -c 3000 gpurun_out/${T}_bench.json
