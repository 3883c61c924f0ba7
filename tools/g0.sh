timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/g0_pytest.log 2>&1; tail -n 3 gpurun_out/g0_pytest.log
timeout 300 python bench.py > gpurun_out/g0_bench.json 2> gpurun_out/g0_bench.err; tail -c 1500 gpurun_out/g0_bench.json
