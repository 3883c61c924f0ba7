set -x
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "conv_pool_tensor_core or conv_tensor_core or first_layer_fused or forward_vehicle or staged or threshold_edges or chunking or first_layer_pooled" > gpurun_out/t22a.log 2>&1 || { tail -30 gpurun_out/t22a.log; PYTHONPATH=. timeout 300 compute-sanitizer --print-limit 5 python tools/repro_first_tma.py 2>&1 | head -60; exit 1; }
tail -3 gpurun_out/t22a.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/t22b.log 2>&1; tail -3 gpurun_out/t22b.log
timeout 300 python bench.py --steps 22 --warmup 3 --no-cpu > gpurun_out/bench22.json 2> gpurun_out/bench22.err; tail -c 300 gpurun_out/bench22.json
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"conv_first_tma|conv_tc4_pool" -c 2 -o gpurun_out/prof_conv22 python bench.py --steps 1 --warmup 1 --no-cpu > gpurun_out/ncu_full22.log 2>&1; tail -2 gpurun_out/ncu_full22.log
