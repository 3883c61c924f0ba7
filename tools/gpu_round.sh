# build-verify round on one box: bash tools/gpu_round.sh TAG
T=${1:-x}
set -x
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "alg1 or weight_images or conv_pool_tensor_core or conv_tensor_core or first_layer_fused or forward_vehicle or staged or threshold_edges or chunking or first_layer_pooled" > gpurun_out/t${T}a.log 2>&1 || { tail -30 gpurun_out/t${T}a.log; PYTHONPATH=. timeout 300 compute-sanitizer --print-limit 5 python tools/repro_first_tma.py 2>&1 | head -60; exit 1; }
tail -1 gpurun_out/t${T}a.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/t${T}b.log 2>&1; tail -1 gpurun_out/t${T}b.log
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu > gpurun_out/bench${T}.json 2> gpurun_out/bench${T}.err; tail -c 300 gpurun_out/bench${T}.json
timeout 300 python bench.py --config latency --steps 10 --warmup 3 > gpurun_out/lat${T}.jsonl 2>&1; tail -c 400 gpurun_out/lat${T}.jsonl
if [ -n "$NCU" ]; then timeout 600 ncu --set full --import-source on --clock-control none -k regex:"$NCU" -c 2 -o gpurun_out/prof_${T} python bench.py --steps 1 --warmup 1 --no-cpu > gpurun_out/ncu_${T}.log 2>&1; tail -2 gpurun_out/ncu_${T}.log; fi
