T=${1:-g3}
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "first_layer_fused_pooled or weight_images or forward_vehicle or luma" > gpurun_out/${T}_a.log 2>&1; tail -n 15 gpurun_out/${T}_a.log
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/${T}_pytest.log 2>&1; tail -n 8 gpurun_out/${T}_pytest.log
timeout 600 python bench.py --no-cpu > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; echo "bench rc=$?"; tail -c 400 gpurun_out/${T}_bench.err
python tools/bench_summary.py gpurun_out/${T}_bench.json
