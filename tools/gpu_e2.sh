# pair-MMA check + A/B: bash tools/gpu_e2.sh
timeout 60 tools/probes/acc_probe > gpurun_out/e2_acc_probe.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "weight_images or forward_vehicle or staged or chunking" > gpurun_out/e2_t1.log 2>&1; tail -3 gpurun_out/e2_t1.log
PYTHONPATH=. timeout 300 python tools/time_opts.py conv_pair=0 conv_pair=1 > gpurun_out/e2_ab.log 2>&1; cat gpurun_out/e2_ab.log | tail -6
timeout 900 python -m pytest tests/test_gpu_operating_point.py -x -q > gpurun_out/e2_t2.log 2>&1; tail -3 gpurun_out/e2_t2.log
