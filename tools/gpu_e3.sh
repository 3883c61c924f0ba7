timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "weight_images or forward_vehicle" > gpurun_out/e3_t1.log 2>&1; tail -3 gpurun_out/e3_t1.log
PYTHONPATH=. timeout 300 python tools/time_opts.py conv_pair=0 conv_pair=1 > gpurun_out/e3_ab.log 2>&1; cat gpurun_out/e3_ab.log | tail -6
