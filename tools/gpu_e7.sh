timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "weight_images or forward_vehicle or conv_pool_tensor_core or forward_cifar or chunking" > gpurun_out/e7_t1.log 2>&1; tail -3 gpurun_out/e7_t1.log
PYTHONPATH=. timeout 300 python tools/time_opts.py conv_pool3=0,conv_pair=1 conv_pool3=1,conv_pair=0 conv_pool3=1,conv_pair=1 > gpurun_out/e7_ab.log 2>&1; cat gpurun_out/e7_ab.log | tail -6
timeout 900 python -m pytest tests/test_gpu_operating_point.py -x -q > gpurun_out/e7_t2.log 2>&1; tail -3 gpurun_out/e7_t2.log
