timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "weight_images or forward_vehicle or conv_pool_tensor_core or forward_cifar or chunking or first_layer" > gpurun_out/e12_t1.log 2>&1; tail -2 gpurun_out/e12_t1.log
bash tools/ab_opts.sh "conv_pair=1 conv_pair=0" base nbg3 l4 l3 > gpurun_out/e12.log 2>&1; cat gpurun_out/e12.log
