T=${1:-g6}
PYTHONPATH=. timeout 300 python tools/time_conv1.py 0 1 2 > gpurun_out/${T}_time.log 2>&1; cat gpurun_out/${T}_time.log
PYTHONPATH=. BNN_TRACE_LIB=1 timeout 300 python tools/trace_conv1.py 1 > gpurun_out/${T}_trace1.log 2>&1; tail -8 gpurun_out/${T}_trace1.log
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "first_layer_fused_pooled or weight_images or forward_vehicle or luma" > gpurun_out/${T}_a.log 2>&1; tail -n 3 gpurun_out/${T}_a.log
