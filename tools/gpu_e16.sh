timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "forward_vehicle or staged or chunking or threshold_edges" > gpurun_out/e16_t.log 2>&1; tail -2 gpurun_out/e16_t.log
PYTHONPATH=. BNN_TRACE_LIB=1 timeout 120 python tools/trace_cluster.py 2>&1 | tail -4
PYTHONPATH=. timeout 120 python tools/time_latency.py 2>&1 | tail -1
PYTHONPATH=. timeout 120 python tools/time_latency.py fused_max_n=8 2>&1 | tail -1
PYTHONPATH=. timeout 120 python tools/time_latency.py fused_max_n=8 fused_cluster=0 2>&1 | tail -1
