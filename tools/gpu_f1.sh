timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "forward_vehicle or staged or chunking or threshold_edges or fused_cluster_shapes" 2>&1 | tail -2
PYTHONPATH=. BNN_TRACE_LIB=1 timeout 120 python tools/trace_cluster.py 2>&1 | tail -3
for i in 1 2; do PYTHONPATH=. timeout 120 python tools/time_latency.py 2>&1 | tail -1; PYTHONPATH=. timeout 120 python tools/time_latency.py fused_max_n=8 2>&1 | tail -1; done
