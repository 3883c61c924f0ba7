timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "forward_vehicle or staged or chunking or threshold_edges or fused_cluster_shapes" 2>&1 | tail -3
PYTHONPATH=. BNN_TRACE_LIB=1 timeout 120 python tools/trace_cluster.py 2>&1 | tail -3
for i in 1 2; do PYTHONPATH=. timeout 300 python tools/time_latency_dev.py 200 2>&1 | tail -3; done
