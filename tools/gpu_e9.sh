export PYTHONPATH=. BNN_TRACE_LIB=1
timeout 120 python tools/trace_conv2.py 0 > gpurun_out/e9_tr2_0.log 2>&1; cat gpurun_out/e9_tr2_0.log
timeout 120 python tools/trace_conv2.py 1 > gpurun_out/e9_tr2_1.log 2>&1; tail -9 gpurun_out/e9_tr2_1.log
