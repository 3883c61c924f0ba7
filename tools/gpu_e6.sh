export PYTHONPATH=. BNN_TRACE_LIB=1
timeout 200 python tools/time_conv1_exp.py 1 0 1 2 3 4 8 12 16 32 48 51 0 > gpurun_out/e6_p1.log 2>&1; cat gpurun_out/e6_p1.log
timeout 200 python tools/time_conv1_exp.py 0 0 3 4 8 16 32 48 51 0 > gpurun_out/e6_p0.log 2>&1; cat gpurun_out/e6_p0.log
