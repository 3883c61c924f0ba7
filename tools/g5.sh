T=${1:-g5}
PYTHONPATH=. BNN_TRACE_LIB=1 timeout 300 python tools/trace_conv1.py 1 > gpurun_out/${T}_trace1.log 2>&1; cat gpurun_out/${T}_trace1.log
PYTHONPATH=. timeout 600 ncu --set full --import-source on --clock-control none -k regex:"conv1_fp4_pool" -c 1 -o gpurun_out/${T}_conv1 python tools/time_conv1.py 1 > gpurun_out/${T}_ncu.log 2>&1; echo "ncu rc=$?"; tail -2 gpurun_out/${T}_ncu.log
