T=${1:-g4}
timeout 300 env PYTHONPATH=. python tools/time_conv1.py 0 1 2 > gpurun_out/${T}_time.log 2>&1; cat gpurun_out/${T}_time.log
PYTHONPATH=. timeout 600 ncu --set full --import-source on --clock-control none -k regex:"conv1_fp4" -c 1 -o gpurun_out/${T}_conv1 python tools/time_conv1.py 1 > gpurun_out/${T}_ncu.log 2>&1; echo "ncu rc=$?"; tail -3 gpurun_out/${T}_ncu.log
