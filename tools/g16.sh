T=${1:-g16}
PYTHONPATH=. timeout 600 ncu --set full --import-source on --clock-control none -k regex:"conv1_fp4_pool" -c 1 -o gpurun_out/${T}_conv1 python tools/time_conv1.py 1 > gpurun_out/${T}_ncu.log 2>&1; echo "ncu rc=$?"; tail -2 gpurun_out/${T}_ncu.log
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/${T}_pytest.log 2>&1; tail -n 3 gpurun_out/${T}_pytest.log
