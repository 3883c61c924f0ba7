for p in 0 1; do
timeout 600 ncu --set full --clock-control none -k regex:"^(conv1_fp4_pool|conv_tc4_pool|dense_tc4_kernel)" -c 3 -o /tmp/e4_pair$p env PYTHONPATH=. python tools/one_forward.py conv_pair=$p > gpurun_out/e4_ncu$p.log 2>&1; tail -1 gpurun_out/e4_ncu$p.log
ncu -i /tmp/e4_pair$p.ncu-rep --page raw --csv > gpurun_out/e4_raw$p.csv 2>&1
done
ls -la gpurun_out
