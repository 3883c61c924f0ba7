nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/e1_smi.txt
timeout 60 tools/probes/acc_probe > gpurun_out/e1_acc_probe.txt 2>&1
bash tools/gpu_final.sh e1
