timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/e13_t.log 2>&1; tail -2 gpurun_out/e13_t.log
bash tools/ab_opts.sh "conv_pair=1 conv_pair=0,conv_pool3=0" cur > gpurun_out/e13.log 2>&1; cat gpurun_out/e13.log
