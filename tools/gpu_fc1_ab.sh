for v in kc8c2 kc8c1; do cp variants/$v.so paper_1808_00209_b200/libbnn.so; echo "== $v"; timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "dense or forward_vehicle" 2>&1 | tail -1; done
cp variants/kc16.so paper_1808_00209_b200/libbnn.so
bash tools/ab_bench_libs.sh kc16 kc8c2 kc8c1
