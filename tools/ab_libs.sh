# A/B timing of library variants: bash tools/ab_libs.sh v4 v5 v7 ...  (variants/<v>.so)
cp paper_1808_00209_b200/libbnn.so /tmp/libbnn_keep.so
for rep in 1 2; do
for v in "$@"; do
  cp variants/$v.so paper_1808_00209_b200/libbnn.so
  echo -n "$v: "; PYTHONPATH=. timeout 120 python tools/time_conv1.py 1 2>&1 | tail -1
done
done
cp /tmp/libbnn_keep.so paper_1808_00209_b200/libbnn.so
