# A/B per-layer timing of library variants: bash tools/ab_stages.sh v1 v2 ...  (variants/<v>.so)
cp paper_1808_00209_b200/libbnn.so /tmp/libbnn_keep.so
for rep in 1 2; do
for v in "$@"; do
  cp variants/$v.so paper_1808_00209_b200/libbnn.so
  echo -n "$v: "; PYTHONPATH=. timeout 120 python tools/time_stages.py 2>&1 | tail -1
done
done
cp /tmp/libbnn_keep.so paper_1808_00209_b200/libbnn.so
