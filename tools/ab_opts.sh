# A/B of library variants (variants/<v>.so) under option settings: bash tools/ab_opts.sh "opts1 opts2" v1 v2 ...
opts=$1; shift
cp paper_1808_00209_b200/libbnn.so /tmp/libbnn_keep.so
for v in "$@"; do
  cp variants/$v.so paper_1808_00209_b200/libbnn.so
  echo "== $v"; PYTHONPATH=. timeout 200 python tools/time_opts.py $opts 2>&1 | tail -4
done
cp /tmp/libbnn_keep.so paper_1808_00209_b200/libbnn.so
