# A/B prebuilt library variants (paper_2401_06089_b200/libdmst_<v>.so) on one workload:
#   bash tools/ab_lib_variants.sh WORKLOAD v1 v2 ...   ("base" = the in-tree build)
wl=$1; shift
cp paper_2401_06089_b200/libdmst.so /tmp/base.so
for v in base "$@"; do
  if [ $v = base ]; then cp /tmp/base.so paper_2401_06089_b200/libdmst.so; else cp paper_2401_06089_b200/libdmst_$v.so paper_2401_06089_b200/libdmst.so; fi
  touch paper_2401_06089_b200/libdmst.so
  timeout 300 python bench.py --workload $wl --no-cpu-baseline --steps 10 > gpurun_out/ab.json 2>/dev/null; echo "== $v"
  python tools/bench_brief.py gpurun_out/ab.json | grep -o "^gpurun_out/ab.json: [0-9.]* ms\|'mi_apply': [0-9.]*\|'mi_split_a': [0-9.]*"
done
cp /tmp/base.so paper_2401_06089_b200/libdmst.so
