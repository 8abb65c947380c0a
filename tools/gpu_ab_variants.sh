# A/B of build-time variants (paper_2401_06089_b200/libdmst_<v>.so) vs the in-tree build, interleaved:
#   bash tools/gpu_ab_variants.sh WORKLOAD REPEATS v1 v2 ...
export PYTHONPATH=$PWD
wl=$1; rep=$2; shift 2
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
cp paper_2401_06089_b200/libdmst.so /tmp/base.so
for r in $(seq $rep); do for v in base "$@"; do
  if [ $v = base ]; then cp /tmp/base.so paper_2401_06089_b200/libdmst.so; else cp paper_2401_06089_b200/libdmst_$v.so paper_2401_06089_b200/libdmst.so; fi
  touch paper_2401_06089_b200/libdmst.so
  timeout 300 python bench.py --workload $wl --no-cpu-baseline --steps 10 > gpurun_out/ab.json 2>/dev/null
  echo "== $v $(python tools/bench_brief.py gpurun_out/ab.json | head -1 | grep -o '[0-9.]* ms/step') $(python tools/bench_brief.py gpurun_out/ab.json | tail -1 | grep -o "'mi_split_a': [0-9.]*\|'link_split': [0-9.]*\|'mi_apply': [0-9.]*\|'v2': [0-9.]*\|'select_edges': [0-9.]*\|'walk': [0-9.]*" | tr '\n' ' ')"
done; done
cp /tmp/base.so paper_2401_06089_b200/libdmst.so
