# chasing-select A/B: library variants (DMST_SEL_CHASE_U) x v0_select, config4 and config5
export PYTHONPATH=$PWD
cp paper_2401_06089_b200/libdmst.so /tmp/base.so
for v in base u1 u4; do
  if [ $v = base ]; then cp /tmp/base.so paper_2401_06089_b200/libdmst.so; else cp paper_2401_06089_b200/libdmst_$v.so paper_2401_06089_b200/libdmst.so; fi
  touch paper_2401_06089_b200/libdmst.so
  for wl in config4 config5; do for p in '{"v0_select":2}' '{"v0_select":1}'; do
    [ $v != base ] && [ "$p" = '{"v0_select":1}' ] && continue
    timeout 300 python bench.py --workload $wl --no-cpu-baseline --steps 10 --paths "$p" > gpurun_out/ab.json 2>/dev/null
    echo "== $v $wl $p"; python tools/bench_brief.py gpurun_out/ab.json | grep -o "^gpurun_out/ab.json: [0-9.]* ms\|'select_edges': [0-9.]*\|'v2': [0-9.]*"
  done; done
done
cp /tmp/base.so paper_2401_06089_b200/libdmst.so
