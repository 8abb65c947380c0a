cp paper_2401_06089_b200/libdmst.so /tmp/base.so
for v in base ls1024 ls4096; do
  if [ $v = base ]; then cp /tmp/base.so paper_2401_06089_b200/libdmst.so; else cp paper_2401_06089_b200/libdmst_$v.so paper_2401_06089_b200/libdmst.so; fi
  touch paper_2401_06089_b200/libdmst.so
  timeout 300 python bench.py --workload config4 --no-cpu-baseline --steps 10 > gpurun_out/ab.json 2>/dev/null; echo "== $v"; python tools/bench_brief.py gpurun_out/ab.json | grep -o "^gpurun_out/ab.json: [0-9.]* ms\|'leafscan': [0-9.]*"
done
cp /tmp/base.so paper_2401_06089_b200/libdmst.so
