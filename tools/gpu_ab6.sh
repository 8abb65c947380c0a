export PYTHONPATH=$PWD
bash tools/gpu_ab_variants.sh config4 2 agg1 agg2
for v in agg1 agg2; do cp paper_2401_06089_b200/libdmst_$v.so paper_2401_06089_b200/libdmst.so; touch paper_2401_06089_b200/libdmst.so; timeout 300 python bench.py --workload config4u --no-cpu-baseline --steps 5 > gpurun_out/ab.json 2>/dev/null; echo "== $v config4u $(python tools/bench_brief.py gpurun_out/ab.json 2>/dev/null| head -1 | grep -o 'ms/step.*parity.*')" | cut -c1-200; done
