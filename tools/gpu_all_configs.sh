# Every BASELINE.json configuration through bench.py (1 GPU), one JSON line each.
for w in config1 config2 config3-path config3-caterpillar random16M config4 config4u config5; do
  timeout 600 python bench.py --workload $w --no-cpu-baseline > gpurun_out/all_$w.json 2>> gpurun_out/all_err.log
  python tools/bench_brief.py gpurun_out/all_$w.json
done
