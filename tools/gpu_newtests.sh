# forced-path parity tests, then A/B of the warp-ranking variants at 128M
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 2400 python -m pytest tests/test_paths_gpu.py tests/test_io.py -x -q -m gpu --durations=10 > gpurun_out/pytest_new.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/pytest_new.log
for p in '{}' '{"sort2_geometry": 3}' '{"sort2_geometry": 4}' '{"sort2_geometry": 1}'; do
  timeout 300 python bench.py --workload config4 --no-cpu-baseline --paths "$p" > gpurun_out/ab.json 2>>gpurun_out/bench_err.log; echo "== $p"; python tools/bench_brief.py gpurun_out/ab.json
done
for p in '{}' '{"sort1_mode": 4}' '{"sort1_mode": 4, "sort2_geometry": 4}'; do
  timeout 300 python bench.py --workload config4u --no-cpu-baseline --paths "$p" > gpurun_out/ab.json 2>>gpurun_out/bench_err.log; echo "== u $p"; python tools/bench_brief.py gpurun_out/ab.json
done
