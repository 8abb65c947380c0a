# round-2 first GPU pass: full -m gpu suite, then config4 / config4u benches
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 2400 python -m pytest tests -q -m gpu --durations=15 > gpurun_out/pytest_gpu_r2a.log 2>&1; echo "pytest rc=$?"
tail -25 gpurun_out/pytest_gpu_r2a.log
for w in config4 config4u; do
  timeout 400 python bench.py --workload $w --no-cpu-baseline > gpurun_out/bench_$w.json 2>>gpurun_out/bench_err.log; echo "== $w"; python tools/bench_brief.py gpurun_out/bench_$w.json
done
tail -5 gpurun_out/bench_err.log
