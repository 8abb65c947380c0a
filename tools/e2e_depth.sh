# e2e leg vs builds in flight (config 4)
for d in 2 3 4; do
  timeout 300 python bench.py --no-cpu-baseline --steps 3 --e2e-depth $d > gpurun_out/e2e_d$d.json 2>>gpurun_out/e2e_err.log
  python tools/bench_brief.py gpurun_out/e2e_d$d.json | head -1
done
