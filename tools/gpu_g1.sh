set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
for g in 0 32 64 128; do ./tools/randbench $g; done > gpurun_out/randbench_l2g.txt 2>&1
for w in config4 config4u; do timeout 300 python bench.py --workload $w --no-cpu-baseline > gpurun_out/bench_$w.json 2>>gpurun_out/bench_err.log; python tools/bench_brief.py gpurun_out/bench_$w.json; done
tail -5 gpurun_out/bench_err.log
