# quick GPU check: parity tests + headline bench + companion workloads
set -x
if [ -z "$NOTEST" ]; then timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log; fi
for w in ${WORKLOADS:-config4 config4u}; do timeout 300 python bench.py --workload $w --no-cpu-baseline > gpurun_out/bench_$w.json 2>>gpurun_out/bench_err.log; python tools/bench_brief.py gpurun_out/bench_$w.json; done
tail -5 gpurun_out/bench_err.log
