# build, quick parity (golden corpus through every forced path + reference digests), then config4 bench
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || echo BUILD FAILED
timeout 900 python -m pytest tests/test_paths_gpu.py tests/test_reference_digests_gpu.py -q -x 2>&1 | tail -3
for wl in ${WL:-config4}; do
timeout 300 python bench.py --workload $wl --no-cpu-baseline --steps 10 > gpurun_out/q_$wl.json 2>>gpurun_out/q_err.log
python tools/bench_brief.py gpurun_out/q_$wl.json
done
