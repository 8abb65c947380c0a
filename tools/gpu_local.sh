# local-sort change: parity (wide-key tests + digests of config4u) and config4u timing
export PYTHONPATH=$PWD
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || echo BUILD FAILED
timeout 900 python -m pytest tests/test_paths_gpu.py -x -q -k "wide_key or v0" > gpurun_out/pt_local.log 2>&1; echo "local rc=$?"; tail -2 gpurun_out/pt_local.log
timeout 900 python -m pytest tests/test_reference_digests_gpu.py -x -q -k "test_reference_digest and not host and not config5" > gpurun_out/dig2.log 2>&1; echo "digests rc=$?"; tail -2 gpurun_out/dig2.log
for i in 1 2; do for wl in config4u config4; do timeout 300 python bench.py --workload $wl --no-cpu-baseline --steps 10 > gpurun_out/ab.json 2>/dev/null; echo "== $wl"; python tools/bench_brief.py gpurun_out/ab.json | grep -o "^gpurun_out/ab.json: [0-9.]* ms\|'sort1_local': [0-9.]*\|'select_edges': [0-9.]*"; done; done
