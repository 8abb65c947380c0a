export PYTHONPATH=$PWD
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || echo BUILD FAILED
timeout 900 python -m pytest tests/test_paths_gpu.py -x -q -k "v0 or deep or default" > gpurun_out/pt_v0.log 2>&1; echo "paths rc=$?"; tail -3 gpurun_out/pt_v0.log
timeout 600 python -m pytest tests/test_reference_digests_gpu.py -x -q > gpurun_out/dig.log 2>&1; echo "digests rc=$?"; tail -3 gpurun_out/dig.log
bash tools/gpu_ab.sh config4 '{"v0_select":1}' '{"v0_select":2}' '{"v0_select":1}' '{"v0_select":2}'
bash tools/gpu_ab.sh config5 '{"v0_select":1}' '{"v0_select":2}'
bash tools/gpu_ab.sh config3-path '{}'
