export PYTHONPATH=$PWD
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || echo BUILD FAILED
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu_last.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu_last.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
