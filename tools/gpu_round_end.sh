# full GPU suite + sanitizer evidence at HEAD
export PYTHONPATH=$PWD
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || echo BUILD FAILED
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu_full.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu_full.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
bash tools/sanitize_full.sh > gpurun_out/sanitizer.txt 2>&1; cat gpurun_out/sanitizer.txt
