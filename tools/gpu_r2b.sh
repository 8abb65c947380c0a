# full -m gpu suite + every configuration's bench line
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 2400 python -m pytest tests -q -m gpu --durations=10 > gpurun_out/pytest_gpu_r2b.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/pytest_gpu_r2b.log
bash tools/gpu_all_configs.sh
