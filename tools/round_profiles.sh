# Refresh every round artefact under gpurun_out/ (copied to profiles/ by hand).
export PYTHONPATH=$PWD
TAG=${TAG:-r01}
bash tools/gpu_profiles.sh > gpurun_out/gpu_profiles.log 2>&1
bash tools/gpu_all_configs.sh > gpurun_out/all_configs.log 2>&1
cat gpurun_out/all_config*.json > /dev/null 2>&1
for n in 100000 1000000; do timeout 300 python tools/mreach_time.py $n; done > gpurun_out/mreach_time.txt 2>&1
timeout 300 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
