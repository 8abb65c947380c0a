# round-2 final evidence at HEAD: GPU suite, smoke, profiles, all configs
export PYTHONPATH=$PWD
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || echo BUILD FAILED
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu_final.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu_final.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
TAG=r02d bash tools/gpu_profiles_r02.sh > gpurun_out/profiles_r02d.log 2>&1
rm -f gpurun_out/all_*.json
bash tools/gpu_all_configs.sh > gpurun_out/all_r02d.txt 2>&1
cat gpurun_out/all_*.json > gpurun_out/all_configs_r02d.jsonl
grep -o "^gpurun_out/all_[a-z0-9-]*.json: [0-9.]* ms/step" gpurun_out/all_r02d.txt
