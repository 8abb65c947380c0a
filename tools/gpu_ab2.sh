export PYTHONPATH=$PWD
timeout 900 python -m pytest tests/test_paths_gpu.py -x -q -k "deep or v0 or generators" > gpurun_out/pt_ab2.log 2>&1; echo "paths rc=$?"; tail -2 gpurun_out/pt_ab2.log
bash tools/gpu_ab_variants.sh config4 2 selldg nokeep
bash tools/gpu_ab_variants.sh config5 2 nokeep
bash tools/gpu_ab_variants.sh random16M 2 nokeep
