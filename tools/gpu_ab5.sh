export PYTHONPATH=$PWD
timeout 900 python -m pytest tests/test_paths_gpu.py -x -q -k "deep or v0 or synthetic" > gpurun_out/pt_ab5.log 2>&1; echo "paths rc=$?"; tail -2 gpurun_out/pt_ab5.log
bash tools/gpu_ab_variants.sh config4 2 oldgrid w2 w4 retkeep
bash tools/gpu_ab_variants.sh config5 1 oldgrid w2
