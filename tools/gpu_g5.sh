# path/plugin/io tests + ncu --set full of the streaming kernels below 3 TB/s at 128M (config 4)
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 2400 python -m pytest tests/test_paths_gpu.py tests/test_plugin_gpu.py tests/test_io.py -x -q -m gpu --durations=10 > gpurun_out/pytest_new.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/pytest_new.log
SKIP=2 bash tools/ncu_full.sh sort2 k_downsweep 1
SKIP=0 bash tools/ncu_full.sh splitA k_split 1
SKIP=0 bash tools/ncu_full.sh fhist k_fine_hist 1
SKIP=2 bash tools/ncu_full.sh upsw k_upsweep 1
SKIP=0 bash tools/ncu_full.sh miapply k_mi_apply 1
ls -la gpurun_out/
