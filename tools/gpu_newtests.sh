# new parity tests of round 2: forced code paths, reference digests at full size, IO fixes
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 2400 python -m pytest tests/test_reference_digests_gpu.py tests/test_paths_gpu.py tests/test_io.py -x -q -m gpu --durations=15 > gpurun_out/pytest_new.log 2>&1; echo "pytest rc=$?"
tail -30 gpurun_out/pytest_new.log
