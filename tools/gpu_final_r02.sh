# round-2 final evidence: sanitizer, profiles (bench lines, ncu kinds/launches, captures), all configs
export PYTHONPATH=$PWD
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || echo BUILD FAILED
which compute-sanitizer || ls /usr/local/cuda/bin/compute-sanitizer
export PATH=$PATH:/usr/local/cuda/bin
for t in memcheck racecheck synccheck initcheck; do
  echo "== $t"; timeout 1500 compute-sanitizer --tool $t --print-limit 20 python tools/sanitize_driver.py > gpurun_out/san_$t.log 2>&1; echo "rc=$?"
  grep -E "ERROR SUMMARY|RACECHECK SUMMARY|mismatches" gpurun_out/san_$t.log | head -5; tail -3 gpurun_out/san_$t.log
done > gpurun_out/sanitizer_r02c.txt 2>&1
cat gpurun_out/sanitizer_r02c.txt
TAG=r02c bash tools/gpu_profiles_r02.sh
bash tools/gpu_all_configs.sh > gpurun_out/all_r02c.txt 2>&1
cat gpurun_out/all_*.json > gpurun_out/all_configs_r02c.jsonl
cat gpurun_out/all_r02c.txt
