# Round profile artefacts: traffic table from an ncu metrics pass over one
# 128M build, the headline bench line (with CPU baseline), and the ncu launch
# list of the bench command.  Outputs in gpurun_out/ (copied to profiles/ by hand).
set -x
TAG=${TAG:-r01}
bash tools/ncu_all.sh traffic tied 128000000
python tools/ncu_traffic.py gpurun_out/ncu_traffic.ncu-rep config4 --out profiles/ncu_traffic.json --csv gpurun_out/ncu_kinds_$TAG.csv > gpurun_out/ncu_kinds_$TAG.txt
cp profiles/ncu_traffic.json gpurun_out/ncu_traffic.json
timeout 600 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 700 --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/bench_under_ncu.log 2>&1
