# Round-2 profile artefacts -> gpurun_out/ (copied to profiles/ by hand)
export PYTHONPATH=$PWD
TAG=${TAG:-r02}
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv
# per-launch DRAM traffic of one 128M build, both weight sets (bench.py roofline.traffic)
bash tools/ncu_all.sh traffic tied 128000000
python tools/ncu_traffic.py gpurun_out/ncu_traffic.ncu-rep config4 --out gpurun_out/ncu_traffic.json --csv gpurun_out/ncu_kinds_$TAG.csv > gpurun_out/ncu_kinds_$TAG.txt
bash tools/ncu_all.sh trafficu random 128000000
python tools/ncu_traffic.py gpurun_out/ncu_trafficu.ncu-rep config4u --out gpurun_out/ncu_traffic.json --csv gpurun_out/ncu_kinds_u_$TAG.csv > gpurun_out/ncu_kinds_u_$TAG.txt
cp gpurun_out/ncu_traffic.json profiles/ncu_traffic.json
# per-launch raw metrics kept (the kind map can be re-applied without a re-capture)
for r in ncu_traffic ncu_trafficu; do ncu -i gpurun_out/$r.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum > gpurun_out/${r}_raw_$TAG.csv; done
rm -f gpurun_out/*.ncu-rep
# headline bench line (CPU baseline: the unmodified reference at full size)
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
timeout 600 python bench.py --workload config4u --no-cpu-baseline > gpurun_out/bench_u_$TAG.json 2>> gpurun_out/bench_$TAG.err
# launch list of the bench command
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/bench_under_ncu.log 2>&1
python tools/launch_summary.py gpurun_out/launches_$TAG.csv --out gpurun_out/launches_${TAG}_summary.csv
# full capture of the dominant kernel (select_edges on view 0) and of the local sort
bash tools/gpu_ncu_one.sh "k_select_edges" 0 tied select_$TAG
bash tools/gpu_ncu_one.sh "k_local_final" 0 random local_$TAG
ls -la gpurun_out | head -40
