# The unmodified reference (baseline/_ref) timed on the GPU box's host at full config-4 size and on
# the bounded sample the default bench uses; rank_edges + pandora as cli.py:82-85 scopes it.
nproc; free -g | head -2; lscpu | grep -E "Model name|^CPU\(s\)|Thread|Socket" 
for spec in "config4 128000000 1" "config4 16000000 3" "config4u 128000000 1"; do
  set -- $spec
  timeout 1500 python bench.py --cpu-worker --workload $1 --n $2 --repeats $3 > gpurun_out/cpuref_$1_$2.json 2> gpurun_out/cpuref_$1_$2.err
  echo "== $1 $2"; cat gpurun_out/cpuref_$1_$2.json; tail -2 gpurun_out/cpuref_$1_$2.err
done
