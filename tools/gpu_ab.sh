# A/B of code-path / kernel-variant settings: bash tools/gpu_ab.sh WORKLOAD 'JSON' ['JSON' ...]
wl=$1; shift
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || echo BUILD FAILED
for p in "$@"; do
  timeout 300 python bench.py --workload $wl --no-cpu-baseline --steps 10 --paths "$p" > gpurun_out/ab.json 2>>gpurun_out/ab_err.log
  echo "== $wl $p"; python tools/bench_brief.py gpurun_out/ab.json
done
