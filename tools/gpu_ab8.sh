export PYTHONPATH=$PWD
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for r in 1 2; do for p in '{}' '{"sort2_geometry":1}' '{"mi_apply_mode":1}'; do
  timeout 300 python bench.py --workload config4 --no-cpu-baseline --steps 10 --paths "$p" > gpurun_out/ab.json 2>/dev/null
  echo "== $p $(python tools/bench_brief.py gpurun_out/ab.json 2>/dev/null | head -1 | grep -o '[0-9.]* ms/step')"
done; done
