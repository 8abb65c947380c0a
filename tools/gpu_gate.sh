# chase-gate A/B on smaller trees: forced V2 vs forced chase
export PYTHONPATH=$PWD
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for r in 1 2; do for wl in random16M config5 config2; do for p in '{"v0_select":1}' '{"v0_select":2}'; do
  timeout 300 python bench.py --workload $wl --no-cpu-baseline --steps 10 --paths "$p" > gpurun_out/ab.json 2>/dev/null
  echo "== $wl $p $(python tools/bench_brief.py gpurun_out/ab.json 2>/dev/null | head -1 | grep -o '[0-9.]* ms/step')"
done; done; done
