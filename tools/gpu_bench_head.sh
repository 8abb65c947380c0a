export PYTHONPATH=$PWD
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || echo BUILD FAILED
timeout 900 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; echo "rc=$?"
python tools/bench_brief.py gpurun_out/bench_final.json 2>/dev/null | head -1
python -c "import json; d=json.load(open('gpurun_out/bench_final.json')); print(d['roofline']); print(d['cpu_baseline'])"
