python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
bash tools/ncu_full.sh local 'k_local_final' 1 random
ncu -i gpurun_out/ncu_local.ncu-rep --page raw --csv > gpurun_out/ncu_local_raw.csv 2>&1
python - <<'PY'
import csv
rows = list(csv.reader(open('gpurun_out/ncu_local_source.csv', errors='ignore')))
print(len(rows)); print(rows[0][:12])
PY
head -c 3000000 gpurun_out/ncu_local_source.csv > gpurun_out/ncu_local_source_head.csv
rm -f gpurun_out/ncu_local_source.csv gpurun_out/ncu_local.ncu-rep
