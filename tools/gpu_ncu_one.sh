# ncu --set full + SASS source of one kernel (regex $1, skip $2 launches) in a 128M build of shape $3
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
TAG=${4:-one}
SKIP=$2 bash tools/ncu_full.sh $TAG "$1" 1 ${3:-tied}
python - <<PY
import csv
rows=list(csv.reader(open('gpurun_out/ncu_${TAG}_source.csv',errors='ignore')))[2:]
rows=[r for r in rows if len(r)>5 and r[2].isdigit()]
with open('gpurun_out/ncu_${TAG}_sass.txt','w') as f:
    for i,r in enumerate(rows): f.write(f"{i:5d} {r[2]:>7} {r[5]:>10} {r[1].strip()}\n")
PY
rm -f gpurun_out/ncu_${TAG}_source.csv gpurun_out/ncu_${TAG}.ncu-rep
