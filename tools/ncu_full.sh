# Full ncu capture (source-level) of kernels matching a regex, one 128M build.
# usage: bash tools/ncu_full.sh <tag> <kernel-regex> [count] [shape] [n]
TAG=$1; KRE=$2; CNT=${3:-1}; SHAPE=${4:-tied}; N=${5:-128000000}
timeout 1200 ncu --set full --import-source on --clock-control none -k "regex:$KRE" --launch-skip ${SKIP:-0} -c $CNT -o gpurun_out/ncu_$TAG -f \
  python tools/prof_driver.py --n $N --shape $SHAPE ${PATHS:+--paths "$PATHS"} > gpurun_out/ncu_$TAG.log 2>&1
ncu -i gpurun_out/ncu_$TAG.ncu-rep --page details > gpurun_out/ncu_${TAG}_details.txt 2>&1
ncu -i gpurun_out/ncu_$TAG.ncu-rep --page source --csv > gpurun_out/ncu_${TAG}_source.csv 2>&1
