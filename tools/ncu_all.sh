# Per-kernel time + DRAM traffic table for one 128M build (ncu, metrics subset).
# usage: bash tools/ncu_all.sh <tag> [shape] [n]
TAG=${1:-all}; SHAPE=${2:-tied}; N=${3:-128000000}
MET="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active,sm__throughput.avg.pct_of_peak_sustained_elapsed,gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed,launch__registers_per_thread,lts__t_sectors.sum"
timeout 900 ncu --metrics $MET --clock-control none -o gpurun_out/ncu_$TAG -f python tools/prof_driver.py --n $N --shape $SHAPE > gpurun_out/ncu_$TAG.log 2>&1
python tools/ncu_summary.py gpurun_out/ncu_$TAG.ncu-rep > gpurun_out/ncu_$TAG.txt 2>&1
