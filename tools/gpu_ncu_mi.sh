# ncu --set full of the sliced maxIncident apply of view 0 (k_mi_atomic) and its V1 (k_v1)
export PYTHONPATH=$PWD
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
bash tools/gpu_ncu_one.sh "k_mi_atomic" 0 tied miatomic_r02
bash tools/gpu_ncu_one.sh "k_v1" 0 tied v1_r02
for t in miatomic_r02 v1_r02; do grep -E "Duration|DRAM Throughput|L2 Cache Throughput|Memory Throughput|L2 Hit Rate|Achieved Occupancy|Registers Per" gpurun_out/ncu_${t}_details.txt | head -9; echo; done
