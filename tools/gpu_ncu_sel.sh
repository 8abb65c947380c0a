# ncu of view 0's label stage: the chasing select vs V2 + the vertex-map select
export PYTHONPATH=$PWD
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
PATHS='{"v0_select":2}' bash tools/gpu_ncu_one.sh "k_select_edges" 0 tied selchase
PATHS='{"v0_select":1}' bash tools/gpu_ncu_one.sh "k_select_edges" 0 tied selvm
PATHS='{"v0_select":1}' bash tools/gpu_ncu_one.sh "k_v2" 0 tied v2v0
for t in selchase selvm v2v0; do grep -E "Duration|DRAM Throughput|L2 Hit Rate|Achieved Occupancy|Registers Per|Memory Throughput|L1/TEX Hit|Theoretical Occ|Warp Cycles Per Issued" gpurun_out/ncu_${t}_details.txt | head -12; echo; done
