# L2 fetch-granularity probe: random 4-B gathers / atomics with the limit at default, 32, 64, 128
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/randbench tools/randbench.cu
for g in "" 32 64 128; do echo "== limit $g"; /tmp/randbench $g; done
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:gather --clock-control none -c 4 /tmp/randbench 32 2>&1 | grep -E "gather|dram__|gpu__time|limit" | head -30
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:gather --clock-control none -c 4 /tmp/randbench 2>&1 | grep -E "gather|dram__|gpu__time|limit" | head -30
