# mma.sync kind throughput probe + ncu full capture of one C2 page-kernel launch.
# Usage: bash tools/gpu_probe.sh TAG
mkdir -p gpurun_out
T=${1:-probe}
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/probe_mma_kinds tools/probe_mma_kinds.cu && /tmp/probe_mma_kinds > gpurun_out/${T}_mma_kinds.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:page_kernel -s 8 -c 1 \
    -o gpurun_out/${T} -f python bench.py --steps 1 --warmup 3 --layers 4 --no-cpu-baseline --no-graph > gpurun_out/${T}_ncu.txt 2>&1
tail -3 gpurun_out/${T}_ncu.txt; cat gpurun_out/${T}_mma_kinds.txt
