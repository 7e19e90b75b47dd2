# ncu full capture of one page-kernel launch at the C2 shape (+ the mma/alu probe).
# Usage: bash tools/gpu_prof.sh [tag] [extra bench args]
mkdir -p gpurun_out
T=${1:-prof}; shift || true
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/probe_mma tools/probe_mma.cu && /tmp/probe_mma > gpurun_out/probe_mma.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:page_kernel -s 8 -c 1 \
    -o gpurun_out/$T -f python bench.py --steps 1 --warmup 3 --layers 4 --no-cpu-baseline --no-graph "$@" > gpurun_out/${T}_ncu.txt 2>&1
tail -3 gpurun_out/${T}_ncu.txt; cat gpurun_out/probe_mma.txt
