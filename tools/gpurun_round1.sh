set -x
mkdir -p gpurun_out
nvidia-smi > gpurun_out/smi.txt 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/probe_mma tools/probe_mma.cu && /tmp/probe_mma > gpurun_out/probe.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q --maxfail=30 -p no:cacheprovider > gpurun_out/pytest_gpu.txt 2>&1
timeout 600 python bench.py --config c1 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c1.txt 2>&1
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_c2.txt 2>&1
tail -3 gpurun_out/*.txt
