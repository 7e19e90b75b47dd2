# Quick GPU check: GPU tests, smoke, one C2 bench line.  Usage: bash tools/gpu_quick.sh [pytest -k expr]
mkdir -p gpurun_out
K=${1:-}
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1
if [ -n "$K" ]; then
  timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -k "$K" > gpurun_out/pytest_gpu.txt 2>&1
else
  timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.txt 2>&1
fi
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c2.txt 2>&1
tail -n 3 gpurun_out/smoke.txt; tail -n 25 gpurun_out/pytest_gpu.txt; tail -n 2 gpurun_out/bench_c2.txt | cut -c1-600
