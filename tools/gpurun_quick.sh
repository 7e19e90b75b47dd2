# quick GPU iteration: smoke, gpu tests, c2 + c1 bench (each under its own timeout)
mkdir -p gpurun_out
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.txt
timeout 600 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.txt 2>&1
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/bench_c2.txt 2>&1
timeout 300 python bench.py --config c1 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c1.txt 2>&1
tail -n 4 gpurun_out/smoke.txt gpurun_out/pytest_gpu.txt gpurun_out/bench_c2.txt gpurun_out/bench_c1.txt
