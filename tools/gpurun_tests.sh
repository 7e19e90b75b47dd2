# GPU test + short bench pass (used from gpurun); writes into gpurun_out/
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q --maxfail=30 -p no:cacheprovider > gpurun_out/pytest_gpu.txt 2>&1
timeout 600 python bench.py --config c1 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c1.txt 2>&1
timeout 900 python bench.py --steps 5 --warmup 3 ${BENCH_ARGS} > gpurun_out/bench_c2.txt 2>&1
tail -n 3 gpurun_out/smoke.txt gpurun_out/pytest_gpu.txt gpurun_out/bench_c1.txt gpurun_out/bench_c2.txt
