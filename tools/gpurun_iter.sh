# quick iteration: gpu tests + c2 bench (+ optional profile)
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.txt 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c2.txt 2>&1
timeout 600 python bench.py --config c1 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c1.txt 2>&1
if [ "$PROFILE" = "1" ]; then
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fast_attention -s 8 -c 1 \
    -o gpurun_out/prof_attn -f python bench.py --steps 1 --warmup 3 --layers 4 --no-cpu-baseline --no-graph > gpurun_out/ncu_full.txt 2>&1
fi
tail -n 3 gpurun_out/smoke.txt gpurun_out/pytest_gpu.txt gpurun_out/bench_c2.txt gpurun_out/bench_c1.txt
