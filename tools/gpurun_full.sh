mkdir -p gpurun_out
nvidia-smi > gpurun_out/smi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q --maxfail=30 -p no:cacheprovider > gpurun_out/pytest_gpu.txt 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_c2.txt 2>&1
timeout 600 python bench.py --config c1 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c1.txt 2>&1
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref.txt 2>&1
bash tools/gpurun_profile.sh
tail -n 3 gpurun_out/smoke.txt gpurun_out/pytest_gpu.txt gpurun_out/bench_c2.txt gpurun_out/bench_c1.txt gpurun_out/bench_ref.txt
