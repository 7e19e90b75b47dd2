mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.txt 2>&1; tail -2 gpurun_out/pytest_gpu.txt
bash tools/ab.sh exp/libPack4.so exp/libComb.so
KITTY_PDL=7 bash tools/ab.sh exp/libPack4.so exp/libComb.so | tail -2
bash tools/ab.sh exp/libPack4.so exp/libComb.so --config c4 | tail -2
KITTY_PDL=7 bash tools/ab.sh exp/libPack4.so exp/libComb.so --config c4 | tail -2
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c2.txt 2>&1; python -c "import json; d=json.loads(open('gpurun_out/bench_c2.txt').read().strip().splitlines()[-1]); print(d['value'], d['e2e'])"
