timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.txt 2>&1; tail -1 gpurun_out/pytest_gpu.txt
bash tools/ab.sh exp/libBase.so exp/libMw.so --config c3 | tail -4
bash tools/ab.sh exp/libBase.so exp/libMw.so | tail -2
bash tools/ab.sh exp/libBase.so exp/libMw.so --config c1 | tail -2
timeout 300 python bench.py --config c1 --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c1', d['value'], d['e2e'])"
