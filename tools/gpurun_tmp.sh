timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.txt 2>&1; tail -1 gpurun_out/pytest_gpu.txt
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for c in c2 c5; do timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline $( [ $c = c5 ] && echo --batch 32 ) 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', d['value'], d['roofline']['avg_launch_ms'], d['roofline']['frac'], d['e2e']['value'])"; done
