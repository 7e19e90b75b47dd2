# iteration: smoke, gpu tests (stop at first failure), c2 bench, trace
mkdir -p gpurun_out
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.txt
timeout 600 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.txt 2>&1
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/bench_c2.txt 2>&1
timeout 120 python tools/trace_tc.py --rows 8 > gpurun_out/trace.txt 2>&1
tail -n 3 gpurun_out/smoke.txt gpurun_out/pytest_gpu.txt
python -c "
import json
try:
    d=json.loads(open('gpurun_out/bench_c2.txt').read().strip().splitlines()[-1]); print('C2', d['value'], 'tok/s', d['roofline']['avg_launch_ms']*1e3, 'us/launch frac', d['roofline']['frac'], 'e2e', d['e2e']['value'])
except Exception as e: print('bench failed', e); print(open('gpurun_out/bench_c2.txt').read()[-2000:])
"
tail -n 16 gpurun_out/trace.txt
