timeout 600 python bench.py --config c3 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c3.txt 2>&1
for b in 0 0.0625 0.25; do timeout 600 python bench.py --config c3 --boost $b --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c3_b$b.txt 2>&1; done
timeout 900 python bench.py --config c5 --batch 32 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c5_b32.txt 2>&1
for f in bench_c3 bench_c3_b0 bench_c3_b0.0625 bench_c3_b0.25 bench_c5_b32; do python -c "import json; d=json.loads(open('gpurun_out/$f.txt').read().strip().splitlines()[-1]); print('$f', d['value'], d['roofline']['avg_launch_ms'], d['roofline']['frac'], d['e2e']['value'])"; done
