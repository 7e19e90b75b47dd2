# Round evidence (one GPU): smoke, GPU tests, benches (C2 default + CPU baseline, C1, C3, C5@32, tc kernel),
# reference arm, ncu launch list and one full capture of the default attention kernel.
mkdir -p gpurun_out
nvidia-smi > gpurun_out/smi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.txt 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_c2.txt 2>&1
timeout 600 python bench.py --config c1 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c1.txt 2>&1
timeout 600 python bench.py --config c3 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c3.txt 2>&1
for b in 0 0.0625 0.25; do  # BASELINE C3 boost fractions (0.125 is bench_c3)
  timeout 600 python bench.py --config c3 --boost $b --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c3_b$b.txt 2>&1
done
timeout 900 python bench.py --config c5 --batch 32 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c5_b32.txt 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --kernel tc > gpurun_out/bench_c2_tc.txt 2>&1
timeout 600 python bench.py --config c4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4.txt 2>&1
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"append|attention|prefill|combine|fp_tokens" -c 2000 --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-graph > gpurun_out/ncu_launch_bench.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fast_attention -s 8 -c 1 \
    -o gpurun_out/prof_attn -f python bench.py --steps 1 --warmup 3 --layers 4 --no-cpu-baseline --no-graph > gpurun_out/ncu_full.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"fp_tokens|combine" -s 4 -c 2 \
    -o gpurun_out/prof_aux -f python bench.py --steps 1 --warmup 3 --layers 4 --no-cpu-baseline --no-graph > gpurun_out/ncu_aux.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:prefill_pack_fast -c 1 \
    -o gpurun_out/prof_pack -f python bench.py --config c4 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_pack.txt 2>&1
tail -n 2 gpurun_out/smoke.txt gpurun_out/pytest_gpu.txt
for f in bench_c2 bench_c1 bench_c3 bench_c3_b0 bench_c3_b0.0625 bench_c3_b0.25 bench_c4 bench_c5_b32 bench_c2_tc bench_ref; do python -c "
import json,sys
try:
    d=json.loads(open('gpurun_out/$f.txt').read().strip().splitlines()[-1]); r=d.get('roofline',{})
    print('$f', d['value'], d['unit'], 'launch_ms', r.get('avg_launch_ms'), 'frac', r.get('frac'), 'e2e', d.get('e2e',{}).get('value'))
except Exception as e: print('$f FAILED', e)
"; done
