# Bench lines for C1/C3/C4/C5 + ncu launch lists (kernel durations) at C2 and C4.
# Usage: bash tools/gpu_configs.sh TAG
mkdir -p gpurun_out
T=${1:-cfg}
for c in c4 c3 c5 c1; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_$c.txt 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/${T}_$c.txt').read().strip().splitlines()[-1]); r=d['roofline']
print('$c value', d['value'], 'launch_ms', r['avg_launch_ms'], 'frac', r['frac'], 'e2e', d['e2e']['value'], 'parity', d.get('parity',{}).get('max_abs'))" || tail -3 gpurun_out/${T}_$c.txt
done
for c in c2 c4; do
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches_$c.csv \
    python bench.py --config $c --layers 2 --steps 1 --warmup 3 --no-cpu-baseline --no-graph --no-parity > /dev/null 2>&1
done
python tools/launch_summary.py gpurun_out/${T}_launches_c4.csv 2>/dev/null | tail -12
