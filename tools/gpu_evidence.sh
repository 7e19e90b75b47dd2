# Round evidence on one box: smoke, full GPU tests, C2 bench (+CPU baseline,
# parity), reference arm, 2-rank KV-head run, C1/C3 x4 boosts/C4/C5 lines,
# launch lists at C2 / C4, one ncu --set full capture of the page kernel.
# Usage: bash tools/gpu_evidence.sh TAG
mkdir -p gpurun_out
T=${1:-ev}
bash tools/gpu_bench.sh $T
for c in c1 c4 c5; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_$c.txt 2>&1
done
for b in 0.0 0.0625 0.125 0.25; do
  timeout 900 python bench.py --config c3 --boost $b --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_c3_b$b.txt 2>&1
done
for f in gpurun_out/${T}_c1.txt gpurun_out/${T}_c4.txt gpurun_out/${T}_c5.txt gpurun_out/${T}_c3_b*.txt; do
  python -c "
import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); r=d['roofline']
print('$f'.split('/')[-1], d['value'], 'launch_ms', r['avg_launch_ms'], 'frac', r['frac'], 'e2e', d['e2e']['value'], 'parity', d.get('parity',{}).get('max_abs'))" || tail -2 $f
done
for c in c2 c4; do
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches_$c.csv \
    python bench.py --config $c --layers 2 --steps 1 --warmup 3 --no-cpu-baseline --no-graph --no-parity > /dev/null 2>&1
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:page_kernel -s 8 -c 1 \
    -o gpurun_out/${T}_page -f python bench.py --steps 1 --warmup 3 --layers 4 --no-cpu-baseline --no-graph --no-parity > gpurun_out/${T}_ncu.txt 2>&1
tail -1 gpurun_out/${T}_ncu.txt
