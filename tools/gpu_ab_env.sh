# A/B of an environment knob on one box.  Usage: bash tools/gpu_ab_env.sh TAG VAR "v1 v2" "c2 c3"
mkdir -p gpurun_out
T=$1; VAR=$2; VALS=$3; CFGS=${4:-c2}
for rep in 1 2; do for v in $VALS; do for c in $CFGS; do
  env $VAR=$v timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-parity > gpurun_out/${T}_${v}_$c.txt 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/${T}_${v}_$c.txt').read().strip().splitlines()[-1]); r=d['roofline']
print('$VAR=$v $c', d['value'], 'ms_step', d['ms_per_step'], 'launch_ms', r['avg_launch_ms'])" || tail -2 gpurun_out/${T}_${v}_$c.txt
done; done; done
