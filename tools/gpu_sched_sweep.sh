# Sweep of the page-queue schedule (KITTY_SCHED = "l1,l2,ppc_max,cs1_div[,ppc_div]") on one config.
# Usage: bash tools/gpu_sched_sweep.sh TAG CONFIG "sched1 sched2 ..."
mkdir -p gpurun_out
T=$1; C=$2; SCHEDS=$3
for rep in 1 2; do for v in $SCHEDS; do
  KITTY_SCHED=$v timeout 600 python bench.py --config $C --steps 10 --warmup 3 --no-cpu-baseline --no-parity > gpurun_out/${T}_$C.txt 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/${T}_$C.txt').read().strip().splitlines()[-1]); r=d['roofline']
print('$v $C', d['value'], 'launch_ms', r['avg_launch_ms'])" || tail -2 gpurun_out/${T}_$C.txt
done; done
