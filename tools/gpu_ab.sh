# A/B of library variants on one box: attention tests on the default build, then
# C2 (and optional extra config) bench for every listed .so.  Usage:
#   bash tools/gpu_ab.sh TAG "libA.so libB.so" [config]
mkdir -p gpurun_out
T=$1; LIBS=$2; CFG=${3:-}
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "attention or cache or pool" > gpurun_out/${T}_pytest.txt 2>&1
tail -n 2 gpurun_out/${T}_pytest.txt
for rep in 1 2; do
for L in $LIBS; do
  for c in c2 $CFG; do
    KITTY_B200_LIB=$PWD/paper_2511_18643_b200/$L timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-parity > gpurun_out/${T}_${L}_$c.txt 2>&1
    python -c "
import json; d=json.loads(open('gpurun_out/${T}_${L}_$c.txt').read().strip().splitlines()[-1]); r=d['roofline']
print('$L $c', d['value'], 'launch_ms', r['avg_launch_ms'], 'frac', r['frac'])" || tail -3 gpurun_out/${T}_${L}_$c.txt
  done
done
done
