# A/B two library builds on the same box: bash tools/ab.sh exp/libA.so exp/libB.so [bench args]
A=$1; B=$2; shift 2
for i in 1 2 3; do for L in $A $B; do
  KITTY_B200_LIB=$L timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline "$@" > /tmp/ab.txt 2>&1
  python -c "import json; d=json.loads(open('/tmp/ab.txt').read().strip().splitlines()[-1]); print('$L', d['value'], d['roofline']['avg_launch_ms'], d['ms_per_step'])" || tail -3 /tmp/ab.txt
done; done
