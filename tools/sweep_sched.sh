# schedule sweep (KITTY_SCHED = "level1 permille, level2 permille, max pages per chunk, level-1 divisor")
# usage: bash tools/sweep_sched.sh [bench args]
mkdir -p gpurun_out
for s in ${SCHEDS:-"850,950,8,4" "800,930,8,4" "880,960,8,4" "850,950,10,4" "850,950,6,4" "850,950,8,2" "900,975,8,4"}; do
  r=$(KITTY_SCHED=$s timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline "$@" 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['avg_launch_ms'])")
  echo "$* $s -> $r" | tee -a gpurun_out/sweep.txt
done
