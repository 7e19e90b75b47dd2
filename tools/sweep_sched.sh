# schedule sweep (KITTY_SCHED = "level1 permille, level2 permille, max pages per chunk, level-1 divisor")
mkdir -p gpurun_out
for s in "850,950,8,4" "900,960,8,4" "880,960,8,8" "900,970,8,8" "850,950,12,4" "900,960,8,2"; do
  r=$(KITTY_SCHED=$s timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['avg_launch_ms'])")
  echo "$s -> $r" | tee -a gpurun_out/sweep.txt
done
