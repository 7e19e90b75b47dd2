# schedule sweep (KITTY_SCHED = "level1 permille, level2 permille, max pages per chunk, level-1 divisor")
mkdir -p gpurun_out
for s in "750,920,8,2" "800,940,8,2" "750,950,8,2" "800,920,8,2" "850,950,8,2" "750,920,8,1"; do
  r=$(KITTY_SCHED=$s timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['avg_launch_ms'])")
  echo "$s -> $r" | tee -a gpurun_out/sweep.txt
done
