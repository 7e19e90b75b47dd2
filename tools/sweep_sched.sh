mkdir -p gpurun_out
for s in "500,800,8,4" "720,930,16,4" "600,900,16,4" "700,900,12,3" "800,950,16,4" "650,920,16,8"; do
  r=$(KITTY_SCHED=$s timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['avg_launch_ms'])")
  echo "$s -> $r" | tee -a gpurun_out/sweep.txt
done
