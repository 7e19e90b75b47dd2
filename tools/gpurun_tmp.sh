mkdir -p gpurun_out
for cfg in c2 c4 c1; do for m in 2 3 6 7 2; do
KITTY_PDL=$m KITTY_B200_LIB=exp/libPdlM.so timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --config $cfg > /tmp/ab.txt 2>&1
python -c "import json; d=json.loads(open('/tmp/ab.txt').read().strip().splitlines()[-1]); print('$cfg pdl=$m', d['value'], d['roofline']['avg_launch_ms'], d['ms_per_step'])" || tail -3 /tmp/ab.txt
done; done
