for c in c2 c3 c4; do for m in 3 7 3 7; do
KITTY_PDL=$m KITTY_B200_LIB=exp/libCur.so timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > /tmp/ab.txt 2>&1
python -c "import json; d=json.loads(open('/tmp/ab.txt').read().strip().splitlines()[-1]); print('$c pdl=$m', d['value'], d['roofline']['avg_launch_ms'])"
done; done
