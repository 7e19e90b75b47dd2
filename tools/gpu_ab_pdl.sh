mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "attention or cache or pool" > gpurun_out/r02i_pytest.txt 2>&1; tail -n 1 gpurun_out/r02i_pytest.txt
for rep in 1 2; do for P in unset 3; do for c in c2 c3; do
  if [ $P = unset ]; then env -u KITTY_PDL python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-parity > gpurun_out/r02i_${P}_$c.txt 2>&1; else KITTY_PDL=$P python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-parity > gpurun_out/r02i_${P}_$c.txt 2>&1; fi
  python -c "
import json; d=json.loads(open('gpurun_out/r02i_${P}_$c.txt').read().strip().splitlines()[-1]); r=d['roofline']
print('pdl=$P $c', d['value'], 'ms_step', d['ms_per_step'], 'launch_ms', r['avg_launch_ms'])"
done; done; done
