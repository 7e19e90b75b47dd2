# Bench evidence: full GPU tests, C2 bench (+ CPU reference), 2-rank gloo smoke of the
# KV-head split on one GPU, reference arm.  Usage: bash tools/gpu_bench.sh TAG
mkdir -p gpurun_out
T=${1:-b}
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/${T}_pytest.txt 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/${T}_c2.txt 2>&1
timeout 900 python bench.py --gpus 2 --dist-backend gloo --config c5 --layers 4 --batch 16 --steps 5 --warmup 3 > gpurun_out/${T}_c5_2rank.txt 2>&1
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${T}_ref.txt 2>&1
tail -n 2 gpurun_out/${T}_smoke.txt; tail -n 3 gpurun_out/${T}_pytest.txt
for f in c2 c5_2rank ref; do python -c "
import json
try:
    d=json.loads(open('gpurun_out/${T}_$f.txt').read().strip().splitlines()[-1]); r=d.get('roofline',{})
    print('$f', d['value'], d['unit'], 'n', d['n_gpus'], 'launch_ms', r.get('avg_launch_ms'), 'frac', r.get('frac'), 'e2e', d.get('e2e',{}).get('value'), 'parity', (d.get('parity') or {}).get('max_abs'), 'cpu', (d.get('cpu_baseline') or {}).get('value'))
except Exception as e: print('$f FAILED', e); print(open('gpurun_out/${T}_$f.txt').read()[-1500:])
"; done
