# Iteration: GPU attention tests, C2 bench line, ncu capture of one page-kernel launch.
# Usage: bash tools/gpu_iter.sh TAG [pytest -k expr]
mkdir -p gpurun_out
T=${1:-iter}; K=${2:-attention or cache}
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "$K" > gpurun_out/${T}_pytest.txt 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_bench.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:page_kernel -s 8 -c 1 \
    -o gpurun_out/$T -f python bench.py --steps 1 --warmup 3 --layers 4 --no-cpu-baseline --no-graph > gpurun_out/${T}_ncu.txt 2>&1
tail -n 3 gpurun_out/${T}_pytest.txt
python -c "
import json; d=json.loads(open('gpurun_out/${T}_bench.txt').read().strip().splitlines()[-1]); r=d['roofline']
print('value', d['value'], 'launch_ms', r['avg_launch_ms'], 'frac', r['frac'], 'e2e', d['e2e']['value'])" || tail -5 gpurun_out/${T}_bench.txt
