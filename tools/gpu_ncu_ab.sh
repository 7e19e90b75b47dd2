mkdir -p gpurun_out
for L in libkitty_base.so libkitty_b200.so; do
  KITTY_B200_LIB=$PWD/paper_2511_18643_b200/$L timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ncuab_$L.csv \
    python bench.py --config c2 --layers 2 --steps 1 --warmup 3 --no-cpu-baseline --no-graph --no-parity > /dev/null 2>&1
  python - <<PY
import csv,collections
rows=list(csv.reader([l for l in open('gpurun_out/ncuab_$L.csv') if not l.startswith('==')]))
h=rows[0]; ki=h.index('Kernel Name'); vi=h.index('Metric Value')
d=collections.defaultdict(list)
for r in rows[1:]:
    if len(r)>vi and ('fastattn' in r[ki] or 'append' in r[ki]): d[r[ki][:60]].append(float(r[vi].replace(',','')))
for k,v in d.items(): print('$L', k, len(v), round(sum(v)/len(v)/1000,2), 'us')
PY
done
