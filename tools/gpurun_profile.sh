# ncu evidence for the attention kernel (one GPU): launch list + one full capture.
# usage (from gpurun): bash tools/gpurun_profile.sh [bench args...]
mkdir -p gpurun_out
ARGS="$@"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"append|attention|prefill|combine" -c 2000 --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-graph $ARGS \
    > gpurun_out/ncu_launch_bench.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fast_attention -s 8 -c 2 \
    -o gpurun_out/prof_attn -f python bench.py --steps 1 --warmup 3 --layers 4 --no-cpu-baseline --no-graph $ARGS \
    > gpurun_out/ncu_full.txt 2>&1
ls -la gpurun_out
