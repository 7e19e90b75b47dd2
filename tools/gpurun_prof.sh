# ncu full capture of one tc attention launch + the launch list (one GPU)
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc_attention -s 4 -c 1 \
    -o gpurun_out/prof_tc -f python bench.py --steps 1 --warmup 3 --layers 4 --no-cpu-baseline --no-graph ${BENCH_ARGS} \
    > gpurun_out/ncu_full.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"append|attention|combine" -c 400 --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-graph ${BENCH_ARGS} \
    > gpurun_out/ncu_launch_bench.txt 2>&1
tail -3 gpurun_out/ncu_full.txt
