mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "bulk_packer or prefill or signed_zero" > gpurun_out/pytest_pack.txt 2>&1; tail -5 gpurun_out/pytest_pack.txt
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:prefill_pack -c 1 python bench.py --steps 3 --warmup 3 --no-cpu-baseline 2>&1 | grep -E "duration|bytes" | head -4
timeout 300 ncu --set full --clock-control none --import-source on -k regex:prefill_pack_fast -c 1 -o gpurun_out/pack_fast3 python bench.py --config c4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_pack.log 2>&1; tail -1 gpurun_out/ncu_pack.log
