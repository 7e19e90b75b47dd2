# compute-sanitizer memcheck / racecheck / synccheck over the decode kernels:
# smoke() (pack, prefill, append, fused attention, merge) and a selection of GPU
# tests (pool / import, odd boost fractions, fp chunks straddling the sink).
# Usage: bash tools/gpu_sanitize.sh TAG
mkdir -p gpurun_out
T=${1:-san}
CS="compute-sanitizer --target-processes all --print-limit 20"
SEL="test_pool_continuous_batching or test_export_import_round_trip or (test_boost_fractions_vs_oracle and (0.1 or 0.25)) or test_fp_chunks_straddling_sink_and_pages or test_golden_cache_step_by_step"
timeout 1200 $CS --tool memcheck python -m pytest tests -m gpu -q -p no:cacheprovider -k "$SEL" > gpurun_out/${T}_memcheck.txt 2>&1
tail -n 4 gpurun_out/${T}_memcheck.txt
for tool in racecheck synccheck; do
  timeout 1200 $CS --tool $tool python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_$tool.txt 2>&1
  tail -n 3 gpurun_out/${T}_$tool.txt
done
timeout 1200 $CS --tool racecheck python -m pytest tests -m gpu -q -p no:cacheprovider -k "test_pool_exhaustion or (test_boost_fractions_vs_oracle and 0.125 and 4)" > gpurun_out/${T}_racecheck_tests.txt 2>&1
tail -n 3 gpurun_out/${T}_racecheck_tests.txt
