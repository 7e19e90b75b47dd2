# Full GPU test suite + smoke + the reference suite against the package.  Usage: bash tools/gpu_tests.sh TAG
mkdir -p gpurun_out
T=${1:-t}
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/${T}_pytest.txt 2>&1
timeout 1200 python tools/run_reference_suite.py > gpurun_out/${T}_refsuite.txt 2>&1
tail -n 2 gpurun_out/${T}_smoke.txt; tail -n 15 gpurun_out/${T}_pytest.txt; tail -n 25 gpurun_out/${T}_refsuite.txt
