mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.txt 2>&1; tail -1 gpurun_out/pytest_gpu.txt
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
bash tools/ab.sh exp/libComb2.so exp/libPvAcc.so | tail -4
bash tools/ab.sh exp/libComb2.so exp/libPvAcc.so --config c5 --batch 32 | tail -2
bash tools/ab.sh exp/libComb2.so exp/libPvAcc.so --config c4 | tail -2
