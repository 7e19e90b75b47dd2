mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.txt 2>&1; tail -1 gpurun_out/pytest_gpu.txt
bash tools/ab.sh exp/libPack4.so exp/libComb2.so | tail -4
KITTY_PDL=7 bash tools/ab.sh exp/libPack4.so exp/libComb2.so | tail -2
bash tools/ab.sh exp/libPack4.so exp/libComb2.so --config c4 | tail -4
KITTY_PDL=7 bash tools/ab.sh exp/libPack4.so exp/libComb2.so --config c4 | tail -2
