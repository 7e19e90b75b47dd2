timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.txt 2>&1; tail -1 gpurun_out/pytest_gpu.txt
bash tools/ab.sh exp/libCur.so exp/libWave2.so --config c4 | tail -4
bash tools/ab.sh exp/libCur.so exp/libWave2.so --config c3 | tail -2
