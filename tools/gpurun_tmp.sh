timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.txt 2>&1; tail -1 gpurun_out/pytest_gpu.txt
bash tools/ab.sh exp/libWave2.so exp/libMpre.so | tail -4
bash tools/ab.sh exp/libWave2.so exp/libMpre.so --config c3 | tail -2
bash tools/ab.sh exp/libWave2.so exp/libMpre.so --config c4 | tail -2
bash tools/ab.sh exp/libWave2.so exp/libMpre.so --config c5 --batch 32 | tail -2
