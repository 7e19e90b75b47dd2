bash tools/ab.sh exp/libWave2.so exp/libF16.so | tail -4
bash tools/ab.sh exp/libWave2.so exp/libF16.so --config c4 | tail -2
