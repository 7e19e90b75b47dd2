for L in exp/libPack3.so exp/libPack4.so; do echo $L; KITTY_B200_LIB=$L PYTHONPATH=. timeout 300 python tools/time_append.py 2>&1 | tail -1; done
