KITTY_B200_LIB=exp/libW5.so timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "attention or decode or ragged or golden or long_units or merge_width" 2>&1 | tail -1
bash tools/ab.sh exp/libW4.so exp/libW5.so | tail -4
bash tools/ab.sh exp/libW4.so exp/libW5.so --config c3 | tail -2
bash tools/ab.sh exp/libW4.so exp/libW5.so --config c4 | tail -2
