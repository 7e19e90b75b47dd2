timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "merge_width or long_units" 2>&1 | tail -3
