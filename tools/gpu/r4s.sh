timeout 900 python -m pytest tests/test_gpu_short_cols.py tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "short or col" 2>&1 | tail -2
for v in spf0 skipid2 spf0 skipid2; do echo "== $v"; python tools/cols_time.py build/variants/$v.so 2>&1 | grep -E "r=(1000|500|1024|2000|300|100|4000) "; done
