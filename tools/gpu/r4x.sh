timeout 900 python -m pytest tests/test_gpu_short_cols.py -x -q -p no:cacheprovider 2>&1 | tail -2
for v in skipid2 skip3 skipid2 skip3; do echo "== $v"; python tools/cols_time.py build/variants/$v.so 2>&1 | grep -E "r=(1000|500|700|1500|2000|100|4000) "; done
