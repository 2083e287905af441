cp build/variants/spf.so paper_2509_06220_b200/libnrmf.so
timeout 600 python -m pytest tests/test_gpu_short_cols.py -x -q -p no:cacheprovider 2>&1 | tail -2
for v in spf0 spf spf0 spf; do echo "== $v"; python tools/cols_time.py build/variants/$v.so 2>&1 | grep -E "r=(1000|500|1024|2000|300|100|4000) "; done
