cp build/variants/pfb.so paper_2509_06220_b200/libnrmf.so
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_short_cols.py tests/test_gpu_unaligned.py -x -q -p no:cacheprovider 2>&1 | tail -2
for v in pfb0 pfb pfb0 pfb; do echo "== $v"; python tools/cols_time.py build/variants/$v.so 2>&1 | grep -E "r=(4000|3000|4096) |ld=4097"; done
