timeout 1200 python -m pytest tests/test_gpu_short_cols.py tests/test_gpu_parity.py tests/test_gpu_unaligned.py tests/test_gpu_safe_mode.py -x -q -p no:cacheprovider 2>&1 | tail -2
for v in spe0 spe2 spe0 spe2; do echo "== $v"; python tools/cols_time.py build/variants/$v.so 2>&1 | grep -E "ld=(301|101|501|1000|4097|4160) "; done
PYTHONPATH=. python tools/unal_time.py > gpurun_out/r5a_unal.txt 2>&1; tail -2 gpurun_out/r5a_unal.txt
