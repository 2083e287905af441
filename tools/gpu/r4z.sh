cp build/variants/spe.so paper_2509_06220_b200/libnrmf.so
timeout 900 python -m pytest tests/test_gpu_short_cols.py tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "short or col" 2>&1 | tail -2
for v in spe0 spe spe0 spe; do echo "== $v"; python tools/cols_time.py build/variants/$v.so 2>&1 | grep -E "ld=(301|101|501|1000|4160|4096) "; done
PYTHONPATH=. python tools/unal_time.py > gpurun_out/r4z_unal.txt 2>&1; tail -4 gpurun_out/r4z_unal.txt
