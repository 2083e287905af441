set -x
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_short_cols.py tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "cols or short" 2>&1 | tail -8 > gpurun_out/r2s_pytest.txt
python tools/cols_time.py > gpurun_out/r2s_cols_new.txt 2>&1
python tools/cols_time.py build/variants/noshort.so > gpurun_out/r2s_cols_old.txt 2>&1
