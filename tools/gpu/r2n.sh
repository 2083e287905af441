set -x
python -c "import __graft_entry__ as g; g.build()"
timeout 1200 python -m pytest tests/test_gpu_defer.py -x -q -p no:cacheprovider 2>&1 | tail -15 > gpurun_out/r2n_defer.txt
python tools/ab.py build/variants/pol.so build/variants/defer.so --rounds 6 > gpurun_out/r2n_ab.txt 2>&1
python tools/c5_time.py > gpurun_out/r2n_c5.txt 2>&1
