set -x
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_safe_mode.py tests/test_gpu_unaligned.py -x -q -p no:cacheprovider 2>&1 | tail -15 > gpurun_out/r3f_pytest.txt
tail -3 gpurun_out/r3f_pytest.txt
python tools/ab.py build/variants/head.so paper_2509_06220_b200/libnrmf.so --rounds 10 > gpurun_out/r3f_ab.txt 2>&1
tail -2 gpurun_out/r3f_ab.txt
