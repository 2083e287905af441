set -x
python -c "import __graft_entry__ as g; g.build()"
python tools/c5_time.py build/variants/safe3.so > gpurun_out/r3e_c5.txt 2>&1
python tools/ab.py build/variants/head.so build/variants/safe3.so --rounds 8 > gpurun_out/r3e_ab.txt 2>&1
cat gpurun_out/r3e_c5.txt; tail -2 gpurun_out/r3e_ab.txt
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -15 > gpurun_out/r3e_pytest.txt
tail -3 gpurun_out/r3e_pytest.txt
