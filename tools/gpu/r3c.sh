set -x
python -c "import __graft_entry__ as g; g.build()"
for v in paper_2509_06220_b200/libnrmf.so build/variants/safe.so; do echo "== $v"; python tools/c5_time.py $v; done > gpurun_out/r3c_c5.txt 2>&1
cat gpurun_out/r3c_c5.txt
python tools/ab.py build/variants/head.so build/variants/safe.so paper_2509_06220_b200/libnrmf.so --rounds 6 > gpurun_out/r3c_ab.txt 2>&1
tail -4 gpurun_out/r3c_ab.txt
cp build/variants/safe.so paper_2509_06220_b200/libnrmf.so
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -15 > gpurun_out/r3c_pytest.txt
tail -3 gpurun_out/r3c_pytest.txt
