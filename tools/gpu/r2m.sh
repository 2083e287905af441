set -x
python -c "import __graft_entry__ as g; g.build()"
timeout 600 python -m pytest tests/test_gpu_split_ll.py -x -q -p no:cacheprovider 2>&1 | tail -4 > gpurun_out/r2m_ll.txt
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -8 > gpurun_out/r2m_pytest.txt
python tools/ab.py paper_2509_06220_b200/libnrmf.so build/variants/elect.so --rounds 6 > gpurun_out/r2m_ab.txt 2>&1
